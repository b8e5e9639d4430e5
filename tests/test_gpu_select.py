"""K2 selection on every GPU path against the oracle: the 8-CTA cluster selection
(n <= 4096 chunks), the one-launch small selection (n <= 8192) and the three-kernel
look-back path beyond,
with duplicates, a known set and the size boundaries; the fused verify-scatter restore on ragged
layouts and several geometries; K5 in bf16."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nchunks", [1, 31, 1023, 1024, 1025, 4096, 4097, 8191, 8192, 8193, 20000,
                                     65536, 65537])
def test_selection_paths_vs_oracle(snap, nchunks):
    rng = np.random.default_rng(nchunks)
    chunk = 4096  # page == chunk: one 4 KiB chunk per slot, cheap to build many
    pool = 64 + nchunks // 3
    nbytes = (pool + nchunks) * chunk
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, pool * chunk, 7 + nchunks, 0)
        # chunk k of the grid = a copy of pool[perm[k]] (many duplicates)
        src = rng.integers(0, pool, nchunks)
        host = c.read(0, pool * chunk)
        img = np.concatenate([host[int(s) * chunk:(int(s) + 1) * chunk] for s in src])
        c.write(pool * chunk, img)
        bufs = [(0, 0, pool * chunk, nchunks * chunk, 1)]
        c.set_buffers(bufs, chunk, chunk)
        known = []
        for rnd in range(2):
            c.snapshot()
            d, lens = c.digests()
            sel, owner, off, tot, nsel = c.selection()
            osel, oown, ooff, otot = O.select(d, lens, np.array(known, np.uint64) if known else None)
            assert np.array_equal(sel, osel) and np.array_equal(owner, oown)
            assert np.array_equal(off, ooff) and tot == otot
            staged = c.read_staging(0, tot) if tot else np.zeros(0, np.uint8)
            exp = np.concatenate([img[g * chunk:(g + 1) * chunk] for g in np.nonzero(osel)[0]]) \
                if otot else np.zeros(0, np.uint8)
            assert np.array_equal(staged, exp)
            known = [int(x) for x in d[rng.integers(0, nchunks, max(1, nchunks // 4))]]
            c.known_clear()
            c.known_add(np.array(known, np.uint64))


@pytest.mark.parametrize("geom", [(4096, 65536), (256, 4096), (1024, 32768), (65536, 65536)])
def test_verify_scatter_ragged(snap, geom):
    """snap_restore / snap_restore_self with verification = one pass that scatters and
    hashes; bit-exact content, and a corrupted image chunk is caught by digest."""
    rng = np.random.default_rng(geom[0])
    arena = 24 << 20
    with snap.Ctx(0, arena) as c:
        c.fill_mix64(0, arena, 3, 0)
        bufs, addr = [], 0
        while True:
            nb = int(rng.integers(1, 900)) * 256
            if addr + nb > arena // 2:
                break
            bufs.append((0, len(bufs), addr, nb, int(rng.integers(0, 4))))
            addr += nb + int(rng.integers(0, 4)) * 256
        host = c.read(0, arena)
        c.set_buffers(bufs, *geom)
        c.snapshot()
        c.write(0, np.zeros(arena // 2, np.uint8))
        c.restore_self(verify=True)
        back = c.read(0, arena)
        for (_r, _s, a, n, _c) in bufs:
            assert np.array_equal(back[a:a + n], host[a:a + n])
        # snap_restore from a host-provided image: flip one byte -> SimFault
        _, _, off, tot, _ = c.selection()
        d, _ = c.digests()
        img = c.read_staging(0, tot)
        dev = c.arena_ptr() + arena // 2
        c.write(arena // 2, img)
        c.restore(dev, tot, off, expect=d, verify=True)
        img[int(rng.integers(0, tot))] ^= 0x5A
        c.write(arena // 2, img)
        with pytest.raises(snap.SnapError) as e:
            c.restore(dev, tot, off, expect=d, verify=True)
        assert e.value.code == snap.SNAP_EFAULT
        assert "1 chunk(s)" in str(e.value)
        # the mismatch state is reset: the intact image verifies again, twice
        img[:] = c.read_staging(0, tot)
        c.write(arena // 2, img)
        c.restore(dev, tot, off, expect=d, verify=True)
        c.restore_self(verify=True)


def test_grad_sum_bf16(snap, ctx):
    rng = np.random.default_rng(21)
    n = 1_000_005
    gs = [((rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8, n)).astype(np.float32)
           .view(np.uint32) >> 16).astype(np.uint16) for _ in range(4)]
    stride = (2 * n + 255) // 256 * 256
    for r, g in enumerate(gs):
        ctx.write(r * stride, g)
    ctx.grad_sum(snap.BF16, [r * stride for r in range(4)], 5 * stride, n)
    got = ctx.read(5 * stride, 2 * n).view(np.uint16)
    assert np.array_equal(got, O.grad_sum_bf16(gs))
    # accumulate: dst (bf16) is the first addend of a new chain
    ctx.grad_sum(snap.BF16, [r * stride for r in range(2)], 5 * stride, n, accumulate=True)
    got2 = ctx.read(5 * stride, 2 * n).view(np.uint16)
    assert np.array_equal(got2, O.grad_sum_bf16([O.grad_sum_bf16(gs), gs[0], gs[1]]))


def test_selection_fuzz_small_ragged(snap):
    """Random ragged layouts of <= 4096 chunks (the 8-CTA cluster selection), duplicate
    chunks across buffers, and random known sets; every round checked against the oracle,
    the staged image against the selected chunks' bytes."""
    rng = np.random.default_rng(77)
    arena = 48 << 20
    with snap.Ctx(0, arena) as c:
        c.fill_mix64(0, arena, 5, 0)
        for rnd in range(12):
            geom = [(4096, 65536), (256, 4096), (1024, 16384)][rnd % 3]
            bufs, addr = [], 0
            while len(bufs) < 200:
                nb = int(rng.integers(1, 6 * geom[1] // 256)) * 256
                if addr + nb > arena // 2:
                    break
                bufs.append((0, len(bufs), addr, nb, int(rng.integers(0, 4))))
                addr += nb + int(rng.integers(0, 3)) * 256
            # duplicate some buffers' leading chunks into others
            host = c.read(0, arena // 2)
            for _ in range(20):
                a, b = rng.integers(0, len(bufs), 2)
                n = min(bufs[a][3], bufs[b][3]) // geom[1] * geom[1]
                if n:
                    host[bufs[b][2]:bufs[b][2] + n] = host[bufs[a][2]:bufs[a][2] + n]
            c.write(0, host)
            n = c.set_buffers(bufs, *geom)
            assert n <= 4096
            c.known_clear()
            known = None
            if rnd % 2:
                c.snapshot()
                d0, _ = c.digests()
                known = d0[rng.integers(0, n, max(1, n // 3))]
                c.known_add(known)
            c.snapshot()
            d, lens = c.digests()
            sel, owner, off, tot, _ = c.selection()
            osel, oown, ooff, otot = O.select(d, lens, known)
            assert np.array_equal(sel, osel) and np.array_equal(owner, oown), rnd
            assert np.array_equal(off, ooff) and tot == otot, rnd
            if otot:
                # each selected chunk's bytes at its offset
                img = c.read_staging(0, tot)
                starts = np.concatenate([[0], np.cumsum(
                    [(b[3] + geom[1] - 1) // geom[1] for b in bufs])])
                for gi in np.nonzero(osel)[0][:64]:
                    bi = int(np.searchsorted(starts, gi, side="right") - 1)
                    k = int(gi - starts[bi])
                    a0 = bufs[bi][2] + k * geom[1]
                    ln = int(lens[gi])
                    assert np.array_equal(img[int(ooff[gi]):int(ooff[gi]) + ln],
                                          host[a0:a0 + ln]), (rnd, gi)


def test_restore_graph_follows_layout_changes(snap):
    """The verified restore replays a cached CUDA graph while the layout is unchanged; a new
    layout must never be served by a stale graph (a corrupted image behind a replayed graph:
    test_verify_scatter_ragged)."""
    rng = np.random.default_rng(5)
    arena = 16 << 20
    with snap.Ctx(0, arena) as c:
        for rnd in range(6):
            c.fill_mix64(0, arena // 2, 100 + rnd, 0)
            nb = int(rng.integers(64, 512)) * 1024
            bufs = [(0, i, i * nb, nb, 0) for i in range((arena // 2) // nb)]
            c.set_buffers(bufs)
            host = c.read(0, arena // 2)
            c.snapshot()
            for _ in range(3):  # replays
                c.write(0, np.zeros(arena // 2, np.uint8))
                c.restore_self(verify=True)
                assert np.array_equal(c.read(0, arena // 2)[:len(bufs) * nb],
                                      host[:len(bufs) * nb]), rnd
