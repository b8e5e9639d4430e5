"""GPU parity tests (B200): K1 hash, K2 select, K3 compact, K4 restore against the
oracle (CPU restatement) and the reference-generated golden fixtures, through the C ABI."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def load_ragged(ctx, golden):
    rag = golden["ragged"]
    arena = O.fill_mix64(rag["arena_bytes"] // 8, rag["seed"], 0)
    src, dst, n = rag["dup"]
    arena[dst // 8:(dst + n) // 8] = arena[src // 8:(src + n) // 8]
    ctx.write(0, arena)
    return arena, [tuple(b) for b in rag["bufs"]]


def test_c1_hash_matches_reference_golden(snap, c1_golden):
    with snap.Ctx(0, 256 << 20) as c:
        c.fill_mix64(0, 256 << 20, 0, 0)  # words[i] = mix64(i)
        bufs = [(0, 0, 0, 256 << 20, 0)]
        assert c.set_buffers(bufs, 4096, 65536) == 4096
        c.hash()
        d, lens, bd = c.digests(buf_digests=True)
        assert np.array_equal(d, c1_golden["merkle"])
        assert int(bd[0]) == int(c1_golden["buf"][0])
        c.set_buffers(bufs, 65536, 65536)
        c.hash()
        d, _ = c.digests()
        assert np.array_equal(d, c1_golden["direct"])
        assert c.launches > 0


@pytest.mark.parametrize("geom", [(4096, 65536), (65536, 65536), (256, 4096), (1024, 32768)])
def test_ragged_hash_golden(snap, ctx, golden, geom):
    arena, bufs = load_ragged(ctx, golden)
    ctx.set_buffers(bufs, *geom)
    ctx.hash()
    d, lens, bd = ctx.digests(buf_digests=True)
    exp = golden["ragged"][f"{geom[0]}_{geom[1]}"]
    assert [f"{x:016x}" for x in d] == exp["chunks"]
    assert [f"{x:016x}" for x in bd] == exp["bufs"]
    od, olens, obd = O.hash_chunks([arena], bufs, *geom)
    assert np.array_equal(d, od) and np.array_equal(lens, olens)


def test_random_layouts_vs_oracle(snap, ctx):
    rng = np.random.default_rng(5)
    arena_bytes = 64 << 20
    for trial in range(4):
        ctx.fill_mix64(0, arena_bytes, 100 + trial, 0)
        host = ctx.read(0, arena_bytes).view(np.uint64)
        # random non-overlapping 256-B aligned buffers
        bufs, addr = [], 0
        while True:
            nb = int(rng.integers(1, 1200)) * 256
            if addr + nb > arena_bytes:
                break
            bufs.append((0, len(bufs), addr, nb, 0))
            addr += nb + int(rng.integers(0, 8)) * 256
        for geom in [(4096, 65536), (256, 8192), (65536, 65536)]:
            ctx.set_buffers(bufs, *geom)
            ctx.hash()
            d, lens = ctx.digests()
            od, olens, _ = O.hash_chunks([host], bufs, *geom)
            assert np.array_equal(d, od), (trial, geom)


def test_select_compact_restore_ragged(snap, ctx, golden):
    arena, bufs = load_ragged(ctx, golden)
    ctx.set_buffers(bufs, 4096, 65536)
    ctx.snapshot()
    sel, owner, off, sbytes, schunks = ctx.selection()
    d, lens = ctx.digests()
    osel, oowner, ooff, ototal = O.select(d, lens)
    assert np.array_equal(sel, osel)
    assert np.array_equal(owner, oowner)
    assert np.array_equal(off, ooff)
    assert sbytes == ototal and schunks == int(osel.sum())
    img = ctx.read_staging(0, sbytes)
    assert np.array_equal(img, O.compact([arena], bufs, 65536, osel, ooff, ototal))
    # restore into a zeroed arena: bit-exact
    ctx.write(0, np.zeros(golden["ragged"]["arena_bytes"], np.uint8))
    ctx.restore_self(verify=True)
    back = ctx.read(0, golden["ragged"]["arena_bytes"]).view(np.uint64)
    for (_r, _s, a, n, _c) in bufs:
        assert np.array_equal(back[a // 8:(a + n) // 8], arena[a // 8:(a + n) // 8])


def test_duplicate_heavy_and_known_set(snap):
    """C1 duplicate-heavy variant (chunk c content = chunk c mod 1024) + incremental
    snapshot against a known set (BlobStore fresh semantics, ckpt.cpp:18-20)."""
    nbytes = 64 << 20
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, 16 << 20, 1, 0)
        base = c.read(0, 16 << 20)
        for k in range(1, 4):
            c.write(k * (16 << 20), base)
        bufs = [(0, 0, 0, nbytes, 0)]
        c.set_buffers(bufs)
        c.snapshot()
        sel, owner, off, sbytes, sch = c.selection()
        assert sch == 256 and sbytes == 16 << 20
        assert (owner[256:] == np.arange(1024)[256:] % 256).all()
        d, lens = c.digests()
        # incremental: everything already known -> nothing staged
        c.known_commit()
        c.hash()
        c.select()
        sel2, owner2, off2, sb2, sc2 = c.selection()
        assert sc2 == 0 and sb2 == 0 and (owner2 == 2**64 - 1).all()
        # dirty 5 % of the distinct chunks -> exactly those staged, canonical order
        rng = np.random.default_rng(9)
        dirty = np.sort(rng.choice(256, size=13, replace=False))
        c.xor_words(dirty.astype(np.uint64) * 65536, 0xDEADBEEF)
        c.hash()
        c.select()
        c.compact()
        sel3, owner3, off3, sb3, sc3 = c.selection()
        d3, lens3 = c.digests()
        osel, oown, ooff, otot = O.select(d3, lens3, known=d)
        assert np.array_equal(sel3, osel) and np.array_equal(off3, ooff) and sb3 == otot
        assert sc3 == 13 and np.array_equal(np.nonzero(sel3)[0], dirty)
        host = c.read(0, nbytes)
        img = c.read_staging(0, sb3)
        assert np.array_equal(img, O.compact([host], bufs, 65536, osel, ooff, otot))


def test_restore_verify_detects_corruption(snap, ctx):
    ctx.fill_mix64(0, 8 << 20, 3, 0)
    bufs = [(0, 0, 0, 4 << 20, 0), (0, 1, 4 << 20, 4 << 20, 1)]
    ctx.set_buffers(bufs)
    ctx.snapshot()
    sel, owner, off, sbytes, _ = ctx.selection()
    d, _ = ctx.digests()
    p, n = ctx.staging_ptr()
    ctx.restore(p, sbytes, off, expect=d, verify=True)
    bad = d.copy()
    bad[7] ^= 1
    with pytest.raises(snap.SnapFault):
        ctx.restore(p, sbytes, off, expect=bad, verify=True)
    # a chunk with no source in the image is a fault, like BlobStore::get (ckpt.cpp:25)
    off2 = off.copy()
    off2[3] = sbytes
    with pytest.raises(snap.SnapFault):
        ctx.restore(p, sbytes, off2, verify=False)


def test_c1_full_round_trip(snap):
    """C1: 256 MiB single-rank image as 64 x 4 MiB buffers, snapshot + restore bit-exact."""
    nbytes = 256 << 20
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, nbytes, 1, 0)
        bufs = [(0, i, i * (4 << 20), 4 << 20, i % 3) for i in range(64)]
        c.set_buffers(bufs)
        c.snapshot()
        sel, owner, off, sbytes, sch = c.selection()
        assert sch == 4096 and sbytes == nbytes and sel.all()
        ref_img = c.read(0, nbytes)
        assert np.array_equal(c.read_staging(0, nbytes), ref_img)  # identity order
        d, lens = c.digests()
        od, _, _ = O.hash_chunks([ref_img], bufs)
        assert np.array_equal(d, od)
        c.write(0, np.zeros(nbytes, np.uint8))
        c.restore_self(verify=True)
        assert np.array_equal(c.read(0, nbytes), ref_img)


@pytest.mark.parametrize("dtype", ["u64", "f32"])
def test_grad_sum(snap, ctx, dtype):
    rng = np.random.default_rng(11)
    n = 1_000_003
    if dtype == "u64":
        gs = [rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64) for _ in range(4)]
        exp = O.grad_sum_u64(gs)
        code = snap.U64
    else:
        gs = [(rng.standard_normal(n) * 10 ** rng.uniform(-3, 3, n)).astype(np.float32)
              for _ in range(4)]
        exp = O.grad_sum_f32(gs)
        code = snap.F32
    nb = gs[0].nbytes
    stride = (nb + 255) // 256 * 256
    for r, g in enumerate(gs):
        ctx.write(r * stride, g)
    dst = 5 * stride
    ctx.grad_sum(code, [r * stride for r in range(4)], dst, n)
    got = np.frombuffer(ctx.read(dst, nb).tobytes(), dtype=gs[0].dtype)
    if dtype == "u64":
        assert np.array_equal(got, exp)
    else:
        # fixed-order fp32: bit-exact with the CPU order; the north-star tolerance is 1e-6 rel
        np.testing.assert_allclose(got, exp, rtol=1e-6, atol=0)
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    # accumulate mode: dst += src_4 ... (time-sliced ranks arriving one by one)
    ctx.write(dst, gs[0])
    for r in range(1, 4):
        ctx.grad_sum(code, [r * stride], dst, n, accumulate=True)
    got2 = np.frombuffer(ctx.read(dst, nb).tobytes(), dtype=gs[0].dtype)
    assert np.array_equal(got2.view(np.uint8), exp.view(np.uint8))


def test_fused_speculation_learns_and_recovers(snap, ctx, golden):
    """Fused hash+compaction: the first snapshot speculates the identity layout, later
    ones reuse the last actual layout; every mispredicted chunk is fixed up from the
    arena, so the staging image always equals the oracle's."""
    arena, bufs = load_ragged(ctx, golden)
    ctx.set_buffers(bufs, 4096, 65536)

    def check(host):
        ctx.snapshot()
        d, lens = ctx.digests()
        sel, owner, off, sbytes, _ = ctx.selection()
        osel, oown, ooff, otot = O.select(d, lens)
        assert np.array_equal(sel, osel) and np.array_equal(off, ooff) and sbytes == otot
        assert np.array_equal(ctx.read_staging(0, sbytes),
                              O.compact([host], bufs, 65536, osel, ooff, otot))

    check(arena)          # identity speculation, fix-up after the duplicate buffer
    check(arena)          # learned layout: no fix-up
    # break the duplicate (buffer 3 becomes unique) -> prediction too small, fix-up again
    src, dst, n = golden["ragged"]["dup"]
    ctx.xor_words([dst + 4096], 0x5A5A)
    host = ctx.read(0, golden["ragged"]["arena_bytes"])
    check(host)
    check(host)
    # make buffer 0 a copy of buffer 5's first 256 B -> new duplicate: holes, fix-up
    b0 = bufs[0]
    ctx.write(b0[2], host[bufs[5][2]:bufs[5][2] + b0[3]])
    host = ctx.read(0, golden["ragged"]["arena_bytes"])
    check(host)


@pytest.mark.parametrize("variant,chunk", [(-1, 65536), (11, 65536), (12, 65536), (13, 65536),
                                           (-1, 16384)])
def test_snapshot_host_pipelined(snap, variant, chunk):
    """snap_snapshot_host (pinned host image -> arena -> K1..K3 -> staging to host), slab
    pipelined: staging image == oracle compaction, through mispredicted, learned and
    incremental layouts, and through the non-pipelined fallback (unsorted buffers).
    variant 11/12: the tensor-core K1 kernels on every slab (grid slices c_begin..c_end).
    16 KiB chunks: 10240 chunks, so K1 also does the K2 insert, slab by slab."""
    snap.set_k1_variant(variant)
    try:
        _host_pipelined(snap, chunk)
    finally:
        snap.set_k1_variant(-1)


def _host_pipelined(snap, chunk=65536):
    nbytes = 160 << 20
    img = O.fill_mix64(nbytes // 8, 21, 0)
    # buffers spanning several 64 MiB slabs, a duplicate (mispredicted speculation)
    bufs = [(0, 0, 0, 48 << 20, 0), (0, 1, 48 << 20, (40 << 20) + 768, 1),
            (0, 2, 100 << 20, 20 << 20, 2), (0, 3, 128 << 20, 8 << 20, 1),
            (0, 4, 150 << 20, 256, 4)]
    img[(128 << 20) // 8:(136 << 20) // 8] = img[(56 << 20) // 8:(64 << 20) // 8]
    pin = snap.PinnedHost(nbytes)
    pin.array[:] = img.view(np.uint8)
    out = snap.PinnedHost(nbytes)
    with snap.Ctx(0, nbytes) as c:
        c.set_buffers(bufs, 4096, chunk)
        dig = np.zeros(c.nchunks, np.uint64)
        od, olens, _ = O.hash_chunks([img], bufs, 4096, chunk)
        osel, oown, ooff, otot = O.select(od, olens)
        exp = O.compact([img], bufs, chunk, osel, ooff, otot)
        for it in range(2):
            staged = c.snapshot_host(pin.ptr, 0, nbytes, out.ptr, nbytes, dig)
            assert staged == otot and np.array_equal(dig, od), it
            assert np.array_equal(out.array[:staged], exp), it
        # incremental: 3 dirty chunks against the committed store
        c.known_commit()
        host2 = img.copy()
        host2[[3 * 8192, 700 * 8192, 1900 * 8192]] ^= np.uint64(0xABCD)  # 3 chunks at any chunk size
        pin.array[:] = host2.view(np.uint8)
        staged = c.snapshot_host(pin.ptr, 0, nbytes, out.ptr, nbytes, dig)
        d2, l2, _ = O.hash_chunks([host2], bufs, 4096, chunk)
        s2, _, o2, t2 = O.select(d2, l2, known=od)
        assert staged == t2 == 3 * chunk
        assert np.array_equal(out.array[:staged], O.compact([host2], bufs, chunk, s2, o2, t2))
    # unsorted buffer order -> sequential fallback, same result
    bufs_u = [bufs[1], bufs[0], bufs[2]]
    with snap.Ctx(0, nbytes) as c:
        pin.array[:] = img.view(np.uint8)
        c.set_buffers(bufs_u, 4096, chunk)
        dig = np.zeros(c.nchunks, np.uint64)
        staged = c.snapshot_host(pin.ptr, 0, nbytes, out.ptr, nbytes, dig)
        od, olens, _ = O.hash_chunks([img], bufs_u, 4096, chunk)
        osel, oown, ooff, otot = O.select(od, olens)
        assert staged == otot
        assert np.array_equal(out.array[:staged], O.compact([img], bufs_u, chunk, osel, ooff, otot))
    pin.free()
    out.free()
