"""Parity at BASELINE.json's full sizes through size-independent properties (the oracle
cannot hash tens of GiB in test time): round trips, the exact dirty set of C4, sampled
chunk digests against the oracle, and staged-byte accounting."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

MIX_SAMPLE = 256  # chunks whose digests are recomputed by the oracle per test


def c2_layout():
    import bench
    return bench.c2_layout()


def sample_digests_vs_oracle(ctx, bufs, d, rng, geom=(4096, 65536)):
    """Recompute a random sample of chunk digests on the CPU from bytes read back."""
    starts = np.concatenate([[0], np.cumsum([(b[3] + geom[1] - 1) // geom[1] for b in bufs])])
    for g in rng.choice(d.size, min(MIX_SAMPLE, d.size), replace=False):
        b = int(np.searchsorted(starts, g, side="right") - 1)
        k = int(g - starts[b])
        off = k * geom[1]
        n = min(geom[1], bufs[b][3] - off)
        host = ctx.read(bufs[b][2] + off, n).view(np.uint64)
        od, _, _ = O.hash_chunks([host], [(0, 0, 0, n, 0)], *geom)
        assert int(od[0]) == int(d[g]), (g, b, k)


def test_c1_256mib_round_trip_dup_heavy(snap):
    # C1 duplicate-heavy variant: chunk c content = chunk (c mod 1024)
    nbytes, chunk = 256 << 20, 65536
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, 1024 * chunk, 1, 0)
        base = c.read(0, 1024 * chunk)
        for r in range(1, nbytes // (1024 * chunk)):
            c.write(r * 1024 * chunk, base)
        bufs = [(0, 0, 0, nbytes, 0)]
        c.set_buffers(bufs)
        c.snapshot()
        _, _, _, sbytes, schunks = c.selection()
        assert schunks == 1024 and sbytes == 1024 * chunk
        d, _ = c.digests()
        assert np.array_equal(d[:1024], d[1024:2048])
        sample_digests_vs_oracle(c, bufs, d, np.random.default_rng(1))
        c.fill_mix64(0, nbytes, 99, 0)
        c.restore_self(verify=True)
        assert np.array_equal(c.read(0, 1024 * chunk), base)


def test_c2_2gib_rank_image_round_trip(snap):
    bufs, rep, per = c2_layout()
    image = rep + per
    with snap.Ctx(0, image + (1 << 20)) as c:
        import bench
        bench.fill_rank(c, 0, rep, per)
        c.set_buffers(bufs)
        for _ in range(2):  # first + learned speculative layout
            c.snapshot()
        _, _, _, sbytes, schunks = c.selection()
        d, lens = c.digests()
        assert schunks == d.size and sbytes == int(lens.sum()) == image  # all unique
        sample_digests_vs_oracle(c, bufs, d, np.random.default_rng(2))
        # staged image == the chunks in canonical order (sampled)
        rng = np.random.default_rng(3)
        _, _, off, _, _ = c.selection()
        starts = np.concatenate([[0], np.cumsum([(b[3] + 65535) // 65536 for b in bufs])])
        for g in rng.choice(d.size, 64, replace=False):
            b = int(np.searchsorted(starts, g, side="right") - 1)
            k = int(g - starts[b])
            n = min(65536, bufs[b][3] - k * 65536)
            assert np.array_equal(c.read_staging(int(off[g]), n), c.read(bufs[b][2] + k * 65536, n))
        c.fill_mix64(0, image, 12345, 0)
        c.restore_self(verify=True)
        c.hash()
        d2, _ = c.digests()
        assert np.array_equal(d, d2)


def test_c4_32gib_incremental_dirty_set_exact(snap):
    """C4: 32 GiB, chunk c dirty iff mix64(seed ^ c) % 20 == 0: the
    incremental selection is exactly that set, in order, with exact staged bytes."""
    gib = 32
    nbytes, nb = gib << 30, 256 << 20
    bufs = [(0, i, i * nb, nb, 1) for i in range(nbytes // nb)]
    with snap.Ctx(0, nbytes + (1 << 20)) as c:
        c.fill_mix64(0, nbytes, 99, 0)
        n = c.set_buffers(bufs)
        c.snapshot()
        c.known_commit()
        mix = np.array([O.mix64(99 ^ k) for k in range(n)], dtype=np.uint64)
        dirty = np.nonzero(mix % np.uint64(20) == 0)[0]
        c.xor_words((dirty * 65536).astype(np.uint64), 0x1234567)
        c.snapshot()
        sel, owner, off, sbytes, schunks = c.selection()
        assert schunks == dirty.size and sbytes == dirty.size * 65536
        assert np.array_equal(np.nonzero(sel)[0], dirty)
        assert np.array_equal(off[dirty], np.arange(dirty.size, dtype=np.uint64) * 65536)
        # unchanged chunks are known (no owner, no offset)
        clean = np.setdiff1d(np.arange(n), dirty)[:1000]
        assert (owner[clean] == np.uint64(2**64 - 1)).all()
        # staged bytes of a few dirty chunks == the mutated arena chunk
        for g in dirty[:: max(1, dirty.size // 16)]:
            assert np.array_equal(c.read_staging(int(off[g]), 65536), c.read(int(g) * 65536, 65536))
