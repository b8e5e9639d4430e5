"""GPU tests of squash-window validation: the mutation set of a window
(digest diff between window open and close, worker.cpp:351-421) computed by K1 on the
auxiliary grid, checked against the CPU oracle, and validated across sharing ranks with
splice::validate_window semantics (splice.cpp:21-61)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

ARENA = 32 << 20
PENDING = 4


def bufs_of(spec):
    return [(0, i, a, n, c, f) for i, (a, n, c, f) in enumerate(spec)]


def oracle_buf_digests(host, bufs):
    live = [b[:5] for b in bufs if not (b[5] & PENDING)]
    return live, O.hash_chunks([host], live)[2]


def test_digest_ranges_vs_oracle_and_grid_untouched(snap):
    with snap.Ctx(0, ARENA) as c:
        c.fill_mix64(0, ARENA, 3, 0)
        host = c.read(0, ARENA).view(np.uint64)
        grid = [(0, 0, 0, 8 << 20, 0), (0, 1, 8 << 20, (4 << 20) + 256, 1)]
        c.set_buffers(grid)
        c.snapshot()
        d0, _ = c.digests()
        ranges = [(0, 0, 1 << 20, 256, 0), (0, 1, 3 << 20, 5 << 20, 0), (0, 2, 20 << 20, 65536, 0)]
        got = c.digest_ranges(ranges)
        assert np.array_equal(got, O.hash_chunks([host], ranges)[2])
        # the installed grid, its digests and its staging are untouched
        d1, _ = c.digests()
        assert np.array_equal(d0, d1)
        c.write(0, np.zeros(1 << 20, np.uint8))
        c.restore_self(verify=True)


def test_window_mutation_set_vs_oracle(snap):
    spec = [(0, 1 << 20, 0, 0), (1 << 20, 2 << 20, 1, 0), (3 << 20, 512 << 10, 2, PENDING),
            (4 << 20, 1 << 20, 1, 0), (6 << 20, 256, 0, 0)]
    with snap.Ctx(0, ARENA) as c:
        c.fill_mix64(0, ARENA, 8, 0)
        b_open = bufs_of(spec)
        c.window_open(1, b_open)
        # in-window work: optimizer touches buffers 1 and 4, the pending gradient changes
        # (skipped), buffer 3 grows, a new buffer appears at 8 MiB
        c.xor_words([(1 << 20) + 4096, 6 << 20, (3 << 20) + 64], 0x77)
        spec2 = list(spec)
        spec2[3] = (4 << 20, (1 << 20) + 256, 1, 0)
        spec2.append((8 << 20, 64 << 10, 3, 0))
        b_close = bufs_of(spec2)
        muts = c.window_close(1, b_close)
        host = c.read(0, ARENA).view(np.uint64)
        live, od = oracle_buf_digests(host, b_close)
        exp = sorted((b[2], b[3], int(d)) for b, d in zip(live, od)
                     if b[2] in {1 << 20, 4 << 20, 6 << 20, 8 << 20})
        assert muts == exp
        # a window with no change has an empty mutation set; close without open is an error
        c.window_open(2, b_close)
        assert c.window_close(2, b_close) == []
        with pytest.raises(snap.SnapError):
            c.window_close(2, b_close)


def test_squash_validation_across_sharing_ranks(snap, oracle_mod):
    """Two time-sliced ranks run the same validation window at the same stable addresses
    (their P/O are swapped in and out of one address range): identical optimizer steps
    validate; a diverging step fails with the reference's reason text."""
    spec = [(0, 2 << 20, 0, 0), (2 << 20, 4 << 20, 1, 0), (6 << 20, 1 << 20, 2, PENDING)]
    b = bufs_of(spec)
    with snap.Ctx(0, ARENA) as c:
        c.fill_mix64(0, 8 << 20, 21, 0)
        start = c.read(0, 8 << 20)
        recs = {}
        for rank, delta in ((0, 0x11), (1, 0x11), (2, 0x12)):
            c.write(0, start)  # the rank's (identical) P/O swapped in
            c.window_open(rank, b)
            c.xor_words([4096, (2 << 20) + 8192], delta)  # the window's optimizer step
            muts = c.window_close(rank, b)
            d2h = [(256, int(c.digest_ranges([(0, 0, 0, 256, 0)])[0]))]  # in-window copy_d2h
            recs[rank] = (muts, d2h)
        ok, why = snap.validate_window({r: recs[r] for r in (0, 1)})
        assert ok and why == ""
        ok, why = snap.validate_window(recs)
        assert not ok and why.startswith("mutation digests differ at addr")
        R = oracle_mod.ref()
        if R is not None:
            from test_capi import _ref_validate
            assert _ref_validate(R, recs) == (ok, why)
