"""GPU edge cases of the C ABI: empty grids, zero-length operations, minimum-size buffers,
buffers ending exactly at the arena end, error codes for bad arguments (the reference's
SimFault / ConfigError behaviour, common.hpp:31-49)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def test_empty_grid_snapshot_restore_persist(snap, ctx, tmp_path):
    assert ctx.set_buffers([]) == 0
    ctx.snapshot()
    sel, owner, off, sbytes, schunks = ctx.selection()
    assert sbytes == 0 and schunks == 0
    ctx.restore_self(verify=True)
    st = ctx.persist(tmp_path)
    assert st["blobs"] == 0 and st["layout_chunks"] == 0
    ctx.load(tmp_path)
    assert ctx.nchunks == 0
    d, _ = ctx.digests()
    assert d.size == 0


def test_single_256_byte_buffer_and_arena_end(snap):
    nbytes = 1 << 20
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, nbytes, 5, 0)
        host = c.read(0, nbytes).view(np.uint64)
        bufs = [(0, 0, 0, 256, 0), (0, 1, nbytes - 256, 256, 1)]  # last byte of the arena
        c.set_buffers(bufs)
        c.snapshot()
        d, lens = c.digests()
        od, olens, _ = O.hash_chunks([host], bufs)
        assert np.array_equal(d, od) and list(lens) == [256, 256]
        c.fill_mix64(0, nbytes, 6, 0)
        c.restore_self(verify=True)
        got = c.read(0, nbytes).view(np.uint64)
        assert np.array_equal(got[:32], host[:32]) and np.array_equal(got[-32:], host[-32:])


def test_bad_arguments_fail_loudly(snap, ctx):
    with pytest.raises(snap.SnapError):  # not 256-byte aligned
        ctx.set_buffers([(0, 0, 128, 256, 0)])
    with pytest.raises(snap.SnapError):  # size not a multiple of 256
        ctx.set_buffers([(0, 0, 0, 300, 0)])
    with pytest.raises(snap.SnapError):  # beyond the arena
        ctx.set_buffers([(0, 0, 0, (64 << 20) + 256, 0)])
    with pytest.raises(snap.SnapError):  # bad geometry
        ctx.set_buffers([(0, 0, 0, 4096, 0)], 4096, 4096 * 64)
    with pytest.raises(snap.SnapError):  # select before hash
        ctx.set_buffers([(0, 0, 0, 4096, 0)])
        ctx.select()
    with pytest.raises(snap.SnapError):  # grad sum: no sources
        ctx.grad_sum(snap.F32, [], 0, 16)
    with pytest.raises(snap.SnapError):  # grad sum range beyond the arena
        ctx.grad_sum(snap.F32, [0], 0, 64 << 20)


def test_grad_sum_zero_and_odd_lengths(snap, ctx):
    for n in (0, 1, 3, 5, 1023):
        a = np.arange(n, dtype=np.float32) + 0.5
        b = np.arange(n, dtype=np.float32) * 2
        ctx.write(0, a if n else np.zeros(1, np.float32))
        ctx.write(1 << 20, b if n else np.zeros(1, np.float32))
        ctx.grad_sum(snap.F32, [0, 1 << 20], 2 << 20, n)
        if n:
            got = np.frombuffer(ctx.read(2 << 20, 4 * n).tobytes(), np.float32)
            assert np.array_equal(got, a + b)


def test_restore_missing_source_is_fault(snap, ctx):
    ctx.fill_mix64(0, 1 << 20, 1, 0)
    ctx.set_buffers([(0, 0, 0, 1 << 20, 0)])
    ctx.snapshot()
    ptr, cap = ctx.staging_ptr()
    # a source offset outside the image: SimFault (missing blob), nothing written
    with pytest.raises(snap.SnapFault):
        ctx.restore(ptr, 65536, [0] * 15 + [65536], verify=False)


def test_splice_rank_without_buffers(snap):
    with snap.Ctx(0, 16 << 20) as c:
        c.splice_init(8 << 20)
        c.splice_set_rank(0, [(0, 0, 0, 1 << 20, 0)])
        c.splice_set_rank(1, [])
        c.fill_mix64(0, 1 << 20, 3, 0)
        st = c.splice_switch(0, 1)
        assert st["hashed_bytes"] == 1 << 20 and st["swap_in_bytes"] == 0
        st = c.splice_switch(1, 0)
        assert st["hashed_bytes"] == 0


def test_no_digest_collisions_10k_buffers(snap):
    # test_simcore.cpp:119-130 on the device: 10^4 random distinct buffers, distinct digests
    rng = np.random.default_rng(7)
    n = 10000
    with snap.Ctx(0, n * 256) as c:
        words = rng.integers(0, 2**64 - 1, size=n * 32, dtype=np.uint64)
        c.write(0, words)
        bufs = [(0, i, i * 256, 256, 0) for i in range(n)]
        d = c.digest_ranges(bufs)
        assert len(set(d.tolist())) == n
        od = O.hash_chunks([words], bufs)[2]
        assert np.array_equal(d, od)
