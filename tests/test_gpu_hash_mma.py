"""GPU parity of the tensor-core K1 (k_hash_mma.cu: 8-bit FNV chain on the CUDA cores +
the linear part of FNV-1a as a tcgen05 int8 MMA) against the reference golden vectors and
the oracle, on the layouts that exercise its paths: TMA-box tasks, per-page bulk tasks
(buffer edges, ragged tails, pages shorter than 4 KiB), partial groups and chunk sizes
from 4 KiB to 128 KiB."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture()
def mma(snap):
    snap.set_k1_variant(11)
    yield snap
    snap.set_k1_variant(-1)


def test_c1_golden_mma(mma, c1_golden):
    with mma.Ctx(0, 256 << 20) as c:
        c.fill_mix64(0, 256 << 20, 0, 0)
        bufs = [(0, 0, 0, 256 << 20, 0)]
        assert c.set_buffers(bufs, 4096, 65536) == 4096
        c.hash()
        d, _, bd = c.digests(buf_digests=True)
        assert np.array_equal(d, c1_golden["merkle"])
        assert int(bd[0]) == int(c1_golden["buf"][0])


def test_ragged_golden_mma(mma, golden):
    rag = golden["ragged"]
    with mma.Ctx(0, 64 << 20) as c:
        arena = O.fill_mix64(rag["arena_bytes"] // 8, rag["seed"], 0)
        src, dst, n = rag["dup"]
        arena[dst // 8:(dst + n) // 8] = arena[src // 8:(src + n) // 8]
        c.write(0, arena)
        bufs = [tuple(b) for b in rag["bufs"]]
        c.set_buffers(bufs, 4096, 65536)
        c.hash()
        d, lens, bd = c.digests(buf_digests=True)
        exp = golden["ragged"]["4096_65536"]
        assert [f"{x:016x}" for x in d] == exp["chunks"]
        assert [f"{x:016x}" for x in bd] == exp["bufs"]


@pytest.mark.parametrize("chunk", [4096, 8192, 16384, 32768, 65536, 131072])
def test_random_layouts_mma(mma, chunk):
    rng = np.random.default_rng(chunk)
    arena_bytes = 96 << 20
    with mma.Ctx(0, arena_bytes) as c:
        for trial in range(3):
            c.fill_mix64(0, arena_bytes, 7 + trial, 0)
            host = c.read(0, arena_bytes)
            bufs, addr, slot = [], 0, 0
            while True:
                kind = rng.integers(0, 4)
                if kind == 0:
                    nb = int(rng.integers(1, 16)) * 256          # sub-page buffers
                elif kind == 1:
                    nb = int(rng.integers(1, 64)) * 4096 + int(rng.integers(0, 16)) * 256
                else:
                    nb = int(rng.integers(1, 700)) * 4096        # page-multiple, TMA tasks
                if addr + nb > arena_bytes:
                    break
                bufs.append((0, slot, addr, nb, int(rng.integers(0, 3))))
                slot += 1
                addr += nb + int(rng.integers(0, 3)) * 256
            c.set_buffers(bufs, 4096, chunk)
            c.hash()
            d, lens = c.digests()
            od, olens, _ = O.hash_chunks([host], bufs, 4096, chunk)
            assert np.array_equal(lens, olens)
            bad = np.nonzero(d != od)[0]
            assert bad.size == 0, f"trial {trial}: {bad.size} chunk digests differ, first {bad[:5]}"


def test_mma_equals_default_large(snap):
    """Same 1 GiB image (one 768 MiB buffer + 64 x 4 MiB): default kernel vs the MMA kernel."""
    nbytes = 1 << 30
    bufs = [(0, 0, 0, 768 << 20, 1)] + [(0, 1 + i, (768 << 20) + i * (4 << 20), 4 << 20, 0)
                                        for i in range(64)]
    out = []
    for v in (-1, 11):
        snap.set_k1_variant(v)
        with snap.Ctx(0, nbytes) as c:
            c.fill_mix64(0, nbytes, 99, 0)
            c.set_buffers(bufs)
            c.hash()
            out.append(c.digests()[0])
    snap.set_k1_variant(-1)
    assert np.array_equal(out[0], out[1])


def _snapshot_check(c, host, bufs):
    c.set_buffers(bufs)
    for rep in range(2):  # second pass: speculation from the previous layout
        c.snapshot()
        d, lens = c.digests()
        sel, owner, off, sbytes, _ = c.selection()
        od, olens, _ = O.hash_chunks([host], bufs)
        osel, oown, ooff, otot = O.select(od, olens)
        assert np.array_equal(d, od), f"pass {rep}: digests differ"
        assert np.array_equal(sel, osel) and np.array_equal(off, ooff) and sbytes == otot
        img = c.read_staging(0, sbytes)
        assert np.array_equal(img, O.compact([host], bufs, 65536, osel, ooff, otot)), \
            f"pass {rep}: staging image differs"


@pytest.mark.parametrize("variant", [11, 12, 13])
def test_fused_snapshot_mma(snap, variant):
    """Fused hash + speculative compaction on the tensor-core kernels (11: 128-B slabs,
    12: the light-write geometry used for striped multi-rank layouts): regular 4 MiB
    buffers, ragged buffers (tails, sub-page buffers), duplicated content (dedup moves
    offsets)."""
    snap.set_k1_variant(variant)
    rng = np.random.default_rng(11)
    nbytes = 160 << 20
    try:
        _fused_case(snap, rng, nbytes)
    finally:
        snap.set_k1_variant(-1)


def _fused_case(mma, rng, nbytes):
    with mma.Ctx(0, nbytes) as c:
        c.fill_mix64(0, nbytes, 21, 0)
        # duplicates: buffer 3 = buffer 1, buffer 7 = buffer 2
        c.write(3 * (4 << 20), c.read(1 * (4 << 20), 4 << 20))
        c.write(7 * (4 << 20), c.read(2 * (4 << 20), 4 << 20))
        host = c.read(0, nbytes)
        regular = [(0, i, i * (4 << 20), 4 << 20, i % 3) for i in range(16)]
        _snapshot_check(c, host, regular)
        bufs, addr, slot = [], 64 << 20, 0
        while True:
            nb = int(rng.integers(1, 900)) * 256 * (1 + 15 * int(rng.integers(0, 2)))
            if addr + nb > nbytes:
                break
            bufs.append((0, slot, addr, nb, int(rng.integers(0, 3))))
            slot += 1
            addr += nb + int(rng.integers(0, 2)) * 4096
        _snapshot_check(c, host, regular[:8] + bufs)


def test_scheduled_groups_mma(mma):
    """The balanced group schedule (mma_schedule: groups with buffer-tail tasks spread over
    the CTAs first, several groups per CTA): 1.5 GiB of buffers of random sizes (~390
    groups over 148 CTAs, heavy and regular groups interleaved) vs the oracle, twice (the
    schedule is built once per grid)."""
    rng = np.random.default_rng(2202)
    arena_bytes = 3 << 29
    with mma.Ctx(0, arena_bytes) as c:
        c.fill_mix64(0, arena_bytes, 31, 0)
        host = c.read(0, arena_bytes)
        bufs, addr, slot = [], 0, 0
        while True:
            nb = int(rng.integers(1, 6 << 20) // 256 + 1) * 256
            if addr + nb > arena_bytes:
                break
            bufs.append((0, slot, addr, nb, 0))
            slot += 1
            addr += nb
        c.set_buffers(bufs)
        od, olens, _ = O.hash_chunks([host], bufs)
        for rep in range(2):
            c.hash()
            d, lens = c.digests()
            assert np.array_equal(lens, olens)
            bad = np.nonzero(d != od)[0]
            assert bad.size == 0, f"rep {rep}: {bad.size} chunk digests differ, first {bad[:5]}"


@pytest.mark.parametrize("cw", ["8", "12"])
def test_mma_other_geometries_whole_suite(cw):
    """The default tensor-core geometry is 16 chain warps x 1 pair (hash-only and fused);
    the 8 x 2 (round-1) and 12 x 2 geometries stay selectable for A/B runs. Every layout
    of this file through them, forced in a child process (read once per process)."""
    import os
    import subprocess
    import sys
    if os.environ.get("SNAP_MMA_CW"):
        pytest.skip("already a forced run")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", __file__, "-k",
                        "not other_geometries"],
                       env=dict(os.environ, SNAP_MMA_CW=cw, SNAP_MMA_FUSED_CW="8"),
                       capture_output=True, text=True, timeout=600, cwd=root)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0


def test_mma_large_grid(snap):
    nbytes = 4 << 30  # 1 M pages, 1024 groups
    bufs = [(0, i, i * (32 << 20), 32 << 20, i % 2) for i in range(nbytes // (32 << 20))]
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, nbytes, 1234, 0)
        c.set_buffers(bufs)
        c.hash()
        d, _ = c.digests()
        host = c.read(0, 64 << 20)
    assert snap.last_k1_kernel().startswith("k_hash_mma")
    od, _, _ = O.hash_chunks([host], bufs[:2])
    assert np.array_equal(d[:od.size], od)
