"""CPU tests of the C-ABI boundary: the library loads, exports every symbol
include/snap.h declares, host-only entry points match the reference, and compute
entry points fail loudly (no CPU fallback) when no GPU is present."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "snap.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(snap_[a-z_0-9]+)\(", src,
                                 re.M)))


def test_header_symbols_exported(snap):
    import ctypes as C
    L = C.CDLL(snap.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/snap.h but not exported"
    # the Python binding covers every declared entry point
    assert set(syms) == set(snap.exported_symbols())


def test_layout_carve_matches_reference(snap, golden):
    # splice::DeviceLayout::carve (splice.cpp:7-19), golden from the reference library
    for case in golden["carve"]:
        if case["rc"] == 0:
            assert list(snap.layout_carve(case["mem"], case["max_buf"], case["slack"])) == case["out"]
        else:
            with pytest.raises(snap.SnapError):
                snap.layout_carve(case["mem"], case["max_buf"], case["slack"])


def test_no_gpu_fails_loudly(snap):
    import torch  # noqa: F401  (only to ask whether a GPU exists)
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(snap.SnapError):
        snap.Ctx(0, 1 << 20)


def test_strerror(snap):
    L = snap.lib()
    assert L.snap_strerror(snap.SNAP_EFAULT) == b"fault (content/digest)"
    assert L.snap_strerror(0) == b"ok"


def test_blob_rel_path_matches_reference(snap, oracle_mod, ref_lib):
    # BlobStore::blob_rel_path (ckpt.cpp:35-40): product, oracle and the reference agree
    import ctypes as C
    import numpy as np
    rng = np.random.default_rng(5)
    ds = [0, 1, 0xff, 0xcbf29ce484222325, 2**64 - 1] + [int(x) for x in
                                                          rng.integers(0, 2**63, 200)]
    for d in ds:
        b = C.create_string_buffer(64)
        assert ref_lib.ref_blob_rel_path(C.c_uint64(d), b, 64) == 0
        assert snap.blob_rel_path(d) == b.value.decode() == oracle_mod.blob_rel_path(d)


def test_persisted_tree_oracle_matches_reference_store(oracle_mod, ref_lib, tmp_path):
    # the oracle's expected directory == what the reference BlobStore::persist writes
    import ctypes as C
    import numpy as np
    st = ref_lib.ref_store_new()
    try:
        blobs = {}
        for i in range(40):
            w = oracle_mod.fill_mix64(512 * (1 + i % 3), seed=11, base=i << 20)
            d = C.c_uint64()
            ref_lib.ref_store_put(st, w.ctypes.data_as(C.c_void_p), w.size, C.byref(d))
            assert d.value == oracle_mod.digest_of_words(w)
            blobs[d.value] = w.tobytes()
        assert ref_lib.ref_store_persist(st, str(tmp_path).encode()) == 0
    finally:
        ref_lib.ref_store_free(st)
    got = {str(p.relative_to(tmp_path)): p.read_bytes() for p in tmp_path.rglob("*") if p.is_file()}
    assert got == oracle_mod.persisted_tree(blobs)


def _ref_validate(ref_lib, records):
    import ctypes as C
    import numpy as np
    ranks = np.array(list(records), np.int32)
    nmut = np.array([len(m) for m, _ in records.values()], np.uint64)
    nd2h = np.array([len(d) for _, d in records.values()], np.uint64)
    muts = np.array([v for m, _ in records.values() for t in m for v in t] or [0], np.uint64)
    d2h = np.array([v for _, d in records.values() for t in d for v in t] or [0], np.uint64)
    reason = C.create_string_buffer(512)
    p = [a.ctypes.data_as(C.c_void_p) for a in (ranks, nmut, muts, nd2h, d2h)]
    ok = ref_lib.ref_validate_window(len(records), *p, reason, 512)
    return ok == 1, reason.value.decode()


def test_validate_window_matches_reference(snap, ref_lib):
    # splice::validate_window (splice.cpp:21-61): pass/fail and the exact reason text
    import numpy as np
    rng = np.random.default_rng(17)
    for trial in range(400):
        nr = int(rng.integers(1, 5))
        base_m = sorted({int(rng.integers(0, 64)) * 256 for _ in range(int(rng.integers(0, 6)))})
        muts = [(a, int(rng.integers(1, 4)) * 256, int(rng.integers(0, 2**63))) for a in base_m]
        d2h = [(int(rng.integers(1, 4)) * 8, int(rng.integers(0, 2**63)))
               for _ in range(int(rng.integers(0, 3)))]
        recs = {}
        for r in rng.permutation(8)[:nr]:
            m, d = [list(x) for x in muts], list(d2h)
            kind = int(rng.integers(0, 7)) if trial % 3 else 0
            if kind == 1 and m:
                m.pop(int(rng.integers(0, len(m))))
            elif kind == 2 and m:
                i = int(rng.integers(0, len(m)))
                m[i][0] += 1 << 20
                m.sort()
            elif kind == 3 and m:
                m[int(rng.integers(0, len(m)))][1] += 256
            elif kind == 4 and m:
                m[int(rng.integers(0, len(m)))][2] ^= 1
            elif kind == 5:
                d = d + [(8, 1)]
            elif kind == 6 and d:
                d[0] = (d[0][0], d[0][1] ^ 2)
            recs[int(r)] = ([tuple(x) for x in m], d)
        assert snap.validate_window(recs) == _ref_validate(ref_lib, recs), (trial, recs)
