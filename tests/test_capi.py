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
