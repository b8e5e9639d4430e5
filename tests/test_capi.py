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
