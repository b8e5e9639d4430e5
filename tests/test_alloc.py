"""CPU parity of the device-proxy memory tracker (host metadata, no GPU): the C++ tracker
behind snap_alloc_* vs the reference's mem::BidiAllocator (oracle/_ref) on random op
sequences, the reference-generated golden op script, and the reference's own unit tests
(proj/tests/test_alloc.cpp) restated."""
import ctypes as C

import numpy as np
import pytest

import oracle as O


def ref_alloc(R, a, nbytes, stable):
    out = C.c_uint64()
    rc = R.ref_alloc_alloc(a, nbytes, 1 if stable else 0, C.byref(out))
    return None if rc == 1 else ("fault" if rc == -1 else out.value)


def test_golden_script(snap, golden):
    A = snap.BidiAllocator(0, 1 << 20)
    for op in golden["alloc"]["ops"]:
        if op[0] == "free":
            _, addr, rc = op
            if rc == 0:
                A.free(addr)
            else:
                with pytest.raises(snap.SnapFault):
                    A.free(addr)
        else:
            _, nb, st, rc, addr = op
            got = A.alloc(nb, bool(st))
            assert got == (addr if rc == 0 else None)
    assert f"{A.stable_state_digest():016x}" == golden["alloc"]["stable_digest"]
    assert list(A.cursors()) == golden["alloc"]["cursors"]


@pytest.mark.parametrize("seed", range(6))
def test_random_vs_reference(snap, seed):
    R = O.ref()
    if R is None:
        pytest.skip("reference library not built here")
    rng = np.random.default_rng(seed)
    region = 1 << 22
    a = R.ref_alloc_new(0, region)
    A = snap.BidiAllocator(0, region)
    live = []
    for _ in range(2000):
        r = rng.random()
        if live and r < 0.45:
            x = live.pop(int(rng.integers(len(live))))
            assert R.ref_alloc_free(a, x) == 0
            A.free(x)
        elif r < 0.47:  # unknown / double free faults on both sides
            bad = int(rng.integers(region)) | 1
            assert R.ref_alloc_free(a, bad) == -1
            with pytest.raises(snap.SnapFault):
                A.free(bad)
        else:
            st = bool(rng.random() < 0.5)
            nb = int(rng.integers(1, 70000)) if rng.random() < 0.9 else int(rng.integers(1, 600000))
            ra = ref_alloc(R, a, nb, st)
            assert A.alloc(nb, st) == ra
            if ra is not None:
                live.append(ra)
        tc, sc, lb = C.c_uint64(), C.c_uint64(), C.c_uint64()
        R.ref_alloc_cursors(a, C.byref(tc), C.byref(sc), C.byref(lb))
        assert A.cursors() == (tc.value, sc.value, lb.value)
    assert A.stable_state_digest() == R.ref_alloc_stable_digest(a)
    R.ref_alloc_free_obj(a)


def test_reference_unit_cases(snap):
    # test_alloc.cpp:9-21 top-down stable / bottom-up transient, 256-B rounding
    A = snap.BidiAllocator(0, 1 << 20)
    assert A.alloc(1000, True) == (1 << 20) - 1024
    assert A.alloc(1, False) == 0 and A.alloc(1, False) == 256
    # :33-42 OOM when the cursors would cross
    B = snap.BidiAllocator(0, 4096)
    assert B.alloc(2048, True) == 2048 and B.alloc(2048, False) == 0
    assert B.alloc(256, True) is None and B.alloc(256, False) is None
    # :82-104 stable coalescing + cursor retreat; transient first-fit gap reuse
    C1 = snap.BidiAllocator(0, 1 << 20)
    s1, s2 = C1.alloc(4096, True), C1.alloc(4096, True)
    C1.free(s2)
    C1.free(s1)
    assert C1.alloc(8192, True) == (1 << 20) - 8192
    D = snap.BidiAllocator(0, 1 << 20)
    t1, t2, t3 = D.alloc(4096, False), D.alloc(4096, False), D.alloc(4096, False)
    D.free(t2)
    assert D.alloc(2048, False) == t2
    # :106-113 faults
    E = snap.BidiAllocator(0, 1 << 20)
    t = E.alloc(1024, False)
    E.free(t)
    with pytest.raises(snap.SnapFault):
        E.free(t)
    with pytest.raises(snap.SnapFault):
        E.alloc(0, True)


def test_identical_stable_addresses_across_replicas(snap):
    # test_alloc.cpp:44-80: stable layout is a pure function of the stable sequence
    def replica(seed):
        rng = np.random.default_rng(seed)
        A = snap.BidiAllocator(0, 1 << 20)
        stable, trans = [], []
        for step in range(40):
            if step % 4 == 0:
                stable.append(A.alloc(1024 + (step // 4) * 256, True))
            for _ in range(1 + int(rng.integers(3))):
                trans.append(A.alloc(256 + int(rng.integers(8192)), False))
            while len(trans) > 4:
                A.free(trans.pop(int(rng.integers(len(trans)))))
        return stable, A.stable_state_digest()

    a, da = replica(11)
    b, db = replica(999)
    assert a == b and da == db


def test_snapshot_round_trip(snap):
    # test_alloc.cpp:115-144
    rng = np.random.default_rng(3)
    A = snap.BidiAllocator(0, 1 << 20)
    live = []
    for _ in range(60):
        if live and rng.integers(3) == 0:
            A.free(live.pop(int(rng.integers(len(live)))))
        else:
            live.append(A.alloc(256 + int(rng.integers(4096)), bool(rng.integers(2))))
    B = snap.BidiAllocator(0, 1 << 20)
    B.restore(A.snapshot())
    for i in range(20):
        assert A.alloc(512 + i * 256, bool(i % 2)) == B.alloc(512 + i * 256, bool(i % 2))
    assert A.stable_state_digest() == B.stable_state_digest()
