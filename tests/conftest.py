import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def c1_golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "c1_digests.npz"))


@pytest.fixture(scope="session")
def snap():
    import paper_2202_07848_b200 as snap
    snap.lib()  # loud failure if the extension was not built
    return snap


@pytest.fixture()
def ctx(snap):
    c = snap.Ctx(0, 64 << 20)
    yield c
    c.close()


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    return oracle


@pytest.fixture(scope="session")
def ref_lib(oracle_mod):
    R = oracle_mod.ref()
    if R is None:
        pytest.skip("reference library (oracle/_ref) not built here")
    return R
