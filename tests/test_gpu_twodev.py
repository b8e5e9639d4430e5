"""Two GPUs driven from one process (one ctx each, the API's ownership model): every K1 kernel
(incl. the tensor-core ones, whose shared-memory attribute and weight table are per device)
hashes identically on both devices. Skips with fewer than 2 GPUs."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _ngpus(snap):
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("variant", [-1, 9, 10, 11])
def test_two_devices_one_process(snap, variant):
    if _ngpus(snap) < 2:
        pytest.skip("needs 2 GPUs")
    snap.set_k1_variant(variant)
    try:
        nbytes = 640 << 20  # >= 512 MiB: the default policy picks the tensor-core kernel
        bufs = [(0, i, i * (5 << 20), 5 << 20, i % 3) for i in range(128)]
        out = []
        ctxs = [snap.Ctx(d, nbytes) for d in (0, 1)]
        try:
            for c in ctxs:
                c.fill_mix64(0, nbytes, 31, 0)
                c.set_buffers(bufs)
            for c in ctxs:  # interleaved: each launch must find its own device's setup
                c.hash()
            for c in ctxs:
                out.append(c.digests()[0])
            host = ctxs[0].read(0, nbytes)
        finally:
            for c in ctxs:
                c.close()
        od, _, _ = O.hash_chunks([host], bufs)
        assert np.array_equal(out[0], od) and np.array_equal(out[1], od)
    finally:
        snap.set_k1_variant(-1)
