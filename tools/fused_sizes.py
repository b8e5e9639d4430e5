"""Fused K1 (hash + speculative stores) time vs image size in units of 'tasks per warp' of the
CfgE geometry (148 SMs x 12 warps, 128 KiB per task): shows the last-wave quantization."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402

warps = 148 * 12
out = {}
with snap.Ctx(0, (3 << 30) + (1 << 20)) as c:
    c.fill_mix64(0, 3 << 30, 9, 0)
    for tpw in (8.0, 8.5, 9.0, 9.25, 9.5, 10.0):
        ntask = int(round(tpw * warps))
        nb = ntask * (128 << 10)
        bufs = [(0, i, i * (128 << 10), 128 << 10, 0) for i in range(ntask)]
        c.set_buffers(bufs)
        for _ in range(3):
            c.snapshot()
        c.sync()
        c.prof_enable(True)
        for _ in range(20):
            c.snapshot()
        ms, n = c.prof_read(snap.PROF_HASH)
        c.prof_enable(False)
        k1 = ms / max(n, 1)
        out[str(tpw)] = {"k1_ms": round(k1, 4), "rw_tbs": round(2 * nb / k1 / 1e9, 3)}
print(json.dumps(out))
