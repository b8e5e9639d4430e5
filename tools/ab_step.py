"""A/B of the C2 single-GPU snapshot step: per-kernel-class medians (CUDA events on the ctx
stream) over many steps. Run once per library build, alternating, on the same box:
  SNAP_LIB_PATH=... python tools/ab_step.py [steps]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402
from bench import c2_layout, fill_rank  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
bufs, rep, per = c2_layout()
image = rep + per
ctx = snap.Ctx(0, image + (64 << 20))
fill_rank(ctx, 0, rep, per)
if len(sys.argv) > 2 and sys.argv[2] == "regular":  # 512 x 4 MiB buffers, same image
    bufs = [(0, i, i * (4 << 20), 4 << 20, 0) for i in range(image // (4 << 20))]
ctx.set_buffers(bufs)
for _ in range(5):
    ctx.snapshot()
ctx.sync()
ctx.prof_enable(True)
tot = []
for _ in range(steps):
    ctx.timer_start()
    ctx.snapshot()
    tot.append(ctx.timer_stop())
res = {"lib": os.path.basename(snap.LIB_PATH), "step_ms": float(np.median(tot))}
for name, k in (("hash", snap.PROF_HASH), ("select", snap.PROF_SELECT),
                ("compact", snap.PROF_COMPACT)):
    ms, n = ctx.prof_read(k)
    res[name + "_ms"] = ms / max(n, 1)
print(json.dumps(res))
