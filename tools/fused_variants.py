"""C2 single-GPU snapshot step per fused-K1 variant (dev tool):
python tools/fused_variants.py 7 14 16 17 [--steps 100]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402
from bench import c2_layout, fill_rank  # noqa: E402

vs = [int(x) for x in sys.argv[1:] if x.lstrip("-").isdigit()] or [-1]
bufs, rep, per = c2_layout()
image = rep + per
ctx = snap.Ctx(0, image + (64 << 20))
fill_rank(ctx, 0, rep, per)
for rnd in range(2):
    for v in vs:
        snap.set_k1_variant(v)
        ctx.set_buffers(bufs)
        for _ in range(5):
            ctx.snapshot()
        ctx.sync()
        ctx.prof_enable(True)
        tot = []
        for _ in range(60):
            ctx.timer_start()
            ctx.snapshot()
            tot.append(ctx.timer_stop())
        ms, n = ctx.prof_read(snap.PROF_HASH)
        ctx.prof_enable(False)
        k = ms / max(n, 1)
        print(json.dumps({"round": rnd, "variant": v, "k1": snap.last_k1_kernel(),
                          "step_ms": round(float(np.median(tot)), 4), "k1_ms": round(k, 4),
                          "k1_frac": round(2 * image / k / 1e6 / 6558.4, 4)}), flush=True)
snap.set_k1_variant(-1)
