"""Fused K1 on one GPU with the staging layout rank 0 of an N-rank job writes
(SNAP_SPEC_STRIPE=N re-predicted every snapshot; the K3 fix-up copies the rest), per K1 variant."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402
from bench import c2_layout, fill_rank  # noqa: E402

bufs, rep, per = c2_layout()
ctx = snap.Ctx(0, rep + per + (64 << 20))
fill_rank(ctx, 0, rep, per)
if len(sys.argv) > 1 and sys.argv[1] == "regular":  # 512 x 4 MiB, all replicated
    bufs = [(0, i, i * (4 << 20), 4 << 20, 0) for i in range((rep + per) // (4 << 20))]
ctx.set_buffers(bufs)
for _ in range(3):
    ctx.snapshot()
ctx.sync()
ctx.prof_enable(True)
for _ in range(30):
    ctx.snapshot()
ms, n = ctx.prof_read(snap.PROF_HASH)
print(json.dumps({"stripe": os.environ.get("SNAP_SPEC_STRIPE"), "variant": os.environ.get("SNAP_HASH_VARIANT"),
                  "k1_ms": round(ms / max(n, 1), 4)}))
