"""Fixed-order allreduce timing under torchrun (dev tool): S sliced ranks per GPU of
GPT-2-medium fp32 gradients; prints strict / hierarchical / NCCL ms from rank 0."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

dist = bench.Dist()
r = bench.grad_allreduce_bench(snap, dist, S=int(os.environ.get("AR_S", "2")))
if dist.rank == 0:
    print(json.dumps({"ctas": os.environ.get("SNAP_AR_CTAS", "4"),
                      "unroll": os.environ.get("SNAP_AR_UNROLL", "1"),
                      **{k: (v["ms"], v["link_frac"]) for k, v in r.items() if isinstance(v, dict)}}))
dist.close()
