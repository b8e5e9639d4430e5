"""C3 splice section of bench.py alone (switch ms for identical / divergent replicas, K5 GB/s)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

r = bench.splice_bench(snap, 0)
print(json.dumps({"swap_ms_identical": r["swap_ms_identical"], "digest_gbs": r["digest_gbs"],
                  "divergent": {k: v["swap_ms"] for k, v in r["swap_ms_divergent"].items()},
                  "grad_sum_gbs": r["grad_sum_gbs"]}))
