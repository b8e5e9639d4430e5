"""C3 identical-replica splice switch time (dev tool)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

r = bench.splice_bench(snap, 0)
print(json.dumps({k: r[k] for k in ("swap_ms_identical", "digest_gbs", "swap_ms_divergent",
                                    "grad_sum_ms")}))
