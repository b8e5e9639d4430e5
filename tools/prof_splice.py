"""ncu driver: C3 identical-replica splice switches (GPT-2-medium fp32 P/m/v, 4 ranks)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

nranks = 4
stable, sbytes, sizes, gbytes = bench.c3_layout()
gregion = sbytes
with snap.Ctx(0, sbytes + (nranks + 1) * gbytes + (1 << 20)) as c:
    c.splice_init(3 * sbytes)
    goffs = np.cumsum([0] + sizes[:-1]).tolist()
    for r in range(nranks):
        g = [(0, 10000 + i, gregion + r * gbytes + off, sz, 2, snap.BUF_PENDING)
             for i, (off, sz) in enumerate(zip(goffs, sizes))]
        c.splice_set_rank(r, stable + g)
    c.fill_mix64(0, sbytes, 5, 0)
    for r in range(nranks):
        c.splice_switch(r, (r + 1) % nranks)
    for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
        c.splice_switch(k % nranks, (k + 1) % nranks)
    c.sync()
print("ok")
