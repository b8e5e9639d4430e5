"""GPU timeline of C3 identical-replica splice switches (dev tool): every kernel and
copy of snap_splice_switch with the idle gap before it (CUPTI via torch.profiler)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402


def main():
    nranks = 4
    stable, sbytes, sizes, gbytes = bench.c3_layout()
    gregion = sbytes
    arena = sbytes + (nranks + 1) * gbytes + (1 << 20)
    torch.cuda.init()
    with snap.Ctx(0, arena) as c:
        c.splice_init(3 * sbytes)
        goffs = np.cumsum([0] + sizes[:-1]).tolist()
        for r in range(nranks):
            g = [(0, 10000 + i, gregion + r * gbytes + off, sz, 2, snap.BUF_PENDING)
                 for i, (off, sz) in enumerate(zip(goffs, sizes))]
            c.splice_set_rank(r, stable + g)
            c.fill_mix64(gregion + r * gbytes, gbytes, 77 + r, 0)
        c.fill_mix64(0, sbytes, 5, 0)
        for r in range(2 * nranks):
            c.splice_switch(r % nranks, (r + 1) % nranks)
        c.sync()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for r in range(3):
                c.splice_switch(r % nranks, (r + 1) % nranks)
            c.sync()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    prev_end = None
    for e in evs:
        s, t = e.time_range.start, e.time_range.end
        gap = "" if prev_end is None else f"gap {s - prev_end:7.2f}"
        print(f"{s:14.2f} {t - s:8.2f} us {gap:14s} {e.name[:90]}")
        prev_end = t if prev_end is None else max(prev_end, t)


if __name__ == "__main__":
    main()
