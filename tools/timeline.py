"""GPU timeline of C1 snapshot / verified-restore calls (dev tool): every kernel and
memcpy/memset the library issues, from CUPTI via torch.profiler, with the idle gap
before each. python tools/timeline.py [snapshot|restore] [calls]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2202_07848_b200 as snap  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "snapshot"
    calls = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    nbytes, nb = 256 << 20, 4 << 20
    bufs = [(0, i, i * nb, nb, 0) for i in range(nbytes // nb)]
    torch.cuda.init()
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, nbytes, 1, 0)
        c.set_buffers(bufs)
        def split():
            c.hash()
            c.sync()
            c.select()
            c.sync()
            c.compact()
            c.sync()
        fn = {"snapshot": c.snapshot, "restore": lambda: c.restore_self(True),
              "split": split}[what]
        for _ in range(3):
            c.snapshot()
            c.restore_self(True)
        c.sync()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(calls):
                fn()
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
