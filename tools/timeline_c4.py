"""GPU timeline of a C4 incremental snapshot (dev tool): 32 GiB, 5 % dirty chunks,
every kernel / copy with the idle gap before it (CUPTI via torch.profiler)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

gib = int(sys.argv[1]) if len(sys.argv) > 1 else 32
nbytes, nb = gib << 30, 256 << 20
bufs = [(0, i, i * nb, nb, 1) for i in range(nbytes // nb)]
torch.cuda.init()
with snap.Ctx(0, nbytes + (1 << 20)) as c:
    c.fill_mix64(0, nbytes, 99, 0)
    n = c.set_buffers(bufs)
    c.snapshot()
    c.known_commit()
    mix = bench.mix64_np(np.uint64(99) ^ np.arange(n, dtype=np.uint64))
    dirty = np.nonzero(mix % np.uint64(20) == 0)[0].astype(np.uint64) * 65536
    c.xor_words(dirty, 0x1234567)
    c.snapshot()
    c.known_commit()
    c.xor_words(dirty, 0x7654321)
    c.sync()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        c.snapshot()
        c.sync()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
prev_end = None
t0 = evs[0].time_range.start
for e in evs:
    s, t = e.time_range.start, e.time_range.end
    gap = "" if prev_end is None else f"gap {s - prev_end:7.2f}"
    print(f"{s - t0:10.2f} {t - s:9.2f} us {gap:14s} {e.name[:90]}")
    prev_end = t if prev_end is None else max(prev_end, t)
