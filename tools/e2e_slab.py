"""e2e (snap_snapshot_host) time of the C2 image for the slab size in SNAP_HOST_SLAB_MB."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

bufs, rep, per = bench.c2_layout()
image = rep + per
c = snap.Ctx(0, image + (16 << 20))
c.set_buffers(bufs)
hi = snap.PinnedHost(image)
hi.array[:] = bench.host_image(0, rep, per).view(np.uint8)
ho = snap.PinnedHost(image)
dig = np.zeros(c.nchunks, np.uint64)
ts = []
for i in range(12):
    t = time.perf_counter()
    c.snapshot_host(hi.ptr, 0, image, ho.ptr, image, dig)
    ts.append(time.perf_counter() - t)
ms = float(np.median(ts[2:])) * 1e3
print(json.dumps({"slab_mb": os.environ.get("SNAP_HOST_SLAB_MB", "64"), "ms": round(ms, 2),
                  "e2e_gbs": round(image / ms / 1e6, 2)}))
