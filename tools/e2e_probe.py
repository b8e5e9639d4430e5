"""Where does snapshot_host time go? (dev tool)"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import bench
import paper_2202_07848_b200 as snap

bufs, rep, per = bench.c2_layout()
image = rep + per
c = snap.Ctx(0, image + (16 << 20))
c.set_buffers(bufs)
hi = snap.PinnedHost(image)
hi.array[:] = bench.host_image(0, rep, per).view(np.uint8)
ho = snap.PinnedHost(image)
dig = np.zeros(c.nchunks, np.uint64)
pdig = snap.PinnedHost(c.nchunks * 8)
for i in range(3):
    t = time.perf_counter(); c.snapshot_host(hi.ptr, 0, image, ho.ptr, image, dig)
    print("snapshot_host", (time.perf_counter() - t) * 1e3, "ms")
t = time.perf_counter(); c._L.snap_write(c.h, 0, snap.C.c_void_p(hi.ptr), image); print("H2D only", (time.perf_counter() - t) * 1e3)
t = time.perf_counter(); c.snapshot(); c.sync(); print("device snapshot", (time.perf_counter() - t) * 1e3)
t = time.perf_counter(); c._L.snap_read_staging(c.h, 0, snap.C.c_void_p(ho.ptr), image); print("D2H only", (time.perf_counter() - t) * 1e3)
os.environ["X"] = "1"
