"""Small driver for ncu: C2 rank image (2 GiB), N snapshots (fused hash+compaction)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
pure = len(sys.argv) > 2 and sys.argv[2] == "hash"
bufs, rep, per = bench.c2_layout()
c = snap.Ctx(0, rep + per + (16 << 20))
bench.fill_rank(c, 0, rep, per)
c.set_buffers(bufs, 4096, 65536)
for _ in range(n):
    if pure:
        c.hash()
    else:
        c.snapshot()
c.sync()
print("ok", c.launches)
