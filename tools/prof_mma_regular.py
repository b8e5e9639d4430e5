"""ncu driver: hash-only tensor-core K1 on a regular layout of the C3 size (1016 groups)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402

nbytes = 4257878016 // (4 << 20) * (4 << 20)
with snap.Ctx(0, nbytes + (1 << 20)) as c:
    c.fill_mix64(0, nbytes, 5, 0)
    c.set_buffers([(0, i, i * (4 << 20), 4 << 20, 0) for i in range(nbytes // (4 << 20))])
    for _ in range(4):
        c.hash()
    c.sync()
print("ok")
