"""ncu driver: hash-only K1 on one buffer shape of tools/hash_variants.py (c2 | c3 | c4)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv += [] if len(sys.argv) > 1 else ["c4"]
import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

shape = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if shape == "c2":
    bufs = [(0, i, i * (4 << 20), 4 << 20, 0) for i in range(512)]
elif shape == "c3":
    bufs, addr = [], 0
    for nparam in bench.gpt2_medium_params():
        nbytes = (nparam * 4 + 255) // 256 * 256
        bufs.append((0, len(bufs), addr, nbytes, 0))
        addr += nbytes
else:
    bufs = [(0, i, i * (256 << 20), 256 << 20, 1) for i in range(32)]
total = max(b[2] + b[3] for b in bufs)
with snap.Ctx(0, total + (1 << 20)) as c:
    c.fill_mix64(0, total, 3, 0)
    c.set_buffers(bufs)
    for _ in range(n):
        c.hash()
    c.sync()
print("ok", shape, total)
