"""Runs one hot-path operation repeatedly (for ncu captures of a single kernel class):
python tools/prof_one.py c1_restore|c1_snapshot|whole|select_small [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402

op = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
nbytes, nb = 256 << 20, 4 << 20
bufs = [(0, i, i * nb, nb, 0) for i in range(nbytes // nb)]
with snap.Ctx(0, nbytes) as c:
    c.fill_mix64(0, nbytes, 1, 0)
    c.set_buffers(bufs)
    c.snapshot()  # one fused K1 + small select
    for _ in range(reps):
        if op == "c1_restore":
            c.restore_self(verify=True)
        elif op in ("c1_snapshot", "select_small"):
            c.snapshot()
        elif op == "whole":
            c.digest_whole([(0, 0, 0, nbytes, 0)])
    c.sync()
print("done", op)
