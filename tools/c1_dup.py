"""C1 duplicate-heavy variant (chunk c = chunk c mod 1024) snapshot time per K1 variant
(dev tool). python tools/c1_dup.py [variants...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402

nbytes, nb = 256 << 20, 4 << 20
bufs = [(0, i, i * nb, nb, 0) for i in range(nbytes // nb)]
for v in [int(x) for x in sys.argv[1:]] or [-1, 12]:
    snap.set_k1_variant(v)
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, nbytes // 4, 1, 0)
        head = c.read(0, nbytes // 4)
        for k in range(1, 4):
            c.write(k * nbytes // 4, head)
        c.set_buffers(bufs)
        for _ in range(3):
            c.snapshot()
        c.sync()
        c.timer_start()
        for _ in range(20):
            c.snapshot()
        ms = c.timer_stop() / 20
        print(v, os.environ.get("SNAP_MMA_FUSED_CW"), snap.last_k1_kernel()[:50], f"{ms * 1e3:.1f} us",
              c.selection()[3], flush=True)
