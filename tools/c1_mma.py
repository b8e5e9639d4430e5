"""C1 snapshot with the tensor-core fused K1 forced (dev tool; SNAP_HASH_VARIANT=12)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402

nbytes, nb = 256 << 20, 4 << 20
bufs = [(0, i, i * nb, nb, 0) for i in range(nbytes // nb)]
with snap.Ctx(0, nbytes) as c:
    c.fill_mix64(0, nbytes, 1, 0)
    c.set_buffers(bufs)
    for name, fn in (("snapshot", c.snapshot), ("hash", c.hash)):
        for _ in range(3):
            fn()
        c.sync()
        c.prof_enable(True)
        c.timer_start()
        for _ in range(20):
            fn()
        ms = c.timer_stop() / 20
        t, n = c.prof_read(snap.PROF_HASH)
        c.prof_enable(False)
        print(name, snap.last_k1_kernel()[:40], f"{ms * 1e3:.1f} us/call, K1 {t / max(n, 1) * 1e3:.1f} us",
              os.environ.get("SNAP_MMA_CW"), os.environ.get("SNAP_MMA_FUSED_CW"), flush=True)
