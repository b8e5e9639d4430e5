"""C1 snapshot / verified restore, device time per call without per-kernel events (dev tool)."""
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
    for _ in range(3):
        c.snapshot()
        c.restore_self(True)
    for name, fn in (("snapshot", c.snapshot), ("restore_verify", lambda: c.restore_self(True)),
                     ("restore_noverify", lambda: c.restore_self(False))):
        best = 9e9
        for _ in range(5):
            c.sync()
            c.timer_start()
            for _ in range(20):
                fn()
            best = min(best, c.timer_stop() / 20)
        print(f"{name:18s} {best * 1e3:8.1f} us  frac {2 * nbytes / best / 1e6 / 6558.4:.3f}",
              os.environ.get("SNAP_SELECT_SMALL", ""), flush=True)

with snap.Ctx(0, nbytes) as c:
    import time
    c.fill_mix64(0, nbytes, 0, 0)
    for bl in ([(0, 0, 0, nbytes, 0)], bufs):
        c.digest_whole(bl)
        t = time.perf_counter()
        d = c.digest_whole(bl)
        print(f"digest_whole {len(bl)} range(s): {(time.perf_counter() - t) * 1e3:.2f} ms",
              hex(int(d[0])))
