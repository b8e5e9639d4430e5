"""Hash-only tensor-core K1 GB/s on 1 GiB images whose buffers end mid-task: 4 MiB buffers
(every task 32 full contiguous pages), 4 MiB - 4 KiB (the last task's second chunk is
partial), 4 MiB - 68 KiB (the last task holds a partial chunk followed by the next buffer's
first chunk), and the C3 GPT-2-medium P/m/v layout. SNAP_LIB_PATH selects the library (A/B)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

out = {"lib": os.environ.get("SNAP_LIB_PATH", "in-tree")}
stable, sbytes, _, _ = bench.c3_layout()
with snap.Ctx(0, max(sbytes, 1 << 30) + (8 << 20)) as c:
    c.fill_mix64(0, max(sbytes, 1 << 30), 5, 0)
    layouts = {}
    for name, nb in (("4MiB", 4 << 20), ("4MiB-4KiB", (4 << 20) - 4096),
                     ("4MiB-68KiB", (4 << 20) - (68 << 10))):
        n = (1 << 30) // (4 << 20)
        layouts[name] = ([(0, i, i * nb, nb, 0) for i in range(n)], n * nb)
    layouts["C3"] = ([b[:5] for b in stable], sbytes)
    for name, (bufs, nbytes) in layouts.items():
        c.set_buffers(bufs)
        c.hash()
        c.sync()
        reps = 20
        c.timer_start()
        for _ in range(reps):
            c.hash()
        ms = c.timer_stop() / reps
        out[name] = round(nbytes / ms / 1e6, 1)
print(json.dumps(out))
