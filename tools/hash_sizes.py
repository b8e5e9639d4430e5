"""Hash-only K1 GB/s vs image size (one layout of 4 MiB buffers), for the kernel policy."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402

out = {"variant": os.environ.get("SNAP_HASH_VARIANT", "default")}
with snap.Ctx(0, (4 << 30) + (1 << 20)) as c:
    c.fill_mix64(0, 4 << 30, 5, 0)
    for mib in (16, 64, 128, 256, 384, 512, 1024, 4096):
        nb = 4 << 20
        bufs = [(0, i, i * nb, nb, 0) for i in range(mib // 4)]
        c.set_buffers(bufs)
        c.hash()
        c.sync()
        reps = max(3, 2048 // mib)
        c.timer_start()
        for _ in range(reps):
            c.hash()
        ms = c.timer_stop() / reps
        out[f"{mib}MiB"] = round(mib * 1048576 / ms / 1e6, 1)
print(json.dumps(out))
