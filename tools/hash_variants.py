"""Hash-only K1 throughput per SNAP_HASH_VARIANT on three buffer shapes (C2 4 MiB buffers,
C3 GPT-2-medium tensors, C4 256 MiB buffers); run once per variant, alternating."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402


def layouts():
    nb = 4 << 20
    yield "c2_4MiB_x512", [(0, i, i * nb, nb, 0) for i in range(512)]
    bufs, addr = [], 0
    for n in bench.gpt2_medium_params():
        nbytes = (n * 4 + 255) // 256 * 256
        bufs.append((0, len(bufs), addr, nbytes, 0))
        addr += nbytes
    yield "c3_gpt2m_fp32_P", bufs
    nb = 256 << 20
    yield "c4_256MiB_x32", [(0, i, i * nb, nb, 1) for i in range(32)]


out = {"variant": os.environ.get("SNAP_HASH_VARIANT", "default")}
with snap.Ctx(0, (8 << 30) + (1 << 20)) as c:
    c.fill_mix64(0, 8 << 30, 3, 0)
    for name, bufs in layouts():
        c.set_buffers(bufs)
        nbytes = sum(b[3] for b in bufs)
        c.hash()
        c.sync()
        c.timer_start()
        for _ in range(10):
            c.hash()
        ms = c.timer_stop() / 10
        out[name] = round(nbytes / ms / 1e6, 1)
print(json.dumps(out))
