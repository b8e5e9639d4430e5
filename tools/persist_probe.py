"""Phase timing of snap_persist / snap_load on this box (SNAP_PERSIST_TRACE=1 prints the
phases): C1-sized image, several writer-thread counts, fresh directory each time."""
import os
import shutil
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402

os.environ.setdefault("SNAP_PERSIST_TRACE", "1")
mib = int(sys.argv[1]) if len(sys.argv) > 1 else 256
nbytes = mib << 20
base = tempfile.mkdtemp(prefix="snap_probe_")
with snap.Ctx(0, nbytes + (1 << 20)) as c:
    c.fill_mix64(0, nbytes, 1, 0)
    c.set_buffers([(0, 0, 0, nbytes, 0)])
    c.snapshot()
    c.sync()
    for th in (1, 4, 8, 16, 32):
        d = os.path.join(base, f"t{th}")
        t = time.perf_counter()
        st = c.persist(d, threads=th)
        dt = time.perf_counter() - t
        print(f"persist threads={th:2d}: {dt * 1e3:8.1f} ms  {nbytes / dt / 1e9:6.2f} GB/s "
              f"files={st['written']}", flush=True)
    for th in (1, 8, 16):
        t = time.perf_counter()
        c.load(os.path.join(base, "t16"), threads=th)
        dt = time.perf_counter() - t
        print(f"load threads={th:2d}: {dt * 1e3:8.1f} ms  {nbytes / dt / 1e9:6.2f} GB/s", flush=True)
# raw python file creation for comparison
d = os.path.join(base, "py")
os.makedirs(d)
buf = os.urandom(65536)
t = time.perf_counter()
for i in range(nbytes // 65536):
    sub = os.path.join(d, f"{i & 255:02x}")
    os.makedirs(sub, exist_ok=True)
    with open(os.path.join(sub, f"{i:016x}"), "wb") as f:
        f.write(buf)
dt = time.perf_counter() - t
print(f"python single-thread create+write: {dt * 1e3:8.1f} ms  {nbytes / dt / 1e9:6.2f} GB/s")
shutil.rmtree(base, ignore_errors=True)
