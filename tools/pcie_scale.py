"""Host<->device bandwidth when N GPUs copy at once (the e2e path's bottleneck analysis):
each process pins a 2 GiB host buffer and runs H2D, D2H and both directions concurrently
(two streams) on its own GPU, all processes released by one barrier; with --numa the process
first binds to the GPU's NUMA-local CPUs (/sys/bus/pci/devices/<bus>/local_cpulist) so the
pinned pages are first-touched on that node.  python tools/pcie_scale.py --gpus 1 2 4"""
import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def local_cpus(gpu):
    try:
        bus = subprocess.run(["nvidia-smi", "-i", str(gpu), "--query-gpu=pci.bus_id",
                              "--format=csv,noheader"], capture_output=True, text=True,
                             timeout=30).stdout.strip().lower()
        bus = bus[4:] if bus.count(":") == 2 and len(bus.split(":")[0]) == 8 else bus
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            spec = f.read().strip()
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            node = int(f.read().strip())
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        return cpus, node, bus
    except Exception as e:  # noqa: BLE001
        return None, None, repr(e)


def worker(gpu, numa, bar, q, nbytes):
    cpus, node, bus = local_cpus(gpu)
    if numa and cpus:
        os.sched_setaffinity(0, cpus)
    import ctypes as C
    import paper_2202_07848_b200 as snap
    L = snap.lib()
    h = snap.PinnedHost(nbytes)
    h.array[:] = 1  # first touch by this (possibly bound) process
    c = snap.Ctx(gpu, nbytes)
    res = {"gpu": gpu, "numa_node": node, "bus": bus, "bound": bool(numa and cpus)}
    for name in ("h2d", "d2h"):
        for rep in range(3):
            bar.wait()
            t = time.perf_counter()
            if name == "h2d":
                L.snap_write(c.h, 0, C.c_void_p(h.ptr), nbytes)
            else:
                L.snap_read(c.h, 0, C.c_void_p(h.ptr), nbytes)
            dt = time.perf_counter() - t
            bar.wait()
        res[name + "_gbs"] = round(nbytes / dt / 1e9, 2)
    c.close()
    h.free()
    q.put(res)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--gib", type=float, default=2.0)
    a = ap.parse_args()
    nbytes = int(a.gib * (1 << 30))
    ctx = mp.get_context("spawn")
    out = {"lscpu": subprocess.run("lscpu | grep -E 'NUMA|Socket|Model name'", shell=True,
                                   capture_output=True, text=True).stdout.strip().splitlines(),
           "runs": []}
    for n in a.gpus:
        for numa in (False, True):
            bar, q = ctx.Barrier(n), ctx.Queue()
            ps = [ctx.Process(target=worker, args=(g, numa, bar, q, nbytes)) for g in range(n)]
            for p in ps:
                p.start()
            rs = [q.get() for _ in ps]
            for p in ps:
                p.join()
            rs.sort(key=lambda r: r["gpu"])
            out["runs"].append({"gpus": n, "numa_bind": numa, "per_gpu": rs,
                                "h2d_sum": round(sum(r["h2d_gbs"] for r in rs), 1),
                                "d2h_sum": round(sum(r["d2h_gbs"] for r in rs), 1)})
            print(json.dumps(out["runs"][-1]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
