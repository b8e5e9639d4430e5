"""Per-kernel timing of the snapshot path (dev tool; the contract bench is bench.py).

python tools/kbench.py [--gib 2] [--reps 10]
Times with CUDA events on the ctx stream (snap_timer_*), inputs > L2 (126 MB).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2202_07848_b200 as snap  # noqa: E402


def timeit(c, fn, reps):
    fn()
    c.sync()
    c.timer_start()
    for _ in range(reps):
        fn()
    return c.timer_stop() / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=2.0)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    nbytes = int(a.gib * (1 << 30)) // (1 << 20) * (1 << 20)
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, nbytes, 1, 0)
        nb = 4 << 20
        bufs = [(0, i, i * nb, nb, 0) for i in range(nbytes // nb)]
        for geom in [(4096, 65536), (65536, 65536)]:
            c.set_buffers(bufs, *geom)
            t = timeit(c, c.hash, a.reps)
            print(f"hash geom={geom}: {t:.3f} ms  {nbytes / t / 1e6:.1f} GB/s (read)")
        c.set_buffers(bufs)
        c.hash()
        t = timeit(c, c.select, a.reps)
        print(f"select ({c.nchunks} chunks): {t * 1e3:.1f} us")
        c.select()
        t = timeit(c, c.compact, a.reps)
        print(f"compact (all unique): {t:.3f} ms  {2 * nbytes / t / 1e6:.1f} GB/s (r+w)")
        t = timeit(c, c.snapshot, a.reps)
        print(f"snapshot hash+select+compact: {t:.3f} ms  R/t {nbytes / t / 1e6:.1f} GB/s  "
              f"(R+W)/t {2 * nbytes / t / 1e6:.1f} GB/s")
        t = timeit(c, lambda: c.restore_self(verify=False), a.reps)
        print(f"restore (scatter): {t:.3f} ms  {2 * nbytes / t / 1e6:.1f} GB/s (r+w)")
        n = nbytes // 4 // 6 // 16 * 16
        t = timeit(c, lambda: c.grad_sum(snap.F32, [0, n * 4, 2 * n * 4, 3 * n * 4], 4 * n * 4, n),
                   a.reps)
        print(f"grad_sum f32 x4 ({n} elems): {t:.3f} ms  {5 * n * 4 / t / 1e6:.1f} GB/s")
        print("launches", c.launches)


if __name__ == "__main__":
    main()
