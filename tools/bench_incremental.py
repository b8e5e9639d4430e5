"""C4 measurement: incremental checkpoint, 5 % dirty chunks, 32 GiB per GPU (independent per
GPU; run plain for N=1 or under torchrun for N GPUs). A first full snapshot is committed to
the store index (known set); then 5 % of the chunks are dirtied (chunk c dirty iff
mix64(seed ^ c) % 20 == 0, first word xor-ed) and the incremental snapshot (K1 hash of all
32 GiB + K2 select against the store + K3 gather of the dirty chunks) is timed.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402


def main():
    gib = float(os.environ.get("C4_GIB", "32"))
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    nbytes = int(gib * (1 << 30))
    nb = 256 << 20  # 128 buffers of 256 MiB
    bufs = [(0, i, i * nb, nb, 1) for i in range(nbytes // nb)]
    ctx = snap.Ctx(local, nbytes + (1 << 20))
    ctx.fill_mix64(0, nbytes, 99 + rank, 0)
    n = ctx.set_buffers(bufs)
    ctx.snapshot()
    ctx.known_commit()  # the first checkpoint is in the store
    mix = np.array([O.mix64(99 ^ c) for c in range(n)], dtype=np.uint64)
    dirty = np.nonzero(mix % np.uint64(20) == 0)[0]
    reps, times, staged = 3, [], 0
    for k in range(reps):
        ctx.xor_words(dirty.astype(np.uint64) * 65536, 0x1234567 + k)
        ctx.sync()
        ctx.timer_start()
        ctx.snapshot()
        ms = ctx.timer_stop()
        times.append(ms)
        _, _, _, staged, nsel = ctx.selection()
        assert nsel == dirty.size, (nsel, dirty.size)
        ctx.known_commit()
    ms = float(np.median(times))
    import bench
    peak, _ = bench.peaks()  # MEASURED_PEAKS.json
    out = {"workload": f"C4: {gib:.0f} GiB/GPU, {n} chunks, {dirty.size} dirty "
                       f"({100 * dirty.size / n:.2f} %), store = previous checkpoint",
           "gpus": world, "ms": round(ms, 3), "R_gbs": round(nbytes / ms / 1e6, 1),
           "W_bytes": int(staged), "rw_gbs": round((nbytes + staged) / ms / 1e6, 1),
           "hbm_frac": round((nbytes + staged) / ms / 1e6 / peak, 4),
           "path": "K1 hash (no speculative stores: dirty set unknown until hashed) + "
                   "K2 select vs known set + K3 gather of the dirty chunks"}
    if rank == 0:
        print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
