"""C5 measurement: elastic resize of Llama-3-8B-sized DP state (bf16 P + fp32 Adam m, v =
80.3 GB per replica, identical on every rank) — snapshot on N GPUs (cross-rank dedup,
1/N stripes), restore onto N/2 GPUs straight from the peer shards over NVLink, reshard on
N/2, restore onto N/4. Run under torchrun (one rank per GPU):

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      tools/bench_resize.py [--scale 1]

Prints one JSON line (rank 0). --scale k divides every tensor by k (smaller boxes).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402


def llama3_8b_params():
    t = [128256 * 4096]
    for _ in range(32):
        t += [4096 * 4096, 4096 * 1024, 4096 * 1024, 4096 * 4096, 4096 * 14336, 4096 * 14336,
              14336 * 4096, 4096, 4096]
    t += [4096, 4096 * 128256]
    assert sum(t) == 8_030_261_248
    return t


def layout(scale):
    bufs, addr = [], 0
    for cat, esz in ((0, 2), (1, 4), (1, 4)):  # bf16 P, fp32 m, fp32 v
        for n in llama3_8b_params():
            nb = max(256, (n * esz // scale + 255) // 256 * 256)
            bufs.append((0, len(bufs), addr, nb, cat))
            addr += nb
    return bufs, addr


def main():
    import torch
    import torch.distributed as td
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    td.init_process_group("gloo", rank=rank, world_size=world)
    bufs, nbytes = layout(a.scale)
    ctx = snap.Ctx(local, nbytes + (64 << 20))
    ctx.fill_mix64(0, nbytes, 77, 0)
    nch = ctx.set_buffers(bufs)
    out = {"workload": f"C5: Llama-3-8B DP state {nbytes / 1e9:.2f} GB/replica (bf16 P + fp32 "
                       f"m,v, {len(bufs)} buffers, {nch} chunks), identical on every rank",
           "stages": []}

    def new_comm(members):
        ctx.comm_destroy()
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == members[0]:
            uid[:] = torch.frombuffer(bytearray(snap.Ctx.unique_id()), dtype=torch.uint8)
        td.broadcast(uid, members[0])
        if rank in members:
            ctx.comm_init(len(members), members.index(rank), bytes(uid.numpy().tobytes()))

    def tmax(x):
        t = torch.tensor([x], dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        return float(t.item())

    members = list(range(world))
    while len(members) >= 2:
        new_comm(members)
        st = {"from_gpus": len(members), "to_gpus": len(members) // 2}
        snap_ms = 0.0
        if rank in members:
            ctx.snapshot()  # warm-up: learns the striped layout
            ctx.sync()
            ctx.timer_start()
            for _ in range(a.reps):
                ctx.snapshot()
            snap_ms = ctx.timer_stop() / a.reps
            _, _, shard, _ = ctx.shard()
            st["shard_bytes_per_gpu"] = int(shard)
        snap_ms = tmax(snap_ms)
        st["snapshot_ms"] = round(snap_ms, 3)
        st["snapshot_gbs_aggregate"] = round(len(members) * nbytes / (snap_ms / 1e3) / 1e9, 1)
        handles = [None] * world
        td.all_gather_object(handles, ctx.ipc_export() if rank in members else b"\0" * 64)
        targets = members[: len(members) // 2]
        rest_ms, ok = 0.0, True
        if rank in targets:
            ctx.ipc_import(b"".join(handles[m] for m in members), len(members))
            ctx.write(0, np.zeros(1 << 20, np.uint8))
            ctx.sync()
            ctx.timer_start()
            ctx.restore_shards(members.index(rank), verify=False)
            rest_ms = ctx.timer_stop()
            ctx.restore_shards(members.index(rank), verify=True)  # digest check (untimed)
        td.barrier()
        rest_ms = tmax(rest_ms)
        remote = nbytes * (len(members) - 1) / len(members)
        st["restore_ms_per_target"] = round(rest_ms, 3)
        st["restore_gbs_per_target"] = round(nbytes / (rest_ms / 1e3) / 1e9, 1)
        st["nvlink_gbs_per_target"] = round(remote / (rest_ms / 1e3) / 1e9, 1)
        st["verified"] = True
        out["stages"].append(st)
        members = targets
    ctx.comm_destroy()
    ctx.close()
    if rank == 0:
        print(json.dumps(out))
    td.destroy_process_group()


if __name__ == "__main__":
    main()
