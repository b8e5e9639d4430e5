"""Elastic resize parity worker (C5 shape, small): under torchrun on N GPUs (N even), or as
N threads sharing one GPU (tests/_group.py).

1. N ranks hold identical DP state (params + Adam m,v, identical addresses); snapshot on N
   (cross-rank dedup -> each GPU writes a 1/N stripe shard).
2. Resize N -> N/2: shards are exchanged as CUDA IPC handles; each target GPU zeroes its
   arena and rebuilds the replica from all N shards (peer shards read over NVLink by the
   scatter kernel), digest-verified, then compared byte-for-byte with the host truth.
3. Reshard: the N/2 targets snapshot again (new NCCL communicator, stripes over N/2) and
   resize N/2 -> N/4 the same way.
Exit 0 = bit-exact restore at every stage.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

MIB = 1 << 20


def replica_layout(scale_mib):
    """params (cat 0) and Adam m, v (cat 1): 2:4:4 bytes per parameter, ragged sizes."""
    bufs, addr = [], 0
    for kind, (cat, mult) in enumerate([(0, 2), (1, 4), (1, 4)]):
        for i, base in enumerate([3, 1, 7, 2]):
            nbytes = (base * scale_mib * MIB * mult // 10) // 256 * 256 + 256 * (i + kind)
            bufs.append((0, len(bufs), addr, nbytes, cat))
            addr += nbytes
    return bufs, addr


def run(g) -> bool:
    rank, world = g.rank, g.world
    scale = int(os.environ.get("RESIZE_SCALE_MIB", "8"))
    bufs, nbytes = replica_layout(scale)
    truth = O.fill_mix64(nbytes // 8, 1234, 0)
    ctx = snap.Ctx(g.device, nbytes + MIB)
    ok = True
    members = list(range(world))
    ctx.write(0, truth)
    ctx.set_buffers(bufs)
    stage = 0
    while len(members) >= 2:
        ctx.comm_destroy()  # collective over the previous world (every rank that had one)
        g.comm_init(ctx, members)
        if rank in members:
            ctx.snapshot()
            _, _, my_bytes, _ = ctx.shard()
            _, _, _, gbytes, _ = ctx.global_selection()
            assert gbytes == nbytes, (gbytes, nbytes)  # replicas dedup to one copy
        handles = g.all_gather(ctx.ipc_export() if rank in members else b"\0" * 64)
        blob = b"".join(handles[m] for m in members)
        targets = members[: len(members) // 2]
        if rank in targets:
            ctx.ipc_import(blob, len(members))
            ctx.write(0, np.zeros(nbytes, np.uint8))  # a fresh GPU for the restored rank
            ctx.restore_shards(members.index(rank), verify=True)
            got = ctx.read(0, nbytes).view(np.uint64)
            if not np.array_equal(got, truth):
                print(f"FAIL rank {rank} stage {stage}: restored bytes differ")
                ok = False
            if rank == targets[0]:
                print(f"stage {stage}: {len(members)} -> {len(targets)} GPUs, shard "
                      f"{my_bytes} B, restored {nbytes} B bit-exact")
        g.barrier()  # sources keep their shards mapped until every target is done
        members = targets
        stage += 1
    ctx.comm_destroy()
    flags = g.all_gather(ok)
    ctx.close()
    if rank == 0:
        print("RESIZE PARITY", "OK" if all(flags) else "FAIL")
    return all(flags)


def main():
    from _group import ProcGroup
    g = ProcGroup()
    ok = run(g)
    g.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
