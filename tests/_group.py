"""Rank plumbing for the multi-rank parity workers, two transports with one API:

* ProcGroup  — one process per GPU under torchrun (gloo for the test's own object
               exchange, NCCL inside libsnap through snap_comm_init);
* ThreadGroup — N ranks as threads of ONE process, every ctx on the same GPU (or
               spread over the visible ones), libsnap's in-process communicator
               (snap_comm_init_local). This is how the driver's 1-GPU test box runs
               the multi-rank product path (K2 cross-rank dedup + stripes, shard
               restore, fixed-order allreduce) instead of skipping it.

Workers implement run(g) -> bool and print their own PASS/FAIL lines.
"""
from __future__ import annotations

import os
import threading


class ProcGroup:
    def __init__(self):
        import torch.distributed as td
        self.td = td
        self.rank = int(os.environ["RANK"])
        self.world = int(os.environ["WORLD_SIZE"])
        self.device = int(os.environ.get("LOCAL_RANK", self.rank))
        self.mode = "nccl"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        td.init_process_group("gloo", rank=self.rank, world_size=self.world)

    def all_gather(self, obj):
        out = [None] * self.world
        self.td.all_gather_object(out, obj)
        return out

    def bcast(self, obj, root=0):
        box = [obj]
        self.td.broadcast_object_list(box, src=root)
        return box[0]

    def barrier(self):
        self.td.barrier()

    def comm_init(self, ctx, members=None):
        """Collective over ALL ranks; the members (default: everyone) join a communicator."""
        members = list(range(self.world)) if members is None else list(members)
        uid = ctx.unique_id() if self.rank == members[0] else None
        uid = self.bcast(uid, members[0])
        if self.rank in members:
            ctx.comm_init(len(members), members.index(self.rank), uid)

    def close(self):
        self.td.destroy_process_group()


class _Shared:
    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world
        self.key = f"snap-threads-{os.getpid()}-{id(self)}"


class ThreadGroup:
    def __init__(self, shared: _Shared, rank: int, device: int):
        self.s = shared
        self.rank = rank
        self.world = shared.world
        self.device = device
        self.mode = "threads"
        self.gen = 0

    def all_gather(self, obj):
        self.s.bar.wait()
        self.s.slots[self.rank] = obj
        self.s.bar.wait()
        out = list(self.s.slots)
        self.s.bar.wait()
        return out

    def bcast(self, obj, root=0):
        return self.all_gather(obj)[root]

    def barrier(self):
        self.s.bar.wait()

    def comm_init(self, ctx, members=None):
        members = list(range(self.world)) if members is None else list(members)
        self.gen += 1  # every thread calls comm_init in the same order: same key
        if self.rank in members:
            ctx.comm_init_local(len(members), members.index(self.rank),
                                f"{self.s.key}-{self.gen}")

    def close(self):
        pass


def run_threads(world, fn, ngpus=1):
    """Runs fn(group) on `world` threads (rank r on device r % ngpus); returns the
    per-rank results (an exception in any rank is re-raised)."""
    shared = _Shared(world)
    res, errs = [None] * world, [None] * world

    def body(r):
        try:
            res[r] = fn(ThreadGroup(shared, r, r % max(ngpus, 1)))
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errs[r] = e
            shared.bar.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errs:
        if e is not None:
            raise e
    return res
