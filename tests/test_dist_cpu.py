"""CPU, world_size 2 (gloo): the N>1 host logic — bench.py's rank plumbing (unique-id
broadcast, max/sum over ranks) and the cross-rank dedup/striping semantics every GPU
computes redundantly after the digest allgather (identical views on every rank, every
unique chunk written exactly once, shards disjoint)."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch
    import torch.distributed as td

    import bench
    import oracle as O
    try:
        d = bench.Dist()
        uid = d.bcast_bytes(bytes(range(128)) if rank == 0 else None, 128)
        assert uid == bytes(range(128))
        assert d.max(float(rank + 1)) == float(world)
        assert d.sum(1.0) == float(world)
        # local image: replicated region (same on all ranks) + per-rank region
        rep = O.fill_mix64(64 * 8192, 5, 0)
        own = O.fill_mix64((16 + 8 * rank) * 8192, 5 ^ (rank << 40), rep.size)
        img = np.concatenate([rep, own])
        bufs = [(0, 0, 0, rep.nbytes, 0), (0, 1, rep.nbytes, own.nbytes, 2)]
        dig, lens, _ = O.hash_chunks([img], bufs)
        # allgather (what snap_select does over NCCL)
        t = torch.from_numpy(dig.view(np.int64).copy())
        sizes = [None] * world
        td.all_gather_object(sizes, int(t.numel()))
        gathered = [None] * world
        td.all_gather_object(gathered, dig)
        gd = np.concatenate(gathered)
        gl = np.full(gd.size, 65536, np.uint32)
        sel, owner, off, total = O.select(gd, gl)
        writer, shoff, shbytes = O.stripe(gd, gl, sizes, sel)
        views = [None] * world
        td.all_gather_object(views, (sel.tobytes(), writer.tobytes(), shoff.tobytes()))
        assert all(v == views[0] for v in views), "ranks disagree on the global selection"
        # replicated chunks: striped round-robin over all ranks; per-rank chunks: own rank
        assert int(sel.sum()) == 64 + sum(16 + 8 * r for r in range(world))
        assert np.bincount(writer[sel == 1], minlength=world).min() > 0
        assert shbytes.sum() == total
        for r in range(world):
            w = writer[(sel == 1)]
        mine = np.nonzero((sel == 1) & (writer == rank))[0]
        offs = np.sort(shoff[mine])
        assert offs.tolist() == list(range(0, 65536 * mine.size, 65536))  # dense shard
        d.close()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
        raise


def test_two_rank_gloo_dedup_and_plumbing():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=240)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: "ok", 1: "ok"}, res
