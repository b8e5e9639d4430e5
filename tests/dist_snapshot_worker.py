"""Multi-rank snapshot parity worker: under torchrun (one rank per GPU, NCCL) or as
threads of one process sharing a GPU (tests/_group.py ThreadGroup, libsnap's in-process
communicator).

Each rank builds a small DP image (replicated P/O buffers + per-rank buffers, unequal chunk
counts, mispredicted replication hints), snapshots it twice through the C ABI with NCCL
allgather of digest vectors, and rank 0 checks every rank's digests, the global
dedup selection, the stripe writers/shard offsets and every shard's bytes against the CPU
oracle (oracle/or_select + or_stripe + or_compact). Exit code 0 = parity.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

MIB = 1 << 20


def layout(rank):
    """(bufs, content) with content[i] = (seed, base) for the fill of buffer i."""
    bufs, fills, addr = [], [], 0

    def add(nbytes, cat, seed, flags=0):
        nonlocal addr
        bufs.append((0, len(bufs), addr, nbytes, cat, flags))
        fills.append((seed, addr // 8))
        addr += (nbytes + 4095) // 4096 * 4096

    add(3 * MIB, 0, 11)                      # params: replicated
    add(5 * MIB + 256, 1, 12)                # Adam m: replicated, ragged tail
    add(2 * MIB, 0, 13, flags=snap_private())  # replicated content, hinted private
    add(1 * MIB + 4096, 2, 100 + rank)       # grads: per rank
    add(1 * MIB, 0, 200 + rank)              # hinted replicated but per-rank content
    if rank % 2 == 1:
        add(768 << 10, 3, 300 + rank)        # extra buffer on odd ranks
    add(64 << 10, 1, 12)                     # duplicate of the start of Adam m (dedup)
    return bufs, fills, addr


def snap_private():
    return 2


def fill_host(bufs, fills, nbytes):
    img = np.zeros(nbytes // 8, np.uint64)
    for (_r, _s, a, n, _c, _f), (seed, base) in zip(bufs, fills):
        img[a // 8:(a + n) // 8] = O.fill_mix64(n // 8, seed, 0)
    return img


def run(g) -> bool:
    rank, world = g.rank, g.world
    bufs, fills, nbytes = layout(rank)
    arena = nbytes + MIB
    ctx = snap.Ctx(g.device, arena)
    host = fill_host(bufs, fills, nbytes)
    ctx.write(0, host)
    sb = snap.bufs_array([b[:5] for b in bufs])
    for i, b in enumerate(bufs):
        sb[i].flags = b[5]
    n = C_set_buffers(ctx, sb, len(bufs))
    g.comm_init(ctx)
    results = []
    for it in range(2):  # second snapshot uses the learned layout
        ctx.snapshot()
        d, lens = ctx.digests()
        gsel, gown, goff, gbytes, gch = ctx.global_selection()
        writer, shard_off, my_bytes, my_chunks = ctx.shard()
        shard = ctx.read_staging(0, my_bytes) if my_bytes else np.zeros(0, np.uint8)
        results.append((d, lens, gsel, gown, goff, gbytes, writer, shard_off, my_bytes, shard))
    _, maxn = ctx.global_info()
    objs = g.all_gather({"rank": rank, "host": host, "bufs": bufs, "res": results,
                         "maxn": maxn})
    ok = True
    if rank == 0:
        objs.sort(key=lambda o: o["rank"])
        per = []
        for o in objs:
            od, ol, _ = O.hash_chunks([o["host"]], [b[:5] for b in o["bufs"]])
            per.append((od, ol))
        npr = [p[0].size for p in per]
        base = np.concatenate([[0], np.cumsum(npr)])
        gd = np.concatenate([p[0] for p in per])
        gl = np.concatenate([p[1] for p in per])
        osel, oown, ooff, otot = O.select(gd, gl)
        owriter, oshoff, oshbytes = O.stripe(gd, gl, npr, osel)
        maxn = objs[0]["maxn"]
        assert maxn == max(npr)
        pad = np.concatenate([r * maxn + np.arange(npr[r]) for r in range(world)])
        for it in range(2):
            for r, o in enumerate(objs):
                d, lens = o["res"][it][0], o["res"][it][1]
                if not (np.array_equal(d, per[r][0]) and np.array_equal(lens, per[r][1])):
                    print(f"FAIL digests rank {r} it {it}")
                    ok = False
            d, lens, gsel, gown, goff, gbytes, writer, shard_off, _, _ = objs[0]["res"][it]
            # map padded owner indices to the oracle's dense indexing
            own = gown[pad].copy()
            live = own != np.uint64(2**64 - 1)
            own_r, own_i = own[live] // maxn, own[live] % maxn
            own[live] = base[own_r.astype(np.int64)] + own_i
            checks = {
                "sel": np.array_equal(gsel[pad], osel),
                "owner": np.array_equal(own, oown),
                "offsets": np.array_equal(goff[pad], ooff),
                "bytes": gbytes == otot,
                "writer": np.array_equal(writer[pad], owriter),
                "shard_off": np.array_equal(shard_off[pad][osel == 1], oshoff[osel == 1]),
            }
            for k, v in checks.items():
                if not v:
                    print(f"FAIL {k} it {it}")
                    ok = False
            # every shard's bytes = oracle compaction of the chunks it writes
            for w in range(world):
                shard = objs[w]["res"][it][9]
                if objs[w]["res"][it][8] != oshbytes[w]:
                    print(f"FAIL shard size w={w}")
                    ok = False
                    continue
                exp = np.zeros(int(oshbytes[w]), np.uint8)
                for gi in np.nonzero((osel == 1) & (owriter == w))[0]:
                    r = int(np.searchsorted(base, gi, side="right") - 1)
                    i = int(gi - base[r])
                    # chunk i of rank r: locate its bytes in rank r's host image
                    o = objs[r]
                    k = i
                    for (_r, _s, a, nb, _c, _f) in o["bufs"]:
                        nc = (nb + 65535) // 65536
                        if k < nc:
                            ln = min(65536, nb - k * 65536)
                            src = o["host"].view(np.uint8)[a + k * 65536:a + k * 65536 + ln]
                            exp[int(oshoff[gi]):int(oshoff[gi]) + ln] = src
                            break
                        k -= nc
                if not np.array_equal(shard, exp):
                    print(f"FAIL shard bytes w={w} it {it}")
                    ok = False
        print("DIST PARITY", "OK" if ok else "FAIL", "world", world, "chunks", npr,
              "unique", int(osel.sum()))
    ok = persist_stage(g, ctx, objs, ok) and ok
    ok = g.bcast(ok, 0)
    ctx.comm_destroy()
    ctx.close()
    return ok


def main():
    from _group import ProcGroup
    g = ProcGroup()
    ok = run(g)
    g.close()
    sys.exit(0 if ok else 1)


def persist_stage(g, ctx, objs, ok):
    """On-disk format across ranks: every rank persists its shard of the (last) snapshot into
    one shared directory (content-addressed, no coordination), then restores the NEXT rank's
    layout from the directory alone into a fresh context and compares it with that rank's
    image. Rank 0 checks that the directory holds exactly the globally unique chunks."""
    import tempfile
    rank, world = g.rank, g.world
    paths = g.all_gather(tempfile.mkdtemp(prefix="snap_persist_") if rank == 0 else None)
    root = paths[0]
    st = ctx.persist(root)
    sts = g.all_gather(st)
    good = True
    peer = (rank + 1) % world
    o = [x for x in objs if x["rank"] == peer][0]
    bufs = [b[:5] for b in o["bufs"]]
    nbytes = max(a + n for (_, _, a, n, _) in bufs)
    with snap.Ctx(g.device, nbytes + MIB) as c2:
        c2.load(root, rank=peer)
        got = c2.read(0, nbytes).view(np.uint64)
        for (_, _, a, n, _) in bufs:
            if not np.array_equal(got[a // 8:(a + n) // 8], o["host"][a // 8:(a + n) // 8]):
                print(f"FAIL persist/load rank {rank} <- layout {peer}")
                good = False
    if rank == 0:
        nfiles = sum(len(fs) for dp, _, fs in os.walk(os.path.join(root, "blobs")))
        uniq = len(set(np.concatenate([O.hash_chunks([x["host"]], [b[:5] for b in x["bufs"]])[0]
                                       for x in objs]).tolist()))
        if nfiles != uniq or sum(s["written"] for s in sts) != uniq:
            print(f"FAIL persist files {nfiles} written {[s['written'] for s in sts]} "
                  f"unique {uniq}")
            good = False
        print("PERSIST", "OK" if good else "FAIL", "files", nfiles)
    flags = g.all_gather(good)
    if rank == 0:
        import shutil
        shutil.rmtree(root, ignore_errors=True)
    return all(flags)


def C_set_buffers(ctx, sb, n):
    import ctypes as C
    g = snap.SnapGeom(4096, 65536)
    out = C.c_uint64()
    ctx._ck(ctx._L.snap_set_buffers(ctx.h, sb, n, C.byref(g), C.byref(out)), "snap_set_buffers")
    ctx.nchunks = out.value
    ctx.nbufs = n
    return out.value


if __name__ == "__main__":
    main()
