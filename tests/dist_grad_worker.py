"""Multi-GPU spliced-DP gradient path (run under torchrun, one rank per GPU).

Each GPU hosts S time-sliced DP ranks (global DP rank = gpu * S + s). Every sliced rank's
issue accumulates its gradient into the GPU's accumulator with K5 in issue order (the
first issue copies — CollectiveEngine::issue sum, collectives.cpp:137-144, worker.cpp:
290-297); the local closer then runs one device-level allreduce over the GPUs
(collectives.cpp:147-154, snap_allreduce over NCCL). Every GPU must end with the sum over
all W * S ranks: u64 bit-exact (mod 2^64), f32 within 1e-6 relative of the oracle's fixed
ascending-order sum (NCCL's cross-GPU order is its own). Exit code 0 = parity.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2202_07848_b200 as snap  # noqa: E402

S = 2  # time-sliced ranks per GPU
N = 1_000_003


def grads(dtype, gr):
    rng = np.random.default_rng(1000 + gr)
    if dtype == "u64":
        return rng.integers(0, 2**64 - 1, size=N, dtype=np.uint64)
    return rng.uniform(0.0, 1.0, N).astype(np.float32)  # same-sign: well conditioned


def main():
    import torch
    import torch.distributed as td
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    td.init_process_group("gloo", rank=rank, world_size=world)
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid[:] = torch.frombuffer(bytearray(snap.Ctx.unique_id()), dtype=torch.uint8)
    td.broadcast(uid, 0)
    ok = True
    stride = (N * 8 + 255) // 256 * 256
    with snap.Ctx(local, (S + 1) * stride) as ctx:
        ctx.comm_init(world, rank, bytes(uid.numpy().tobytes()))
        for dtype, code in (("u64", snap.U64), ("f32", snap.F32)):
            acc = S * stride
            for s in range(S):  # each sliced rank's issue, in slice order
                g = grads(dtype, rank * S + s)
                ctx.write(s * stride, g)
                ctx.grad_sum(code, [s * stride], acc, N, accumulate=(s > 0))
            ctx.allreduce(code, acc, N)
            ctx.sync()
            got = np.frombuffer(ctx.read(acc, N * (8 if dtype == "u64" else 4)).tobytes(),
                                dtype=np.uint64 if dtype == "u64" else np.float32)
            every = [grads(dtype, gr) for gr in range(world * S)]
            if dtype == "u64":
                good = np.array_equal(got, O.grad_sum_u64(every))
            else:
                exp = O.grad_sum_f32(every)
                rel = np.max(np.abs(got.astype(np.float64) - exp) / np.abs(exp.astype(np.float64)))
                good = bool(rel <= 1e-6)
                print(f"rank {rank} f32 max rel {rel:.3e}")
            if not good:
                print(f"FAIL grad {dtype} rank {rank}")
                ok = False
        ctx.comm_destroy()
    flags = [None] * world
    td.all_gather_object(flags, ok)
    if rank == 0:
        print("GRAD PARITY", "OK" if all(flags) else "FAIL", "world", world, "sliced", S)
    td.destroy_process_group()
    sys.exit(0 if all(flags) else 1)


if __name__ == "__main__":
    main()
