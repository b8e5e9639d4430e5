"""Spliced-DP gradient path across GPUs: under torchrun (one rank per GPU) or as threads of
one process sharing a GPU (tests/_group.py).

Each GPU hosts S time-sliced DP ranks (global DP rank = gpu * S + s). Checks, on every GPU:

1. NCCL path (collectives.cpp:137-154 as NCCL does it): K5 accumulates the co-sliced ranks
   in issue order (worker.cpp:290-297), the local closer runs snap_allreduce. u64 is
   bit-exact (mod 2^64); f32 is only within 1e-6 relative on well-conditioned data, since
   NCCL picks its own cross-GPU order.
2. Fixed-order path (snap_allreduce_ordered, one fused peer-memory kernel per GPU): the sum
   over all W * S ranks in ascending dp order on mixed-sign, heavily cancelling data —
   bit-identical to the oracle's left-to-right sum for u64, f32 and bf16, on every GPU;
   also in place (dst = a source) and in the hierarchical order (one K5 partial sum per
   GPU, key = GPU index).
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
ESZ = {"u64": 8, "f32": 4, "bf16": 2}
NP = {"u64": np.uint64, "f32": np.float32, "bf16": np.uint16}
CODE = {"u64": snap.U64, "f32": snap.F32, "bf16": snap.BF16}


def _base(gr):
    rng = np.random.default_rng(1000 + gr)
    return (rng.standard_normal(N) * 10.0 ** rng.integers(-4, 4, N)).astype(np.float32)


def grads(dtype, gr, cancelling=True):
    if dtype == "u64":
        return np.random.default_rng(1000 + gr).integers(0, 2**64 - 1, size=N, dtype=np.uint64)
    if not cancelling:
        x = np.random.default_rng(1000 + gr).uniform(0.0, 1.0, N).astype(np.float32)
    else:
        # mixed sign, magnitudes over 8 decades, and every odd rank nearly cancels the
        # previous one: the partial sums cancel, so any other order gives other bits
        x = _base(gr)
        if gr % 2 == 1:
            x = (-_base(gr - 1) + x * np.float32(1e-3)).astype(np.float32)
    if dtype == "bf16":
        return (x.view(np.uint32) >> 16).astype(np.uint16)
    return x


def run(g) -> bool:
    rank, world = g.rank, g.world
    ok = True
    stride = (N * 8 + 255) // 256 * 256
    with snap.Ctx(g.device, (S + 2) * stride) as ctx:
        g.comm_init(ctx)
        acc = S * stride
        # 1. K5 + NCCL allreduce (well-conditioned f32)
        for dtype in ("u64", "f32"):
            code = CODE[dtype]
            for s in range(S):
                ctx.write(s * stride, grads(dtype, rank * S + s, cancelling=False))
                ctx.grad_sum(code, [s * stride], acc, N, accumulate=(s > 0))
            ctx.allreduce(code, acc, N)
            ctx.sync()
            got = np.frombuffer(ctx.read(acc, N * ESZ[dtype]).tobytes(), dtype=NP[dtype])
            every = [grads(dtype, gr, cancelling=False) for gr in range(world * S)]
            if dtype == "u64":
                good = np.array_equal(got, O.grad_sum_u64(every))
            else:
                exp = O.grad_sum_f32(every)
                rel = np.max(np.abs(got.astype(np.float64) - exp) / np.abs(exp.astype(np.float64)))
                good = bool(rel <= 1e-6)
                if rank == 0:
                    print(f"nccl f32 max rel {rel:.3e} (well conditioned)")
            if not good:
                print(f"FAIL nccl grad {dtype} rank {rank}")
                ok = False
        # 2. fixed order over every sliced rank of every GPU
        sums = {"u64": O.grad_sum_u64, "f32": O.grad_sum_f32, "bf16": O.grad_sum_bf16}
        for dtype in ("u64", "f32", "bf16"):
            code = CODE[dtype]
            mine = [grads(dtype, rank * S + s) for s in range(S)]
            for s in range(S):
                ctx.write(s * stride, mine[s])
            every = [grads(dtype, gr) for gr in range(world * S)]
            exp = sums[dtype](every)
            keys = [rank * S + s for s in range(S)]
            for mode in ("strict", "inplace", "hier"):
                if mode == "hier":
                    # K5 partial per GPU (ascending slice order), then one key per GPU
                    for s in range(S):
                        ctx.write(s * stride, mine[s])
                    ctx.grad_sum(code, [s * stride for s in range(S)], acc, N)
                    ctx.allreduce_ordered(code, [rank], [acc], acc, N)
                    partial = [sums[dtype]([grads(dtype, q * S + s) for s in range(S)])
                               for q in range(world)]
                    want = sums[dtype](partial)
                    dst = acc
                else:
                    for s in range(S):
                        ctx.write(s * stride, mine[s])
                    dst = 0 if mode == "inplace" else acc
                    ctx.allreduce_ordered(code, keys, [s * stride for s in range(S)], dst, N)
                    want = exp
                ctx.sync()
                got = np.frombuffer(ctx.read(dst, N * ESZ[dtype]).tobytes(), dtype=NP[dtype])
                if not np.array_equal(got, want):
                    bad = int(np.count_nonzero(got != want))
                    print(f"FAIL ordered {dtype} {mode} rank {rank}: {bad} elements differ")
                    ok = False
                g.barrier()  # every GPU read this round's sources before they change
        if rank == 0:
            f = O.grad_sum_f32([grads("f32", gr) for gr in range(world * S)])
            d = O.grad_sum_f32([grads("f32", gr) for gr in reversed(range(world * S))])
            print("f32 reversed-order sum differs from the fixed order in",
                  int(np.count_nonzero(f != d)), "of", N, "elements (the data is order-sensitive)")
        ctx.comm_destroy()
    flags = g.all_gather(ok)
    if rank == 0:
        print("GRAD PARITY", "OK" if all(flags) else "FAIL", "world", world, "sliced", S,
              "transport", g.mode)
    return all(flags)


def main():
    from _group import ProcGroup
    g = ProcGroup()
    ok = run(g)
    g.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
