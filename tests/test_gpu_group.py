"""The multi-rank product path on ONE GPU: N ranks as threads of this process, each with
its own ctx, joined by libsnap's in-process communicator (snap_comm_init_local). The same
worker code runs under torchrun on N GPUs with NCCL (test_gpu_multi.py); here it runs on
the driver's 1-GPU box (up to 8 ranks: the host logic of the 8-GPU configurations), so
cross-rank dedup + striped shards (K2), shard restore over
peer memory (K4, resize), persist/load across ranks and the fixed-order gradient allreduce
(K5 + ordered reduce) are checked against the oracle every round instead of skipping."""
import pytest

from _group import run_threads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_threads_snapshot_parity(world, capsys):
    import dist_snapshot_worker as W
    assert all(run_threads(world, W.run))
    out = capsys.readouterr().out
    assert "DIST PARITY OK" in out and "PERSIST OK" in out


@pytest.mark.parametrize("world", [2, 4, 8])
def test_threads_resize_reshard(world, capsys):
    import dist_resize_worker as W
    assert all(run_threads(world, W.run))
    assert "RESIZE PARITY OK" in capsys.readouterr().out


@pytest.mark.parametrize("world", [2, 3, 8])
def test_threads_fixed_order_allreduce(world, capsys):
    import dist_grad_worker as W
    assert all(run_threads(world, W.run))
    assert "GRAD PARITY OK" in capsys.readouterr().out


def test_threads_ordered_allreduce_uneven_sources():
    """Uneven slicing: 3 GPUs (threads) holding 2, 0 and 3 sliced ranks with non-contiguous
    order keys; every rank ends with the left-to-right sum in key order (f32, odd length)."""
    import numpy as np

    import oracle as O
    import paper_2202_07848_b200 as snap
    n = 77_777
    keys = {0: [5, 1], 1: [], 2: [9, 0, 3]}
    rng = np.random.default_rng(12)
    g = {k: (rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, n)).astype(np.float32)
         for r in keys for k in keys[r]}
    want = O.grad_sum_f32([g[k] for k in sorted(g)])
    stride = 1 << 20

    def run(grp):
        with snap.Ctx(0, 6 * stride) as c:
            grp.comm_init(c)
            mine = keys[grp.rank]
            for i, k in enumerate(mine):
                c.write(i * stride, g[k])
            c.allreduce_ordered(snap.F32, mine, [i * stride for i in range(len(mine))],
                                5 * stride, n)
            got = c.read(5 * stride, 4 * n).view(np.float32)
            c.comm_destroy()
            return bool(np.array_equal(got, want))

    assert all(run_threads(3, run))
