"""The multi-rank product path on ONE GPU: N ranks as threads of this process, each with
its own ctx, joined by libsnap's in-process communicator (snap_comm_init_local). The same
worker code runs under torchrun on N GPUs with NCCL (test_gpu_multi.py); here it runs on
the driver's 1-GPU box, so cross-rank dedup + striped shards (K2), shard restore over
peer memory (K4, resize), persist/load across ranks and the fixed-order gradient allreduce
(K5 + ordered reduce) are checked against the oracle every round instead of skipping."""
import pytest

from _group import run_threads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
def test_threads_snapshot_parity(world, capsys):
    import dist_snapshot_worker as W
    assert all(run_threads(world, W.run))
    out = capsys.readouterr().out
    assert "DIST PARITY OK" in out and "PERSIST OK" in out


@pytest.mark.parametrize("world", [2, 4])
def test_threads_resize_reshard(world, capsys):
    import dist_resize_worker as W
    assert all(run_threads(world, W.run))
    assert "RESIZE PARITY OK" in capsys.readouterr().out


@pytest.mark.parametrize("world", [2, 3])
def test_threads_fixed_order_allreduce(world, capsys):
    import dist_grad_worker as W
    assert all(run_threads(world, W.run))
    assert "GRAD PARITY OK" in capsys.readouterr().out
