"""The N>1 bench path (replicas only) on CPU: 2 gloo ranks, barrier + max-over-ranks timing."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench

    w, r, _ = bench.dist_setup()
    assert (w, r) == (world, rank)
    bench.barrier(w)
    mx = bench.max_over_ranks(10.0 + rank, w)
    out[rank] = (mx, bench.aggregate_value(1000, mx, w))
    import torch.distributed as dist

    dist.destroy_process_group()


def test_two_rank_gloo_max_and_aggregate():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == 11.0  # slowest rank's time
    assert out[0][1] == pytest.approx(2 * 1000**2 / 11e-3)
