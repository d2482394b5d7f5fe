"""World-size-2 CPU (gloo) test of the scene-batch bookkeeping used for N > 1 GPUs."""

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2308_09400_b200 import scene_batch, workloads

    seed = scene_batch.replica_seed(100, rank)
    qb = workloads.config2_batch(n=500, seed=seed)
    units = float(len(qb.ee))
    ms = 2.0 + rank  # the slower rank decides
    total, ms_max = scene_batch.aggregate(units, ms, dist)
    results[rank] = (seed, float(qb.positions.sum()), total, ms_max)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_replicas_aggregate():
    world, port = 2, 29000 + os.getpid() % 2000
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
        r0, r1 = results[0], results[1]
    assert (r0[0], r1[0]) == (100, 101)
    assert r0[1] != r1[1]                      # independent scenes
    assert r0[2] == r1[2] == 1000.0            # units summed over ranks
    assert r0[3] == r1[3] == 3.0               # slowest rank's time
    assert torch.distributed.is_available()
