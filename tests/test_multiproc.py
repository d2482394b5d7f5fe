"""World-size-2 CPU (gloo) tests of the scene-batch path used for N > 1 GPUs: the same functions bench.py is
built on (scene_batch.init / timed_steps / aggregate / launch), and bench.py's own launcher end to end."""

import json
import os
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2308_09400_b200 import scene_batch, workloads

    r, w, local, d = scene_batch.init(backend="gloo")
    assert (r, w, local) == (rank, world, rank) and d is not None and d.get_world_size() == world
    seed = scene_batch.replica_seed(100, rank)
    state = {}

    def step():
        state["qb"] = workloads.config2_batch(n=500, seed=seed)
        state["calls"] = state.get("calls", 0) + 1

    ms_own = scene_batch.timed_steps(step, 4, 2, d, cuda=False)
    assert state["calls"] == 6 and ms_own > 0.0
    units = float(len(state["qb"].ee))
    ms = 2.0 + rank  # the slower rank decides
    total, ms_max = scene_batch.aggregate(units, ms, d)
    results[rank] = (seed, float(state["qb"].positions.sum()), total, ms_max,
                     scene_batch.throughput(total, ms_max, 4))
    scene_batch.finish(d)
    assert not dist.is_initialized()


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
    assert r0[4] == pytest.approx(1000.0 * 4 / 3e-3)
    assert torch.distributed.is_available()


def test_single_process_is_the_identity():
    from paper_2308_09400_b200 import scene_batch

    assert scene_batch.aggregate(7.0, 2.5, None) == (7.0, 2.5)
    assert scene_batch.throughput(10.0, 2.0, 4) == pytest.approx(20000.0)
    calls = []
    ms = scene_batch.timed_steps(lambda: calls.append(1), 3, 2, None, cuda=False)
    assert len(calls) == 5 and ms >= 0.0


@pytest.mark.timeout(300)
def test_bench_gpus_2_spawns_two_ranks():
    """`python bench.py --gpus 2` with no rank environment re-executes itself under torch.distributed.run
    (scene_batch.launch) and prints ONE line with n_gpus = 2 -- rehearsed on CPUs (--dry-run, gloo)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "3",
                          "--warmup", "1"], capture_output=True, text=True, env=env, timeout=280)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["dry_run"] is True
    assert lines[0]["units_per_step_all_ranks"] == 4000.0      # 2000 queries per replica, summed over two ranks


@pytest.mark.timeout(300)
def test_reference_arm_under_two_ranks_prints_once():
    """Under N > 1 ranks the reference arm runs on rank 0 alone; the other ranks exit 0 without work."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--steps", "2", "--warmup", "1", "--n-stencils", "4000", "--skip-newton"],
                         capture_output=True, text=True, env=env, timeout=280)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    assert lines[0]["config"]["stencils_per_gpu"] == 4000 and lines[0]["e2e"]["h2d_bytes_per_step"] == 0
