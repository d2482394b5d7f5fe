"""Scene-batch scaling: one independent scene (replica) per GPU, no data-path collective.

A single scene does not shard (assembly / SpMV / PCG couple all vertices every iteration and a
100k-330k vertex problem is smaller than one GPU's sweet spot), so multi-GPU throughput comes from
batches of independent scenes -- BASELINE.json north_star: "replicas only".  The only
cross-rank traffic is this bookkeeping: the slowest rank's time and the total unit count.

``bench.py --gpus N`` is built on exactly these functions: ``launch`` (re-exec under
``torch.distributed.run`` when no rank environment exists), ``init`` (rank / device / process group),
``timed_steps`` (the contract's barrier + synchronize bracket) and ``aggregate``.  The CPU test
(tests/test_multiproc.py) drives the same code with the gloo backend.
"""

import os
import socket
import subprocess
import sys
import time


def replica_seed(base_seed, rank):
    """Seed of the rank's own scene: replicas differ, runs are reproducible."""
    return int(base_seed) + int(rank)


def free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch(n_ranks, argv, python=None):
    """Run ``argv`` (script + arguments) as ``n_ranks`` processes on this node, one per GPU, the way the
    driver does: ``python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1
    --master-port P script args``.  Returns the launcher's exit code.  Called when ``--gpus N > 1`` is
    asked for and no rank environment (WORLD_SIZE) exists yet."""
    cmd = [python or sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={int(n_ranks)}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port())] + list(argv)
    return subprocess.call(cmd)


def init(backend="nccl"):
    """(rank, world, local_rank, dist) from the torchrun environment.  ``dist`` is the initialised
    ``torch.distributed`` module when world > 1, else None.  With the nccl backend the process is bound to
    GPU ``local_rank`` first (one process per GPU)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if backend == "nccl":
        import torch

        have = torch.cuda.device_count()
        if local >= have:
            raise SystemExit(f"rank {rank}: local rank {local} needs GPU {local}, but this node has {have} "
                             f"(one process per GPU: --gpus must not exceed the GPUs of the node)")
        torch.cuda.set_device(local)
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local, dist


def barrier(dist):
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def timed_steps(fn, steps, warmup, dist=None, cuda=True):
    """``warmup`` untimed calls of ``fn``, then exactly ``steps`` timed ones bracketed by a barrier and a
    device synchronize on both sides -> this rank's milliseconds for all ``steps``.  On a GPU the clock is a
    pair of CUDA events on the current (launching) stream; the CPU rehearsal uses the wall clock."""
    for _ in range(warmup):
        fn()
    if cuda:
        import torch

        barrier(dist)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        barrier(dist)
        return e0.elapsed_time(e1)
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    ms = (time.perf_counter() - t0) * 1e3
    barrier(dist)
    return ms


def aggregate(units_local, ms_local, dist=None, device="cpu"):
    """(total units over ranks, max time over ranks).  ``dist``: an initialised
    ``torch.distributed`` module (nccl on GPUs, gloo in CPU tests) or None for one process."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(units_local), float(ms_local)
    import torch

    t = torch.tensor([float(ms_local)], dtype=torch.float64, device=device)
    u = torch.tensor([float(units_local)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(u.item()), float(t.item())


def throughput(units_total, ms_max, steps):
    """Whole-job units per second: all ranks' units over the slowest rank's time."""
    return units_total * steps / (ms_max * 1e-3)


def finish(dist):
    if dist is not None and dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
