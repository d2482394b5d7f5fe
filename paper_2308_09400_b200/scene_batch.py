"""Scene-batch scaling: one independent scene (replica) per GPU, no data-path collective.

A single scene does not shard (assembly / SpMV / PCG couple all vertices every iteration and a
100k-330k vertex problem is smaller than one GPU's sweet spot), so multi-GPU throughput comes from
batches of independent scenes -- BASELINE.json north_star: "replicas only".  The only
cross-rank traffic is this bookkeeping: the slowest rank's time and the total unit count.
"""


def replica_seed(base_seed, rank):
    """Seed of the rank's own scene: replicas differ, runs are reproducible."""
    return int(base_seed) + int(rank)


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
