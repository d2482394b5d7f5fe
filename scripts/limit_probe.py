"""One Newton direction of the stepper past the factor-descriptor limit (a family with >= 2^27 / 12 four-vertex
blocks): the stepper must take the dense path there (NewtonSystem.factors_fit) and still produce a converged
direction.   python scripts/limit_probe.py [layers n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2308_09400_b200 import barrier, stepper, workloads

layers, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8, 450)
scene = workloads.cloth_stack(layers=layers, n=n, seed=3, d_hat_rel=0.2, jitter_rel=0.01, kappa=1e5)
cfg = stepper.SolverConfig(dt=scene.dt, barrier=barrier.BarrierParams(d_hat=scene.d_hat, kappa=scene.kappa),
                           preconditioner="mas")
state = stepper.SimState(scene.as_scene(), cfg)
x = state.x
table = state.detect(x)
counts = {s: table.family_count(s) for s in (2, 3, 4)}
print("vertices", x.shape[0], "contacts", table.n, "family counts", counts, "factors_fit", state.system.factors_fit(counts), flush=True)
xt = x + 1e-4 * torch.randn_like(x)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d, iters, ok = stepper._search_direction(state, x, xt, x, table)
    torch.cuda.synchronize()
    print("direction %d: %.1f ms, pcg iters %d converged %s, |d|_inf %.3e, finite %s, peak mem %.1f GB" % (
        rep, (time.perf_counter() - t0) * 1e3, iters, ok, float(d.abs().max()), bool(torch.isfinite(d).all()),
        torch.cuda.max_memory_allocated() / 2**30), flush=True)
state.close()
