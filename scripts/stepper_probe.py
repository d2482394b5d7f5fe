"""Scratch: full time steps of a cloth stack through stepper.SimState.
usage: stepper_probe.py n d_hat_rel gap_rel jitter_rel steps newton_cap kappa"""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2308_09400_b200 import barrier, stepper, workloads
a = sys.argv[1:] + [None] * 7
n = int(a[0] or 140); dh = float(a[1] or 0.2); gap = float(a[2] or 0.6); jit = float(a[3] or 0.05)
steps = int(a[4] or 3); cap = int(a[5] or 30)
cloth = workloads.cloth_stack(layers=4, n=n, seed=1, d_hat_rel=dh, gap_rel=gap, jitter_rel=jit, kappa=float(a[6] or 2e8))
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
cfg = stepper.SolverConfig(dt=cloth.dt, barrier=params, newton_max_iters=cap)
state = stepper.SimState(cloth.as_scene(), cfg)
print("verts", state.n, "fixed", int(cloth.fixed.sum()), "d_hat", cloth.d_hat, "kappa", cloth.kappa, "dt", cloth.dt,
      "contacts", state.detect(state.x).n)
for k in range(steps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st = stepper.advance_time_step(state)
    torch.cuda.synchronize()
    print(k, "newton", st.newton_iters, "pcg", st.pcg_iters, "min_d %.3g" % st.min_distance, "alpha_min %.3g" % st.alpha_min,
          st.warning or "converged", "%.1f ms" % ((time.perf_counter() - t0) * 1e3), "contacts", state.detect(state.x).n)
