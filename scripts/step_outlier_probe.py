"""Scratch: the bench's three time steps, repeated in one process -- is a slow second step a first-use cost?"""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import barrier, stepper, workloads
soft = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2, jitter_rel=0.01, kappa=1e5)
cfg = stepper.SolverConfig(dt=soft.dt, barrier=barrier.BarrierParams(d_hat=soft.d_hat, kappa=soft.kappa))
for rep in range(4):
    state = stepper.SimState(soft.as_scene(), cfg)
    out = []
    for _ in range(3):
        st = stepper.advance_time_step(state)
        out.append((st.newton_iters, round(st.wall_ms, 1)))
    state.close()
    print("rep", rep, out, flush=True)
