"""Scratch: time steps of the cube-drop scene (elastic + barrier + friction families together)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2308_09400_b200 import barrier, device, elasticity, stepper, workloads
k = int(sys.argv[1]) if len(sys.argv) > 1 else 12
mu_f = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
sc = workloads.cube_drop(k=k, tilt=0.5)
cfg = stepper.SolverConfig(dt=sc.dt, barrier=barrier.BarrierParams(sc.d_hat, sc.kappa), friction_mu=mu_f)
state = stepper.SimState(sc, cfg, elasticity.ElasticMaterial(1e5, 0.4))
state.v = device.to_device(sc.v0.copy())
print(sc.name, "verts", state.n, "tets", sc.tets.shape[0], "contacts", state.detect(state.x).n)
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 5):
    st = stepper.advance_time_step(state)
    fr = 0 if state.friction_state is None else state.friction_state.n
    print(i, "newton", st.newton_iters, "pcg", st.pcg_iters, "min_d/d_hat %.3f" % (st.min_distance / sc.d_hat), "alpha_min %.3g" % st.alpha_min,
          st.warning or "converged", "%.1f ms" % st.wall_ms, "contacts", state.detect(state.x).n, "friction data", fr)
