"""Scratch for ncu / timing: the symbolic phase alone at bench scale (set_pattern x 4)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads

which = sys.argv[1] if len(sys.argv) > 1 else "stack"
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2) if which == "stack" else workloads.cloth_on_sphere()
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
pos = device.to_device(cloth.positions)
bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
vt, ee = bp.query(pos)
table, _ = contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
batch = stencils.evaluate(table, pos, params, dt=cloth.dt, want_factors=True)
fams = [batch.families[s] for s in sorted(batch.families)]
sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
for mode in (0, 1, 0):
    sysm.set_symbolic_mode(mode)
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        sysm.set_pattern([(f.s, f.vids) for f in fams])
        torch.cuda.synchronize(); print(mode, (time.perf_counter() - t0) * 1e3, sysm.stats())
