"""Scratch: time the numeric assembly kernels on the bench scene."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads
import bench
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
vt, ee = bp.query(cloth.positions)
table, _ = contacts.narrow_phase_device(cloth.positions, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
batch = stencils.evaluate(table, cloth.positions, params, dt=cloth.dt, want_factors=True)
fams = [batch.families[s] for s in sorted(batch.families)]
sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
sysm.set_pattern([(f.s, f.vids) for f in fams])
hess, fac = [f.hess for f in fams], [f.fac for f in fams]
noop = lambda: None
print("dense ms", bench.time_steps(torch, lambda: sysm.assemble(hess), 50, 5, noop) / 50,
      "factors ms", bench.time_steps(torch, lambda: sysm.assemble_from_factors(fac), 50, 5, noop) / 50)
