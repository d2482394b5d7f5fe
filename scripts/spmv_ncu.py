"""Scratch: a few streamed SpMV launches on the bench scene, for ncu."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
vt, ee = workloads.broad_phase(cloth)
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
pos = device.to_device(cloth.positions)
table, _ = contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
batch = stencils.evaluate(table, pos, params, dt=cloth.dt)
fams = [batch.families[s] for s in sorted(batch.families)]
sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
sysm.set_pattern([(f.s, f.vids) for f in fams])
sysm.assemble([f.hess for f in fams])
x = device.to_device(np.random.default_rng(0).normal(size=3 * sysm.n)); y = device.empty((3 * sysm.n,))
for _ in range(4):
    sysm.spmv(x, out=y)
import torch; torch.cuda.synchronize()
