"""Scratch for ncu: each Newton-step kernel launched a few times at bench scale."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads

cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
pos = device.to_device(cloth.positions)
bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
for _ in range(2):
    vt, ee = bp.query(pos)
    table, _ = contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
dirs = device.to_device(0.3 * cloth.d_hat * np.random.default_rng(3).normal(size=cloth.positions.shape))
for _ in range(2):
    bp.ccd_step_bound(pos, dirs)
batch = stencils.evaluate(table, pos, params, dt=cloth.dt, want_factors=True)
fams = [batch.families[s] for s in sorted(batch.families)]
sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
sysm.set_pattern([(f.s, f.vids) for f in fams])
hess = [f.hess for f in fams]
for variant in (0, 4, 0):
    sysm.set_numeric_variant(variant)
    for _ in range(2):
        sysm.assemble(hess)
for _ in range(2):
    sysm.assemble_from_factors([f.fac for f in fams])
x = device.to_device(np.random.default_rng(0).normal(size=3 * sysm.n))
for _ in range(3):
    y = sysm.spmv(x)
xt = device.to_device(cloth.positions + 1e-4 * np.random.default_rng(1).normal(size=cloth.positions.shape))
for _ in range(2):
    g = sysm.gradient(pos, xt, [f.grad for f in fams])
from paper_2308_09400_b200 import elasticity, friction
raw = stencils.evaluate(table, pos, params, dt=1.0, want_energy=False, want_hess=False)
fstate = friction.update_state(table, pos, 0.4, 1e-3, cloth.dt, barrier_batch=raw)
xm = device.to_device(cloth.positions + 5e-6 * np.random.default_rng(4).normal(size=cloth.positions.shape))
for _ in range(2):
    friction.evaluate(fstate, xm, pos)
rng_e = np.random.default_rng(11)      # the bench's elastic workload: 400k private tets
n_tet = 400_000
rest_t = rng_e.normal(size=(4 * n_tet, 3))
mesh_t = elasticity.TetMesh(rest_t, np.arange(4 * n_tet).reshape(n_tet, 4), 3.7e4, 8.6e4)
x_t = device.to_device(rest_t + 0.1 * rng_e.normal(size=rest_t.shape))
for _ in range(2):
    mesh_t.evaluate(x_t, dt=cloth.dt)
sysm.block_jacobi()
sysm.set_symbolic_mode(1)          # the sort-based symbolic phase, for comparison with the row-wise one above
sysm.set_pattern([(f.s, f.vids) for f in fams])
sysm.set_symbolic_mode(0)
sysm.set_pattern([(f.s, f.vids) for f in fams])
sysm.assemble_from_factors([f.fac for f in fams])
if "--pcg" in sys.argv:
    sysm.pcg(-g, 1e-30, 20)
    sysm.mas_order(pos)
    for levels in (1, 2):
        sysm.mas_setup(levels)
        sysm._mas_stale = False
        sysm.pcg(-g, 1e-30, 20, preconditioner="mas", mas_levels=levels)
    sysm.mas_setup(1)
    sysm.mas_apply(g)
torch.cuda.synchronize()
