"""Scratch: time Newton-step kernels on the bench's cloth stack for a few tuning knobs."""
import os, sys, time, json
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads
import bench

cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
vt, ee = workloads.broad_phase(cloth)
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
pos = device.to_device(cloth.positions)
table, _ = contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
batch = stencils.evaluate(table, pos, params, dt=cloth.dt, want_factors=True)
fams = [batch.families[s] for s in sorted(batch.families)]
sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
nnzb = sysm.set_pattern([(f.s, f.vids) for f in fams])
hess = [f.hess for f in fams]
noop = lambda: None
for variant in (0, 1, 4):
    sysm.set_numeric_variant(variant)
    ms = bench.time_steps(torch, lambda: sysm.assemble(hess), 20, 3, noop) / 20
    print("assemble variant", variant, "ms", ms, flush=True)
fac = [f.fac for f in fams]
print("assemble from factors ms", bench.time_steps(torch, lambda: sysm.assemble_from_factors(fac), 20, 3, noop) / 20, flush=True)
lean = stencils.evaluate(table, pos, params, dt=cloth.dt, want_hess=False, want_factors=True)
print("stencils factors-only ms", bench.time_steps(torch, lambda: stencils.evaluate(table, pos, params, dt=cloth.dt, want_hess=False, want_factors=True, out=lean), 20, 3, noop) / 20, flush=True)
print("stencils dense ms", bench.time_steps(torch, lambda: stencils.evaluate(table, pos, params, dt=cloth.dt, want_factors=True, out=batch), 20, 3, noop) / 20, flush=True)
sysm.set_numeric_variant(0); sysm.assemble(hess)
x = device.to_device(np.random.default_rng(0).normal(size=3 * sysm.n)); y = device.empty((3 * sysm.n,))
print("spmv ms", bench.time_steps(torch, lambda: sysm.spmv(x, out=y), 50, 5, noop) / 50, flush=True)
xt = device.to_device(cloth.positions + 1e-4 * np.random.default_rng(1).normal(size=cloth.positions.shape))
rhs = -sysm.gradient(pos, xt, [f.grad for f in fams])
sysm.block_jacobi()
for per_sm in ("1", "2", "4", "8"):
    os.environ["B200IPC_PCG_CTAS_PER_SM"] = per_sm
    sysm.pcg(rhs, 1e-30, 5)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d, iters, ok, _, _ = sysm.pcg(rhs, 1e-30, 100)
    print("pcg ctas/sm", per_sm, "ms/iter", (time.perf_counter() - t0) * 1e3 / iters, flush=True)
