"""Scratch: per-phase PCG timers (library built with B200IPC_PCG_TIMING=1)."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
vt, ee = workloads.broad_phase(cloth)
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
pos = device.to_device(cloth.positions)
table, _ = contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
batch = stencils.evaluate(table, pos, params, dt=cloth.dt)
fams = [batch.families[s] for s in sorted(batch.families)]
sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
sysm.set_pattern([(f.s, f.vids) for f in fams]); sysm.assemble([f.hess for f in fams])
xt = device.to_device(cloth.positions + 1e-4 * np.random.default_rng(1).normal(size=cloth.positions.shape))
rhs = -sysm.gradient(pos, xt, [f.grad for f in fams])
sysm.block_jacobi()
for _ in range(3): sysm.spmv(rhs)
sysm.pcg(rhs, 1e-30, 5)
torch.cuda.synchronize(); t0 = time.perf_counter()
d, iters, ok, _, _ = sysm.pcg(rhs, 1e-30, 200)
torch.cuda.synchronize(); print("ms/iter", (time.perf_counter() - t0) * 1e3 / iters)
ws = device.to_host(sysm._pcg_ws)
part = ws[21 * sysm.n:]
for k, name in enumerate(("product+blocksum", "sync1+sumparts", "update+blocksum", "sync2+sumparts")):
    t = part[1024 + 512 * k: 1024 + 512 * k + 148] / iters / 1e3
    print(name, "us/iter: min %.2f mean %.2f max %.2f" % (t.min(), t.mean(), t.max()))
dbg = part[3072:3072 + 3 * 148].view(np.uint64).reshape(148, 3).astype(np.float64) / iters / 1.965e3
for k, name in enumerate(("consumer warp0 wait-full", "consumer warp0 compute", "producer wait-empty")):
    print(name, "us/iter: min %.2f mean %.2f max %.2f" % (dbg[:, k].min(), dbg[:, k].mean(), dbg[:, k].max()))
