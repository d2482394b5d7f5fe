"""Scratch: A/B the streamed (TMA-staged) SpMV / PCG against the direct-load kernels on the bench scene."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads
import bench

layers = int(os.environ.get("PROBE_LAYERS", "4")); n = int(os.environ.get("PROBE_N", "140"))
cloth = workloads.cloth_stack(layers=layers, n=n, seed=1, d_hat_rel=0.2)
vt, ee = workloads.broad_phase(cloth)
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
pos = device.to_device(cloth.positions)
table, _ = contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
batch = stencils.evaluate(table, pos, params, dt=cloth.dt)
fams = [batch.families[s] for s in sorted(batch.families)]
sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
nnzb = sysm.set_pattern([(f.s, f.vids) for f in fams])
sysm.assemble([f.hess for f in fams])
rp = device.to_host(sysm.rowptr).astype(np.int64)
rl = np.diff(rp)
print("n", sysm.n, "nnzb", nnzb, "row len mean/max", rl.mean(), rl.max(), flush=True)
for R in (16, 24, 32):
    cb = rp[np.minimum(np.arange(0, sysm.n + R, R), sysm.n)]
    c = np.diff(cb)
    print("R", R, "chunk blocks mean/max", c.mean(), c.max(), "over 888:", int((c > 888).sum()), "of", len(c), flush=True)
noop = lambda: None
x = device.to_device(np.random.default_rng(0).normal(size=3 * sysm.n)); y = device.empty((3 * sysm.n,))
os.environ["B200IPC_SPMV_MODE"] = "legacy"
sysm.spmv(x, out=y); ref = device.to_host(y).copy()
print("legacy spmv ms", bench.time_steps(torch, lambda: sysm.spmv(x, out=y), 100, 5, noop) / 100, flush=True)
os.environ["B200IPC_SPMV_MODE"] = "stream"
for R, PF in (("12", "0"), ("18", "0"), ("24", "0"), ("30", "0")):
    os.environ["B200IPC_SPMV_ROWS_PER_CHUNK"] = R
    os.environ["B200IPC_SPMV_PREFETCH_X"] = PF
    y.zero_(); sysm.spmv(x, out=y); got = device.to_host(y)
    print("stream R", R, "pf", PF, "bitwise equal", bool(np.array_equal(got, ref)), "max abs diff", float(np.abs(got - ref).max()),
          "ms", bench.time_steps(torch, lambda: sysm.spmv(x, out=y), 100, 5, noop) / 100, flush=True)
del os.environ["B200IPC_SPMV_ROWS_PER_CHUNK"]; del os.environ["B200IPC_SPMV_PREFETCH_X"]
xt = device.to_device(cloth.positions + 1e-4 * np.random.default_rng(1).normal(size=cloth.positions.shape))
rhs = -sysm.gradient(pos, xt, [f.grad for f in fams])
sysm.block_jacobi()
res = {}
for mode in ("legacy", "stream"):
    os.environ["B200IPC_SPMV_MODE"] = mode
    sysm.pcg(rhs, 1e-30, 5)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d, iters, ok, _, _ = sysm.pcg(rhs, 1e-30, 200)
    torch.cuda.synchronize()
    print("pcg", mode, "ms/iter", (time.perf_counter() - t0) * 1e3 / iters, flush=True)
    d, iters, ok, d0, dn = sysm.pcg(rhs, 1e-4, 2000)
    res[mode] = (device.to_host(d).copy() if hasattr(d, "device") else np.asarray(d), iters, ok)
    print("pcg", mode, "to 1e-4: iters", iters, "converged", ok, flush=True)
print("pcg solutions bitwise equal", bool(np.array_equal(res["legacy"][0], res["stream"][0])),
      "max abs diff", float(np.abs(res["legacy"][0] - res["stream"][0]).max()))
