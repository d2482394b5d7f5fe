"""Scratch: time streamed SpMV and PCG/iter for tuning builds (one subprocess per library)."""
import os, subprocess, sys, time
import numpy as np
sys.path.insert(0, ".")
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads
    import bench
    cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
    z = np.load("/tmp/variant_scene.npz"); vt, ee = z["vt"], z["ee"]
    params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
    pos = device.to_device(cloth.positions)
    table, _ = contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
    batch = stencils.evaluate(table, pos, params, dt=cloth.dt)
    fams = [batch.families[s] for s in sorted(batch.families)]
    sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
    sysm.set_pattern([(f.s, f.vids) for f in fams]); sysm.assemble([f.hess for f in fams])
    x = device.to_device(np.random.default_rng(0).normal(size=3 * sysm.n)); y = device.empty((3 * sysm.n,))
    out = []
    for R in os.environ.get("PROBE_R", "0").split(","):
        if R != "0": os.environ["B200IPC_SPMV_ROWS_PER_CHUNK"] = R
        sp = bench.time_steps(torch, lambda: sysm.spmv(x, out=y), 100, 5) / 100
        xt = device.to_device(cloth.positions + 1e-4 * np.random.default_rng(1).normal(size=cloth.positions.shape))
        rhs = -sysm.gradient(pos, xt, [f.grad for f in fams])
        sysm.block_jacobi(); sysm.pcg(rhs, 1e-30, 5)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        d, iters, ok, _, _ = sysm.pcg(rhs, 1e-30, 300)
        torch.cuda.synchronize(); pc = (time.perf_counter() - t0) * 1e3 / iters
        out.append("R=%s spmv %.2f us pcg %.2f us/iter" % (R, sp * 1e3, pc * 1e3))
    print(os.path.basename(os.environ.get("B200IPC_LIB", "default")), " | ".join(out), flush=True)
    sys.exit(0)
from paper_2308_09400_b200 import workloads
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
vt, ee = workloads.broad_phase(cloth)
np.savez("/tmp/variant_scene.npz", vt=vt, ee=ee)
for spec in sys.argv[1:]:
    lib, _, rs = spec.partition(":")
    env = dict(os.environ, B200IPC_LIB=os.path.abspath(lib), PROBE_R=rs or "0")
    subprocess.run([sys.executable, __file__, "--child"], env=env)
