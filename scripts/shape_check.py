"""Scratch: Newton direction on other scene shapes, cross-checked (SpMV vs matrix-free, PCG residual)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import barrier, contacts, device, kernels, solver, stencils, workloads
for layers, n, rel in ((8, 100, 0.2), (2, 224, 0.2), (6, 60, 0.5), (12, 40, 0.35)):
    cloth = workloads.cloth_stack(layers=layers, n=n, seed=3, d_hat_rel=rel)
    bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
    vt, ee = bp.query(cloth.positions)
    table, _ = contacts.narrow_phase_device(cloth.positions, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
    params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
    batch = stencils.evaluate(table, cloth.positions, params, dt=cloth.dt, want_factors=True)
    fams = [batch.families[s] for s in sorted(batch.families)]
    sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
    nnzb = sysm.set_pattern([(f.s, f.vids) for f in fams])
    a1 = sysm.assemble([f.hess for f in fams]).clone()
    a2 = sysm.assemble_from_factors([f.fac for f in fams])
    rp = device.to_host(sysm.rowptr); rl = np.diff(rp)
    t = torch
    rng = np.random.default_rng(0)
    x = device.to_device(rng.normal(size=3 * sysm.n)); y = sysm.spmv(x)
    free = t.from_numpy(~cloth.fixed).cuda().repeat_interleave(3)
    xm = t.where(free, x, t.zeros_like(x)); out = t.repeat_interleave(sysm.masses, 3) * xm
    for f in fams: kernels.matvec_blocks_device(f.hess, f.vids, xm, out)
    out = t.where(free, out, x)
    xt = device.to_device(cloth.positions + 1e-4 * rng.normal(size=cloth.positions.shape))
    rhs = -sysm.gradient(cloth.positions, xt, [f.grad for f in fams])
    sysm.pcg(rhs, 1e-4, 3)   # warm: workspace allocation, lazy module load
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d, iters, ok, d0, dn = sysm.pcg(rhs, 1e-4, 5000)
    torch.cuda.synchronize(); ms = (time.perf_counter() - t0) * 1e3
    alpha = bp.ccd_step_bound(cloth.positions, device.to_host(d).reshape(-1, 3))
    print(f"{layers}x{n}: verts {sysm.n} contacts {table.n} nnzb {nnzb} rowlen mean {rl.mean():.1f} max {rl.max()} | "
          f"dense==factor {bool((a1 == a2).all())} spmv err {float((y - out).abs().max() / out.abs().max()):.2e} | "
          f"pcg {iters} it {ms:.2f} ms ok {ok} | ccd alpha {alpha:.4f} | penetrating {batch.summary()[2]}", flush=True)
    sysm.close(); bp.close()
