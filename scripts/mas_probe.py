"""Scratch: block-Jacobi vs MAS PCG on the bench scenes (iterations, wall ms incl. setup)."""
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
sysm.set_pattern([(f.s, f.vids) for f in fams])
sysm.assemble_from_factors([f.fac for f in fams])
xt = device.to_device(cloth.positions + 1e-4 * np.random.default_rng(1).normal(size=cloth.positions.shape))
g = sysm.gradient(pos, xt, [f.grad for f in fams])
rhs = -g

def wall(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best, out

t, out = wall(lambda: sysm.pcg(rhs, 1e-4, 5000))
print(f"block-jacobi: {t:.3f} ms, iters {out[1]}, {t/max(out[1],1)*1e3:.1f} us/iter")
t, _ = wall(lambda: sysm.mas_order(pos))
print(f"mas_order: {t:.3f} ms")
for levels in (1, 2):
    t, _ = wall(lambda: sysm.mas_setup(levels))
    print(f"mas_setup levels={levels}: {t:.3f} ms")
    sysm._mas_stale = False
    t, out = wall(lambda: sysm.pcg(rhs, 1e-4, 5000, preconditioner="mas", mas_levels=levels))
    print(f"mas pcg levels={levels}: {t:.3f} ms, iters {out[1]}, {t/max(out[1],1)*1e3:.1f} us/iter, converged {out[2]}")
r = device.to_device(np.random.default_rng(0).normal(size=3 * sysm.n))
sysm.mas_setup(1)
t, _ = wall(lambda: sysm.mas_apply(r))
print(f"mas_apply (standalone, 1 level): {t*1e3:.1f} us")
