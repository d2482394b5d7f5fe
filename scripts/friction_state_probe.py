"""Scratch: where update_state's time goes (per stage, synchronised)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import barrier, contacts, device, friction, stencils, workloads
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
vt, ee = workloads.broad_phase(cloth)
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
pos = device.to_device(cloth.positions)
table, _ = contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
raw = stencils.evaluate(table, pos, params, dt=1.0, want_energy=False, want_hess=False)
def T(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best, out
print("update_state total %.3f ms" % T(lambda: friction.update_state(table, pos, 0.4, 1e-3, cloth.dt, barrier_batch=raw))[0])
st = friction.update_state(table, pos, 0.4, 1e-3, cloth.dt, barrier_batch=raw)
n = table.n
status = torch.zeros(n, dtype=torch.uint8, device="cuda")
frame = torch.empty((n, 12), dtype=torch.float64, device="cuda")
ok = status == 0
print("cumsum+cat %.3f" % T(lambda: torch.cat([torch.zeros(1, dtype=torch.int64, device="cuda"), torch.cumsum(ok, 0, dtype=torch.int64)]))[0])
print("nonzero %.3f" % T(lambda: torch.nonzero(ok).squeeze(1))[0])
keep = torch.nonzero(ok).squeeze(1)
print("frame index_select %.3f" % T(lambda: frame.index_select(0, keep))[0])
print("frame [keep] %.3f" % T(lambda: frame[keep].contiguous())[0])
print("verts index_select %.3f" % T(lambda: table.verts.index_select(0, keep))[0])
print("sub/eps index_select %.3f" % T(lambda: (table.sub.index_select(0, keep), table.eps_x.index_select(0, keep)))[0])
print("alloc frame+status %.3f" % T(lambda: (device.empty((n, 12)), device.empty((n,), np.uint8)))[0])
