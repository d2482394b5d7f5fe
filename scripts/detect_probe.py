"""Scratch: time the detect stages (broad, narrow, CCD sweep + filter) on the bench scene."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import contacts, device, workloads
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
pos = device.to_device(cloth.positions)
rest = device.to_device(cloth.rest_positions)
bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
dirs = device.to_device(0.3 * cloth.d_hat * np.random.default_rng(3).normal(size=cloth.positions.shape))
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): out = fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3 / reps, out
ms, (vt, ee) = timed(lambda: bp.query(pos)); print("broad ms", ms, vt.shape[0], ee.shape[0])
ms, _ = timed(lambda: contacts.narrow_phase_device(pos, rest, vt, ee, cloth.d_hat, want_origin=False)); print("narrow ms", ms)
ms, (svt, see) = timed(lambda: bp.sweep(pos, dirs)); print("sweep ms", ms, svt.shape[0], see.shape[0])
ms, a = timed(lambda: contacts.ccd_filter_device(svt, see, pos, dirs)); print("ccd filter ms", ms, a)
med = float(np.median(np.linalg.norm(cloth.positions[cloth.edges[:, 1]] - cloth.positions[cloth.edges[:, 0]], axis=1)))
print("median edge", med, "d_hat", cloth.d_hat, "default cell", bp.cell)
for f in (0.25, 0.4, 0.5, 0.7, 1.0, 1.5):
    b2 = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions, cell=f * med)
    ms, (v2, e2) = timed(lambda: b2.query(pos)); print("cell", f, "x median edge: broad ms", ms, v2.shape[0], e2.shape[0])
    b2.close()
