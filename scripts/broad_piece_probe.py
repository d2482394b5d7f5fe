"""Scratch: host-side pieces of BroadPhase.query on the settled cloth stack."""
import sys, time, ctypes as C; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2308_09400_b200 import workloads, contacts, device, _lib
gap = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2, jitter_rel=0.01, gap_rel=gap)
cf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
bp = contacts.BroadPhase(np.unique(cloth.tris), cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
if cf:
    bp.cell *= cf
print('cell', bp.cell)
pos = device.to_device(cloth.positions)
def t(fn, reps=50):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): r = fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3, r
ms, r = t(lambda: bp.query(pos)); print("query %.3f ms" % ms, r[0].shape[0], r[1].shape[0])
ms, _ = t(lambda: pos.amin(dim=0).cpu().numpy()); print("amin+cpu %.3f ms" % ms)
lo = pos.amin(dim=0).cpu().numpy() - 2.0 * bp.cell
origin = (C.c_double * 3)(*[float(v) for v in lo]); n_vt, n_ee = C.c_int64(0), C.c_int64(0); L = _lib.lib()
def count():
    L.b200ipc_broad_phase_count(bp._h, pos.shape[0], device.ptr(pos), bp.surf_verts.shape[0], device.ptr(bp.surf_verts),
        bp.tris.shape[0], device.ptr(bp.tris), bp.edges.shape[0], device.ptr(bp.edges), bp.d_hat, bp.cell, origin,
        C.byref(n_vt), C.byref(n_ee), device.stream())
ms, _ = t(count); print("count call %.3f ms" % ms)
def fill():
    vt = device.empty((max(int(n_vt.value), 1), 4), np.int32); ee = device.empty((max(int(n_ee.value), 1), 4), np.int32)
    L.b200ipc_broad_phase_fill(bp._h, device.ptr(vt), device.ptr(ee), device.stream())
ms, _ = t(fill); print("alloc+fill %.3f ms" % ms)
