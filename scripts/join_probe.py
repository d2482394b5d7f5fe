"""Scratch: one broad-phase query of the bench cloth stack (for ncu -k regex:join_kernel)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import contacts, device, workloads
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2) if len(sys.argv) < 2 or sys.argv[1] == "stack" else workloads.cloth_on_sphere()
pos = device.to_device(cloth.positions)
bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
for _ in range(2):
    vt, ee = bp.query(pos)
torch.cuda.synchronize()
import numpy as np
x = cloth.positions; e = np.asarray(cloth.edges)
el = np.linalg.norm(x[e[:, 1]] - x[e[:, 0]], axis=1)
print("cell", bp.cell, "d_hat", cloth.d_hat, "edge length median %.4g max %.4g" % (np.median(el), el.max()), "bbox", x.min(0), x.max(0))
print("edges", len(cloth.edges), "tris", len(cloth.tris), "vt", int(vt.shape[0]), "ee", int(ee.shape[0]))
