"""Scratch: one broad-phase query of the bench cloth stack (for ncu -k regex:join_kernel)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import contacts, device, workloads
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
pos = device.to_device(cloth.positions)
bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
for _ in range(2):
    vt, ee = bp.query(pos)
torch.cuda.synchronize()
print("edges", len(cloth.edges), "tris", len(cloth.tris), "vt", int(vt.shape[0]), "ee", int(ee.shape[0]))
