"""Scratch: narrow-phase time on the bench cloth stack."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2308_09400_b200 import workloads, contacts, device
for kw in (dict(d_hat_rel=0.2), dict(d_hat_rel=0.2, jitter_rel=0.01, gap_rel=3.0)):
    cloth = workloads.cloth_stack(layers=4, n=140, seed=1, **kw)
    bp = contacts.BroadPhase(np.unique(cloth.tris), cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
    pos, rest = device.to_device(cloth.positions), device.to_device(cloth.rest_positions)
    vt, ee = bp.query(pos)
    f = lambda: contacts.narrow_phase_device(pos, rest, vt, ee, cloth.d_hat, want_origin=False)
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(30): tab, _ = f()
    torch.cuda.synchronize(); print("narrow %.3f ms" % ((time.perf_counter() - t0) / 30 * 1e3), "queries", vt.shape[0] + ee.shape[0], "contacts", tab.n)
