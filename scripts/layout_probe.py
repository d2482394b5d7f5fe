"""Dense-block device layout: the reference's row-major (nb,3s,3s) against sub-block-major (nb,s,s,3,3) on the
bench cloth stack (1.03 M contacts) -- stencil kernel and numeric assembly, both layouts, same matrix bit for bit."""
import os
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import bench
from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads

which = sys.argv[1] if len(sys.argv) > 1 else "stack"
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2) if which == "stack" else workloads.cloth_on_sphere()
vt, ee = workloads.broad_phase(cloth)
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
pos = device.to_device(cloth.positions)
table, _ = contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
out = {}
vals = {}
N, W = (1, 0) if os.environ.get("LAYOUT_PROBE_QUICK") else (50, 5)   # under ncu: one launch of each
for layout in ("dense", "subblock"):
    batch = stencils.evaluate(table, pos, params, dt=cloth.dt, hess_layout=layout)
    fams = [batch.families[s] for s in sorted(batch.families)]
    sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
    sysm.set_pattern([(f.s, f.vids) for f in fams], tiled=[f.tiled for f in fams])
    hess = [f.hess for f in fams]
    ms_st = bench.time_steps(torch, lambda: stencils.evaluate(table, pos, params, dt=cloth.dt, out=batch, hess_layout=layout), N, W) / N
    for variant in ((1,) if N == 1 else (1, 2)):
        sysm.set_numeric_variant(variant)
        ms = bench.time_steps(torch, lambda: sysm.assemble(hess), N, W) / N
        out[(layout, variant)] = ms
        vals[(layout, variant)] = device.to_host(sysm.vals).copy()
    out[(layout, "stencil")] = ms_st
    print(layout, "contacts", table.n, "nnzb", sysm.nnzb, "stencil %.4f ms" % ms_st,
          "numeric walker1 %.4f ms walker2 %.4f ms" % (out[(layout, 1)], out.get((layout, 2), float("nan"))), flush=True)
    sysm.close()
for variant in ((1,) if N == 1 else (1, 2)):
    assert np.array_equal(vals[("dense", variant)], vals[("subblock", variant)])
print("bitwise equal matrices")
