"""Per-stage wall times (synchronised) of the bench's Newton direction e2e on a cloth stack, several calls in a row.
    python scripts/direction_stage_probe.py [layers n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads

layers, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8, 180)
cloth = workloads.cloth_stack(layers=layers, n=n, seed=3, d_hat_rel=0.2)
params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
d_rest = device.to_device(cloth.rest_positions)
bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
x_host = np.ascontiguousarray(cloth.positions)
xt_host = x_host + 1e-4 * np.random.default_rng(0).normal(size=x_host.shape)


def run(prec):
    marks = []

    def mark(name):
        torch.cuda.synchronize()
        marks.append((name, time.perf_counter()))

    mark("start")
    px, pxt = device.to_device(x_host), device.to_device(xt_host)
    mark("h2d")
    cvt, cee = bp.query(px)
    mark("broad")
    tab, _ = contacts.narrow_phase_device(px, d_rest, cvt, cee, cloth.d_hat, want_origin=False)
    mark("narrow")
    b = stencils.evaluate(tab, px, params, dt=cloth.dt, want_hess=False, want_factors=True)
    mark("stencils")
    fl = [b.families[s_] for s_ in sorted(b.families)]
    sysm.set_pattern([(f.s, f.vids) for f in fl])
    mark("symbolic")
    sysm.assemble_from_factors([f.fac for f in fl])
    mark("numeric")
    g = sysm.gradient(px, pxt, [f.grad for f in fl])
    mark("gradient")
    sysm.block_jacobi()
    mark("block_jacobi")
    if prec == "mas":
        sysm.mas_order(px)
        mark("mas_order")
    dd, its, okk, _, _ = sysm.pcg(-g, 1e-4, 4000, preconditioner=prec)
    mark("pcg")
    out = device.to_host(dd)
    e = float(b.summary()[0])
    mark("d2h")
    return [(b_[0], (b_[1] - a_[1]) * 1e3) for a_, b_ in zip(marks, marks[1:])], its


for prec in ("block_jacobi", "mas", "block_jacobi"):
    for rep in range(4):
        stages, its = run(prec)
        print(prec, rep, "iters", its, "total %.2f ms |" % sum(v for _, v in stages),
              " ".join("%s %.2f" % kv for kv in stages), flush=True)
