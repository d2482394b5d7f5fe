"""Scratch timing of the stencil kernel (NOT bench.py): table built by the GPU narrow phase."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch

from paper_2308_09400_b200 import barrier, contacts, proximity, stencils, workloads, device, _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
which = sys.argv[2] if len(sys.argv) > 2 else "c2"
t0 = time.time()
qb = workloads.config2_batch(n=n) if which == "c2" else workloads.config1_batch(n_pt=n // 2, n_ee=n // 2)
dt, extra = contacts.narrow_phase_device(qb.positions, qb.rest_positions, qb.vt, qb.ee, qb.d_hat, want_origin=False)
tab = {"kind": device.to_host(extra.kind)}
print("setup s", time.time() - t0, "rows", dt.n, "kinds", np.diff(dt.kind_off).tolist(), flush=True)
params = barrier.BarrierParams(d_hat=qb.d_hat, kappa=qb.kappa)
pos = device.to_device(qb.positions)
batch = stencils.evaluate(dt, pos, params)
torch.cuda.synchronize()
for label, kw in (("all", {}), ("hess_only", dict(want_energy=False, want_grad=False)), ("energy_only", dict(want_grad=False, want_hess=False))):
    b = stencils.evaluate(dt, pos, params, **kw)
    for _ in range(3):
        stencils.evaluate(dt, pos, params, out=b, **kw)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    reps = 20
    ev[0].record()
    for _ in range(reps):
        stencils.evaluate(dt, pos, params, out=b, **kw)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    nbytes = sum(1272 if s == 4 else (740 if s == 3 else 352) for s in proximity.KIND_SIZE[tab["kind"]])
    print(json.dumps({"case": label, "ms": ms, "stencils_per_s": dt.n / ms * 1e3, "GBps_alg": nbytes / ms / 1e6}), flush=True)
print("launches", _lib.lib().b200ipc_launch_count())
