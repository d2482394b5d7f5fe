"""Scratch: numeric assembly variants at bench scale (CUDA-event times, values compared)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
exec(open("scripts/mas_probe.py").read().split("xt = device.to_device")[0])
import torch
def ev(fn, reps=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
hess = [f.hess for f in fams] if fams[0].hess is not None else None
if hess is None:
    batch = stencils.evaluate(table, pos, params, dt=cloth.dt, want_factors=True)
    fams = [batch.families[s] for s in sorted(batch.families)]
    hess = [f.hess for f in fams]
fac = [f.fac for f in fams]
ref = None
for variant in (1, 2, 4):
    sysm.set_numeric_variant(variant)
    t = ev(lambda: sysm.assemble(hess))
    v = sysm.vals.clone()
    if ref is None: ref = v
    print(f"dense variant {variant}: {t*1e3:.1f} us   max|diff| vs v1 = {(v-ref).abs().max().item():.3e} (scale {ref.abs().max().item():.3e})")
for variant in (1, 0):
    sysm.set_numeric_variant(variant)
    t = ev(lambda: sysm.assemble_from_factors(fac))
    v = sysm.vals.clone()
    print(f"factors variant {variant}: {t*1e3:.1f} us   max|diff| vs dense v1 = {(v-ref).abs().max().item():.3e}")
