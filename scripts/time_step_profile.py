"""Scratch: one time step of the bench's soft cloth stack under torch.profiler -- wall clock against the sum of
kernel times (is the stepper GPU-bound or host-bound?) and the kernels by total time."""
import sys, time
sys.path.insert(0, ".")
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2308_09400_b200 import barrier, stepper, workloads
soft = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2, jitter_rel=0.01, kappa=1e5)
cfg = stepper.SolverConfig(dt=soft.dt, barrier=barrier.BarrierParams(d_hat=soft.d_hat, kappa=soft.kappa))
state = stepper.SimState(soft.as_scene(), cfg)
for _ in range(2):
    st = stepper.advance_time_step(state)
    print("step", st.newton_iters, st.pcg_iters, "%.1f ms" % st.wall_ms)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    st = stepper.advance_time_step(state)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
tot = sum(e.device_time for e in ev) / 1e3 if ev and hasattr(ev[0], "device_time") else sum(e.cuda_time for e in ev) / 1e3
print("profiled step: newton %d pcg %d wall %.1f ms (under profiler), sum of device activities %.2f ms, %d activities" % (st.newton_iters, st.pcg_iters, wall, tot, len(ev)))
agg = {}
for e in ev:
    d = getattr(e, "device_time", None) or getattr(e, "cuda_time", 0)
    a = agg.setdefault(e.name[:70], [0, 0.0]); a[0] += 1; a[1] += d / 1e3
for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:28]:
    print("%8.3f ms %5d  %s" % (ms, n, name))
