"""Scratch: where a steady-state Newton iteration of the stepper spends its wall time."""
import sys, time, collections; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2308_09400_b200 import barrier, stepper, workloads, contacts, stencils, solver
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2, jitter_rel=0.01, kappa=1e5)
cfg = stepper.SolverConfig(dt=cloth.dt, barrier=barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa))
state = stepper.SimState(cloth.as_scene(), cfg)
acc = collections.defaultdict(float); cnt = collections.Counter()
def wrap(obj, name, label=None):
    fn = getattr(obj, name)
    def timed(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize(); acc[label or name] += time.perf_counter() - t0; cnt[label or name] += 1
        return r
    setattr(obj, name, timed)
wrap(state.broad, "query", "broad.query"); wrap(contacts, "narrow_phase_device"); wrap(stencils, "evaluate", "stencils.evaluate")
wrap(state.system, "set_pattern"); wrap(state.system, "assemble"); wrap(state.system, "gradient"); wrap(state.system, "pcg")
wrap(state.broad, "ccd_step_bound"); wrap(state, "evaluate_energy"); wrap(state, "min_distance")
for k in range(5):
    if k == 2:
        acc.clear(); cnt.clear(); torch.cuda.synchronize(); t_all = time.perf_counter(); it0 = sum(s.newton_iters for s in state.stats)
    stepper.advance_time_step(state)
torch.cuda.synchronize(); total = time.perf_counter() - t_all
its = sum(s.newton_iters for s in state.stats) - it0
print(f"3 steps, {its} Newton iterations, {total*1e3:.1f} ms total, {total*1e3/its:.2f} ms per iteration")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:22s} {v*1e3:8.2f} ms  {cnt[k]:4d} calls  {v*1e3/cnt[k]:.3f} ms/call")
