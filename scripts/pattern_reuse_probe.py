"""Scratch: how often do consecutive Newton iterations see the identical contact families?"""
import sys; sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import barrier, stepper, workloads, device, elasticity
def run(state, steps, label):
    sysm = state.system; orig = sysm.set_pattern; last = [None]; hits = [0, 0]
    def probe(fams):
        fams = list(fams)
        same = last[0] is not None and len(last[0]) == len(fams) and all(
            a[0] == b[0] and a[1].shape == b[1].shape and bool(torch.equal(a[1], b[1])) for a, b in zip(last[0], fams))
        hits[0] += int(same); hits[1] += 1; last[0] = [(s, v.clone()) for s, v in fams]
        return orig(fams)
    sysm.set_pattern = probe
    for _ in range(steps): stepper.advance_time_step(state)
    print(label, "identical pattern in %d of %d Newton iterations" % tuple(hits))
cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2, jitter_rel=0.01, kappa=1e5)
st = stepper.SimState(cloth.as_scene(), stepper.SolverConfig(dt=cloth.dt, barrier=barrier.BarrierParams(cloth.d_hat, cloth.kappa)))
run(st, 5, "cloth stack")
sc = workloads.cube_drop(k=12, tilt=0.5)
st = stepper.SimState(sc, stepper.SolverConfig(dt=sc.dt, barrier=barrier.BarrierParams(sc.d_hat, sc.kappa), friction_mu=0.3), elasticity.ElasticMaterial(1e5, 0.4))
st.v = device.to_device(sc.v0.copy())
run(st, 40, "cube drop")
