"""The GPU time stepper (the Newton / line-search loop around the hot path) against
trajectories of the reference's own ``advance_time_step`` (tests/golden/stepper_*.npz, made by
``make_golden.py --stepper-only``), and the reference's dynamics tests (tests/test_solver.py:166-215)
restated on the device path."""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

# the reference's own bound between its PCG path and a dense direct solve, per step
# (tests/test_solver.py:223-254) is 1e-6 l; measured here: 1e-16 l per step (printed), so the gate is 1e-9 l
# and the Newton / PCG iteration counts must be the reference's.
POS_TOL = 1e-9


@pytest.fixture(scope="module")
def S():
    from paper_2308_09400_b200 import barrier, device, stepper

    return SimpleNamespace(barrier=barrier, device=device, stepper=stepper)


def scene_of(z, positions=None):
    return SimpleNamespace(positions=z["positions"] if positions is None else positions,
                           rest_positions=z["rest_positions"], masses=z["masses"], fixed=z["fixed"], tets=z["tets"],
                           surf_tris=z["surf_tris"], surf_edges=z["surf_edges"], surf_verts=z["surf_verts"],
                           gravity=z["gravity"], bbox_diagonal=float(z["bbox_diagonal"]))


def state_of(S, z, **kw):
    params = S.barrier.BarrierParams(d_hat=float(z["d_hat"]), kappa=float(z["kappa"]))
    cfg = S.stepper.SolverConfig(dt=float(z["dt"]), barrier=params, friction_mu=float(z["friction_mu"]),
                                 friction_eps_v=float(z["friction_eps_v"]), **kw)
    state = S.stepper.SimState(scene_of(z), cfg, (z["tet_mu"], z["tet_lam"]))
    state.v = S.device.to_device(z["v0"].copy())
    return state


@pytest.mark.parametrize("name", ["drop", "slide", "stack"])
def test_trajectory_matches_reference(S, name):
    z = load_golden("stepper_" + name)
    state = state_of(S, z)
    l = state.l
    worst = 0.0
    for k in range(z["xs"].shape[0] - 1):
        # every step starts from the reference's state, so one knife-edge Newton decision cannot
        # compound; the free-running trajectory is checked below
        state.x = S.device.to_device(z["xs"][k].copy())
        state.v = S.device.to_device(z["vs"][k].copy())
        if state.config.friction_mu > 0.0:
            state._refresh_friction(state.x)
        stats = S.stepper.advance_time_step(state)
        err = np.abs(state.positions() - z["xs"][k + 1]).max() / l
        worst = max(worst, err)
        ref = z["stats"][k]
        assert err < POS_TOL, (name, k, err)
        assert stats.converged == bool(ref[5]) and stats.warning == ""
        assert stats.newton_iters == int(ref[0]) and stats.pcg_iters == int(ref[1])
        assert (np.isnan(ref[2]) and np.isnan(stats.min_distance)) or abs(stats.min_distance - ref[2]) < 1e-5 * l
        assert abs(stats.energy - ref[3]) <= 1e-6 * max(abs(ref[3]), 1e-12)
        np.testing.assert_allclose(state.velocities(), z["vs"][k + 1], atol=POS_TOL * l / float(z["dt"]))
    print(f"{name}: worst per-step position error {worst:.2e} l")


@pytest.mark.parametrize("name", ["drop", "slide", "stack"])
def test_free_running_trajectory_stays_close(S, name):
    z = load_golden("stepper_" + name)
    state = state_of(S, z)
    for k in range(z["xs"].shape[0] - 1):
        S.stepper.advance_time_step(state)
    err = np.abs(state.positions() - z["xs"][-1]).max() / state.l
    print(f"{name}: free-running error after {z['xs'].shape[0] - 1} steps {err:.2e} l")
    assert err < 10 * POS_TOL


def test_free_fall_matches_implicit_euler(S):
    """tests/test_solver.py:167-180: no contacts, the step map is x += dt (v += dt g)."""
    z = load_golden("stepper_drop")
    free = ~z["fixed"]
    x_start = z["positions"].copy()
    x_start[free, 2] += 5.0
    params = S.barrier.BarrierParams(d_hat=float(z["d_hat"]), kappa=float(z["kappa"]))
    cfg = S.stepper.SolverConfig(dt=0.02, barrier=params)
    state = S.stepper.SimState(scene_of(z, x_start), cfg, (z["tet_mu"], z["tet_lam"]))
    x0, v = x_start.copy(), np.zeros_like(x_start)
    for _ in range(3):
        stats = S.stepper.advance_time_step(state)
        assert stats.newton_iters <= 2 and np.isnan(stats.min_distance)
        v[free] += cfg.dt * z["gravity"]
        x0 = x0 + cfg.dt * v
        np.testing.assert_allclose(state.positions(), x0, atol=1e-10 * state.l)


def test_newton_step_decreases_energy_and_stays_feasible(S):
    """tests/test_solver.py:182-192."""
    z = load_golden("stepper_drop")
    state = state_of(S, z)
    x0 = state.x.clone()
    x_tilde = state._inertia_target(x0)
    e0 = state.evaluate_energy(x0, x_tilde, x0)
    x1, e1, info = S.stepper.newton_step(state, x0, x_tilde, x0, e0)
    assert info["accepted"] and e1 <= e0 and info["n_contacts"] > 0
    table = state.detect(x1)
    assert state.min_distance(x1, table) > 0.0


def test_drop_lands_without_interpenetration(S):
    """tests/test_solver.py:194-204 on the stacked cubes: 40 steps, every end-of-step distance positive,
    nothing falls through, no line-search collapse."""
    z = load_golden("stepper_stack")
    state = state_of(S, z)
    for _ in range(40):
        stats = S.stepper.advance_time_step(state)
        assert not (stats.min_distance <= 0.0)
    x = state.positions()
    assert x[~z["fixed"], 2].min() > 0.0
    assert not any(s.warning == "line-search-collapse" for s in state.stats)


def test_reference_mode_is_refused(S):
    params = S.barrier.BarrierParams(d_hat=1e-2, kappa=1.0)
    with pytest.raises(NotImplementedError):
        S.stepper.SolverConfig(dt=0.01, barrier=params, mode="reference-ipc")
    with pytest.raises(ValueError):
        S.stepper.SolverConfig(dt=0.0, barrier=params)


def test_time_step_at_bench_scale(S):
    """One whole time step of a 78 400-vertex cloth stack (~1 M contacts at the start): the Newton loop
    converges, every accepted iterate is intersection-free, and the incremental potential does not rise."""
    from paper_2308_09400_b200 import workloads

    cloth = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2, jitter_rel=0.01, kappa=1e5)
    cfg = S.stepper.SolverConfig(dt=cloth.dt, barrier=S.barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa))
    state = S.stepper.SimState(cloth.as_scene(), cfg)
    x0 = state.x.clone()
    assert state.detect(x0).n > 500_000
    e0 = state.evaluate_energy(x0, state._inertia_target(x0), x0)
    stats = S.stepper.advance_time_step(state)
    assert stats.converged and stats.warning == "" and stats.newton_iters < cfg.newton_max_iters
    assert stats.energy <= e0
    assert stats.min_distance > 0.0
    fixed = cloth.fixed
    np.testing.assert_array_equal(state.positions()[fixed], cloth.positions[fixed])
    assert np.all(state.velocities()[fixed] == 0.0)
    state.close()
