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


def test_host_arrays_are_accepted_like_the_reference(S):
    """The reference passes NumPy arrays around; the device path takes them at its entry points."""
    z = load_golden("stepper_drop")
    state = state_of(S, z)
    x0 = z["positions"].copy()
    state.v = z["v0"].copy()                                  # a host array, as reference code would assign
    x_tilde = state._inertia_target(x0)
    e0 = state.evaluate_energy(x0, S.device.to_host(x_tilde), x0)
    x1, e1, info = S.stepper.newton_step(state, x0, S.device.to_host(x_tilde), x0, e0)
    assert info["accepted"] and e1 <= e0
    state.x = x0
    stats = S.stepper.advance_time_step(state)
    assert abs(np.abs(state.positions() - z["xs"][1]).max()) < POS_TOL * state.l and stats.converged


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


def _cube_state(S, k, friction_mu):
    from paper_2308_09400_b200 import elasticity, workloads

    sc = workloads.cube_drop(k=k, tilt=0.5)
    cfg = S.stepper.SolverConfig(dt=sc.dt, barrier=S.barrier.BarrierParams(sc.d_hat, sc.kappa), friction_mu=friction_mu)
    state = S.stepper.SimState(sc, cfg, elasticity.ElasticMaterial(1e5, 0.4))
    state.v = S.device.to_device(sc.v0.copy())
    return sc, state


def test_all_seven_families_in_one_newton_matrix(S):
    """Elastic tets + barrier 6/9/12 + friction 6/9/12 blocks of a cube-drop scene through one pattern:
    the assembled SpMV equals mass + the sum of the families' block products (an independent kernel)."""
    from paper_2308_09400_b200 import kernels

    t = S.device.torch()
    sc, state = _cube_state(S, 6, 0.3)
    rng = np.random.default_rng(5)
    x0 = state.x
    x = x0 + S.device.to_device(np.where(sc.fixed[:, None], 0.0, 2e-4 * rng.normal(size=sc.positions.shape)))
    table = state.detect(x)
    fams = state.assemble_local_quadratics(x, x0, table)
    sizes = sorted(f.s for f in fams)
    assert sizes.count(4) >= 3 and len(fams) >= 4, sizes          # elastic, barrier and friction 12x12 at least
    assert state.friction_state.n > 0 and table.n > 0
    sysm = state.system
    sysm.set_pattern([(f.s, f.vids) for f in fams])
    sysm.assemble([f.hess for f in fams])
    v = S.device.to_device(rng.normal(size=3 * state.n))
    y = sysm.spmv(v)
    free = (~state._fixed_dev).repeat_interleave(3)
    vm = t.where(free, v, t.zeros_like(v))
    ref = t.repeat_interleave(sysm.masses, 3) * vm
    for f in fams:
        kernels.matvec_blocks_device(f.hess, f.vids, vm, ref)
    ref = t.where(free, ref, v)
    assert float((y - ref).abs().max()) <= 1e-11 * float(ref.abs().max())
    # and the gradient: M (x - x~) + scattered family gradients, fixed rows zero
    x_tilde = state._inertia_target(x0)
    g = state.gradient(x, x_tilde, fams).reshape(-1, 3)
    want = sysm.masses[:, None] * (x - x_tilde)
    for f in fams:
        want.index_add_(0, f.vids.reshape(-1), f.grad.reshape(-1, 3))
    want[state._fixed_dev] = 0.0
    assert float((g - want).abs().max()) <= 1e-11 * float(want.abs().max())
    state.close()


def test_cube_drop_with_friction_bounces_without_interpenetration(S):
    """144 elastic cubes dropping on a floor with friction 0.3, eight steps: every step converges, contacts
    switch on and off, nothing crosses the floor, fixed vertices stay put."""
    sc, state = _cube_state(S, 12, 0.3)
    seen_contact = seen_free = False
    for _ in range(8):
        stats = S.stepper.advance_time_step(state)
        assert stats.converged and stats.warning == ""
        assert np.isnan(stats.min_distance) or stats.min_distance > 0.0
        seen_contact |= not np.isnan(stats.min_distance)
        seen_free |= bool(np.isnan(stats.min_distance))
    x = state.positions()
    assert seen_contact and seen_free
    assert x[~sc.fixed, 2].min() > 0.0
    np.testing.assert_array_equal(x[sc.fixed], sc.positions[sc.fixed])
    state.close()


def test_assembly_path_raises_on_interpenetration(S):
    """The reference's assemble_local_quadratics -> _barrier_block -> build_diagonal_jacobian raises
    InterpenetrationError on d2 <= 0 (gap.py:61-62); the device path must not hand back a direction built from
    silently zeroed blocks."""
    from paper_2308_09400_b200 import proximity
    from paper_2308_09400_b200.gap import InterpenetrationError

    z = load_golden("stepper_drop")
    state = state_of(S, z)
    x = state.positions().copy()
    # a point-point stencil over two coincident vertices: d2 = 0
    x[1] = x[0]
    table = proximity.StencilTable(np.array([4], np.uint8), np.array([[0, 1, -1, -1]], np.int32), np.zeros(1, np.uint8),
                                   np.zeros(1))
    from paper_2308_09400_b200.stencils import DeviceStencilTable

    dev = DeviceStencilTable.from_host(table)
    xd = S.device.to_device(x)
    with pytest.raises(InterpenetrationError):
        state.assemble_local_quadratics(xd, xd, dev)
    state.close()


def test_mas_preconditioner_through_the_time_stepper(S):
    """SolverConfig.preconditioner = "mas": same stopping rules (PCG and Newton), so the trajectory stays within the
    Newton tolerance of the block-Jacobi run, with fewer PCG iterations on a contact-dominated cloth stack."""
    from paper_2308_09400_b200 import workloads

    soft = workloads.cloth_stack(layers=4, n=40, seed=1, d_hat_rel=0.2, jitter_rel=0.01, kappa=1e5)
    out = {}
    for prec in ("block_jacobi", "mas"):
        cfg = S.stepper.SolverConfig(dt=soft.dt, barrier=S.barrier.BarrierParams(d_hat=soft.d_hat, kappa=soft.kappa),
                                     preconditioner=prec)
        state = S.stepper.SimState(soft.as_scene(), cfg)
        stats = [S.stepper.advance_time_step(state) for _ in range(2)]
        out[prec] = (state.positions(), sum(st.pcg_iters for st in stats), [st.converged for st in stats], state.l)
        state.close()
    (xa, ita, oka, l), (xb, itb, okb, _) = out["block_jacobi"], out["mas"]
    assert all(oka) and all(okb)
    # both runs stop Newton at |d|_inf <= eps_d l dt (solver.py:393): they agree to that tolerance per step
    assert np.abs(xa - xb).max() <= 2 * 2 * cfg.eps_d * l * soft.dt
    assert itb < ita, (itb, ita)


def test_mas_on_a_seven_family_matrix(S):
    """Elastic + barrier + friction families in one matrix (the row-wise numeric kernel, > 3 families) solved with the
    MAS preconditioner, two levels: same steps converge, the cubes land in the same place to the Newton tolerance."""
    out = {}
    for prec in ("block_jacobi", "mas"):
        sc, state = _cube_state(S, 8, 0.3)
        state.config.preconditioner = prec
        state.config.mas_levels = 2
        stats = [S.stepper.advance_time_step(state) for _ in range(6)]
        assert all(st.converged and st.warning == "" for st in stats)
        out[prec] = (state.positions(), state.l, state.config)
        state.close()
    (xa, l, cfg), (xb, _, _) = out["block_jacobi"], out["mas"]
    assert np.abs(xa - xb).max() <= 2 * 6 * cfg.eps_d * l * cfg.dt


def test_auto_preconditioner_switches_on_hard_solves_only(S):
    """SolverConfig.preconditioner = "auto" (the paper's "trial both, keep the faster"): a stiff contact stack whose
    block-Jacobi solves exceed the threshold switches to MAS inside the step; below the threshold it never does."""
    from paper_2308_09400_b200 import workloads

    for kappa, threshold, expect_switch in ((2e8, 40, True), (1e5, 1000, False)):
        sc = workloads.cloth_stack(layers=4, n=40, seed=1, d_hat_rel=0.2, jitter_rel=0.01, kappa=kappa)
        cfg = S.stepper.SolverConfig(dt=sc.dt, barrier=S.barrier.BarrierParams(d_hat=sc.d_hat, kappa=sc.kappa),
                                     preconditioner="auto", auto_switch_iters=threshold, newton_max_iters=6)
        state = S.stepper.SimState(sc.as_scene(), cfg)
        S.stepper.advance_time_step(state)
        assert state._auto_mas == expect_switch, (kappa, state._auto_mas)
        state.close()
