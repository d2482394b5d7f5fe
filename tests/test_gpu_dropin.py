"""The reference package itself (``tetipc``, unmodified) running on this backend -- SURVEY.md section 2 row 6b:
"the caller that must keep working unmodified" -- through the seam of ``kernels/__init__.py:13-32`` and the
``SimState`` subclass of INTEGRATION.md (``paper_2308_09400_b200.integration``).

(i) the assertions of the reference's own ``tests/test_kernels.py:16-75`` with
``paper_2308_09400_b200.kernels`` as the second backend; (ii) the reference's ``find_contact_pairs`` /
``stencil_distance`` / ``build_diagonal_jacobian`` running over the swapped seam; (iii) the reference's own
``advance_time_step`` (``solver.py:365-422``) on ``B200SimState`` for bundled scenes, against the pure-reference
run of the same scene.

``tetipc`` is looked for under ``/root/reference/pkg/src`` (build container) and ``baseline/_ref`` (the
unmodified package installed with pip, git-ignored, travels to the GPU box); the module is skipped where
neither exists.
"""

import copy
import importlib
import json
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _import_tetipc():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "tetipc")):
            if path not in sys.path:
                sys.path.insert(0, path)
            return importlib.import_module("tetipc")
    return None


@pytest.fixture(scope="module")
def T():
    tetipc = _import_tetipc()
    if tetipc is None:
        pytest.skip("the reference package is not importable here (no baseline/_ref, no /root/reference)")
    import tetipc.kernels, tetipc.proximity, tetipc.gap, tetipc.barrier, tetipc.solver, tetipc.scenes  # noqa: F401,E401
    from tetipc.kernels import _numpy

    from paper_2308_09400_b200 import integration, kernels

    class NS:
        pass

    ns = NS()
    ns.tetipc, ns.numpy_backend, ns.integration, ns.b200 = tetipc, _numpy, integration, kernels
    return ns


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)          # the reference's tests/conftest.py:9-11


def _random_points(rng, n):
    return [rng.normal(size=(n, 3)) for _ in range(4)]


# ---- (i) tests/test_kernels.py of the reference, with the B200 backend in the place of `_core` ----------------

def test_pt_classify_parity(T, rng):
    p, a, b, c = _random_points(rng, 2000)
    got = T.b200.pt_classify_batch(p, a, b, c)
    ref = T.numpy_backend.pt_classify_batch(p, a, b, c)
    np.testing.assert_array_equal(got[0], ref[0])
    for i in (1, 2, 3):
        np.testing.assert_allclose(got[i], ref[i], rtol=1e-13, atol=1e-13)


def test_ee_classify_parity(T, rng):
    p, a, b, c = _random_points(rng, 2000)
    got = T.b200.ee_classify_batch(p, a, b, c)
    ref = T.numpy_backend.ee_classify_batch(p, a, b, c)
    np.testing.assert_array_equal(got[0], ref[0])
    for i in (1, 2, 3):
        np.testing.assert_allclose(got[i], ref[i], rtol=1e-13, atol=1e-13)


def test_cross_sq_parity(T, rng):
    p, a, b, c = _random_points(rng, 500)
    got = T.b200.cross_sq_batch(p, a, b, c)
    ref = T.numpy_backend.cross_sq_batch(p, a, b, c)
    np.testing.assert_allclose(got[0], ref[0], rtol=1e-13)
    np.testing.assert_allclose(got[1], ref[1], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("s", [2, 3, 4])
def test_matvec_parity(T, rng, s):
    nb, n = 40, 30
    hess = rng.normal(size=(nb, 3 * s, 3 * s))
    hess = hess + hess.transpose(0, 2, 1)
    vids = np.stack([rng.choice(n, size=s, replace=False) for _ in range(nb)]).astype(np.int64)
    x = rng.normal(size=3 * n)
    out_a = np.zeros(3 * n)
    out_b = np.zeros(3 * n)
    T.b200.matvec_blocks(hess, vids, x, out_a)
    T.numpy_backend.matvec_blocks(hess, vids, x, out_b)
    np.testing.assert_allclose(out_a, out_b, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("pair", [0, 1, 2, 3])
def test_accd_parity(T, rng, pair):
    k = T.tetipc.kernels
    s = {k.PAIR_PT: 4, k.PAIR_EE: 4, k.PAIR_PE: 3, k.PAIR_PP: 2}[pair]
    for _ in range(50):
        x = rng.normal(size=(s, 3)) * 2.0
        x[0] += np.array([0.0, 0.0, 5.0])  # keep the pair separated
        dx = rng.normal(size=(s, 3)) * 0.5
        got = T.b200.accd_max_step(x, dx, pair, 0.9)
        ref = T.numpy_backend.accd_max_step(x, dx, pair, 0.9)
        assert got == pytest.approx(ref, rel=1e-12, abs=1e-12)


def test_accd_rejects_touching(T, rng):
    x = np.zeros((2, 3))
    dx = rng.normal(size=(2, 3))
    with pytest.raises(ValueError):
        T.b200.accd_max_step(x, dx, T.tetipc.kernels.PAIR_PP, 0.9)


# ---- (ii) the reference's own callers over the swapped seam ---------------------------------------------------

def _scene_state(T, tmp_path, name, cls=None, **overrides):
    """A bundled scene of the reference, written by the reference's own generators, as a SimState (or `cls`)."""
    sc = T.tetipc.scenes
    scene_dir = tmp_path / "scenes"
    if not scene_dir.exists():
        sc.write_bundled_scenes(str(scene_dir))
    with open(scene_dir / f"{name}.json") as fh:
        config = json.load(fh)
    state, steps, _ = sc.build_simulation(config, str(scene_dir), overrides or None)
    if cls is not None:
        v = state.v.copy()
        state = cls(state.scene, state.config, _materials(T, config, str(scene_dir)))
        state.v = v
    return state


def _materials(T, config, base_dir):
    return [T.tetipc.scenes.load_body(entry, base_dir)[1] for entry in config["bodies"]]


def test_reference_callers_run_on_the_b200_seam(T, tmp_path):
    """find_contact_pairs, stencil_distance, build_diagonal_jacobian, the barrier blocks and matvec_matrix_free
    of the reference, executed by the reference's code with tetipc.kernels dispatching to libb200ipc.so."""
    tet = T.tetipc
    state = _scene_state(T, tmp_path, "cube-align")
    x = state.x.copy()
    x[state.scene.body_offsets[1]:, 2] -= 0.0075          # bring the upper cube within d_hat of the lower one
    d_hat = state.config.barrier.d_hat
    ref_list = tet.proximity.find_contact_pairs(state.scene, x, d_hat)
    assert len(ref_list) > 10
    ref_blocks = [state._barrier_block(st, x) for st in ref_list]
    grouped = tet.solver.group_blocks(ref_blocks)
    v = np.random.default_rng(1).normal(size=3 * x.shape[0])
    ref_mv = tet.solver.matvec_matrix_free(grouped, state.masses, state.fixed, v)
    with T.integration.kernel_backend(tet) as seam:
        assert seam.BACKEND == "b200" and tet.kernels.pt_classify_batch is T.b200.pt_classify_batch
        got_list = tet.proximity.find_contact_pairs(state.scene, x, d_hat)
        got_blocks = [state._barrier_block(st, x) for st in got_list]
        got_mv = tet.solver.matvec_matrix_free(grouped, state.masses, state.fixed, v)
    assert tet.kernels.BACKEND in ("core", "numpy")                       # restored
    assert got_list == ref_list                                           # same dataclasses, same order
    for a, b in zip(got_blocks, ref_blocks):
        np.testing.assert_array_equal(a.vert_ids, b.vert_ids)
        np.testing.assert_allclose(a.grad, b.grad, rtol=1e-12, atol=1e-12 * np.abs(b.grad).max())
        np.testing.assert_allclose(a.hess, b.hess, rtol=1e-12, atol=1e-12 * np.abs(b.hess).max())
    np.testing.assert_allclose(got_mv, ref_mv, rtol=1e-12, atol=1e-12 * np.abs(ref_mv).max())


# ---- (iii) the reference's advance_time_step on B200SimState --------------------------------------------------

@pytest.mark.parametrize("name,steps,kw", [("pt-drop", 6, {}), ("ee-parallel-drop", 6, {}), ("cube-align", 4, {}),
                                            ("boxes-stiff", 3, {"friction.mu": 0.3})])
def test_reference_time_stepper_on_b200_simstate(T, tmp_path, name, steps, kw):
    """INTEGRATION.md's subclass, as code: the reference's own newton_step / advance_time_step drive
    B200SimState (detect, barrier energy, gradients and blocks batched on the GPU) and reproduce the
    pure-reference trajectory of the same bundled scene."""
    tet = T.tetipc
    B200SimState = T.integration.b200_sim_state(tet)
    ref_state = _scene_state(T, tmp_path, name, **kw)
    dev_state = _scene_state(T, tmp_path, name, cls=B200SimState, **kw)
    assert isinstance(dev_state, tet.solver.SimState)
    bat_state = copy.deepcopy(dev_state)
    contacts_seen = 0
    for _ in range(steps):
        rs = tet.solver.advance_time_step(ref_state)
        ds = tet.solver.advance_time_step(dev_state)
        with T.integration.batched_solver(tet):                           # + PCG and CCD on the device
            bs = tet.solver.advance_time_step(bat_state)
        l = ref_state.l
        assert (ds.newton_iters, ds.pcg_iters, ds.converged, ds.warning) == (rs.newton_iters, rs.pcg_iters,
                                                                              rs.converged, rs.warning)
        assert np.abs(dev_state.x - ref_state.x).max() <= 1e-9 * l
        assert ds.energy == pytest.approx(rs.energy, rel=1e-9, abs=1e-12)
        assert (np.isnan(ds.min_distance) and np.isnan(rs.min_distance)) or ds.min_distance == pytest.approx(rs.min_distance, rel=1e-9)
        # device PCG (FMA, per-entry sums) may stop an iteration apart at pcg_rel_tol = 1e-4, so its Newton
        # directions differ at the level of the PCG tolerance, not of round-off: same Newton iteration counts,
        # trajectory within 1e-5 l (the reference's own PCG-vs-dense-solve bound is 1e-6 l on its softer scene,
        # tests/test_solver.py:223-254; boxes-stiff with friction is the stiffest bundled scene)
        assert bs.converged == rs.converged and bs.newton_iters == rs.newton_iters
        assert np.abs(bat_state.x - ref_state.x).max() <= 1e-5 * l
        contacts_seen += len(ref_state.detect(ref_state.x))
    assert contacts_seen > 0 or name == "pt-drop"
