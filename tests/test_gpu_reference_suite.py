"""The reference's OWN test-suite (``/root/reference/pkg/tests``, unmodified) run against this backend: a child
pytest imports the reference package, swaps every function this package mirrors for the mirror
(``integration.function_overlay`` -- per-stencil distance / Jacobian / barrier scalars / blocks / mollified
eigensystem / friction / elasticity / contact detection / CCD / matvec / preconditioner / PCG, plus the kernel
seam) and runs the reference's tests as they are.  What passes there is the reference's own statement of
correctness for the functions on the path -- finite-difference checks, eigenvalue identities, golden scenes,
error behaviour -- evaluated on the GPU.

The reference's tests are not part of this repository: ``__graft_entry__.build()`` copies them next to the
unmodified package under the git-ignored ``baseline/_ref`` (which travels to the GPU box); the module is skipped
where neither that copy nor ``/root/reference`` exists."""

import json
import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _locate():
    for pkg, tests in ((os.path.join(ROOT, "baseline", "_ref"), os.path.join(ROOT, "baseline", "_ref", "_reference_tests")),
                       ("/root/reference/pkg/src", "/root/reference/pkg/tests")):
        if os.path.isdir(os.path.join(pkg, "tetipc")) and os.path.isfile(os.path.join(tests, "test_barrier.py")):
            return pkg, tests
    return None, None


# every family of mirrored functions must actually have been exercised by the reference's tests
MUST_BE_CALLED = ["barrier.barrier_value", "barrier.lambda1", "barrier.build_local_quadratic", "gap.build_diagonal_jacobian",
                  "gap.gap_function", "proximity.stencil_distance", "proximity.parallel_measure",
                  "proximity.find_contact_pairs", "proximity.accd_step_bound", "proximity.global_ccd_filter",
                  "mollifier.mollified_eigensystem", "mollifier.build_mollified_local_quadratic",
                  "mollifier.mollified_gradient", "friction.friction_hessian_psd", "friction.update_friction_state",
                  "elasticity.batch_grad_hess", "elasticity.tet_energy_grad_hess", "solver.pcg_solve",
                  "solver.matvec_matrix_free", "solver.block_jacobi_preconditioner", "kernels.pt_classify_batch",
                  "kernels.ee_classify_batch"]


def _run_reference_suite(tmp_path, pkg, tests, select, batched):
    report = tmp_path / "overlay_calls.json"
    env = dict(os.environ)
    if batched:
        env["B200_OVERLAY_BATCHED"] = "1"
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "plugins"), ROOT, pkg] + env.get("PYTHONPATH", "").split(os.pathsep))
    env["B200_OVERLAY_REPORT"] = str(report)
    env["HYPOTHESIS_STORAGE_DIRECTORY"] = str(tmp_path / "hypothesis")
    cmd = [sys.executable, "-m", "pytest", select, "-q", "-p", "reference_overlay_plugin", "-p", "no:cacheprovider",
           "--rootdir", tests, "-o", "addopts=", "--tb=short",
           # fails on the unmodified reference alone (a CLI diagnostic curve, 9.0e-5 against its own 1e-6 bound; no
           # function of the path is involved): 170 of the reference's 171 tests pass on the reference itself
           "-k", "not test_norms_curve_ratio_vanishes"]
    run = subprocess.run(cmd, env=env, cwd=str(tmp_path), capture_output=True, text=True, timeout=3000)
    tail = "\n".join(run.stdout.splitlines()[-60:])
    m = re.search(r"(\d+) passed", run.stdout)
    assert run.returncode == 0, f"reference test-suite on the B200 backend:\n{tail}\n{run.stderr[-2000:]}"
    return (int(m.group(1)) if m else 0), json.loads(report.read_text()), tail


def test_reference_test_suite_passes_on_this_backend(tmp_path):
    pkg, tests = _locate()
    if pkg is None:
        pytest.skip("the reference package and its tests are not available here")
    passed, calls, tail = _run_reference_suite(tmp_path, pkg, tests, tests, batched=False)
    assert passed >= 170, tail
    missing = [k for k in MUST_BE_CALLED if calls.get(k, 0) == 0]
    assert not missing, f"mirrors the reference's tests never reached: {missing}\n{json.dumps(calls, indent=1)}"
    print(json.dumps(calls, sort_keys=True))


def test_reference_solver_tests_pass_on_the_batched_sim_state(tmp_path):
    """The reference's ``tests/test_solver.py`` once more, with ``SimState`` itself replaced by the batched
    subclass (``integration.b200_sim_state``): detect, barrier energy and the barrier blocks of every Newton
    iteration are single device launches under the reference's own ``newton_step`` / ``advance_time_step``."""
    pkg, tests = _locate()
    if pkg is None:
        pytest.skip("the reference package and its tests are not available here")
    passed, calls, tail = _run_reference_suite(tmp_path, pkg, tests, os.path.join(tests, "test_solver.py"), batched=True)
    assert passed >= 15, tail
    for k in ("SimState.detect", "SimState._barrier_energy", "SimState.assemble_local_quadratics", "solver.pcg_solve"):
        assert calls.get(k, 0) > 0, f"{k} never ran\n{json.dumps(calls, indent=1)}"
    print(json.dumps({k: v for k, v in calls.items() if k.startswith("SimState")}, sort_keys=True))
