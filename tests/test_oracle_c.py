"""The plain-C oracle (oracle/oracle_c.c) and the reference's own compiled kernels (oracle/_ref)
against the frozen reference outputs and the NumPy oracle."""

import numpy as np
import pytest

from conftest import block_rel_err, load_golden
from oracle import c_oracle
from oracle import tetipc_oracle as o

pytestmark = pytest.mark.skipif(not c_oracle.available(), reason="liboracle_c.so not built (make -C oracle)")


def test_c_classify_bit_exact_with_reference_core():
    z = load_golden("classify")
    pts = [z[f"in{j}"] for j in range(4)]
    for op in ("pt", "ee"):
        codes, d2, grad, w = c_oracle.classify(op, *pts)
        np.testing.assert_array_equal(codes, z[f"{op}_core_codes"])
        np.testing.assert_array_equal(d2, z[f"{op}_core_d2"])
        np.testing.assert_array_equal(grad, z[f"{op}_core_grad"])
        np.testing.assert_array_equal(w, z[f"{op}_core_w"])


def _run(z, d_hat, kappa, dt, scale_pos=1.0, threads=1):
    c_oracle.set_threads(threads)
    koff = np.searchsorted(z["kind"], np.arange(8)).astype(np.int64)
    prm = c_oracle.make_params(d_hat, kappa, dt=dt)
    out = c_oracle.barrier_stencils(prm, z["positions"] * scale_pos, koff, z["verts"], z["sub"], z["eps_x"])
    n = len(z["kind"])
    grad, hess = np.zeros((n, 12)), np.zeros((n, 12, 12))
    fam4 = np.concatenate([np.arange(koff[k], koff[k + 1]) for k in (0, 1, 3, 5, 6)])
    grad[fam4], hess[fam4] = out["grad4"], out["hess4"]
    grad[koff[2]:koff[3], :9], hess[koff[2]:koff[3], :9, :9] = out["grad3"], out["hess3"]
    grad[koff[4]:koff[5], :6], hess[koff[4]:koff[5], :6, :6] = out["grad2"], out["hess2"]
    return out["energy"], out["status"], grad, hess


@pytest.mark.parametrize("pset,d_hat,kappa,dt", [("unit", 1.0, 1.0, 1.0), ("scene", 5e-3, 2e8, 0.01)])
def test_c_blocks_vs_reference_golden(pset, d_hat, kappa, dt):
    z = load_golden("blocks_plain")
    energy, status, grad, hess = _run(z, d_hat, kappa, dt, scale_pos=d_hat, threads=3)
    np.testing.assert_array_equal(status, z[f"{pset}_ref_status"])
    np.testing.assert_allclose(energy, z[f"{pset}_ref_energy"], rtol=1e-12)
    assert block_rel_err(grad, z[f"{pset}_ref_grad"]) < 1e-12
    assert block_rel_err(hess, z[f"{pset}_ref_hess"]) < 1e-12


def test_c_parallel_blocks_vs_reference_golden():
    z = load_golden("blocks_parallel")
    energy, status, grad, hess = _run(z, 1.0, 1.0, 1.0)
    np.testing.assert_array_equal(status, z["unit_ref_status"])
    np.testing.assert_allclose(energy, z["unit_ref_energy"], rtol=1e-12)
    assert block_rel_err(grad, z["unit_ref_grad"]) < 1e-11
    assert block_rel_err(hess, z["unit_ref_hess"]) < 1e-10


def test_c_matches_numpy_oracle_on_config2_sample():
    from paper_2308_09400_b200 import workloads

    qb = workloads.config2_batch(n=5000)
    tab = o.narrow_phase(qb.positions, qb.rest_positions, qb.vt, qb.ee, qb.d_hat)
    tab["positions"] = qb.positions
    energy, status, grad, hess = _run(tab, qb.d_hat, qb.kappa, 1.0, threads=4)
    ref = o.local_quadratics_batch(tab["kind"], tab["verts"], tab["sub"], tab["eps_x"], qb.positions, qb.d_hat, qb.kappa)
    np.testing.assert_array_equal(status, ref["status"])
    np.testing.assert_allclose(energy, ref["energy"], rtol=1e-12, atol=1e-300)
    assert block_rel_err(grad, ref["grad"]) < 1e-10
    assert np.mean(np.abs(hess - ref["hess"]).reshape(len(hess), -1).max(axis=1)
                   <= 1e-9 * np.maximum(np.abs(ref["hess"]).reshape(len(hess), -1).max(axis=1), 1e-300)) > 0.99


def test_reference_core_binary_matches_golden():
    """oracle/_ref holds the reference's own kernels, compiled from /root/reference (binary only)."""
    core = c_oracle.reference_core()
    if core is None:
        pytest.skip("oracle/_ref not built (needs /root/reference: build container only)")
    z = load_golden("classify")
    pts = [z[f"in{j}"] for j in range(4)]
    for op, fn in (("pt", core.pt_classify_batch), ("ee", core.ee_classify_batch)):
        got = fn(*pts)
        for a, key in zip(got, ("codes", "d2", "grad", "w")):
            np.testing.assert_array_equal(a, z[f"{op}_core_{key}"])
    out = np.zeros(90)
    core.matvec_blocks(z["mv_hess"], z["mv_vids"], z["mv_x"], out)
    np.testing.assert_array_equal(out, z["mv_core_out"])
    out_c = np.zeros(90)
    c_oracle.matvec_blocks(z["mv_hess"], z["mv_vids"], z["mv_x"], out_c)
    np.testing.assert_array_equal(out_c, out)
