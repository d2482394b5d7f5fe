"""GPU stable neo-Hookean blocks against the reference's frozen outputs."""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import block_rel_err, load_golden, rel_err
from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def E():
    from paper_2308_09400_b200 import device, elasticity, solver

    return SimpleNamespace(device=device, elasticity=elasticity, solver=solver)


def grad_err(got, ref):
    """Per-entry error relative to the tet's gradient scale; tets at rest have an analytically zero
    gradient (round-off of O(1e4) terms), so the scale is floored at 1e-6 of the batch maximum."""
    scale = np.maximum(np.abs(ref).max(axis=1), 1e-6 * np.abs(ref).max())
    return float((np.abs(got - ref) / scale[:, None]).max())


def test_rest_data_and_blocks_match_reference(E):
    z = load_golden("elastic")
    rest_inv, vols, g = E.elasticity.rest_data(z["rest"], z["tets"])
    assert block_rel_err(rest_inv, z["rest_inv"]) < 1e-12 and rel_err(vols, z["vols"]) < 1e-12
    assert g.shape == (len(vols), 9, 12)
    e, grad, hess = E.elasticity.batch_grad_hess(z["x"], z["tets"], z["rest_inv"], z["vols"], g, z["mu"], z["lam"])
    assert rel_err(e, z["energy"]) < TOL
    assert grad_err(grad, z["grad"]) < TOL
    assert block_rel_err(hess, z["hess"]) < TOL                       # Jacobi projection == LAPACK eigh projection
    _, _, raw = E.elasticity.batch_grad_hess(z["x"], z["tets"], z["rest_inv"], z["vols"], g, z["mu"], z["lam"], project=False)
    assert block_rel_err(raw[::5], z["hess_raw"]) < TOL
    # projected blocks: symmetric, PSD
    assert np.abs(hess - np.swapaxes(hess, 1, 2)).max() <= 1e-12 * np.abs(hess).max()
    ev = np.linalg.eigvalsh(0.5 * (hess + np.swapaxes(hess, 1, 2)))
    assert (ev.min(axis=1) >= -1e-10 * ev.max(axis=1)).all()


def test_device_mesh_dt_scaling_and_single_tet(E):
    z = load_golden("elastic")
    mesh = E.elasticity.TetMesh(z["rest"], z["tets"], z["mu"], z["lam"])
    dt = 0.01
    energy, fam = mesh.evaluate(z["x"], dt=dt)
    assert rel_err(E.device.to_host(energy), z["energy"]) < TOL
    assert grad_err(E.device.to_host(fam.grad), dt * dt * z["grad"]) < TOL
    assert block_rel_err(E.device.to_host(fam.hess), dt * dt * z["hess"]) < TOL
    assert np.array_equal(E.device.to_host(fam.vids), z["tets"])
    # zero gradient and PSD Hessian at rest (the reference's own sanity property)
    e0, fam0 = mesh.evaluate(z["rest"])
    assert np.abs(E.device.to_host(fam0.grad)).max() <= 1e-9 * np.abs(z["grad"]).max()
    mat = E.elasticity.ElasticMaterial(youngs_E=1.0e5, poisson_nu=0.3)
    k = 7
    ids = z["tets"][k]
    e1, g1, h1 = E.elasticity.tet_energy_grad_hess(z["rest_inv"][k], z["x"][ids], mat)
    eo, go, ho = o.elastic_blocks(z["x"][ids], np.array([[0, 1, 2, 3]]), z["rest_inv"][k:k + 1],
                                  np.array([1.0 / (6.0 * np.linalg.det(z["rest_inv"][k]))]),
                                  np.array([mat.lame_mu]), np.array([mat.lame_lambda]))
    assert abs(e1 - eo[0]) <= TOL * abs(eo[0]) and block_rel_err(g1[None], go) < TOL and block_rel_err(h1[None], ho) < TOL
    with pytest.raises(ValueError):
        E.elasticity.ElasticMaterial(youngs_E=-1.0, poisson_nu=0.3)


def test_elastic_family_through_the_assembly(E):
    z = load_golden("elastic")
    mesh = E.elasticity.TetMesh(z["rest"], z["tets"], z["mu"], z["lam"])
    _, fam = mesh.evaluate(z["x"], dt=0.01)
    nv = z["rest"].shape[0]
    masses, fixed = np.full(nv, 0.3), np.zeros(nv, bool)
    fixed[::17] = True
    grouped = [(E.device.to_host(fam.hess), E.device.to_host(fam.vids))]
    rowptr, colidx, vals = E.solver.assemble_bsr(grouped, masses, fixed)
    ref = o.assemble_dense(grouped, masses, fixed)
    dense = np.zeros_like(ref)
    for r, (a, b) in enumerate(zip(rowptr[:-1], rowptr[1:])):
        for c, blk in zip(colidx[a:b], vals[a:b]):
            dense[3 * r:3 * r + 3, 3 * c:3 * c + 3] = blk
    assert np.abs(dense - ref).max() <= TOL * np.abs(ref).max()
