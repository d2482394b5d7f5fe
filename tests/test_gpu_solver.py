"""GPU parity of assembly, SpMV, matrix-free matvec, block-Jacobi, gradient scatter and PCG
against the reference's frozen outputs (tests/golden/scene.npz) and the oracle."""

import numpy as np
import pytest

from conftest import block_rel_err, load_golden, rel_err
from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def S():
    from paper_2308_09400_b200 import barrier, device, proximity, solver, stencils

    class NS:
        pass

    ns = NS()
    ns.barrier, ns.device, ns.proximity, ns.solver, ns.stencils = barrier, device, proximity, solver, stencils
    return ns


@pytest.fixture(scope="module")
def scene():
    z = load_golden("scene")
    z["grouped"] = [(z[f"fam{s}_hess"], z[f"fam{s}_vids"]) for s in (2, 3, 4) if f"fam{s}_hess" in z]
    return z


def bsr_to_dense(n, rowptr, colidx, vals):
    a = np.zeros((3 * n, 3 * n))
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    for r, c, blk in zip(rows, colidx, vals):
        a[3 * r:3 * r + 3, 3 * c:3 * c + 3] = blk
    return a


def test_assembled_matrix_equals_reference_dense(S, scene):
    n = scene["masses"].shape[0]
    rowptr, colidx, vals = S.solver.assemble_bsr(scene["grouped"], scene["masses"], scene["fixed"])
    # sparsity pattern: bit-exact with the oracle's definition
    o_rowptr, o_colidx, o_vals = o.assemble_bsr(scene["grouped"], scene["masses"], scene["fixed"])
    np.testing.assert_array_equal(rowptr, o_rowptr)
    np.testing.assert_array_equal(colidx, o_colidx)
    assert rowptr.dtype == np.int32 and colidx.dtype == np.int32 and vals.shape == (len(colidx), 3, 3)
    # columns ascend within each row, every row has its diagonal
    for r in range(n):
        cols = colidx[rowptr[r]:rowptr[r + 1]]
        assert np.all(np.diff(cols) > 0) and r in cols
    ref = scene["ref_dense"]
    got = bsr_to_dense(n, rowptr, colidx, vals)
    assert np.abs(got - ref).max() <= TOL * np.abs(ref).max()
    assert block_rel_err(vals, o_vals) < 1e-12   # same order of summation family by family
    # fixed rows reduced to the identity diagonal
    for r in np.flatnonzero(scene["fixed"]):
        assert rowptr[r + 1] - rowptr[r] == 1 and np.array_equal(vals[rowptr[r]], np.eye(3))
    assert np.array_equal(got, got.T) or np.abs(got - got.T).max() <= 1e-14 * np.abs(got).max()


def test_spmv_and_matrix_free_matvec(S, scene):
    sysm = S.solver._system_from_grouped(scene["grouped"], scene["masses"], scene["fixed"])
    v = scene["v"]
    y = S.device.to_host(sysm.spmv(v))
    ref = scene["ref_dense"] @ v
    assert np.abs(y - ref).max() <= TOL * np.abs(ref).max()
    assert rel_err(y, scene["ref_matvec"], floor=1e-6) < 1e-8
    mf = S.solver.matvec_matrix_free(scene["grouped"], scene["masses"], scene["fixed"], v)
    assert np.abs(mf - scene["ref_matvec"]).max() <= TOL * np.abs(scene["ref_matvec"]).max()
    assert np.array_equal(mf.reshape(-1, 3)[scene["fixed"]], v.reshape(-1, 3)[scene["fixed"]])
    z = S.solver.matvec_matrix_free(scene["grouped"], scene["masses"], scene["fixed"], np.zeros_like(v))
    assert np.all(z == 0.0)
    # determinism of the assembled path: bitwise identical on repeat
    assert np.array_equal(S.device.to_host(sysm.spmv(v)), y)
    sysm.close()


def test_block_jacobi(S, scene):
    pinv = S.solver.block_jacobi_preconditioner(scene["grouped"], scene["masses"], scene["fixed"])
    assert pinv.shape == scene["ref_pinv"].shape
    # 3x3 blocks with kappa = 2e8 are ill conditioned: compare through P^-1 D = I
    n = scene["masses"].shape[0]
    diag = np.stack([scene["ref_dense"][3 * i:3 * i + 3, 3 * i:3 * i + 3] for i in range(n)])
    prod = np.einsum("nij,njk->nik", pinv, diag)
    cond = np.linalg.cond(diag)
    assert np.all(np.abs(prod - np.eye(3)).reshape(n, -1).max(axis=1) <= 1e-13 * cond + 1e-12)
    assert block_rel_err(pinv, scene["ref_pinv"]) < 1e-6
    for r in np.flatnonzero(scene["fixed"]):
        assert np.array_equal(pinv[r], np.eye(3))


def test_gradient_scatter(S, scene):
    table = S.proximity.StencilTable(scene["kind"], scene["verts"], scene["sub"], scene["eps_x"])
    params = S.barrier.BarrierParams(d_hat=float(scene["d_hat"]), kappa=float(scene["kappa"]))
    batch = S.stencils.evaluate(table, scene["positions"], params, dt=float(scene["dt"]))
    assert batch.summary()[0] == pytest.approx(float(scene["ref_energy"]), rel=TOL)
    sysm = S.solver.NewtonSystem(scene["masses"], scene["fixed"])
    fams = [batch.families[s] for s in sorted(batch.families)]
    sysm.set_pattern([(f.s, f.vids) for f in fams])
    g = S.device.to_host(sysm.gradient(scene["positions"], scene["x_tilde"], [f.grad for f in fams]))
    ref = scene["ref_gradient"]
    assert np.abs(g - ref).max() <= TOL * np.abs(ref).max()
    assert np.all(g.reshape(-1, 3)[scene["fixed"]] == 0.0)
    # blocks straight from the stencil kernel assemble to the reference matrix too
    sysm.assemble([f.hess for f in fams])
    got = bsr_to_dense(sysm.n, *sysm.to_scipy_like())
    assert np.abs(got - scene["ref_dense"]).max() <= TOL * np.abs(scene["ref_dense"]).max()
    for s, f in zip(sorted(batch.families), fams):
        np.testing.assert_array_equal(S.device.to_host(f.vids), scene[f"fam{s}_vids"])
        assert block_rel_err(S.device.to_host(f.hess), scene[f"fam{s}_hess"]) < TOL
    sysm.close()


def test_factor_path_equals_dense_path(S, scene):
    """Rank-1 factors: hess == z z^T bit for bit, and the matrix assembled from z alone equals the
    one assembled from the dense blocks (bitwise for the per-block-run kernel, 1e-13 otherwise)."""
    table = S.proximity.StencilTable(scene["kind"], scene["verts"], scene["sub"], scene["eps_x"])
    params = S.barrier.BarrierParams(d_hat=float(scene["d_hat"]), kappa=float(scene["kappa"]))
    full = S.stencils.evaluate(table, scene["positions"], params, dt=float(scene["dt"]), want_factors=True)
    lean = S.stencils.evaluate(table, scene["positions"], params, dt=float(scene["dt"]), want_hess=False,
                               want_factors=True)
    fams = [full.families[s] for s in sorted(full.families)]
    for f, g in zip(fams, [lean.families[s] for s in sorted(lean.families)]):
        z = S.device.to_host(f.fac)
        assert g.hess is None and np.array_equal(z, S.device.to_host(g.fac))
        assert np.array_equal(S.device.to_host(f.hess), z[:, :, None] * z[:, None, :])
    sysm = S.solver.NewtonSystem(scene["masses"], scene["fixed"])
    sysm.set_pattern([(f.s, f.vids) for f in fams])
    sysm.set_numeric_variant(1)
    dense = S.device.to_host(sysm.assemble([f.hess for f in fams])).copy()
    fused = S.device.to_host(sysm.assemble_from_factors([f.fac for f in fams])).copy()
    assert np.array_equal(dense, fused)
    sysm.set_numeric_variant(4)
    rows = S.device.to_host(sysm.assemble([f.hess for f in fams]))
    assert block_rel_err(fused, rows) < 1e-12
    got = bsr_to_dense(sysm.n, S.device.to_host(sysm.rowptr), S.device.to_host(sysm.colidx), fused)
    assert np.abs(got - scene["ref_dense"]).max() <= TOL * np.abs(scene["ref_dense"]).max()
    sysm.close()


def test_pcg_matches_reference(S, scene):
    rhs = -scene["ref_gradient"]
    d, iters, ok = S.solver.pcg_solve(scene["grouped"], scene["masses"], scene["fixed"], rhs, 1e-4, 2000)
    # kappa = 2e8: round-off (summation order of the assembly, of the SpMV, of the dot products) moves
    # the stopping iteration.  delta = r.s is not monotone: with the streamed SpMV (FMA, per-entry sums)
    # it dips to 0.97e-4 * delta0 at iteration 65, where the reference's arithmetic stays a hair above
    # 1e-4 until iteration 83.  So the count is bounded from above only; that the stop is legitimate is
    # checked right below with the reference's own matrix and preconditioner, and the 1e-12 solve
    # further down must agree with the reference within a few percent of its ~1000 iterations.
    ref_it = int(scene["ref_pcg_iters"])
    assert ok == bool(scene["ref_pcg_ok"]) and 0 < iters <= ref_it + 2 + 0.05 * ref_it, (iters, ref_it)
    assert np.all(d.reshape(-1, 3)[scene["fixed"]] == 0.0)
    # the stopping criterion itself, re-evaluated with the reference's own matrix and preconditioner
    a = scene["ref_dense"]
    n = scene["masses"].shape[0]
    r0 = rhs.copy()
    r0.reshape(n, 3)[scene["fixed"]] = 0.0
    prec = lambda r: np.einsum("nij,nj->ni", scene["ref_pinv"], r.reshape(n, 3)).reshape(-1)  # noqa: E731
    delta0 = r0 @ prec(r0)
    res = r0 - a @ d
    assert res @ prec(res) <= 1.01e-4 * delta0
    # same Krylov iterate up to the few iterations by which round-off moves the stop
    diff = d - scene["ref_pcg_d"]
    assert np.sqrt(diff @ a @ diff) <= 0.1 * np.sqrt(scene["ref_pcg_d"] @ a @ scene["ref_pcg_d"])
    d12, it12, ok12 = S.solver.pcg_solve(scene["grouped"], scene["masses"], scene["fixed"], rhs, 1e-12, 5000)
    # ~1000 iterations on a kappa = 2e8 system: round-off reorders convergence by a few percent
    assert ok12 and abs(it12 - int(scene["ref_pcg12_iters"])) <= 0.05 * int(scene["ref_pcg12_iters"])
    r = rhs.copy()
    r.reshape(-1, 3)[scene["fixed"]] = 0.0
    res, ref_res = a @ d12 - r, a @ scene["ref_pcg12_d"] - r
    assert np.linalg.norm(res) <= 10.0 * max(np.linalg.norm(ref_res), 1e-12 * np.linalg.norm(r))
    # solver contracts of the reference's own tests (test_solver.py:129-142)
    d0, it0, ok0 = S.solver.pcg_solve(scene["grouped"], scene["masses"], scene["fixed"], np.zeros_like(rhs), 1e-4, 50)
    assert it0 == 0 and ok0 and np.all(d0 == 0.0)
    capped = S.solver.pcg_solve(scene["grouped"], scene["masses"], scene["fixed"], rhs, 1e-30, 3)
    assert capped[1] == 3 and capped[2] is False


def test_pcg_diagonal_system_one_iteration(S):
    """Mass-only system: block-Jacobi is exact, PCG converges in one iteration (test_solver.py:136-142)."""
    rng = np.random.default_rng(3)
    n = 500
    masses = rng.uniform(0.5, 2.0, n)
    fixed = np.zeros(n, bool)
    fixed[::17] = True
    rhs = rng.normal(size=3 * n)
    d, iters, ok = S.solver.pcg_solve([], masses, fixed, rhs, 1e-10, 10)
    assert iters == 1 and ok
    expect = (rhs.reshape(n, 3) / masses[:, None])
    expect[fixed] = 0.0
    np.testing.assert_allclose(d.reshape(n, 3), expect, rtol=1e-14)


@pytest.mark.parametrize("n,nb", [(2000, 15000), (50000, 200000)])
def test_random_blocks_assembly_vs_oracle(S, n, nb):
    """Random symmetric blocks of all three sizes, random fixed set, against the oracle's BSR."""
    rng = np.random.default_rng(n)
    masses = rng.uniform(0.1, 1.0, n)
    fixed = rng.uniform(size=n) < 0.02
    grouped = []
    for s, cnt in ((2, nb // 10), (3, nb // 5), (4, nb)):
        u = rng.normal(size=(cnt, 3 * s))
        hess = u[:, :, None] * u[:, None, :] * rng.uniform(0.1, 5.0, size=(cnt, 1, 1))
        base = rng.integers(0, n - 8, size=(cnt, 1))
        vids = (base + np.stack([rng.permutation(8)[:s] for _ in range(cnt)])).astype(np.int64)
        if s == 4:  # a hub vertex with several hundred neighbours: rows longer than one smem window
            hub = np.stack([np.concatenate([[7], rng.choice(np.arange(8, n), size=3, replace=False)]) for _ in range(300)])
            vids[:300] = hub
        grouped.append((hess, vids))
    fixed[7] = False
    rowptr, colidx, vals = S.solver.assemble_bsr(grouped, masses, fixed)
    o_rowptr, o_colidx, o_vals = o.assemble_bsr(grouped, masses, fixed)
    np.testing.assert_array_equal(rowptr, o_rowptr)
    np.testing.assert_array_equal(colidx, o_colidx)
    assert rowptr[8] - rowptr[7] > 500
    assert block_rel_err(vals, o_vals) < 1e-12
    # the alternative numeric kernels give the same matrix
    for variant in (1, 4):
        alt = S.solver._system_from_grouped(grouped, masses, fixed, variant=variant)
        assert block_rel_err(S.device.to_host(alt.vals), o_vals) < 1e-12, variant
        alt.close()
    x = rng.normal(size=3 * n)
    sysm = S.solver._system_from_grouped(grouped, masses, fixed)
    y = S.device.to_host(sysm.spmv(x))
    ref = o.bsr_matvec(o_rowptr, o_colidx, o_vals, x)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    mf = S.solver.matvec_matrix_free(grouped, masses, fixed, x)
    ref_mf = o.matvec_matrix_free(grouped, masses, fixed, x)
    assert np.abs(mf - ref_mf).max() <= 1e-11 * np.abs(ref_mf).max()
    assert np.abs(mf - y).max() <= 1e-11 * np.abs(y).max()
    rhs = rng.normal(size=3 * n)
    d, iters, ok, delta0, delta_new = sysm.pcg(rhs, 1e-8, 500)
    od, oit, ook = o.pcg_solve(grouped, masses, fixed, rhs, 1e-8, 500)
    assert ok == ook and abs(iters - oit) <= 2
    np.testing.assert_allclose(S.device.to_host(d), od, rtol=1e-5, atol=1e-7 * np.abs(od).max())
    sysm.close()


def test_group_blocks_matches_reference_layout(S, scene):
    table = S.proximity.StencilTable(scene["kind"], scene["verts"], scene["sub"], scene["eps_x"])
    params = S.barrier.BarrierParams(d_hat=float(scene["d_hat"]), kappa=float(scene["kappa"]))
    batch = S.stencils.evaluate(table, scene["positions"], params, dt=float(scene["dt"]))
    grouped = S.solver.group_blocks(batch.to_local_quadratics())
    assert [h.shape[1] for h, _ in grouped] == [6, 9, 12]
    for (h, v), s in zip(grouped, (2, 3, 4)):
        np.testing.assert_array_equal(v, scene[f"fam{s}_vids"])
        assert block_rel_err(h, scene[f"fam{s}_hess"]) < TOL


def test_direct_load_fallback_kernels_agree_with_the_streamed_ones(S, scene, monkeypatch):
    """B200IPC_SPMV_MODE=legacy selects the direct-load SpMV / PCG kernels (the fallback for arrays that
    are not 16-byte aligned): same operator, same solve."""
    rhs = -scene["ref_gradient"]
    d_s, it_s, ok_s = S.solver.pcg_solve(scene["grouped"], scene["masses"], scene["fixed"], rhs, 1e-12, 5000)
    monkeypatch.setenv("B200IPC_SPMV_MODE", "legacy")
    d_l, it_l, ok_l = S.solver.pcg_solve(scene["grouped"], scene["masses"], scene["fixed"], rhs, 1e-12, 5000)
    assert ok_s and ok_l and abs(it_s - it_l) <= 0.05 * it_l
    a = scene["ref_dense"]
    diff = d_s - d_l
    assert np.sqrt(diff @ a @ diff) <= 1e-5 * np.sqrt(d_l @ a @ d_l)
    v = scene["v"]
    mv_l = S.solver.matvec_matrix_free(scene["grouped"], scene["masses"], scene["fixed"], v)
    monkeypatch.delenv("B200IPC_SPMV_MODE")
    mv_s = S.solver.matvec_matrix_free(scene["grouped"], scene["masses"], scene["fixed"], v)
    assert np.abs(mv_l - mv_s).max() <= 1e-12 * np.abs(mv_s).max()
