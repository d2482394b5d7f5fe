"""GPU friction against the reference's frozen outputs (tests/golden/friction.npz) and the oracle."""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import block_rel_err, load_golden, rel_err
from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def F():
    from paper_2308_09400_b200 import barrier, device, friction, proximity, solver, stencils

    return SimpleNamespace(barrier=barrier, device=device, friction=friction, proximity=proximity, solver=solver,
                           stencils=stencils)


@pytest.fixture(scope="module", params=["a", "b"])
def z(request):
    """(a) golden cloth scene, (b) nearly-parallel edge-edge batch (parallel kinds, skipped stencils)."""
    full = load_golden("friction")
    return {k[2:]: v for k, v in full.items() if k.startswith(request.param + "_")}


def _state(F, z):
    table = F.proximity.StencilTable(z["kind"], z["verts"], z["sub"], z["eps_x"])
    params = F.barrier.BarrierParams(d_hat=float(z["d_hat"]), kappa=float(z["kappa"]))
    return table, F.friction.update_state(table, z["x0"], float(z["mu"]), float(z["eps_v"]), float(z["dt"]), params=params)


def test_friction_state_matches_reference(F, z):
    table, state = _state(F, z)
    assert np.array_equal(state.rows, z["rows"])                     # same data kept, same order
    fr = F.device.to_host(state.frame)
    assert rel_err(fr[:, 10], z["lambda_n"]) < TOL
    size = F.proximity.KIND_SIZE[z["kind"]][state.rows]
    worst = 0.0
    for i in range(len(fr)):
        s = int(size[i])
        basis = np.zeros((3 * s, 2))
        for v in range(s):
            basis[3 * v:3 * v + 3, 0] = fr[i, v] * fr[i, 4:7]
            basis[3 * v:3 * v + 3, 1] = fr[i, v] * fr[i, 7:10]
        worst = max(worst, float(np.abs(basis - z["basis"][i, :3 * s]).max()))
    assert worst < TOL                                                # basis columns are unit vectors
    # the oracle agrees too (all seven kinds are present in the scene)
    ref = o.friction_state(z["kind"], z["verts"], z["sub"], z["x0"], z["raw_grad"])
    assert np.array_equal(np.flatnonzero(ref["status"] == 0), state.rows)
    assert len(np.unique(z["kind"])) >= 5


def test_friction_blocks_match_reference(F, z):
    table, state = _state(F, z)
    batch = F.friction.evaluate(state, z["x1"], z["x0"])
    dt2 = float(z["dt"]) ** 2
    assert rel_err(F.device.to_host(batch.energy), z["potential"]) < TOL
    kinds = z["kind"][state.rows]
    off = np.searchsorted(kinds, np.arange(8))
    n_hess = 0
    for s, fam in batch.families.items():
        rows = np.concatenate([np.arange(off[k], off[k + 1]) for k in F.stencils.FAMILY_KINDS[s]])
        grad, hess = F.device.to_host(fam.grad), F.device.to_host(fam.hess)
        assert np.array_equal(F.device.to_host(fam.vids), z["verts"][state.rows][rows][:, :s])
        assert block_rel_err(grad, -dt2 * z["force"][rows][:, :3 * s]) < TOL
        pick = np.flatnonzero(np.isin(rows, z["hess_rows"]))
        ref = dt2 * z["hess"][np.searchsorted(z["hess_rows"], rows[pick])][:, :3 * s, :3 * s]
        assert block_rel_err(hess[pick], ref) < TOL
        n_hess += len(pick)
        # PSD, rank <= 2, symmetric
        for blk in hess[:: max(1, len(hess) // 40)]:
            assert np.array_equal(blk, blk.T)
            ev = np.linalg.eigvalsh(blk)
            assert ev.min() >= -1e-12 * max(ev.max(), 1e-300) and (ev > 1e-9 * ev.max()).sum() <= 2
    assert n_hess == len(z["hess_rows"])
    assert abs(batch.total_energy() - z["potential"].sum()) <= TOL * z["potential"].sum()


def test_friction_blocks_flow_through_the_assembly(F, z):
    """Friction families are ordinary (hess, vids) families: assembled next to nothing else here,
    the matrix equals the dense sum of the reference's friction blocks."""
    table, state = _state(F, z)
    batch = F.friction.evaluate(state, z["x1"], z["x0"])
    nv = z["x0"].shape[0]
    masses, fixed = np.ones(nv), np.zeros(nv, bool)
    grouped = [(F.device.to_host(h), F.device.to_host(v)) for h, v in batch.grouped()]
    rowptr, colidx, vals = F.solver.assemble_bsr(grouped, masses, fixed)
    dense = np.zeros((3 * nv, 3 * nv))
    for r, (a, b) in enumerate(zip(rowptr[:-1], rowptr[1:])):
        for c, blk in zip(colidx[a:b], vals[a:b]):
            dense[3 * r:3 * r + 3, 3 * c:3 * c + 3] = blk
    ref = np.eye(3 * nv)
    dt2 = float(z["dt"]) ** 2
    o_st = o.friction_state(z["kind"], z["verts"], z["sub"], z["x0"], z["raw_grad"])
    rows = state.rows
    size = o.KIND_SIZE[z["kind"]][rows]
    blocks = o.friction_blocks(z["verts"][rows], size, o_st["lambda_n"][rows], o_st["cn"][rows], o_st["t1"][rows],
                               o_st["t2"][rows], z["x1"], z["x0"], float(z["mu"]), float(z["eps_v"]), float(z["dt"]))
    for i, r in enumerate(rows):
        s = int(size[i])
        idx = np.concatenate([[3 * v, 3 * v + 1, 3 * v + 2] for v in z["verts"][r, :s]])
        ref[np.ix_(idx, idx)] += blocks["hess"][i, :3 * s, :3 * s]
    assert np.abs(dense - ref).max() <= TOL * np.abs(ref).max()
    assert dt2 > 0


def test_reference_shaped_entry_points(F, z):
    """update_friction_state / potential / friction_force / friction_hessian_psd / f0_f1 twins."""
    table = F.proximity.StencilTable(z["kind"], z["verts"], z["sub"], z["eps_x"], z["origin_type"], z["origin"])
    stencils = table.to_stencils()
    size = F.proximity.KIND_SIZE[z["kind"]]
    grads = [z["raw_grad"][i, :3 * int(size[i])] for i in range(len(stencils))]
    data = F.friction.update_friction_state(stencils, grads, z["x0"], float(z["mu"]), float(z["eps_v"]), float(z["dt"]))
    assert len(data) == len(z["rows"])
    hess_at = {int(r): k for k, r in enumerate(z["hess_rows"])}
    for i in list(range(0, len(data), 211)) + [len(data) - 1]:
        d = data[i]
        s = len(d.stencil.verts)
        assert abs(d.lambda_n - z["lambda_n"][i]) <= TOL * z["lambda_n"][i]
        assert np.abs(d.basis_T - z["basis"][i, :3 * s]).max() < TOL
        u = F.friction.tangential_displacement(d, z["x1"], z["x0"])
        assert np.abs(u - z["u"][i]).max() <= 1e-12 * max(np.abs(z["u"][i]).max(), 1e-300) + 1e-18
        assert abs(F.friction.potential(d, u) - z["potential"][i]) <= TOL * z["potential"][i]
        f = F.friction.friction_force(d, u)
        assert np.abs(f - z["force"][i, :3 * s]).max() <= TOL * max(np.abs(z["force"][i]).max(), 1e-300)
        if i in hess_at:
            blk = F.friction.friction_hessian_psd(d, u)
            ref = z["hess"][hess_at[i]][:3 * s, :3 * s]
            assert np.abs(blk.hess - ref).max() <= TOL * np.abs(ref).max()
            assert np.array_equal(blk.vert_ids, np.asarray(d.stencil.verts)) and not blk.grad.any()
    h = float(z["dt"]) * float(z["eps_v"])
    for un in (0.0, 0.3 * h, h, 2.5 * h):
        f0, f1, f1p = F.friction.f0_f1(un, float(z["eps_v"]), float(z["dt"]))
        r0, r1, r1p = o.f0_f1(un, float(z["eps_v"]), float(z["dt"]))
        assert abs(f0 - r0) <= 1e-12 * abs(r0) and abs(f1 - r1) <= 1e-12 and abs(f1p - r1p) <= 1e-12 * max(abs(r1p), 1)
    assert F.friction.update_friction_state(stencils, grads, z["x0"], 0.0, 1e-2, 0.01) == []
    # the reference accepts the stencils in ANY order with a positionally matched gradient list (friction.py:148-171):
    # a shuffled call returns the same data, in the caller's order
    perm = np.random.default_rng(0).permutation(len(stencils))[:400]
    sub_st, sub_g = [stencils[i] for i in perm], [grads[i] for i in perm]
    shuffled = F.friction.update_friction_state(sub_st, sub_g, z["x0"], float(z["mu"]), float(z["eps_v"]), float(z["dt"]))
    by_key = {(d.stencil.kind, tuple(d.stencil.verts)): d for d in data}
    kept = [st for st in sub_st if (st.kind, tuple(st.verts)) in by_key]
    assert [(d.stencil.kind, tuple(d.stencil.verts)) for d in shuffled] == [(st.kind, tuple(st.verts)) for st in kept]
    for d in shuffled[::37]:
        ref_d = by_key[(d.stencil.kind, tuple(d.stencil.verts))]
        assert d.lambda_n == ref_d.lambda_n and np.array_equal(d.basis_T, ref_d.basis_T)


def test_barrier_and_friction_families_assemble_together(F, z):
    """Six families (barrier 6/9/12 + friction 6/9/12), as group_blocks would hand them to the solver:
    pattern, values, SpMV and gradient scatter against the dense sum of the oracle's blocks."""
    table, state = _state(F, z)
    params = F.barrier.BarrierParams(d_hat=float(z["d_hat"]), kappa=float(z["kappa"]))
    dt = float(z["dt"])
    bar = F.stencils.evaluate(table, z["x1"], params, dt=dt)
    st = F.device.to_host(bar.status)
    if (st == 2).any():
        pytest.skip("displaced pose penetrates")
    fri = F.friction.evaluate(state, z["x1"], z["x0"])
    fams = [bar.families[s] for s in sorted(bar.families)] + [fri.families[s] for s in sorted(fri.families)]
    nv = z["x0"].shape[0]
    rng = np.random.default_rng(3)
    masses = rng.uniform(0.5, 2.0, size=nv)
    fixed = rng.uniform(size=nv) < 0.05
    sysm = F.solver.NewtonSystem(masses, fixed)
    sysm.set_pattern([(f.s, f.vids) for f in fams])
    vals = F.device.to_host(sysm.assemble([f.hess for f in fams]))
    rowptr, colidx = F.device.to_host(sysm.rowptr), F.device.to_host(sysm.colidx)
    grouped = [(F.device.to_host(f.hess), F.device.to_host(f.vids)) for f in fams]
    ref = o.assemble_dense(grouped, masses, fixed)
    dense = np.zeros_like(ref)
    for r, (a, b) in enumerate(zip(rowptr[:-1], rowptr[1:])):
        for c, blk in zip(colidx[a:b], vals[a:b]):
            dense[3 * r:3 * r + 3, 3 * c:3 * c + 3] = blk
    assert np.abs(dense - ref).max() <= TOL * np.abs(ref).max()
    x = rng.normal(size=3 * nv)
    y = F.device.to_host(sysm.spmv(x))
    assert np.abs(y - ref @ x).max() <= 1e-11 * np.abs(ref @ x).max()
    xt = z["x0"]
    g = F.device.to_host(sysm.gradient(z["x1"], xt, [f.grad for f in fams]))
    gref = o.scatter_gradient(masses, fixed, z["x1"], xt, [(f.s, None, F.device.to_host(f.vids), F.device.to_host(f.grad), None) for f in fams])
    assert np.abs(g - gref).max() <= TOL * np.abs(gref).max()
    sysm.close()


def test_gather_rows_matches_indexing():
    """``b200ipc_gather_rows`` (the row compaction of the lagged friction state): any row width that is a multiple of
    4 bytes, 16- / 8- / 4-byte word paths, repeated and out-of-order indices, empty inputs."""
    import torch

    from paper_2308_09400_b200 import device

    g = torch.Generator(device="cuda").manual_seed(5)
    for shape, dtype in (((5000, 12), torch.float64), ((5000, 4), torch.int32), ((5000,), torch.float64),
                         ((4097, 3), torch.int32), ((300, 3, 3), torch.float64), ((1000, 5), torch.float32)):
        src = (torch.rand(shape, generator=g, device="cuda", dtype=torch.float64) * 1000).to(dtype)
        idx = torch.randint(0, shape[0], (7001,), generator=g, device="cuda")
        assert torch.equal(device.gather_rows(src, idx), src[idx])
        assert torch.equal(device.gather_rows(src[1:], idx.clamp(max=shape[0] - 2)), src[1:][idx.clamp(max=shape[0] - 2)])
        assert device.gather_rows(src, idx[:0]).shape == (0,) + tuple(shape[1:])
    u8 = torch.randint(0, 255, (100,), device="cuda", dtype=torch.uint8)       # byte rows fall back to torch
    assert torch.equal(device.gather_rows(u8, torch.arange(99, -1, -1, device="cuda")), u8.flip(0))
