"""Multilevel additive Schwarz preconditioner (not in the reference package, which has
block-Jacobi only).  The operator is checked piece by piece against the oracle's restatement of the published
algorithm (domain order, stored inverses through their action, one- and two-level application), and the solve
is pinned to the REFERENCE: the direction of a MAS-driven PCG must meet the reference's stopping rule
(solver.py:302: r . P_bj r <= tol * r0 . P_bj r0) evaluated with the reference-defined dense matrix and
block-Jacobi inverses, and agree with a direct solve at a tight tolerance."""

import numpy as np
import pytest

from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    from paper_2308_09400_b200 import barrier, contacts, device, solver, stencils, workloads

    class NS:
        pass

    ns = NS()
    ns.barrier, ns.contacts, ns.device, ns.solver, ns.stencils, ns.workloads = barrier, contacts, device, solver, stencils, workloads
    return ns


def cloth_system(M, layers, n, seed, kappa=2e8):
    """(scene, NewtonSystem with assembled values, grouped host blocks, rhs)."""
    cloth = M.workloads.cloth_stack(layers=layers, n=n, seed=seed, kappa=kappa)
    pos = M.device.to_device(cloth.positions)
    bp = M.contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
    vt, ee = bp.query(pos)
    bp.close()
    table, _ = M.contacts.narrow_phase_device(pos, cloth.rest_positions, vt, ee, cloth.d_hat, want_origin=False)
    params = M.barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
    batch = M.stencils.evaluate(table, pos, params, dt=cloth.dt)
    fams = [batch.families[s] for s in sorted(batch.families)]
    sysm = M.solver.NewtonSystem(cloth.masses, cloth.fixed)
    sysm.set_pattern([(f.s, f.vids) for f in fams])
    sysm.assemble([f.hess for f in fams])
    xt = cloth.positions + 1e-4 * np.random.default_rng(seed).normal(size=cloth.positions.shape)
    g = M.device.to_host(sysm.gradient(pos, xt, [f.grad for f in fams]))
    return cloth, sysm, -g


@pytest.mark.parametrize("use_positions", [True, False], ids=["morton", "index"])
def test_domain_order_matches_oracle(M, use_positions):
    cloth = M.workloads.cloth_stack(layers=3, n=21, seed=4)
    sysm = M.solver.NewtonSystem(cloth.masses, cloth.fixed)
    sysm.mas_order(cloth.positions if use_positions else None)
    got = M.device.to_host(sysm.mas_rank())
    ref = o.mas_order(cloth.positions if use_positions else None, len(cloth.masses))
    assert np.array_equal(got, ref)
    assert np.array_equal(np.sort(got), np.arange(len(got)))
    sysm.close()


@pytest.mark.parametrize("levels", [1, 2])
@pytest.mark.parametrize("layers,n", [(3, 21), (4, 40)], ids=["1323v", "6400v"])
def test_apply_matches_oracle(M, layers, n, levels):
    """z = M^-1 r for random r: the device inverts in fp64 and stores fp32, as the oracle does; what is left is
    the rounding of the stored entries that differ by one fp32 ulp."""
    cloth, sysm, rhs = cloth_system(M, layers, n, seed=3)
    sysm.mas_order(cloth.positions)
    sysm.mas_setup(levels)
    rowptr, colidx, vals = sysm.to_scipy_like()
    lv = o.mas_setup(rowptr, colidx, vals, o.mas_order(cloth.positions), levels, cloth.fixed)
    assert len(lv) == levels
    rng = np.random.default_rng(0)
    for _ in range(3):
        r = rng.normal(size=3 * sysm.n)
        got = M.device.to_host(sysm.mas_apply(r))
        ref = o.mas_apply(lv, r)
        assert np.abs(got - ref).max() <= 2e-6 * np.abs(ref).max()
    # the operator is symmetric positive definite: u.Mv == v.Mu, v.Mv > 0
    u, v = rng.normal(size=3 * sysm.n), rng.normal(size=3 * sysm.n)
    mu, mv = M.device.to_host(sysm.mas_apply(u)), M.device.to_host(sysm.mas_apply(v))
    assert abs(u @ mv - v @ mu) <= 1e-9 * abs(u @ mv) and v @ mv > 0
    sysm.close()


@pytest.mark.parametrize("levels", [1, 2])
def test_mas_pcg_meets_the_reference_stopping_rule(M, levels):
    """The reference's rule on the reference's matrix: r = rhs - A d with the dense assembly of
    tests/test_solver.py:71-84 and its block-Jacobi inverses."""
    cloth, sysm, rhs = cloth_system(M, 3, 21, seed=5)
    n = sysm.n
    rowptr, colidx, vals = sysm.to_scipy_like()
    a = np.zeros((3 * n, 3 * n))
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    for r_, c_, blk in zip(rows, colidx, vals):
        a[3 * r_:3 * r_ + 3, 3 * c_:3 * c_ + 3] = blk
    pinv = np.linalg.inv(np.stack([a[3 * i:3 * i + 3, 3 * i:3 * i + 3] for i in range(n)]))
    prec = lambda r: np.einsum("nij,nj->ni", pinv, r.reshape(n, 3)).reshape(-1)  # noqa: E731
    b = rhs.copy()
    b.reshape(n, 3)[cloth.fixed] = 0.0
    sysm.mas_order(cloth.positions)
    d_bj, it_bj, ok_bj, _, _ = sysm.pcg(rhs, 1e-4, 5000)
    d, iters, ok, d0, dn = sysm.pcg(rhs, 1e-4, 5000, preconditioner="mas", mas_levels=levels)
    d = M.device.to_host(d)
    res = b - a @ d
    assert ok and 0 < iters
    assert abs(d0 - b @ prec(b)) <= 1e-9 * d0
    assert res @ prec(res) <= 1.01e-4 * (b @ prec(b))
    assert abs(res @ prec(res) - dn) <= 1e-6 * d0          # the reported residual norm is the true one
    # same iteration as the oracle's restatement (fp32-stored inverses on both sides): same count +- 2
    lv = o.mas_setup(rowptr, colidx, vals, o.mas_order(cloth.positions), levels, cloth.fixed)
    d_o, it_o, ok_o = o.pcg_solve_mas(rowptr, colidx, vals, pinv, cloth.fixed, rhs, 1e-4, 5000, lv)
    assert ok_o and abs(it_o - iters) <= 2
    # tight tolerance: the solution of the linear system
    d, iters, ok, _, _ = sysm.pcg(rhs, 1e-22, 20000, preconditioner="mas", mas_levels=levels)
    sol = np.linalg.solve(a, b)
    assert ok and np.abs(M.device.to_host(d) - sol).max() <= 1e-7 * np.abs(sol).max()
    assert np.all(M.device.to_host(d).reshape(n, 3)[cloth.fixed] == 0.0)
    sysm.close()


def test_mas_cuts_the_iteration_count_on_a_contact_stack(M):
    """Layers in contact: domains that follow the Morton order across the layers capture the contact coupling."""
    cloth, sysm, rhs = cloth_system(M, 4, 60, seed=1)
    _, it_bj, ok_bj, _, _ = sysm.pcg(rhs, 1e-4, 5000)
    sysm.mas_order(cloth.positions)
    _, it_mas, ok_mas, _, _ = sysm.pcg(rhs, 1e-4, 5000, preconditioner="mas", mas_levels=1)
    assert ok_bj and ok_mas
    assert it_mas < 0.6 * it_bj, (it_mas, it_bj)
    # deterministic: fixed summation orders, no atomics -- a second solve returns the same bits
    d_a, it_a, _, _, _ = sysm.pcg(rhs, 1e-4, 5000, preconditioner="mas", mas_levels=1)
    d_b, it_b, _, _, _ = sysm.pcg(rhs, 1e-4, 5000, preconditioner="mas", mas_levels=1)
    assert it_a == it_b == it_mas and bool((d_a == d_b).all())
    # zero right-hand side: no iterations, converged (solver.py:296-297)
    d, iters, ok, _, _ = sysm.pcg(np.zeros(3 * sysm.n), 1e-4, 100, preconditioner="mas")
    assert ok and iters == 0 and not M.device.to_host(d).any()
    # values change -> the stored inverses are rebuilt on the next solve
    sysm.vals.mul_(2.0)
    sysm.pinv = None
    sysm._mas_stale = True
    d2, it2, ok2, _, _ = sysm.pcg(rhs, 1e-4, 5000, preconditioner="mas")
    assert ok2 and abs(it2 - it_mas) <= 3
    sysm.close()


@pytest.mark.parametrize("n", [1, 5, 32, 33])
def test_tiny_systems(M, n):
    """Fewer vertices than one domain (MAS is then the exact inverse: one iteration), exactly one domain, one vertex
    into the second domain; two levels requested where only one domain exists fall back to one."""
    rng = np.random.default_rng(n)
    grouped = []
    if n >= 2:
        nb = 3 * n
        vids = np.stack([rng.choice(n, size=2, replace=False) for _ in range(nb)]).astype(np.int64)
        z = rng.normal(size=(nb, 6))
        grouped.append((z[:, :, None] * z[:, None, :], vids))
    masses, fixed = rng.uniform(0.5, 2.0, size=n), np.zeros(n, bool)
    if n >= 5:
        fixed[2] = True
    sysm = M.solver.NewtonSystem(masses, fixed)
    sysm.set_pattern([(v.shape[1], v) for _, v in grouped])
    sysm.assemble([h for h, _ in grouped])
    rhs = rng.normal(size=3 * n)
    a = o.assemble_dense(grouped, masses, fixed)
    b = rhs.copy()
    b.reshape(n, 3)[fixed] = 0.0
    sol = np.linalg.solve(a, b)
    for levels in (1, 2):
        d, iters, ok, _, _ = sysm.pcg(rhs, 1e-20, 200, preconditioner="mas", mas_levels=levels)
        assert ok and np.abs(M.device.to_host(d) - sol).max() <= 1e-9 * max(np.abs(sol).max(), 1e-300)
        if n <= 32:
            assert iters <= 2          # one domain holds the whole matrix (fp32-stored inverse: a second sweep at most)
    sysm.close()
