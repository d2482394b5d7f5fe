"""The two symbolic assembly phases -- row-wise (shared-memory column sets per block-row, the default) and
sort-by-key -- build the same pattern, the same source runs and therefore bitwise the same matrices, and both
match the oracle's restatement of the reference's dense assembly (tests/test_solver.py:71-84) bit for bit in
the pattern.  Edge cases: empty families, vertices without contacts, fixed rows and columns, a hub vertex whose
row overflows the per-warp set (fallback to the sort path), rows beyond the 16-bit limit of the row-wise
NUMERIC kernel (typed error instead of a silently wrong matrix)."""

import numpy as np
import pytest

from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2308_09400_b200 import _lib, device, solver

    class NS:
        pass

    ns = NS()
    ns.lib, ns.device, ns.solver = _lib, device, solver
    return ns


def random_families(rng, n, counts, hub=None):
    """[(hess (nb,3s,3s), vids (nb,s))] with distinct vertices per block; ``hub`` = (vertex, nb2) adds a
    two-vertex family tying ``vertex`` to nb2 different vertices."""
    grouped = []
    for s, nb in counts:
        if nb == 0:
            continue
        vids = np.stack([rng.choice(n, size=s, replace=False) for _ in range(nb)]).astype(np.int64)
        z = rng.normal(size=(nb, 3 * s))
        hess = z[:, :, None] * z[:, None, :] + 0.01 * rng.normal(size=(nb, 3 * s, 3 * s))
        grouped.append((hess, vids))
    if hub is not None:
        v, nb = hub
        others = rng.choice(np.setdiff1d(np.arange(n), [v]), size=nb, replace=False)
        vids = np.stack([np.full(nb, v), others], axis=1).astype(np.int64)
        vids[::2] = vids[::2, ::-1]
        z = rng.normal(size=(nb, 6))
        grouped.insert(0, (z[:, :, None] * z[:, None, :], vids))
    return grouped


def build(S, grouped, masses, fixed, mode, variant=0):
    sysm = S.solver.NewtonSystem(masses, fixed)
    sysm.set_symbolic_mode(mode)
    sysm.set_numeric_variant(variant)
    sysm.set_pattern([(v.shape[1], v) for _, v in grouped])
    sysm.assemble([h for h, _ in grouped])
    return sysm


CASES = [
    ("no-blocks", 50, [], None, 0.1),
    ("pairs-only", 300, [(2, 900)], None, 0.05),
    ("all-sizes", 2000, [(2, 3000), (3, 4000), (4, 9000)], None, 0.02),
    ("dense-small", 40, [(2, 500), (3, 500), (4, 2000)], None, 0.1),      # every row touches almost every column
    ("sparse-large", 50000, [(4, 30000)], None, 0.01),                     # most vertices have no contact
    ("long-rows", 600, [(4, 40000)], None, 0.0),                           # ~270 incidences per row, rows of ~400 columns: overflow
    ("hub", 5000, [(3, 2000), (4, 6000)], (17, 3000), 0.01),               # one row with 3000+ columns: overflow
]


@pytest.mark.parametrize("name,n,counts,hub,fixed_frac", CASES, ids=[c[0] for c in CASES])
def test_row_wise_symbolic_equals_sort_path_and_oracle(S, name, n, counts, hub, fixed_frac):
    rng = np.random.default_rng(len(name) * 1000 + n)
    grouped = random_families(rng, n, counts, hub)
    masses = rng.uniform(0.5, 2.0, size=n)
    fixed = rng.uniform(size=n) < fixed_frac
    a = build(S, grouped, masses, fixed, mode=0)
    b = build(S, grouped, masses, fixed, mode=1)
    assert b.stats()["symbolic"] == "sort"
    expect_rows = name not in ("long-rows", "hub", "dense-small") or a.stats()["max_row"] <= 256
    if name in ("long-rows", "hub"):
        assert a.stats()["symbolic"] == "sort"          # a row beyond the per-warp set: rebuilt by the sort path
    elif expect_rows:
        assert a.stats()["symbolic"] == "rows"
    ra, ca, va = a.to_scipy_like()
    rb, cb, vb = b.to_scipy_like()
    assert np.array_equal(ra, rb) and np.array_equal(ca, cb)
    assert np.array_equal(va, vb)                          # same runs in the same order: bitwise the same sums
    o_rowptr, o_colidx, o_vals = o.assemble_bsr(grouped, masses, fixed)
    assert np.array_equal(ra, o_rowptr) and np.array_equal(ca, o_colidx)
    assert np.abs(va - o_vals).max() <= 1e-12 * max(np.abs(o_vals).max(), 1.0)
    if a.stats()["symbolic"] == "rows":
        st = a.stats()
        assert st["max_row"] == int(np.diff(ra).max()) and st["nnzb"] == len(ca)
        assert st["sources"] == b.stats()["sources"]      # same runs: the numeric walker choice cannot differ
    # the factor path and the row-wise numeric kernel on the row-wise pattern
    if grouped and a.stats()["symbolic"] == "rows":
        r4 = build(S, grouped, masses, fixed, mode=0, variant=4)
        assert np.abs(S.device.to_host(r4.vals) - va).max() <= 1e-12 * max(np.abs(va).max(), 1.0)
        r4.close()
    # gradient runs are shared by both phases
    x, xt = rng.normal(size=(n, 3)), rng.normal(size=(n, 3))
    grads = [rng.normal(size=(h.shape[0], h.shape[1])) for h, _ in grouped]
    ga = S.device.to_host(a.gradient(x, xt, grads))
    gb = S.device.to_host(b.gradient(x, xt, grads))
    assert np.array_equal(ga, gb)
    a.close()
    b.close()


def test_factor_descriptors_from_the_row_wise_phase(S):
    """assemble_from_factors reads the descriptor table the row-wise phase wrote: same matrix as the dense path."""
    rng = np.random.default_rng(5)
    n = 3000
    fams = []
    for s, nb in ((2, 2000), (3, 3000), (4, 8000)):
        vids = np.stack([rng.choice(n, size=s, replace=False) for _ in range(nb)]).astype(np.int64)
        fams.append((rng.normal(size=(nb, 3 * s)), vids))
    masses, fixed = rng.uniform(0.5, 2.0, size=n), rng.uniform(size=n) < 0.02
    out = {}
    for mode in (0, 1):
        sysm = S.solver.NewtonSystem(masses, fixed)
        sysm.set_symbolic_mode(mode)
        sysm.set_pattern([(v.shape[1], v) for _, v in fams])
        vf = S.device.to_host(sysm.assemble_from_factors([z for z, _ in fams])).copy()
        vd = S.device.to_host(sysm.assemble([z[:, :, None] * z[:, None, :] for z, _ in fams])).copy()
        assert np.array_equal(vf, vd)
        out[mode] = vf
        sysm.close()
    assert np.array_equal(out[0], out[1])


def test_row_wise_numeric_kernel_refuses_rows_beyond_16_bits(S):
    """rs_dst holds a destination's position inside its row in 16 bits.  A hub row of >= 65535 blocks
    must be a typed error on that kernel (and still assemble correctly on the per-block-run kernel)."""
    rng = np.random.default_rng(9)
    n = 70001
    vids = np.stack([np.zeros(n - 1, np.int64), np.arange(1, n, dtype=np.int64)], axis=1)
    z = rng.normal(size=(n - 1, 6))
    hess = z[:, :, None] * z[:, None, :]
    masses, fixed = np.ones(n), np.zeros(n, bool)
    sysm = S.solver.NewtonSystem(masses, fixed)
    sysm.set_pattern([(2, vids)])
    assert sysm.stats()["symbolic"] == "sort"
    vals = S.device.to_host(sysm.assemble([hess]))
    rowptr, colidx, _ = sysm.to_scipy_like()
    assert rowptr[1] == n and np.array_equal(colidx[:n], np.arange(n))
    assert np.allclose(vals[0], np.eye(3) + np.einsum("bi,bj->ij", z[:, :3], z[:, :3]), rtol=1e-12, atol=1e-9)
    assert np.array_equal(vals[1:n], hess[:, :3, 3:])
    sysm.set_numeric_variant(4)
    with pytest.raises(S.lib.B200IpcError):
        sysm.assemble([hess])
    sysm.close()


def test_random_scenes_both_phases_and_oracle(S):
    """Randomised stress (scripts/symbolic_stress.py, shortened): clustered vertex choices so that rows get long
    and share columns, 0 - 30 % Dirichlet vertices -- both symbolic phases and the oracle, pattern and values."""
    rng = np.random.default_rng(12345)
    for case in range(25):
        n = int(rng.integers(2, 3000))
        fams = []
        for s in (2, 3, 4):
            nb = int(rng.integers(0, 6 * n))
            if n < s or nb == 0:
                continue
            centre = rng.integers(0, n, size=nb)
            width = max(s, int(rng.integers(s, max(s + 1, n // int(rng.integers(1, 40)) + s))))
            vids = np.stack([(c + rng.choice(width, size=s, replace=False)) % n for c in centre]).astype(np.int64)
            vids = vids[np.array([len(set(v)) == s for v in vids])]
            if len(vids):
                z = rng.normal(size=(len(vids), 3 * s))
                fams.append((z[:, :, None] * z[:, None, :], vids))
        masses = rng.uniform(0.5, 2.0, size=n)
        fixed = rng.uniform(size=n) < rng.choice([0.0, 0.02, 0.3])
        a, b = build(S, fams, masses, fixed, mode=0), build(S, fams, masses, fixed, mode=1)
        ra, ca, va = a.to_scipy_like()
        rb, cb, vb = b.to_scipy_like()
        o_rowptr, o_colidx, o_vals = o.assemble_bsr(fams, masses, fixed)
        assert np.array_equal(ra, rb) and np.array_equal(ca, cb) and np.array_equal(va, vb), case
        assert np.array_equal(ra, o_rowptr) and np.array_equal(ca, o_colidx), case
        assert np.abs(va - o_vals).max() <= 1e-12 * max(np.abs(o_vals).max(), 1.0), case
        a.close()
        b.close()
