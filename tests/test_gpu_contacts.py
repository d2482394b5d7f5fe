"""GPU narrow phase: bit-exact ordered contact lists (kind, verts, sub, eps_x, origin)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu

KEYS = ("kind", "verts", "sub", "eps_x", "origin_type", "origin")


@pytest.fixture(scope="module")
def Cn():
    from paper_2308_09400_b200 import contacts, proximity, workloads

    class NS:
        pass

    ns = NS()
    ns.contacts, ns.proximity, ns.workloads = contacts, proximity, workloads
    return ns


def all_pairs(tris, edges):
    verts = np.unique(tris)
    vv, tt = np.meshgrid(verts, np.arange(tris.shape[0]), indexing="ij")
    vt = np.concatenate([vv.reshape(-1, 1), tris[tt.reshape(-1)]], axis=1)
    vt = vt[(vt[:, :1] != vt[:, 1:]).all(axis=1)]
    i, j = np.triu_indices(edges.shape[0], 1)
    ee = np.concatenate([edges[i], edges[j]], axis=1)
    ee = ee[(ee[:, 0] != ee[:, 2]) & (ee[:, 0] != ee[:, 3]) & (ee[:, 1] != ee[:, 2]) & (ee[:, 1] != ee[:, 3])]
    return vt, ee


def assert_same_table(got, ref):
    for key in KEYS:
        np.testing.assert_array_equal(getattr(got, key), ref[key], err_msg=key)


def test_golden_scene_list_is_bit_exact(Cn):
    """The reference's find_contact_pairs output on the golden cloth scene, row for row."""
    z = load_golden("scene")
    vt, ee = all_pairs(z["tris"], z["edges"])
    got = Cn.contacts.narrow_phase(z["positions"], z["rest_positions"], vt, ee, float(z["d_hat"]))
    assert_same_table(got, z)
    # grid broad phase instead of all pairs: identical list
    scene = type("S", (), dict(surf_tris=z["tris"], surf_edges=z["edges"], rest_positions=z["rest_positions"]))()
    stencils = Cn.contacts.find_contact_pairs(scene, z["positions"], float(z["d_hat"]))
    table = Cn.proximity.StencilTable.from_stencils(stencils)
    assert_same_table(table, z)
    assert stencils == sorted(stencils, key=lambda s: s.sort_key())
    # no promotion: plain kinds only, same queries
    plain = Cn.contacts.narrow_phase(z["positions"], z["rest_positions"], vt, ee, float(z["d_hat"]), promote_parallel=False)
    ref = o.narrow_phase(z["positions"], z["rest_positions"], vt, ee, float(z["d_hat"]), promote_parallel=False)
    assert_same_table(plain, ref)
    assert not np.any(np.isin(plain.kind, (1, 3, 5)))


def test_config2_kinds_and_order_vs_oracle(Cn):
    qb = Cn.workloads.config2_batch(n=60000)
    got = Cn.contacts.narrow_phase(qb.positions, qb.rest_positions, qb.vt, qb.ee, qb.d_hat)
    ref = o.narrow_phase(qb.positions, qb.rest_positions, qb.vt, qb.ee, qb.d_hat)
    assert_same_table(got, ref)
    assert {1, 3, 5} <= set(got.kind.tolist())
    np.testing.assert_array_equal(got.kind_offsets(), np.searchsorted(ref["kind"], np.arange(8)))


def test_config1_and_empty(Cn):
    qb = Cn.workloads.config1_batch(n_pt=3000, n_ee=3000)
    got = Cn.contacts.narrow_phase(qb.positions, qb.rest_positions, qb.vt, qb.ee, qb.d_hat)
    ref = o.narrow_phase(qb.positions, qb.rest_positions, qb.vt, qb.ee, qb.d_hat)
    assert_same_table(got, ref)
    far = Cn.contacts.narrow_phase(qb.positions, qb.rest_positions, qb.vt, qb.ee, 1e-6)
    assert len(far) == 0
    none = Cn.contacts.narrow_phase(qb.positions, qb.rest_positions, np.zeros((0, 4), int), np.zeros((0, 4), int), 1.0)
    assert len(none) == 0


def test_cloth_stack_grid_broad_phase_vs_all_pairs(Cn):
    """Conservative grid candidates give the same list as all pairs on a 4-layer cloth stack."""
    cloth = Cn.workloads.cloth_stack(layers=4, n=10, seed=5)
    vt_all, ee_all = all_pairs(cloth.tris, cloth.edges)
    ref = o.narrow_phase(cloth.positions, cloth.rest_positions, vt_all, ee_all, cloth.d_hat)
    vt, ee = Cn.workloads.broad_phase(cloth)
    assert len(vt) < len(vt_all) and len(ee) < len(ee_all)
    got = Cn.contacts.narrow_phase(cloth.positions, cloth.rest_positions, vt, ee, cloth.d_hat)
    assert_same_table(got, ref)
    assert len(got) > 2000


def _rows(a):
    a = np.asarray(a, dtype=np.int64).reshape(-1, 4)
    return a[np.lexsort(a.T[::-1])]


@pytest.mark.parametrize("layers,n,seed", [(4, 10, 5), (3, 14, 2), (1, 9, 3)])
def test_gpu_broad_phase_equals_reference_aabb_candidates(Cn, layers, n, seed):
    """The grid join reports exactly the reference's AABB-overlap candidates, each once."""
    from paper_2308_09400_b200 import device

    cloth = Cn.workloads.cloth_stack(layers=layers, n=n, seed=seed)
    surf = np.unique(cloth.tris)
    ref_vt, ref_ee = o.aabb_candidates(cloth.positions, surf, cloth.tris, cloth.edges, cloth.d_hat)
    for cell in (None, 0.37 * cloth.d_hat, 11.0 * cloth.d_hat):   # cell size is a speed knob only
        bp = Cn.contacts.BroadPhase(surf, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions, cell=cell)
        vt, ee = bp.query(cloth.positions)
        bp.close()
        vt, ee = device.to_host(vt), device.to_host(ee)
        assert vt.dtype == np.int32 and ee.dtype == np.int32
        np.testing.assert_array_equal(_rows(vt), _rows(ref_vt))
        np.testing.assert_array_equal(_rows(ee), _rows(ref_ee))
    assert len(ref_vt) > 0 and (layers == 1 or len(ref_ee) > 100)


def test_gpu_broad_phase_list_regrows_and_shrinks(Cn):
    """The appending join keeps its candidate list between queries: a sparse pose first (short list), then
    a pose with many times more candidates (the pass only counts, the list is regrown, the pass repeats),
    then the sparse pose again (long list, few rows) -- every answer is the reference's candidate set, and
    sheets with many hits per probe (more than the four a thread holds in registers) flush correctly."""
    from paper_2308_09400_b200 import device

    cloth = Cn.workloads.cloth_stack(layers=4, n=12, seed=11)
    surf = np.unique(cloth.tris)
    sparse = cloth.positions.copy()
    sparse[:, 2] *= 40.0                      # sheets far apart: only in-sheet neighbours overlap
    dense = cloth.positions.copy()
    dense[:, 2] *= 0.05                       # sheets almost coincident
    # a d_hat of several cell widths makes every box overlap dozens of others
    d_hat = 3.0 * cloth.d_hat
    bp = Cn.contacts.BroadPhase(surf, cloth.tris, cloth.edges, d_hat, cloth.positions)
    sizes = []
    for x in (sparse, dense, sparse, dense):
        vt, ee = bp.query(device.to_device(x))
        ref_vt, ref_ee = o.aabb_candidates(x, surf, cloth.tris, cloth.edges, d_hat)
        np.testing.assert_array_equal(_rows(device.to_host(vt)), _rows(ref_vt))
        np.testing.assert_array_equal(_rows(device.to_host(ee)), _rows(ref_ee))
        sizes.append(len(ref_ee))
    # a cell-count hint far too small for the scene (coordinates clamp into the boundary cells, which
    # merge): slower, same candidate set
    from paper_2308_09400_b200 import _lib

    grid = bp._grid

    def tiny(span, margin):
        origin = grid(span, margin)
        _lib.check(_lib.lib().b200ipc_broad_set_grid_cells(bp._h, 3, 2, 1), "broad_set_grid_cells")
        return origin

    bp._grid = tiny
    vt, ee = bp.query(device.to_device(dense))
    np.testing.assert_array_equal(_rows(device.to_host(vt)), _rows(ref_vt))
    np.testing.assert_array_equal(_rows(device.to_host(ee)), _rows(ref_ee))

    # a grid of more than 2^21 cells (here: the widest hint, 63 key bits) has no dense cell table: the join finds
    # its column runs by binary search instead -- same candidate set
    def huge(span, margin):
        origin = grid(span, margin)
        _lib.check(_lib.lib().b200ipc_broad_set_grid_cells(bp._h, 1 << 21, 1 << 21, 1 << 21), "broad_set_grid_cells")
        return origin

    bp._grid = huge
    for x in (dense, sparse):
        vt, ee = bp.query(device.to_device(x))
        ref_vt, ref_ee = o.aabb_candidates(x, surf, cloth.tris, cloth.edges, d_hat)
        np.testing.assert_array_equal(_rows(device.to_host(vt)), _rows(ref_vt))
        np.testing.assert_array_equal(_rows(device.to_host(ee)), _rows(ref_ee))
    bp.close()
    assert sizes[1] > 3 * sizes[0] and sizes[1] > 9 * 4 * len(cloth.edges)   # > 4 hits per (box, slot) on average


def test_gpu_broad_phase_two_size_classes(Cn):
    """Cloth draped on a coarse sphere (collider edges many cells long): the broad phase files the long boxes on a
    coarse grid of their own and joins every A box with both bin lists -- the candidate set is still exactly the
    reference's, for the static query and for the swept one, and whatever the class boundary does to the split
    (coarse cell barely above / far above the threshold, classes off)."""
    from paper_2308_09400_b200 import _lib, device

    scene = Cn.workloads.cloth_on_sphere(n=26, subdiv=2, seed=4)
    surf = np.unique(scene.tris)
    ref_vt, ref_ee = o.aabb_candidates(scene.positions, surf, scene.tris, scene.edges, scene.d_hat)
    assert len(ref_vt) > 50 and len(ref_ee) > 50
    bp = Cn.contacts.BroadPhase(surf, scene.tris, scene.edges, scene.d_hat, scene.positions)
    assert bp.coarse_cell > 2.0 * bp.cell                       # the scene does trigger the second class
    for coarse in (bp.coarse_cell, 2.01 * bp.cell, 40.0 * bp.cell, 0.0):
        _lib.check(_lib.lib().b200ipc_broad_set_coarse_cell(bp._h, coarse), "broad_set_coarse_cell")
        vt, ee = bp.query(scene.positions)
        np.testing.assert_array_equal(_rows(device.to_host(vt)), _rows(ref_vt))
        np.testing.assert_array_equal(_rows(device.to_host(ee)), _rows(ref_ee))
    _lib.check(_lib.lib().b200ipc_broad_set_coarse_cell(bp._h, bp.coarse_cell), "broad_set_coarse_cell")
    rng = np.random.default_rng(8)
    d = 0.4 * scene.d_hat * rng.normal(size=scene.positions.shape)
    s_vt, s_ee = bp.sweep(scene.positions, d)
    r_vt, r_ee = o.sweep_candidates(scene.positions, d, surf, scene.tris, scene.edges, scene.d_hat)
    np.testing.assert_array_equal(_rows(device.to_host(s_vt)), _rows(r_vt))
    np.testing.assert_array_equal(_rows(device.to_host(s_ee)), _rows(r_ee))
    bp.close()


def test_gpu_broad_phase_moving_scene_and_find_contact_pairs(Cn):
    """One handle, several detects (positions change); find_contact_pairs end to end on the GPU."""
    from types import SimpleNamespace

    from paper_2308_09400_b200 import device

    cloth = Cn.workloads.cloth_stack(layers=3, n=12, seed=9)
    surf = np.unique(cloth.tris)
    bp = Cn.contacts.BroadPhase(surf, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
    rng = np.random.default_rng(4)
    for step in range(3):
        x = cloth.positions + step * 0.1 * cloth.d_hat * rng.normal(size=cloth.positions.shape)
        vt, ee = bp.query(device.to_device(x))
        ref_vt, ref_ee = o.aabb_candidates(x, surf, cloth.tris, cloth.edges, cloth.d_hat)
        np.testing.assert_array_equal(_rows(device.to_host(vt)), _rows(ref_vt))
        np.testing.assert_array_equal(_rows(device.to_host(ee)), _rows(ref_ee))
        got = Cn.contacts.narrow_phase(x, cloth.rest_positions, vt, ee, cloth.d_hat)
        ref = o.narrow_phase(x, cloth.rest_positions, ref_vt, ref_ee, cloth.d_hat)
        assert_same_table(got, ref)
    bp.close()
    scene = SimpleNamespace(surf_tris=cloth.tris, surf_edges=cloth.edges, surf_verts=surf,
                            rest_positions=cloth.rest_positions)
    stencils = Cn.contacts.find_contact_pairs(scene, cloth.positions, cloth.d_hat)
    ref = o.narrow_phase(cloth.positions, cloth.rest_positions, *o.aabb_candidates(
        cloth.positions, surf, cloth.tris, cloth.edges, cloth.d_hat), cloth.d_hat)
    assert len(stencils) == len(ref["kind"]) > 1000
    assert [tuple(v for v in s.verts) for s in stencils[:50]] == [
        tuple(int(v) for v in row if v >= 0) for row in ref["verts"][:50]]


def test_gpu_broad_phase_empty_inputs(Cn):
    bp = Cn.contacts.BroadPhase(np.zeros(0, int), np.zeros((0, 3), int), np.zeros((0, 2), int), 0.1)
    vt, ee = bp.query(np.zeros((4, 3)))
    assert vt.shape == (0, 4) and ee.shape == (0, 4)
    bp.close()


@pytest.mark.parametrize("tag", ["a", "b"])
def test_gpu_detect_matches_frozen_reference(Cn, tag):
    """Broad + narrow phase on the GPU against the reference's frozen candidates and contact list."""
    from paper_2308_09400_b200 import device

    z = load_golden("broad")
    x, tris, edges, d_hat = z[f"{tag}_positions"], z[f"{tag}_tris"], z[f"{tag}_edges"], float(z[f"{tag}_d_hat"])
    bp = Cn.contacts.BroadPhase(np.unique(tris), tris, edges, d_hat, x)
    vt, ee = bp.query(x)
    np.testing.assert_array_equal(_rows(device.to_host(vt)), _rows(z[f"{tag}_vt"]))
    np.testing.assert_array_equal(_rows(device.to_host(ee)), _rows(z[f"{tag}_ee"]))
    got = Cn.contacts.narrow_phase(x, z[f"{tag}_rest_positions"], vt, ee, d_hat)
    bp.close()
    for key in KEYS:
        np.testing.assert_array_equal(getattr(got, key), z[f"{tag}_list_{key}"], err_msg=key)


def test_long_tie_runs_are_ordered_by_origin(Cn):
    """Two cones whose apexes almost touch: every (upper spoke, lower spoke) edge query and every
    apex-triangle query reduces to the same point-point stencil, a run of ~m*m + 2m equal (kind, vertices)
    keys that the narrow phase must order by origin exactly as the reference's sort_key does -- in random
    candidate order, as the broad phase delivers them."""
    m = 14
    ang = 2.0 * np.pi * np.arange(m) / m
    rng = np.random.default_rng(12)
    up = np.stack([np.cos(ang), np.sin(ang), np.full(m, 1.0)], axis=1) + 0.01 * rng.normal(size=(m, 3))
    dn = np.stack([np.cos(ang + 0.2), np.sin(ang + 0.2), np.full(m, -1.0)], axis=1) + 0.01 * rng.normal(size=(m, 3))
    pos = np.concatenate([[[0.0, 0.0, 0.004]], up, [[0.001, -0.002, -0.004]], dn])   # apex A = 0, apex B = m + 1
    a, b = 0, m + 1
    tris = np.array([[a, 1 + i, 1 + (i + 1) % m] for i in range(m)] + [[b, b + 1 + i, b + 1 + (i + 1) % m] for i in range(m)])
    edges = np.unique(np.sort(np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]]), axis=1), axis=0)
    d_hat = 0.05
    vt, ee = all_pairs(tris, edges)
    ref = o.narrow_phase(pos, pos, vt, ee, d_hat)
    key = np.concatenate([ref["kind"][:, None].astype(np.int64), ref["verts"]], axis=1)
    _, counts = np.unique(key, axis=0, return_counts=True)
    assert counts.max() >= 200                                              # one very long run of ties (210 of the 224 queries)
    vt_s, ee_s = vt[rng.permutation(len(vt))], ee[rng.permutation(len(ee))]  # unordered candidate sets
    got = Cn.contacts.narrow_phase(pos, pos, vt_s, ee_s, d_hat)
    assert_same_table(got, ref)
