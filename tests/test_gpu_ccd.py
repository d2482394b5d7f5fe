"""GPU additive CCD: per-pair bounds bit-identical to the reference's compiled
accd_max_step, swept-AABB candidates identical as sets, global step bound identical."""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import load_golden
from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_2308_09400_b200 import contacts, device, kernels, workloads

    return SimpleNamespace(contacts=contacts, device=device, kernels=kernels, workloads=workloads)


def _rows(a):
    a = np.asarray(a, dtype=np.int64).reshape(-1, 4)
    return a[np.lexsort(a.T[::-1])]


def _batch(G, x, dx, kind, slack, max_iter=512):
    n, s = x.shape[0], x.shape[1]
    ids = np.zeros((n, 4), np.int32)
    ids[:, :s] = np.arange(n * s).reshape(n, s)
    step, status = G.kernels.accd_max_step_device(G.device.to_device(ids), kind, G.device.to_device(x.reshape(-1, 3)),
                                                  G.device.to_device(dx.reshape(-1, 3)), slack, max_iter)
    return G.device.to_host(step), G.device.to_host(status)


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_accd_batch_bit_exact_with_reference(G, kind):
    z = load_golden("ccd")
    x, dx = z[f"k{kind}_x"], z[f"k{kind}_dx"]
    step, status = _batch(G, x, dx, kind, 0.9)
    assert not status.any()
    np.testing.assert_array_equal(step, z[f"k{kind}_step"])
    capped, _ = _batch(G, x, dx, kind, 0.5, 3)
    np.testing.assert_array_equal(capped, z[f"k{kind}_step_s05_it3"])
    # mixed kinds in one launch (per-pair kind array)
    if kind == 0:
        xs = [z[f"k{k}_x"][:50] for k in range(4)]
        ds = [z[f"k{k}_dx"][:50] for k in range(4)]
        pos = np.concatenate([a.reshape(-1, 3) for a in xs])
        dirs = np.concatenate([a.reshape(-1, 3) for a in ds])
        ids, kinds, base = [], [], 0
        for k, a in enumerate(xs):
            s = a.shape[1]
            row = np.zeros((50, 4), np.int32)
            row[:, :s] = base + np.arange(50 * s).reshape(50, s)
            ids.append(row); kinds.append(np.full(50, k, np.uint8)); base += 50 * s
        step, status = G.kernels.accd_max_step_device(
            G.device.to_device(np.concatenate(ids)), G.device.to_device(np.concatenate(kinds)),
            G.device.to_device(pos), G.device.to_device(dirs), 0.9)
        np.testing.assert_array_equal(G.device.to_host(step), np.concatenate([z[f"k{k}_step"][:50] for k in range(4)]))


def test_accd_single_pair_twin_and_errors(G):
    """kernels.accd_max_step keeps the reference signature; a touching pair raises ValueError."""
    z = load_golden("ccd")
    for kind in range(4):
        for i in (0, 25, 200):
            got = G.kernels.accd_max_step(z[f"k{kind}_x"][i], z[f"k{kind}_dx"][i], kind, 0.9)
            assert got == z[f"k{kind}_step"][i]
    # accd_step_bound(stencil, ...) twin (proximity.py:372-385): parallel kinds run as EE pairs
    from paper_2308_09400_b200.proximity import ContactStencil, StencilKind

    x, dx = z["k1_x"][30], z["k1_dx"][30]
    st = ContactStencil(kind=StencilKind.EDGE_EDGE_PARALLEL, verts=(0, 1, 2, 3), eps_x=1.0, sub=(0, 1, 2, 3))
    assert G.contacts.accd_step_bound(st, x, dx) == z["k1_step"][30]
    st = ContactStencil(kind=StencilKind.POINT_POINT, verts=(1, 0))
    assert G.contacts.accd_step_bound(st, z["k3_x"][40][::-1], z["k3_dx"][40][::-1]) == G.kernels.accd_max_step(
        z["k3_x"][40], z["k3_dx"][40], 3, 0.9)
    with pytest.raises(ValueError):
        G.kernels.accd_max_step(np.zeros((2, 3)), np.array([[1.0, 0, 0], [-1.0, 0, 0]]), G.kernels.PAIR_PP, 0.9)


def test_sweep_candidates_and_ccd_filter_match_reference(G):
    z = load_golden("ccd")
    x, d, tris, edges, d_hat = (z["scene_positions"], z["scene_directions"], z["scene_tris"], z["scene_edges"],
                                float(z["scene_d_hat"]))
    kinds, ref_ids = z["scene_cand_kind"], z["scene_cand_ids"]
    bp = G.contacts.BroadPhase(np.unique(tris), tris, edges, d_hat, x)
    vt, ee = bp.sweep(x, d)
    np.testing.assert_array_equal(_rows(G.device.to_host(vt)), _rows(ref_ids[kinds == 0]))
    np.testing.assert_array_equal(_rows(G.device.to_host(ee)), _rows(ref_ids[kinds == 1]))
    alpha = bp.ccd_step_bound(x, d)
    assert alpha == float(z["scene_alpha"])
    bp.close()
    # reference-shaped entry points
    scene = SimpleNamespace(surf_tris=tris, surf_edges=edges, surf_verts=np.unique(tris))
    cands = G.contacts.sweep_candidates(scene, x, d, d_hat)
    assert sorted(cands) == sorted((int(k), tuple(int(v) for v in ids)) for k, ids in zip(kinds, ref_ids))
    assert G.contacts.global_ccd_filter(scene, x, d, cands) == float(z["scene_alpha"])
    assert G.contacts.global_ccd_filter(scene, x, d, []) == 1.0


def test_ccd_filter_large_scene_against_oracle(G):
    """A 4 x 24 x 24 stack: device candidates == all-pairs oracle, global bound bit-identical, and the
    verified step really keeps every candidate's distance positive."""
    cloth = G.workloads.cloth_stack(layers=4, n=24, seed=21)
    rng = np.random.default_rng(5)
    x = cloth.positions
    d = 0.6 * cloth.d_hat * rng.normal(size=x.shape)
    surf = np.unique(cloth.tris)
    vt, ee = o.sweep_candidates(x, d, surf, cloth.tris, cloth.edges, cloth.d_hat)
    bp = G.contacts.BroadPhase(surf, cloth.tris, cloth.edges, cloth.d_hat, x)
    g_vt, g_ee = bp.sweep(x, d)
    np.testing.assert_array_equal(_rows(G.device.to_host(g_vt)), _rows(vt))
    np.testing.assert_array_equal(_rows(G.device.to_host(g_ee)), _rows(ee))
    alpha = bp.ccd_step_bound(x, d)
    bp.close()
    assert alpha == o.global_ccd_filter(x, d, vt, ee)
    assert 0.0 < alpha <= 1.0
    xe = x + alpha * d
    d2 = o.pt_classify_batch(xe[vt[:, 0]], xe[vt[:, 1]], xe[vt[:, 2]], xe[vt[:, 3]])[1]
    assert d2.min() > 0.0


def test_superset_filter_equals_the_reference_candidate_filter(G):
    """One swept join with a margin of 0.51 d_hat, cut down by the reference's own swept-box test at 1e-3 d_hat on
    the device, gives the bound of sweep_candidates + global_ccd_filter bit for bit; and it contains every pair a
    static detection finds anywhere on the step (the line search then skips its broad phase)."""
    cloth = G.workloads.cloth_stack(layers=4, n=24, seed=21)
    rng = np.random.default_rng(3)
    dirs = 0.4 * cloth.d_hat * rng.normal(size=cloth.positions.shape)
    bp = G.contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
    pos, dd = G.device.to_device(cloth.positions), G.device.to_device(dirs)
    exact = bp.ccd_step_bound(pos, dd)
    vt, ee = bp.sweep(pos, dd, margin=0.51 * cloth.d_hat)
    ref_vt, ref_ee = bp.sweep(pos, dd)
    assert vt.shape[0] > ref_vt.shape[0] and ee.shape[0] > ref_ee.shape[0]
    got = G.contacts.ccd_filter_superset_device(vt, ee, pos, dd, 1e-3 * cloth.d_hat)
    assert got == exact
    as_set = lambda t: set(map(tuple, G.device.to_host(t).tolist()))  # noqa: E731
    big_vt, big_ee = as_set(vt), as_set(ee)
    for alpha in (0.0, 0.37, 1.0):
        q_vt, q_ee = bp.query(G.device.to_device(cloth.positions + alpha * dirs))
        assert as_set(q_vt) <= big_vt and as_set(q_ee) <= big_ee
    bp.close()
