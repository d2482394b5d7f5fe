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
