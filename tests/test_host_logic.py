"""Host-side logic that needs no GPU: stencil table, kind order, broad phase, generators, params."""

import numpy as np
import pytest

from oracle import tetipc_oracle as o
from paper_2308_09400_b200 import barrier, proximity, scene_batch, solver, workloads
from paper_2308_09400_b200.proximity import ContactStencil, StencilKind, StencilTable


def test_kind_codes_follow_reference_list_order():
    assert [k.value for k in proximity.KIND_ORDER] == list(o.KIND_NAMES)
    assert (proximity.EE, proximity.EEP, proximity.PE, proximity.PEP, proximity.PP, proximity.PPP, proximity.PT) == (
        o.EE, o.EEP, o.PE, o.PEP, o.PP, o.PPP, o.PT)
    np.testing.assert_array_equal(proximity.KIND_SIZE, o.KIND_SIZE)
    np.testing.assert_array_equal(proximity.IS_PARALLEL, o.IS_PARALLEL)


def test_table_roundtrip_and_validation():
    stencils = [
        ContactStencil(kind=StencilKind.POINT_TRIANGLE, verts=(3, 0, 1, 2), origin=("vt", 3, 0, 1, 2)),
        ContactStencil(kind=StencilKind.EDGE_EDGE, verts=(0, 1, 4, 5), origin=("ee", 0, 1, 4, 5)),
        ContactStencil(kind=StencilKind.POINT_EDGE_PARALLEL, verts=(0, 1, 6, 7), eps_x=1e-3, sub=(2, 0, 1),
                       edge_pair=((0, 1), (6, 7)), origin=("ee", 0, 1, 6, 7)),
        ContactStencil(kind=StencilKind.POINT_POINT, verts=(1, 6), origin=("ee", 0, 1, 6, 7)),
    ]
    table = StencilTable.from_stencils(stencils, sort=True)
    assert table.kind.tolist() == [0, 3, 4, 6]
    assert table.verts[2].tolist() == [1, 6, -1, -1]
    assert table.sub[1] == o.pack_sub((2, 0, 1)) and table.eps_x[1] == 1e-3
    back = table.to_stencils()
    assert back == sorted(stencils, key=lambda s: s.sort_key())
    np.testing.assert_array_equal(table.kind_offsets(), [0, 1, 1, 1, 2, 3, 3, 4])
    assert table.family_rows(4).tolist() == [0, 1, 3] and table.family_rows(2).tolist() == [2]
    with pytest.raises(proximity.ProximityError):
        StencilTable([6, 0], np.zeros((2, 4)), np.zeros(2), np.zeros(2))  # not kind sorted
    with pytest.raises(proximity.ProximityError):
        ContactStencil(kind=StencilKind.POINT_EDGE, verts=(0, 1))
    with pytest.raises(proximity.ProximityError):
        ContactStencil(kind=StencilKind.EDGE_EDGE_PARALLEL, verts=(0, 1, 2, 3))


def test_params_mirror_reference_expressions():
    with pytest.raises(ValueError):
        barrier.BarrierParams(d_hat=1.0, d_thr_ratio=1.5)
    with pytest.raises(ValueError):
        barrier.BarrierParams(d_hat=1.0, form="cubic")
    p = barrier.BarrierParams(d_hat=5e-3, kappa=2e8)
    assert p.eps_g == 0.1 * 0.1 and p.d_thr == 0.1 * 5e-3
    c = barrier.c_params(p, dt=0.01)
    assert c.d_hat_sq == 5e-3 * 5e-3 and c.d_hat_pow2 == 5e-3**2 and c.scale == 2e8 * 5e-3**4
    assert c.dt2 == 0.01**2 and c.use_filter == 1 and c.form == 0


def all_pairs(tris, edges):
    verts = np.unique(tris)
    vv, tt = np.meshgrid(verts, np.arange(tris.shape[0]), indexing="ij")
    vt = np.concatenate([vv.reshape(-1, 1), tris[tt.reshape(-1)]], axis=1)
    vt = vt[(vt[:, :1] != vt[:, 1:]).all(axis=1)]
    i, j = np.triu_indices(edges.shape[0], 1)
    ee = np.concatenate([edges[i], edges[j]], axis=1)
    return vt, ee[(ee[:, 0] != ee[:, 2]) & (ee[:, 0] != ee[:, 3]) & (ee[:, 1] != ee[:, 2]) & (ee[:, 1] != ee[:, 3])]


@pytest.mark.parametrize("seed,layers,n", [(5, 4, 9), (2, 2, 12)])
def test_grid_broad_phase_is_a_duplicate_free_superset(seed, layers, n):
    cloth = workloads.cloth_stack(layers=layers, n=n, seed=seed)
    vt, ee = workloads.broad_phase(cloth)
    assert len(np.unique(vt, axis=0)) == len(vt) and len(np.unique(ee, axis=0)) == len(ee)
    vt_all, ee_all = all_pairs(cloth.tris, cloth.edges)
    ref = o.narrow_phase(cloth.positions, cloth.rest_positions, vt_all, ee_all, cloth.d_hat)
    got = o.narrow_phase(cloth.positions, cloth.rest_positions, vt, ee, cloth.d_hat)
    for key in ref:
        np.testing.assert_array_equal(got[key], ref[key], err_msg=key)
    assert len(ref["kind"]) > 500 and len(vt) < len(vt_all) // 4


def test_generators_are_seeded_and_hit_their_distances():
    a, b = workloads.config1_batch(n_pt=50, n_ee=50), workloads.config1_batch(n_pt=50, n_ee=50)
    np.testing.assert_array_equal(a.positions, b.positions)
    tab = o.narrow_phase(a.positions, a.rest_positions, a.vt, a.ee, a.d_hat)
    assert np.bincount(tab["kind"], minlength=7).tolist() == [50, 0, 0, 0, 0, 0, 50]
    rng = np.random.default_rng(0)
    d = rng.uniform(0.1, 0.9, 200)
    x = workloads.gen_point_triangle(rng, 200, d)
    codes, d2, _, _ = o.pt_classify_batch(x[:, 0], x[:, 1], x[:, 2], x[:, 3])
    assert np.all(codes == 0)
    np.testing.assert_allclose(np.sqrt(d2), d, rtol=1e-9)
    x = workloads.gen_edge_edge(rng, 200, d)
    codes, d2, _, _ = o.ee_classify_batch(x[:, 0], x[:, 1], x[:, 2], x[:, 3])
    assert np.all(codes == 8)
    np.testing.assert_allclose(np.sqrt(d2), d, rtol=1e-9)
    x = workloads.gen_exact_parallel_edge_edge(rng, 50, rng.integers(13, 58, 50))
    c, _ = o.cross_sq_batch(x[:, 0], x[:, 1], x[:, 2], x[:, 3])
    assert np.all(c == 0.0)
    qb = workloads.config2_batch(n=4000)
    kinds = set(o.narrow_phase(qb.positions, qb.rest_positions, qb.vt, qb.ee, qb.d_hat)["kind"].tolist())
    assert {o.EEP, o.PEP, o.PPP} <= kinds


def test_group_blocks_layout():
    rng = np.random.default_rng(1)
    blocks = []
    for s in (4, 2, 3, 4, 2):
        blocks.append(barrier.LocalQuadratic(vert_ids=np.arange(s, dtype=np.int64), grad=rng.normal(size=3 * s),
                                             hess=rng.normal(size=(3 * s, 3 * s))))
    grouped = solver.group_blocks(blocks)
    assert [h.shape for h, _ in grouped] == [(2, 6, 6), (1, 9, 9), (2, 12, 12)]
    np.testing.assert_array_equal(grouped[2][0][1], blocks[3].hess)
    assert solver.group_blocks([]) == []


def test_scene_batch_single_process():
    assert scene_batch.replica_seed(10, 3) == 13
    assert scene_batch.aggregate(5.0, 2.0) == (5.0, 2.0)
    assert scene_batch.throughput(8e6, 2.0, 4) == pytest.approx(1.6e10)


def test_cloth_on_sphere_generator():
    """configs[2] scene at a small size: closed icosphere, seeded, sheets outside the sphere, contacts of
    several kinds and no penetration (oracle narrow phase on all-pairs candidates)."""
    from oracle import tetipc_oracle as o
    from paper_2308_09400_b200 import workloads

    v, f = workloads._icosphere(2)
    assert v.shape == (162, 3) and f.shape == (320, 3) and np.abs(np.linalg.norm(v, axis=1) - 1.0).max() < 1e-15
    e = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), axis=1)
    assert (np.unique(e, axis=0, return_counts=True)[1] == 2).all()          # closed surface
    a = workloads.cloth_on_sphere(n=36, layers=2, subdiv=2, seed=4)
    b = workloads.cloth_on_sphere(n=36, layers=2, subdiv=2, seed=4)
    assert np.array_equal(a.positions, b.positions) and a.positions.shape[0] == 162 + 2 * 36 * 36
    assert a.fixed[:162].all() and (np.linalg.norm(a.positions[162:], axis=1) > 1.0).all()
    vt, ee = o.aabb_candidates(a.positions, np.unique(a.tris), a.tris, a.edges, a.d_hat)
    tab = o.narrow_phase(a.positions, a.rest_positions, vt, ee, a.d_hat)
    out = o.local_quadratics_batch(tab["kind"], tab["verts"], tab["sub"], tab["eps_x"], a.positions, a.d_hat, a.kappa)
    assert len(tab["kind"]) > 1000 and len(np.unique(tab["kind"])) >= 4 and not (out["status"] == 2).any()


def test_stepper_config_and_reexport():
    """SolverConfig validation like solver.py:46-51; the stepper is reachable under the reference's
    import path; the baseline mode is refused, not silently substituted."""
    from paper_2308_09400_b200 import stepper

    params = barrier.BarrierParams(d_hat=1e-2, kappa=1.0)
    cfg = solver.SolverConfig(dt=0.01, barrier=params)
    assert (cfg.eps_d, cfg.pcg_rel_tol, cfg.pcg_max_iters, cfg.newton_max_iters) == (1e-2, 1e-4, 2000, 100)
    assert (cfg.accd_slack, cfg.line_search_floor, cfg.mollify, cfg.mode) == (0.9, 1e-12, True, "gipc")
    assert solver.SimState is stepper.SimState and solver.advance_time_step is stepper.advance_time_step
    for bad in (dict(dt=0.0), dict(dt=0.01, eps_d=0.0), dict(dt=0.01, pcg_rel_tol=-1.0)):
        with pytest.raises(ValueError):
            stepper.SolverConfig(barrier=params, **bad)
    with pytest.raises(ValueError):
        stepper.SolverConfig(dt=0.01, barrier=params, mode="nonsense")
    with pytest.raises(NotImplementedError):
        stepper.SolverConfig(dt=0.01, barrier=params, mode="reference-ipc")
    with pytest.raises(AttributeError):
        solver.no_such_name


def test_stepper_materials_per_body_and_per_tet():
    from types import SimpleNamespace

    from paper_2308_09400_b200 import elasticity, stepper

    soft, hard = elasticity.ElasticMaterial(1e4, 0.3), elasticity.ElasticMaterial(1e6, 0.45)
    bodies = [SimpleNamespace(tets=np.zeros((2, 4), int)), SimpleNamespace(tets=np.zeros((0, 4), int)),
              SimpleNamespace(tets=np.zeros((3, 4), int))]
    scene = SimpleNamespace(bodies=bodies)
    mu, lam = stepper._tet_materials(scene, [soft, None, hard], 5)
    np.testing.assert_array_equal(mu, [soft.lame_mu] * 2 + [hard.lame_mu] * 3)
    np.testing.assert_array_equal(lam, [soft.lame_lambda] * 2 + [hard.lame_lambda] * 3)
    with pytest.raises(ValueError):
        stepper._tet_materials(scene, [None, None, hard], 5)
    mu, lam = stepper._tet_materials(SimpleNamespace(), soft, 4)
    assert np.all(mu == soft.lame_mu) and np.all(lam == soft.lame_lambda)
    mu, lam = stepper._tet_materials(SimpleNamespace(), (np.arange(4.0), 2 * np.arange(4.0)), 4)
    np.testing.assert_array_equal(lam, 2 * mu)
    with pytest.raises(ValueError):
        stepper._tet_materials(SimpleNamespace(), None, 4)


def test_cloth_scene_as_scene():
    cloth = workloads.cloth_stack(layers=2, n=8, seed=3)
    sc = cloth.as_scene()
    assert sc.tets.shape == (0, 4) and sc.surf_tris is cloth.tris and sc.surf_edges is cloth.edges
    np.testing.assert_array_equal(sc.surf_verts, np.arange(cloth.positions.shape[0]))
    assert sc.bbox_diagonal == pytest.approx(np.linalg.norm(np.ptp(cloth.positions, axis=0)))


def test_cube_drop_workload_is_well_formed():
    sc = workloads.cube_drop(k=3)
    p = sc.positions[sc.tets]
    det = np.einsum("ij,ij->i", np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), p[:, 3] - p[:, 0])
    assert det.min() > 0.0                                                     # positively oriented tets
    np.testing.assert_allclose(det.reshape(-1, 5).sum(axis=1) / 6.0, 0.4 ** 3)  # five tets fill each cube
    tris, edges = workloads.tet_boundary(sc.tets[:5])
    assert tris.shape == (12, 3) and edges.shape == (18, 2)                    # a cube's surface
    np.testing.assert_allclose(sc.masses[:8].sum(), 1000.0 * 0.4 ** 3)
    assert sc.fixed[72:].all() and not sc.fixed[:72].any() and sc.surf_verts.size == sc.positions.shape[0]


def test_factor_path_limit_is_a_host_side_choice():
    """The factor descriptors hold a 27-bit element index (assembly.cu): the stepper picks the rank-1 factor path
    only while every family fits and assembles from the dense blocks beyond that, instead of running into the
    C ABI's EINVAL."""
    fit = solver.NewtonSystem.factors_fit
    assert fit({2: 0, 3: 0, 4: 0}) and fit({2: 10**6, 3: 10**6, 4: 10**6})
    assert fit({4: (1 << 27) // 12 - 1 + (1 if ((1 << 27) % 12) else 0)})
    assert not fit({4: (1 << 27) // 12 + 1})
    assert not fit({2: 1, 3: (1 << 27) // 9 + 1, 4: 1})
