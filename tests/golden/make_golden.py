#!/usr/bin/env python
"""Freeze outputs of the REAL reference (`tetipc`) into tests/golden/*.npz.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

The reference package is imported unmodified.  Its compiled backend
(``tetipc.kernels._core``) is the canonical arithmetic (scalar, left-to-right,
no FMA); because /root/reference is read-only the script copies ``pkg/`` to
/tmp/refprobe and builds the extension there with the reference's own setup.py,
then imports from that copy (``kernels.BACKEND == "core"``).  The ``_numpy``
fallback outputs of the three classify kernels are stored next to the ``_core``
ones: they differ in the last bits (einsum uses FMA/SIMD), region codes agree.

Inputs come from ``paper_2308_09400_b200.workloads`` (seeded); every array the
parity tests need is stored in the .npz, so the GPU box needs neither
/root/reference nor this script.
"""

import os
import shutil
import subprocess
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg"
PROBE = "/tmp/refprobe/pkg"


def _import_reference():
    so = [f for f in os.listdir(os.path.join(PROBE, "src/tetipc/kernels"))
          if f.startswith("_core") and f.endswith(".so")] if os.path.isdir(PROBE) else []
    if not so:
        os.makedirs(os.path.dirname(PROBE), exist_ok=True)
        shutil.copytree(REF_SRC, PROBE, dirs_exist_ok=True)
        subprocess.check_call([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=PROBE)
    sys.path.insert(0, os.path.join(PROBE, "src"))
    import tetipc  # noqa: F401
    from tetipc import kernels

    assert kernels.BACKEND == "core", kernels.BACKEND
    return kernels


kernels = _import_reference()
sys.path.insert(0, ROOT)

from tetipc import barrier as rb  # noqa: E402
from tetipc import mollifier as rm  # noqa: E402
from tetipc import proximity as rp  # noqa: E402
from tetipc import solver as rs  # noqa: E402
from tetipc.gap import build_diagonal_jacobian  # noqa: E402
from tetipc.kernels import _numpy as k_numpy  # noqa: E402
from tetipc.mesh import Scene  # noqa: E402

from paper_2308_09400_b200 import workloads as wl  # noqa: E402

KIND_CODE = {
    rp.StencilKind.EDGE_EDGE: 0,
    rp.StencilKind.EDGE_EDGE_PARALLEL: 1,
    rp.StencilKind.POINT_EDGE: 2,
    rp.StencilKind.POINT_EDGE_PARALLEL: 3,
    rp.StencilKind.POINT_POINT: 4,
    rp.StencilKind.POINT_POINT_PARALLEL: 5,
    rp.StencilKind.POINT_TRIANGLE: 6,
}

PARAM_SETS = {
    # name: (d_hat, kappa, dt)   second set = bundled-scene values (scenes.py:223-225)
    "unit": (1.0, 1.0, 1.0),
    "scene": (5e-3, 2e8, 0.01),
}


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}.npz: {os.path.getsize(path) / 1024:.0f} KiB, keys={sorted(arrays)}")


def table_of(stencils):
    n = len(stencils)
    kind = np.zeros(n, np.uint8)
    verts = np.full((n, 4), -1, np.int32)
    sub = np.zeros(n, np.uint8)
    eps = np.zeros(n)
    otype = np.zeros(n, np.uint8)
    origin = np.full((n, 4), -1, np.int32)
    for i, st in enumerate(stencils):
        kind[i] = KIND_CODE[st.kind]
        verts[i, : len(st.verts)] = st.verts
        if st.sub is not None:
            for k, loc in enumerate(st.sub):
                sub[i] |= (loc & 3) << (2 * k)
        if st.eps_x is not None:
            eps[i] = st.eps_x
        if st.origin is not None:
            otype[i] = {"ee": 1, "vt": 2}[st.origin[0]]
            origin[i] = st.origin[1:]
    return dict(kind=kind, verts=verts, sub=sub, eps_x=eps, origin_type=otype, origin=origin)


def fake_state(d_hat, kappa, dt, masses=None, fixed=None, **kw):
    """Just enough of SimState for its unbound hot-path methods (solver.py:127-226)."""
    params = rb.BarrierParams(d_hat=d_hat, kappa=kappa, **kw)
    cfg = rs.SolverConfig(dt=dt, barrier=params)
    scene = types.SimpleNamespace(tets=np.zeros((0, 4), np.int64))
    st = types.SimpleNamespace(config=cfg, scene=scene, friction_data=[], masses=masses, fixed=fixed, l=1.0)
    st._barrier_block = lambda stencil, x: rs.SimState._barrier_block(st, stencil, x)
    return st


def reference_blocks(stencils, x, d_hat, kappa, dt, **kw):
    """Per-stencil reference outputs padded to 4 vertices."""
    st = fake_state(d_hat, kappa, dt, **kw)
    n = len(stencils)
    energy = np.zeros(n)
    grad = np.zeros((n, 12))
    hess = np.zeros((n, 12, 12))
    status = np.zeros(n, np.uint8)
    for i, s in enumerate(stencils):
        dist = rp.stencil_distance(s, x)
        if dist.d2 <= 0.0:
            status[i] = 2
            continue
        if dist.d2 >= d_hat**2:
            status[i] = 1
            continue
        energy[i] = rs.SimState._barrier_energy(st, x, [s])
        blk = rs.SimState.assemble_local_quadratics(st, x, x, [s])[0]
        k = blk.grad.shape[0]
        grad[i, :k] = blk.grad
        hess[i, :k, :k] = blk.hess
    return dict(ref_energy=energy, ref_grad=grad, ref_hess=hess, ref_status=status)


# ---------------------------------------------------------------------------

def golden_scalars():
    g = np.concatenate([np.linspace(0.01, 0.99, 99), [1e-6, 1e-4, 0.0025, 0.25, 1 - 1e-6, 1 - 1e-12]])
    out = {"g": g}
    for name, (d_hat, kappa, _) in PARAM_SETS.items():
        for form in ("qlog", "log"):
            p = rb.BarrierParams(d_hat=d_hat, kappa=kappa, form=form)
            tag = f"{name}_{form}"
            out[tag + "_b"] = rb.barrier_value(g, p)
            out[tag + "_bg"] = rb.barrier_dg(g, p)
            out[tag + "_bgg"] = rb.barrier_d2g(g, p)
            out[tag + "_lam1"] = rb.lambda1(g, p)
            out[tag + "_lam23"] = rb.lambda23(g, p)
            out[tag + "_lam1f"] = rb.filtered_lambda1(g, p)
    save("scalars", **out)


def golden_classify():
    rng = np.random.default_rng(20240817)
    n = 768
    pts = [rng.normal(size=(n, 3)) for _ in range(4)]
    # a block of exact-distance PT / EE stencils, and near-degenerate rows
    xp = wl.gen_point_triangle(rng, 128, rng.uniform(0.1, 0.9, 128))
    xe = wl.gen_edge_edge(rng, 128, rng.uniform(0.1, 0.9, 128))
    xq = wl.gen_parallel_edge_edge(rng, 120, rng.uniform(0.2, 0.9, 120),
                                   np.exp(rng.uniform(np.log(1e-7), np.log(1e-2), 120)))
    xz = wl.gen_exact_parallel_edge_edge(rng, 8, rng.integers(13, 58, 8))
    for j in range(4):
        pts[j][:128] = xp[:, j]
        pts[j][128:256] = xe[:, j]
        pts[j][256:376] = xq[:, j]
        pts[j][376:384] = xz[:, j]
    out = {f"in{j}": pts[j] for j in range(4)}
    for tag, mod in (("core", kernels.get_backend("core")), ("numpy", k_numpy)):
        c, d2, g, w = mod.pt_classify_batch(*pts)
        out.update({f"pt_{tag}_codes": c, f"pt_{tag}_d2": d2, f"pt_{tag}_grad": g, f"pt_{tag}_w": w})
        c, d2, g, w = mod.ee_classify_batch(*pts)
        out.update({f"ee_{tag}_codes": c, f"ee_{tag}_d2": d2, f"ee_{tag}_grad": g, f"ee_{tag}_w": w})
        cv, cg = mod.cross_sq_batch(*pts)
        out.update({f"cs_{tag}_c": cv, f"cs_{tag}_grad": cg})
        hess = rng.normal(size=(40, 12, 12)) if tag == "core" else out["mv_hess"]
        if tag == "core":
            hess = hess + hess.transpose(0, 2, 1)
            out["mv_hess"] = hess
            out["mv_vids"] = np.stack([rng.choice(30, size=4, replace=False) for _ in range(40)]).astype(np.int64)
            out["mv_x"] = rng.normal(size=90)
        acc = np.zeros(90)
        mod.matvec_blocks(out["mv_hess"], out["mv_vids"], out["mv_x"], acc)
        out[f"mv_{tag}_out"] = acc
    save("classify", **out)


def golden_plain_blocks():
    pos, ids = wl.mixed_kind_batch(n_each=48, seed=11)
    kinds = {"pp": rp.StencilKind.POINT_POINT, "pe": rp.StencilKind.POINT_EDGE,
             "pt": rp.StencilKind.POINT_TRIANGLE, "ee": rp.StencilKind.EDGE_EDGE}
    stencils = []
    for name in ("ee", "pe", "pp", "pt"):  # reference list order
        for row in ids[name]:
            stencils.append(rp.ContactStencil(kind=kinds[name], verts=tuple(int(v) for v in row)))
    # off-branch PT/EE rows: move some points sideways so the closest feature is an edge/vertex
    rng = np.random.default_rng(5)
    x = pos.copy()
    for row in ids["pt"][::4]:
        x[row[0]] += (x[row[2]] - x[row[1]]) * rng.uniform(1.0, 2.0)
    for row in ids["ee"][::4]:
        x[row[2:]] += (x[row[1]] - x[row[0]]) * rng.uniform(0.8, 1.6)
    out = dict(table_of(stencils), positions=x)
    for name, (d_hat, kappa, dt) in PARAM_SETS.items():
        xs = x * d_hat  # d/d_hat preserved; geometry shrinks with d_hat
        ref = reference_blocks(stencils, xs, d_hat, kappa, dt)
        out.update({f"{name}_{k}": v for k, v in ref.items()})
        ref = reference_blocks(stencils, xs, d_hat, kappa, dt, use_filter=False)
        out[f"{name}_nofilter_ref_hess"] = ref["ref_hess"]
    save("blocks_plain", **out)


def golden_parallel_blocks():
    batch = wl.config2_batch(n=320, seed=20240818)
    x = batch.positions
    stencils, cvals, eig = [], [], []
    for q in batch.ee:
        ea, eb = q[:2], q[2:]
        eps = rp.edge_parallel_eps(batch.rest_positions, ea, eb)
        kind, local, res, c = rp.classify_edge_edge(x[q[0]], x[q[1]], x[q[2]], x[q[3]], eps_x=eps)
        if res.d2 >= batch.d_hat**2:
            continue
        gids = tuple(int(v) for v in q)
        if kind in rp.PARALLEL_KINDS:
            st = rp.ContactStencil(kind=kind, verts=gids, eps_x=eps, sub=local, origin=("ee",) + gids,
                                   edge_pair=(gids[:2], gids[2:]))
        else:
            st = rp.ContactStencil(kind=kind, verts=tuple(gids[k] for k in local), origin=("ee",) + gids)
        stencils.append(st)
        cvals.append(c)
    stencils.sort(key=lambda s: s.sort_key())
    out = dict(table_of(stencils), positions=x)
    for name, (d_hat, kappa, dt) in PARAM_SETS.items():
        if name == "scene":
            continue  # eps_x is tied to the unit geometry
        ref = reference_blocks(stencils, x, d_hat, kappa, dt)
        out.update({f"{name}_{k}": v for k, v in ref.items()})
        params = rb.BarrierParams(d_hat=d_hat, kappa=kappa)
        rows = []
        for s in stencils:
            if s.kind not in rp.PARALLEL_KINDS:
                rows.append([np.nan] * 8)
                continue
            jac = build_diagonal_jacobian(s, x, d_hat)
            sysm = rm.mollified_eigensystem(jac.f * jac.f, jac.sqrt_c * jac.sqrt_c, params, s.eps_x)
            rows.append([sysm.lambda_gamma[0], sysm.lambda_g[0], sysm.t, sysm.p, sysm.lambda7p,
                         sysm.lambda8p, sysm.q8p[4], sysm.q8p[8]])
        out[f"{name}_eig"] = np.array(rows)
    save("blocks_parallel", **out)


def _reference_scene(cloth):
    nv = cloth.positions.shape[0]
    return Scene(
        bodies=[], gravity=np.array([0.0, 0.0, -9.81]), bbox_diagonal=float(np.linalg.norm(np.ptp(cloth.positions, axis=0))),
        positions=cloth.positions, rest_positions=cloth.rest_positions, masses=cloth.masses, fixed=cloth.fixed,
        tets=np.zeros((0, 4), np.int64), surf_tris=cloth.tris, surf_edges=cloth.edges,
        surf_verts=np.unique(cloth.tris), body_offsets=np.array([0, nv]), tet_volumes=np.zeros(0),
    )


def golden_scene():
    cloth = wl.cloth_stack(layers=3, n=6, seed=3, twist_deg=5.0)
    scene = _reference_scene(cloth)
    stencils = rp.find_contact_pairs(scene, cloth.positions, cloth.d_hat)
    kinds = sorted({s.kind.value for s in stencils})
    print(f"scene: {cloth.positions.shape[0]} verts, {len(stencils)} contacts, kinds={kinds}")
    st = fake_state(cloth.d_hat, cloth.kappa, cloth.dt, masses=cloth.masses, fixed=cloth.fixed)
    x = cloth.positions
    rng = np.random.default_rng(9)
    x_tilde = x + rng.normal(size=x.shape) * 1e-4
    blocks = rs.SimState.assemble_local_quadratics(st, x, x, stencils)
    grouped = rs.group_blocks(blocks)
    grad = rs.SimState.gradient(st, x, x_tilde, blocks)
    energy = rs.SimState._barrier_energy(st, x, stencils)
    v = rng.normal(size=3 * x.shape[0])
    mv = rs.matvec_matrix_free(grouped, cloth.masses, cloth.fixed, v)
    pinv = rs.block_jacobi_preconditioner(grouped, cloth.masses, cloth.fixed)
    d, iters, ok = rs.pcg_solve(grouped, cloth.masses, cloth.fixed, -grad, 1e-4, 2000)
    d12, iters12, ok12 = rs.pcg_solve(grouped, cloth.masses, cloth.fixed, -grad, 1e-12, 5000)
    # dense assembly exactly as the reference's own test oracle does it (tests/test_solver.py:71-84)
    n = x.shape[0]
    a = np.zeros((3 * n, 3 * n))
    for i in range(n):
        a[3 * i:3 * i + 3, 3 * i:3 * i + 3] = cloth.masses[i] * np.eye(3)
    for blk in blocks:
        idx = np.concatenate([[3 * i, 3 * i + 1, 3 * i + 2] for i in blk.vert_ids])
        a[np.ix_(idx, idx)] += blk.hess
    fd = np.repeat(cloth.fixed, 3)
    a[fd, :] = 0.0
    a[:, fd] = 0.0
    a[fd, fd] = 1.0
    out = dict(table_of(stencils), positions=x, rest_positions=cloth.rest_positions, tris=cloth.tris,
               edges=cloth.edges, masses=cloth.masses, fixed=cloth.fixed, x_tilde=x_tilde,
               d_hat=cloth.d_hat, kappa=cloth.kappa, dt=cloth.dt,
               ref_gradient=grad, ref_energy=energy, v=v, ref_matvec=mv, ref_pinv=pinv,
               ref_pcg_d=d, ref_pcg_iters=iters, ref_pcg_ok=ok,
               ref_pcg12_d=d12, ref_pcg12_iters=iters12, ref_pcg12_ok=ok12,
               ref_dense=a.astype(np.float64))
    for s, (hess, vids) in zip((int(h.shape[1]) // 3 for h, _ in grouped), grouped):
        out[f"fam{s}_hess"] = hess
        out[f"fam{s}_vids"] = vids
    save("scene", **out)


def golden_broad():
    """Candidate queries of the reference's broad phase: its own box construction
    (proximity.py:276-281, :304-307) fed to its own ``_aabb_overlap_pairs`` (:232-248) and its own
    incidence filters (:283-286, :310-317), on two poses of a small cloth stack."""
    out = {}
    for tag, (layers, n, seed, push) in {"a": (3, 6, 3, 0.0), "b": (2, 9, 11, 0.3)}.items():
        cloth = wl.cloth_stack(layers=layers, n=n, seed=seed, twist_deg=5.0)
        x = cloth.positions + push * cloth.d_hat * np.random.default_rng(seed).normal(size=cloth.positions.shape)
        d_hat = cloth.d_hat
        verts, tris, edges = np.unique(cloth.tris), cloth.tris, cloth.edges
        p = x[verts]
        tri_stack = np.stack([x[tris[:, 0]], x[tris[:, 1]], x[tris[:, 2]]], axis=1)
        pairs = rp._aabb_overlap_pairs(p - d_hat, p + d_hat, tri_stack.min(axis=1), tri_stack.max(axis=1))
        vid, tv = verts[pairs[:, 0]], tris[pairs[:, 1]]
        keep = (vid != tv[:, 0]) & (vid != tv[:, 1]) & (vid != tv[:, 2])
        vt = np.concatenate([vid[keep, None], tv[keep]], axis=1)
        e1, e2 = x[edges[:, 0]], x[edges[:, 1]]
        lo_e, hi_e = np.minimum(e1, e2) - d_hat * 0.5, np.maximum(e1, e2) + d_hat * 0.5
        pairs = rp._aabb_overlap_pairs(lo_e, hi_e, lo_e, hi_e)
        pairs = pairs[pairs[:, 0] < pairs[:, 1]]
        ea, eb = edges[pairs[:, 0]], edges[pairs[:, 1]]
        keep = (ea[:, 0] != eb[:, 0]) & (ea[:, 0] != eb[:, 1]) & (ea[:, 1] != eb[:, 0]) & (ea[:, 1] != eb[:, 1])
        ee = np.concatenate([ea[keep], eb[keep]], axis=1)
        # the list the reference builds from them
        scene = _reference_scene(cloth)
        stencils = rp.find_contact_pairs(scene, x, d_hat)
        print(f"broad {tag}: {len(vt)} vt + {len(ee)} ee candidates -> {len(stencils)} contacts")
        tab = table_of(stencils)
        out.update({f"{tag}_positions": x, f"{tag}_rest_positions": cloth.rest_positions, f"{tag}_tris": tris,
                    f"{tag}_edges": edges, f"{tag}_d_hat": d_hat, f"{tag}_vt": vt.astype(np.int32),
                    f"{tag}_ee": ee.astype(np.int32)})
        out.update({f"{tag}_list_{k}": v for k, v in tab.items()})
    save("broad", **out)


def golden_ccd():
    """accd_max_step of the reference's compiled backend on seeded pairs of all four kinds (including
    zero motion, head-on approach, iteration-cap and step<1e-14 exits), and sweep_candidates +
    global_ccd_filter of the reference on a small cloth stack pushed along a random direction."""
    rng = np.random.default_rng(20240819)
    out = {}
    n = 400
    recipes = {
        kernels.PAIR_PT: lambda d: wl.gen_point_triangle(rng, n, d),
        kernels.PAIR_EE: lambda d: wl.gen_edge_edge(rng, n, d),
        kernels.PAIR_PE: lambda d: wl.gen_point_edge(rng, n, d),
        kernels.PAIR_PP: lambda d: wl.gen_point_point(rng, n, d),
    }
    for kind, gen in recipes.items():
        dist = rng.uniform(0.05, 0.6, size=n)
        x = gen(dist)
        s = x.shape[1]
        dx = rng.normal(size=x.shape) * rng.choice([0.02, 0.3, 2.0], size=(n, 1, 1))
        dx[:10] = 0.0                                   # lp == 0 -> 1.0
        dx[10:20] = dx[10:20, :1]                       # rigid translation: mean-free part is zero
        # first vertex moves straight at the rest: forces contact-limited steps
        dx[20:120, 0] = (x[20:120, 1:].mean(axis=1) - x[20:120, 0]) * rng.uniform(0.5, 3.0, size=(100, 1))
        steps = np.array([kernels.accd_max_step(x[i], dx[i], kind, 0.9) for i in range(n)])
        capped = np.array([kernels.accd_max_step(x[i], dx[i], kind, 0.5, 3) for i in range(n)])
        out.update({f"k{kind}_x": x, f"k{kind}_dx": dx, f"k{kind}_step": steps, f"k{kind}_step_s05_it3": capped})
        print(f"ccd kind {kind}: s={s}, full steps {np.mean(steps == 1.0):.2f}, min {steps.min():.3g}")
    cloth = wl.cloth_stack(layers=3, n=7, seed=13, twist_deg=4.0)
    scene = _reference_scene(cloth)
    x = cloth.positions
    d = rng.normal(size=x.shape) * 0.8 * cloth.d_hat
    d[:, 2] -= 0.5 * cloth.d_hat * (x[:, 2] > x[:, 2].mean())   # push the upper sheets down
    cands = rp.sweep_candidates(scene, x, d, cloth.d_hat)
    alpha = rp.global_ccd_filter(scene, x, d, cands)
    per_pair = np.array([kernels.accd_max_step(x[list(ids)], d[list(ids)], pair, 0.9) for pair, ids in cands])
    print(f"ccd scene: {len(cands)} candidates, alpha = {alpha:.6g}")
    out.update(scene_positions=x, scene_rest_positions=cloth.rest_positions, scene_directions=d, scene_tris=cloth.tris,
               scene_edges=cloth.edges, scene_d_hat=cloth.d_hat,
               scene_cand_kind=np.array([p for p, _ in cands], np.uint8),
               scene_cand_ids=np.array([ids for _, ids in cands], np.int32), scene_cand_step=per_pair,
               scene_alpha=alpha)
    save("ccd", **out)


def _friction_case(rf, stencils, x0, x1, d_hat, kappa, mu, eps_v, dt, hess_stride):
    st = fake_state(d_hat, kappa, dt, masses=np.ones(x0.shape[0]), fixed=np.zeros(x0.shape[0], bool))
    grads = rs.SimState.barrier_gradient_blocks(st, x0, stencils)
    data = rf.update_friction_state(stencils, grads, x0, mu, eps_v, dt)
    index = {id(s): i for i, s in enumerate(stencils)}
    rows = np.array([index[id(d.stencil)] for d in data])
    n = len(data)
    lam = np.array([d.lambda_n for d in data])
    basis, u, pot = np.zeros((n, 12, 2)), np.zeros((n, 2)), np.zeros(n)
    force, hess = np.zeros((n, 12)), np.zeros((n, 12, 12))
    for i, d in enumerate(data):
        s = len(d.stencil.verts)
        basis[i, :3 * s] = d.basis_T
        u[i] = rf.tangential_displacement(d, x1, x0)
        pot[i] = rf.potential(d, u[i])
        force[i, :3 * s] = rf.friction_force(d, u[i])
        hess[i, :3 * s, :3 * s] = rf.friction_hessian_psd(d, u[i]).hess
    raw = np.zeros((len(stencils), 12))
    for i, g in enumerate(grads):
        raw[i, :len(g)] = g
    h = dt * eps_v
    kinds = sorted({s.kind.value for s in stencils})
    print(f"friction: {len(stencils)} stencils {kinds} -> {n} data, |u|/h up to {(np.linalg.norm(u, axis=1) / h).max():.3g}, "
          f"zero-motion data {(np.linalg.norm(u, axis=1) == 0).sum()}")
    return dict(table_of(stencils), x0=x0, x1=x1, raw_grad=raw, mu=mu, eps_v=eps_v, dt=dt, d_hat=d_hat, kappa=kappa,
                rows=rows, lambda_n=lam, basis=basis, u=u, potential=pot, force=force,
                hess_rows=np.arange(0, n, hess_stride), hess=hess[::hess_stride])


def golden_friction():
    """update_friction_state / tangential_displacement / potential / friction_force /
    friction_hessian_psd of the reference, with the reference's own raw barrier gradients, at a displaced
    pose with stick, slip and zero-motion data: (a) the golden cloth scene, (b) a nearly-parallel
    edge-edge batch (edge-edge-parallel / point-edge-parallel / point-point-parallel stencils)."""
    from tetipc import friction as rf

    rng = np.random.default_rng(77)
    cloth = wl.cloth_stack(layers=3, n=6, seed=3, twist_deg=5.0)
    x0 = cloth.positions
    stencils = rp.find_contact_pairs(_reference_scene(cloth), x0, cloth.d_hat)
    mu, eps_v, dt = 0.4, 1e-2, cloth.dt
    h = dt * eps_v
    x1 = x0 + rng.normal(size=x0.shape) * h * rng.choice([0.05, 0.5, 5.0], size=(x0.shape[0], 1))
    for st_ in stencils[::97]:                      # a few data with exactly zero tangential motion
        x1[list(st_.verts)] = x0[list(st_.verts)]
    out = {f"a_{k}": v for k, v in _friction_case(rf, stencils, x0, x1, cloth.d_hat, cloth.kappa, mu, eps_v, dt, 3).items()}

    batch = wl.config2_batch(n=240, seed=20240820)
    x0 = batch.positions
    stencils = []
    for q in batch.ee:
        ea, eb = q[:2], q[2:]
        eps = rp.edge_parallel_eps(batch.rest_positions, ea, eb)
        kind, local, res, c = rp.classify_edge_edge(x0[q[0]], x0[q[1]], x0[q[2]], x0[q[3]], eps_x=eps)
        if res.d2 >= batch.d_hat**2:
            continue
        gids = tuple(int(v) for v in q)
        if kind in rp.PARALLEL_KINDS:
            stencils.append(rp.ContactStencil(kind=kind, verts=gids, eps_x=eps, sub=local, origin=("ee",) + gids,
                                              edge_pair=(gids[:2], gids[2:])))
        else:
            stencils.append(rp.ContactStencil(kind=kind, verts=tuple(gids[k] for k in local), origin=("ee",) + gids))
    stencils.sort(key=lambda s: s.sort_key())
    dt, eps_v = 0.01, 1.0
    h = dt * eps_v
    x1 = x0 + rng.normal(size=x0.shape) * h * rng.choice([0.05, 0.5, 5.0], size=(x0.shape[0], 1))
    out.update({f"b_{k}": v for k, v in _friction_case(rf, stencils, x0, x1, batch.d_hat, batch.kappa, 0.3, eps_v, dt, 2).items()})
    save("friction", **out)


def golden_elastic():
    """rest_data / batch_grad_hess of the reference on random tetrahedra: mildly deformed, strongly
    compressed (indefinite dPsi/dF^2: the projection matters), inverted, and at rest."""
    from tetipc import elasticity as re_

    rng = np.random.default_rng(20240821)
    t = 300
    rest = rng.normal(size=(4 * t, 3))
    tets = np.arange(4 * t).reshape(t, 4)
    # make every rest tet positively oriented and not too flat
    dm = np.stack([rest[tets[:, k]] - rest[tets[:, 0]] for k in (1, 2, 3)], axis=2)
    flip = np.linalg.det(dm) < 0
    tets[flip] = tets[flip][:, [0, 2, 1, 3]]
    x = rest.copy()
    amp = rng.choice([0.0, 0.05, 0.6], size=(t, 1, 1), p=[0.1, 0.5, 0.4])
    a = np.eye(3)[None] + amp * rng.normal(size=(t, 3, 3))
    a[20:40] = np.diag([1.0, 1.0, -0.7])[None] @ a[20:40]      # inverted elements
    a[40:80] *= rng.uniform(0.2, 0.5, size=(40, 1, 1))         # strong compression
    for k in range(t):
        c = rest[tets[k]].mean(axis=0)
        x[tets[k]] = (rest[tets[k]] - c) @ a[k].T + c
    mat = re_.ElasticMaterial(youngs_E=2.0e5, poisson_nu=0.35)
    mu = np.full(t, mat.lame_mu) * rng.uniform(0.5, 2.0, size=t)
    lam = np.full(t, mat.lame_lambda) * rng.uniform(0.5, 2.0, size=t)
    rest_inv, vols, g = re_.rest_data(rest, tets)
    e, grad, hess = re_.batch_grad_hess(x, tets, rest_inv, vols, g, mu, lam)
    _, _, hess_raw = re_.batch_grad_hess(x, tets, rest_inv, vols, g, mu, lam, project=False)
    neg = (np.linalg.eigvalsh(hess_raw).min(axis=1) < -1e-9 * np.abs(hess_raw).max(axis=(1, 2))).sum()
    print(f"elastic: {t} tets, {neg} with an indefinite raw Hessian, energy range [{e.min():.3g}, {e.max():.3g}]")
    save("elastic", rest=rest, x=x, tets=tets, mu=mu, lam=lam, rest_inv=rest_inv, vols=vols, energy=e, grad=grad,
         hess=hess, hess_raw=hess_raw[::5])


def golden_stepper():
    """Trajectories of the reference's own ``advance_time_step`` on small drop scenes (the bodies of
    tests/test_solver.py): per-step positions, velocities and StepStats, plus the scene arrays a
    duck-typed scene needs.  One file per case: stepper_<name>.npz."""
    import tempfile

    from tetipc.elasticity import ElasticMaterial
    from tetipc.mesh import compute_lumped_masses, load_obj_surface, load_tet_mesh
    from tetipc.scenes import box_5tet, flat_tet, floor_quad, write_node_ele, write_obj

    tmp = tempfile.mkdtemp(prefix="golden_stepper_")
    mat = ElasticMaterial(youngs_E=1e5, poisson_nu=0.4)

    def tet_mesh(name, verts_tets, translate, density=1000.0):
        base = os.path.join(tmp, name)
        write_node_ele(base, *verts_tets)
        mesh = load_tet_mesh(base + ".node", base + ".ele").transformed(translate=translate)
        mesh.vertex_mass = compute_lumped_masses(mesh, density)
        return mesh

    def floor(half=1.5):
        path = os.path.join(tmp, "floor.obj")
        write_obj(path, *floor_quad(half))
        return load_obj_surface(path, fixed=True)

    def run(name, bodies, materials, v0, steps, **cfg_kw):
        scene = Scene.build(bodies)
        params = rb.BarrierParams(d_hat=5e-3 * scene.bbox_diagonal, kappa=2e8)
        cfg = rs.SolverConfig(dt=0.01, barrier=params, **cfg_kw)
        state = rs.SimState(scene, cfg, materials)
        state.v[:] = v0(scene)
        xs, vs, stats = [state.x.copy()], [state.v.copy()], []
        for _ in range(steps):
            st = rs.advance_time_step(state)
            xs.append(state.x.copy())
            vs.append(state.v.copy())
            stats.append([st.newton_iters, st.pcg_iters, st.min_distance, st.energy, st.alpha_min, float(st.converged)])
        tet_mu = np.asarray(state.tet_mu)
        tet_lam = np.asarray(state.tet_lam)
        print(f"stepper {name}: {scene.positions.shape[0]} verts, {scene.tets.shape[0]} tets, newton iters "
              f"{[int(s[0]) for s in stats]}, pcg iters {[int(s[1]) for s in stats]}")
        save("stepper_" + name, positions=scene.positions, rest_positions=scene.rest_positions, masses=scene.masses,
             fixed=scene.fixed, tets=scene.tets, surf_tris=scene.surf_tris, surf_edges=scene.surf_edges,
             surf_verts=scene.surf_verts, gravity=scene.gravity, bbox_diagonal=scene.bbox_diagonal, tet_mu=tet_mu,
             tet_lam=tet_lam, d_hat=params.d_hat, kappa=params.kappa, dt=cfg.dt, friction_mu=cfg.friction_mu,
             friction_eps_v=cfg.friction_eps_v, v0=vs[0], xs=np.stack(xs), vs=np.stack(vs), stats=np.array(stats))

    def down(vz, vx=0.0):
        def f(scene):
            v = np.zeros_like(scene.positions)
            v[~scene.fixed] = [vx, 0.0, vz]
            return v
        return f

    # the reference's drop_state with the initial velocity of test_pcg_vs_dense_per_step_positions
    run("drop", [tet_mesh("tet", flat_tet(0.5), (0.0, 0.0, 0.004)), floor()], [mat, None], down(-0.3), 6)
    # a sliding cube with lagged friction
    run("slide", [tet_mesh("cube", box_5tet(0.4, 0.4, 0.4), (0.0, 0.0, 0.004)), floor()], [mat, None],
        down(-0.2, 0.5), 6, friction_mu=0.5)
    # two cubes stacked over the floor: body-body and body-floor contacts in the same system
    run("stack", [tet_mesh("cube_a", box_5tet(0.4, 0.4, 0.4), (0.0, 0.0, 0.004)),
                  tet_mesh("cube_b", box_5tet(0.3, 0.3, 0.3), (0.03, 0.02, 0.409)), floor()], [mat, mat, None],
        down(-0.25), 5)
    shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    if "--stepper-only" in sys.argv:
        golden_stepper()
        sys.exit(0)
    if "--elastic-only" in sys.argv:
        golden_elastic()
        sys.exit(0)
    if "--friction-only" in sys.argv:
        golden_friction()
        sys.exit(0)
    if "--broad-only" in sys.argv:
        golden_broad()
        sys.exit(0)
    if "--ccd-only" in sys.argv:
        golden_ccd()
        sys.exit(0)
    golden_scalars()
    golden_classify()
    golden_plain_blocks()
    golden_parallel_blocks()
    golden_scene()
    golden_broad()
    golden_ccd()
    golden_friction()
    golden_elastic()
    golden_stepper()
