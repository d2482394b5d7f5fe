"""Synthetic input generators for the configurations BASELINE.json names.

Host-side NumPy only: these build *inputs* (vertex positions, candidate queries,
masses) for tests and ``bench.py``; nothing here evaluates the barrier path.
The stencil constructions follow the recipes the reference's test fixtures use
(exact-distance point/triangle, skew edges, nearly-parallel edges --
``/root/reference/pkg/tests/conftest.py:25-101``) but are written
batched: every generator returns whole arrays.

Conventions: a *query batch* is ``positions (4n,3)`` plus ``quads (n,4) int64``
indexing it; point-triangle quads are (p, t1, t2, t3), edge-edge quads are
(a1, a2, b1, b2).
"""

from dataclasses import dataclass

import numpy as np


def _unit(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _unit_avoiding(rng, ref, min_cross):
    """Unit vectors whose cross product with ``ref`` exceeds ``min_cross``."""
    n = ref.shape[0]
    out = _unit(rng, n)
    for _ in range(64):
        bad = np.linalg.norm(np.cross(out, ref), axis=1) <= min_cross
        if not bad.any():
            break
        out[bad] = _unit(rng, int(bad.sum()))
    return out


def gen_point_triangle(rng, n, dist, scale=1.0):
    """(n,4,3): point at exact distance ``dist`` (n,) over a triangle interior."""
    t1 = scale * rng.normal(size=(n, 3))
    e2 = _unit(rng, n)
    e3 = _unit_avoiding(rng, e2, 0.35)
    t2 = t1 + scale * rng.uniform(0.5, 2.0, size=(n, 1)) * e2
    t3 = t1 + scale * rng.uniform(0.5, 2.0, size=(n, 1)) * e3
    nrm = np.cross(t2 - t1, t3 - t1)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    w1 = rng.uniform(0.15, 0.6, size=n)
    w2 = rng.uniform(0.15, 0.6, size=n)
    big = w1 + w2 > 0.85
    w1, w2 = np.where(big, 0.5 * w1, w1), np.where(big, 0.5 * w2, w2)
    base = (1 - w1 - w2)[:, None] * t1 + w1[:, None] * t2 + w2[:, None] * t3
    sign = np.where(rng.uniform(size=n) < 0.5, 1.0, -1.0)
    p = base + (sign * dist)[:, None] * nrm
    return np.stack([p, t1, t2, t3], axis=1)


def gen_edge_edge(rng, n, dist, scale=1.0):
    """(n,4,3): skew segments, interior-interior closest pair at ``dist``."""
    ua = _unit(rng, n)
    ub = _unit_avoiding(rng, ua, 0.4)
    nrm = np.cross(ua, ub)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    ca = scale * rng.normal(size=(n, 3))
    cb = ca + np.asarray(dist)[:, None] * nrm
    la = scale * rng.uniform(0.6, 1.5, size=(n, 1))
    lb = scale * rng.uniform(0.6, 1.5, size=(n, 1))
    return np.stack([ca - la * ua, ca + la * ua, cb - lb * ub, cb + lb * ub], axis=1)


def gen_point_edge(rng, n, dist, scale=1.0):
    """(n,3,3): point at ``dist`` from a segment interior."""
    e1 = scale * rng.normal(size=(n, 3))
    ue = _unit(rng, n)
    edge = scale * rng.uniform(0.5, 2.0, size=(n, 1)) * ue
    perp = _unit_avoiding(rng, ue, 0.3)
    perp -= np.sum(perp * ue, axis=1, keepdims=True) * ue
    perp /= np.linalg.norm(perp, axis=1, keepdims=True)
    t = rng.uniform(0.2, 0.8, size=(n, 1))
    p = e1 + t * edge + np.asarray(dist)[:, None] * perp
    return np.stack([p, e1, e1 + edge], axis=1)


def gen_point_point(rng, n, dist, scale=1.0):
    """(n,2,3): two points at exact distance ``dist``."""
    x0 = scale * rng.normal(size=(n, 3))
    return np.stack([x0, x0 + np.asarray(dist)[:, None] * _unit(rng, n)], axis=1)


def gen_parallel_edge_edge(rng, n, dist, angle):
    """(n,4,3): segments at ``dist`` whose directions differ by ``angle`` rad.

    Half-lengths U(0.6,1.2), centres offset along the common normal, as in the
    reference fixture (conftest.py:82-101).  A random slide of segment b along its
    own direction (up to 12 % past the end of a) makes endpoint regions (PE, PP)
    occur as well as interior ones.
    """
    ua = _unit(rng, n)
    perp = _unit_avoiding(rng, ua, 0.3)
    perp -= np.sum(perp * ua, axis=1, keepdims=True) * ua
    perp /= np.linalg.norm(perp, axis=1, keepdims=True)
    ang = np.asarray(angle)[:, None]
    ub = np.cos(ang) * ua + np.sin(ang) * perp
    off = np.cross(ua, perp)
    off /= np.linalg.norm(off, axis=1, keepdims=True)
    ca = rng.normal(size=(n, 3))
    la = rng.uniform(0.6, 1.2, size=(n, 1))
    lb = rng.uniform(0.6, 1.2, size=(n, 1))
    slide = rng.uniform(-1.12, 1.12, size=(n, 1)) * (la + lb)
    cb = ca + np.asarray(dist)[:, None] * off + slide * ub
    return np.stack([ca - la * ua, ca + la * ua, cb - lb * ub, cb + lb * ub], axis=1)


def gen_exact_parallel_edge_edge(rng, n, dist_steps):
    """(n,4,3) axis-aligned dyadic segments: the cross product is exactly zero.

    ``dist_steps`` (n,) integers: separation in units of 1/64.
    """
    axis = rng.integers(0, 3, size=n)
    other = (axis + 1 + rng.integers(0, 2, size=n)) % 3
    base = rng.integers(-64, 64, size=(n, 3)) / 16.0
    la = rng.integers(40, 77, size=n) / 64.0
    lb = rng.integers(40, 77, size=n) / 64.0
    sl = rng.integers(-32, 33, size=n) / 64.0
    x = np.zeros((n, 4, 3))
    x[:] = base[:, None, :]
    rows = np.arange(n)
    x[rows, 0, axis] -= la
    x[rows, 1, axis] += la
    x[rows, 2, axis] += sl - lb
    x[rows, 3, axis] += sl + lb
    x[rows, 2, other] += np.asarray(dist_steps) / 64.0
    x[rows, 3, other] += np.asarray(dist_steps) / 64.0
    return x


def _as_queries(x):
    """(n,s,3) per-stencil coordinates -> (positions (s*n,3), ids (n,s))."""
    n, s, _ = x.shape
    return x.reshape(n * s, 3).copy(), np.arange(n * s, dtype=np.int64).reshape(n, s)


@dataclass
class QueryBatch:
    """Independent narrow-phase queries over a private vertex set."""

    positions: np.ndarray        # (nv,3)
    rest_positions: np.ndarray   # (nv,3)
    vt: np.ndarray               # (m,4) int64 point-triangle queries
    ee: np.ndarray               # (k,4) int64 edge-edge queries
    d_hat: float
    kappa: float
    dt: float = 1.0
    name: str = ""


def config1_batch(n_pt=5000, n_ee=5000, seed=20240817, d_hat=1.0, kappa=1.0, dt=1.0, scale=1.0):
    """BASELINE config 1: PT + EE stencils at d = U(0.15,0.95) d_hat."""
    rng = np.random.default_rng(seed)
    xp = gen_point_triangle(rng, n_pt, rng.uniform(0.15, 0.95, n_pt) * d_hat, scale)
    xe = gen_edge_edge(rng, n_ee, rng.uniform(0.15, 0.95, n_ee) * d_hat, scale)
    pos = np.concatenate([xp.reshape(-1, 3), xe.reshape(-1, 3)])
    vt = np.arange(4 * n_pt, dtype=np.int64).reshape(n_pt, 4)
    ee = 4 * n_pt + np.arange(4 * n_ee, dtype=np.int64).reshape(n_ee, 4)
    return QueryBatch(pos, pos.copy(), vt, ee, d_hat, kappa, dt, "config1-pt+ee")


def config2_batch(n=1_000_000, seed=20240818, d_hat=1.0, kappa=1.0):
    """BASELINE config 2: nearly-parallel edge-edge stress set.

    angle log-uniform in [1e-6, 2e-2], d/d_hat in U(0.2,0.9); 1 % exactly parallel
    rows (c == 0) and 1 % rows at angle 0.2 rad (c >= eps_x: stay plain kinds).
    eps_x comes from the same positions taken as rest positions.
    """
    rng = np.random.default_rng(seed)
    angle = np.exp(rng.uniform(np.log(1e-6), np.log(2e-2), size=n))
    wide = rng.uniform(size=n) < 0.01
    angle[wide] = 0.2
    x = gen_parallel_edge_edge(rng, n, rng.uniform(0.2, 0.9, n) * d_hat, angle)
    exact = np.flatnonzero(rng.uniform(size=n) < 0.01)
    x[exact] = gen_exact_parallel_edge_edge(rng, exact.size, rng.integers(13, 58, exact.size))
    pos, ee = _as_queries(x)
    return QueryBatch(pos, pos.copy(), np.zeros((0, 4), np.int64), ee, d_hat, kappa, 1.0,
                      "config2-parallel-ee")


def mixed_kind_batch(n_each=256, seed=7, d_hat=1.0, kappa=1.0):
    """Per-kind exact-distance stencils as direct tables (no narrow phase).

    Returns (positions, kind-coded lists) for PP / PE / PT / EE so tests can hit
    every plain kind including the 6x6 and 9x9 families.
    """
    rng = np.random.default_rng(seed)
    d = lambda: rng.uniform(0.03, 0.97, n_each) * d_hat  # noqa: E731
    parts = [
        ("pp", gen_point_point(rng, n_each, d())),
        ("pe", gen_point_edge(rng, n_each, d())),
        ("pt", gen_point_triangle(rng, n_each, d())),
        ("ee", gen_edge_edge(rng, n_each, d())),
    ]
    pos, ids, off = [], {}, 0
    for name, x in parts:
        n, s, _ = x.shape
        pos.append(x.reshape(-1, 3))
        ids[name] = off + np.arange(n * s, dtype=np.int64).reshape(n, s)
        off += n * s
    return np.concatenate(pos), ids


# ----------------------------------------------------------------------------
# cloth scenes (configs 3-5) and a conservative host broad phase
# ----------------------------------------------------------------------------

@dataclass
class ClothScene:
    positions: np.ndarray       # (N,3)
    rest_positions: np.ndarray  # (N,3)
    tris: np.ndarray            # (F,3) int64
    edges: np.ndarray           # (E,2) int64
    masses: np.ndarray          # (N,)
    fixed: np.ndarray           # (N,) bool
    d_hat: float
    kappa: float
    dt: float
    name: str = ""

    def as_scene(self, gravity=(0.0, 0.0, -9.81)):
        """The reference ``Scene`` fields (mesh.py:76-141) ``stepper.SimState`` reads: a shell-only scene."""
        from types import SimpleNamespace

        lo, hi = self.positions.min(axis=0), self.positions.max(axis=0)
        return SimpleNamespace(positions=self.positions, rest_positions=self.rest_positions, masses=self.masses,
                               fixed=self.fixed, tets=np.zeros((0, 4), dtype=np.int64), surf_tris=self.tris,
                               surf_edges=self.edges, surf_verts=np.unique(self.tris),
                               gravity=np.asarray(gravity, dtype=np.float64),
                               bbox_diagonal=float(np.linalg.norm(hi - lo)))


def _grid_mesh(n):
    """n x n vertex grid: (tris (2(n-1)^2,3), edges) in local indices."""
    idx = np.arange(n * n, dtype=np.int64).reshape(n, n)
    a, b, c, d = idx[:-1, :-1], idx[1:, :-1], idx[:-1, 1:], idx[1:, 1:]
    tris = np.concatenate([np.stack([a, b, d], -1).reshape(-1, 3), np.stack([a, d, c], -1).reshape(-1, 3)])
    e = np.concatenate([
        np.stack([idx[:-1, :], idx[1:, :]], -1).reshape(-1, 2),
        np.stack([idx[:, :-1], idx[:, 1:]], -1).reshape(-1, 2),
        np.stack([a, d], -1).reshape(-1, 2),
    ])
    return tris, np.sort(e, axis=1)


def cloth_stack(layers=4, n=64, seed=1, h=0.01, gap_rel=0.6, d_hat_rel=0.5, jitter_rel=0.05,
                twist_deg=7.0, kappa=2e8, dt=0.01, density=0.2, fixed_frac=0.01):
    """Teaser-style stack of ``layers`` n x n cloth sheets.

    Sheet k is rotated by k*twist_deg in its plane and jittered by
    jitter_rel*h so that generic and nearly-parallel edge pairs both occur;
    sheets are gap_rel*d_hat apart with d_hat = d_hat_rel*h.  Rest positions are
    the unjittered sheets.  Masses are lumped area density; ``fixed_frac`` of the
    vertices are pinned.
    """
    rng = np.random.default_rng(seed)
    d_hat = d_hat_rel * h
    tris_l, edges_l = _grid_mesh(n)
    u = (np.arange(n) - 0.5 * (n - 1)) * h
    gx, gy = np.meshgrid(u, u, indexing="ij")
    flat = np.stack([gx.reshape(-1), gy.reshape(-1), np.zeros(n * n)], axis=1)
    pos, rest, tris, edges = [], [], [], []
    for k in range(layers):
        th = np.deg2rad(twist_deg * k)
        rot = np.array([[np.cos(th), -np.sin(th), 0.0], [np.sin(th), np.cos(th), 0.0], [0.0, 0.0, 1.0]])
        sheet = flat @ rot.T
        sheet[:, 2] = k * gap_rel * d_hat
        rest.append(sheet.copy())
        jit = rng.normal(size=sheet.shape) * (jitter_rel * h)
        # out-of-plane: sigma 0.1 d_hat clipped at 0.25 d_hat, so sheets never cross
        jit[:, 2] = np.clip(rng.normal(size=sheet.shape[0]) * 0.1 * d_hat, -0.25 * d_hat, 0.25 * d_hat)
        pos.append(sheet + jit)
        tris.append(tris_l + k * n * n)
        edges.append(edges_l + k * n * n)
    pos, rest = np.concatenate(pos), np.concatenate(rest)
    nv = pos.shape[0]
    masses = np.full(nv, density * h * h)
    fixed = rng.uniform(size=nv) < fixed_frac
    return ClothScene(pos, rest, np.concatenate(tris), np.concatenate(edges), masses, fixed,
                      d_hat, kappa, dt, f"cloth-stack-{layers}x{n}x{n}")


def _icosphere(subdiv):
    """Unit icosphere: (verts (V,3), tris (F,3)); V = 10*4^subdiv + 2."""
    t = (1.0 + np.sqrt(5.0)) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], dtype=np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4], [11, 10, 2],
                  [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5],
                  [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    for _ in range(subdiv):
        e = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), axis=1)
        ue, inv = np.unique(e, axis=0, return_inverse=True)
        mid = v[ue[:, 0]] + v[ue[:, 1]]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        m = inv.reshape(3, -1) + v.shape[0]          # midpoint ids of edges (01, 12, 20) per face
        v = np.concatenate([v, mid])
        a, b, c = f[:, 0], f[:, 1], f[:, 2]
        ab, bc, ca = m[0], m[1], m[2]
        f = np.concatenate([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1), np.stack([c, ca, bc], 1),
                            np.stack([ab, bc, ca], 1)])
    return v, f


def cloth_on_sphere(n=316, layers=1, subdiv=5, seed=1, radius=1.0, span=0.8, gap_rel=0.6, d_hat_rel=0.2,
                    jitter_rel=0.02, twist_deg=7.0, kappa=2e8, dt=0.01, density=0.2, fixed_frac=0.01):
    """BASELINE configs[2]: cloth draped over a sphere.

    ``layers`` n x n sheets of side 2*span*radius conform to the upper cap of an icosphere
    (subdivision ``subdiv``) at offsets (k + 1) * gap_rel * d_hat along the sphere normal, d_hat =
    d_hat_rel * h with h the sheet spacing, each sheet rotated by twist_deg against the previous one;
    outside the cap the sheets continue flat.  Defaults (the scene SURVEY 8d
    describes): 10 242 + 316^2 = 110 098 vertices and 273 110 active contacts.  The sphere's
    vertices are fixed.  Rest positions are the unjittered sheets.
    """
    rng = np.random.default_rng(seed)
    h = 2.0 * span * radius / (n - 1)
    d_hat = d_hat_rel * h
    sv, sf = _icosphere(subdiv)
    sv = sv * radius
    se = np.unique(np.sort(np.concatenate([sf[:, [0, 1]], sf[:, [1, 2]], sf[:, [2, 0]]]), axis=1), axis=0)
    tris_l, edges_l = _grid_mesh(n)
    u = (np.arange(n) - 0.5 * (n - 1)) * h
    gx, gy = np.meshgrid(u, u, indexing="ij")
    gx0, gy0 = gx.reshape(-1), gy.reshape(-1)
    pos, rest, tris, edges = [sv], [sv.copy()], [sf], [se]
    base = sv.shape[0]
    rim = 0.95 * radius
    for k in range(layers):
        th = np.deg2rad(twist_deg * (k + 1))      # sheets rotated against each other: no vertex-on-vertex alignment
        gx, gy = np.cos(th) * gx0 - np.sin(th) * gy0, np.sin(th) * gx0 + np.cos(th) * gy0
        rho2 = gx * gx + gy * gy
        r_k = radius + (k + 1) * gap_rel * d_hat
        inside = rho2 < rim * rim
        z = np.where(inside, np.sqrt(np.maximum(r_k * r_k - rho2, 0.0)), np.sqrt(r_k * r_k - rim * rim))
        sheet = np.stack([gx, gy, z], axis=1)
        rest.append(sheet.copy())
        jit = rng.normal(size=sheet.shape) * (jitter_rel * h)
        jit[:, 2] = np.clip(rng.normal(size=n * n) * 0.05 * d_hat, -0.12 * d_hat, 0.12 * d_hat)
        pos.append(sheet + jit)
        tris.append(tris_l + base)
        edges.append(edges_l + base)
        base += n * n
    pos, rest = np.concatenate(pos), np.concatenate(rest)
    nv = pos.shape[0]
    masses = np.full(nv, density * h * h)
    fixed = rng.uniform(size=nv) < fixed_frac
    fixed[:sv.shape[0]] = True
    return ClothScene(pos, rest, np.concatenate(tris), np.concatenate(edges), masses, fixed, d_hat, kappa, dt,
                      f"cloth-on-sphere-{layers}x{n}x{n}-ico{subdiv}")


def _cells_of_boxes(lo, hi, cell, origin):
    """All (box, cell) incidences of axis-aligned boxes on a uniform grid."""
    ilo = np.floor((lo - origin) / cell).astype(np.int64)
    ihi = np.floor((hi - origin) / cell).astype(np.int64)
    span = ihi - ilo + 1
    count = span.prod(axis=1)
    box = np.repeat(np.arange(lo.shape[0], dtype=np.int64), count)
    start = np.cumsum(count) - count
    local = np.arange(count.sum(), dtype=np.int64) - np.repeat(start, count)
    sx, sy = span[box, 0], span[box, 1]
    cx = ilo[box, 0] + local % sx
    cy = ilo[box, 1] + (local // sx) % sy
    cz = ilo[box, 2] + local // (sx * sy)
    return box, (cx << 42) | (cy << 21) | cz


def _overlap_join(lo_a, hi_a, lo_b, hi_b, cell, origin, chunk=4_000_000):
    """All (a, b) with overlapping boxes, each exactly once.

    Boxes are binned into grid cells; a pair that shares several cells is reported only from the
    cell holding the lower corner of the boxes' intersection, so no de-duplication pass is needed.
    """
    box_a, key_a = _cells_of_boxes(lo_a, hi_a, cell, origin)
    box_b, key_b = _cells_of_boxes(lo_b, hi_b, cell, origin)
    ob = np.argsort(key_b, kind="stable")
    kb, box_b = key_b[ob], box_b[ob]
    first = np.searchsorted(kb, key_a, side="left")
    cnt = np.searchsorted(kb, key_a, side="right") - first
    out = []
    order = np.flatnonzero(cnt > 0)
    csum = np.cumsum(cnt[order])
    lo_i = 0
    while lo_i < order.size:
        base = csum[lo_i - 1] if lo_i else 0
        hi_i = int(np.searchsorted(csum, base + chunk, side="right"))
        hi_i = max(hi_i, lo_i + 1)
        sel = order[lo_i:hi_i]
        c = cnt[sel]
        rep = np.repeat(np.arange(sel.size), c)
        local = np.arange(c.sum(), dtype=np.int64) - np.repeat(np.cumsum(c) - c, c)
        ia = box_a[sel][rep]
        ib = box_b[first[sel][rep] + local]
        lo_int = np.maximum(lo_a[ia], lo_b[ib])
        ok = np.all(lo_int <= np.minimum(hi_a[ia], hi_b[ib]), axis=1)
        own = np.floor((lo_int - origin) / cell).astype(np.int64)
        ok &= ((own[:, 0] << 42) | (own[:, 1] << 21) | own[:, 2]) == key_a[sel][rep]
        out.append(np.stack([ia[ok], ib[ok]], axis=1))
        lo_i = hi_i
    return np.concatenate(out) if out else np.zeros((0, 2), np.int64)


def broad_phase(scene, positions=None, surf_verts=None):
    """Conservative uniform-grid broad phase -> (vt (m,4), ee (k,4)) candidate queries.

    Replaces the reference's O(n^2) AABB sweep (proximity.py:232-248, :275-319) with
    a grid join that returns a superset of the same overlapping boxes, minus
    incident vertex/triangle and adjacent edge pairs (proximity.py:286, :312-317).
    Any duplicate-free superset yields the identical contact list after the
    narrow phase.
    """
    x = scene.positions if positions is None else positions
    d_hat = scene.d_hat
    tris, edges = scene.tris, scene.edges
    if tris.shape[0] == 0 and edges.shape[0] < 2:
        return np.zeros((0, 4), np.int64), np.zeros((0, 4), np.int64)
    verts = np.unique(tris) if surf_verts is None else np.asarray(surf_verts)
    tx = x[tris]
    elen = np.linalg.norm(x[edges[:, 1]] - x[edges[:, 0]], axis=1)
    cell = max(2.0 * d_hat, 1.0 * float(np.median(elen)))
    origin = x.min(axis=0) - 2.0 * cell
    lo_v, hi_v = x[verts] - d_hat, x[verts] + d_hat
    pairs = _overlap_join(lo_v, hi_v, tx.min(axis=1), tx.max(axis=1), cell, origin)
    vid, tv = verts[pairs[:, 0]], tris[pairs[:, 1]]
    ok = (vid != tv[:, 0]) & (vid != tv[:, 1]) & (vid != tv[:, 2])
    vt = np.concatenate([vid[ok, None], tv[ok]], axis=1)
    vt = vt[np.lexsort((pairs[ok, 1], pairs[ok, 0]))]

    e1, e2 = x[edges[:, 0]], x[edges[:, 1]]
    lo_e = np.minimum(e1, e2) - 0.5 * d_hat
    hi_e = np.maximum(e1, e2) + 0.5 * d_hat
    pairs = _overlap_join(lo_e, hi_e, lo_e, hi_e, cell, origin)
    pairs = pairs[pairs[:, 0] < pairs[:, 1]]
    ea, eb = edges[pairs[:, 0]], edges[pairs[:, 1]]
    ok = (ea[:, 0] != eb[:, 0]) & (ea[:, 0] != eb[:, 1]) & (ea[:, 1] != eb[:, 0]) & (ea[:, 1] != eb[:, 1])
    ee = np.concatenate([ea[ok], eb[ok]], axis=1)
    ee = ee[np.lexsort((pairs[ok, 1], pairs[ok, 0]))]
    return vt, ee


# ---- volumetric scene: a grid of elastic cubes over a tessellated floor -------------------------------

_CUBE_CORNERS = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]],
                         dtype=np.float64)
# five-tet split of the unit cube (four corner tets around one central tet), positively oriented
_CUBE_TETS = np.array([[0, 1, 3, 4], [1, 2, 3, 6], [1, 5, 6, 4], [3, 6, 7, 4], [1, 6, 3, 4]], dtype=np.int64)


def tet_boundary(tets):
    """Boundary triangles (faces that belong to one tet) and their unique edges, global vertex ids."""
    tets = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    faces = np.concatenate([tets[:, [1, 2, 3]], tets[:, [0, 3, 2]], tets[:, [0, 1, 3]], tets[:, [0, 2, 1]]])
    key = np.sort(faces, axis=1)
    _, first, count = np.unique(key, axis=0, return_index=True, return_counts=True)
    tris = faces[np.sort(first[count == 1])]
    e = np.sort(np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]]), axis=1)
    return tris, np.unique(e, axis=0)


def cube_drop(k=12, size=0.4, pitch=0.6, z0=0.004, d_hat=0.02, kappa=2e8, dt=0.01, density=1000.0, seed=1,
              tilt=0.0):
    """k x k elastic cubes (five tets each) hovering ``z0`` above a fixed tessellated floor, as a
    reference-``Scene``-shaped namespace (tets, surface arrays, lumped masses, gravity) plus ``d_hat``,
    ``kappa``, ``dt`` and ``v0`` (free vertices moving down).  ``tilt`` jitters the cube heights (relative
    to z0) so that contacts do not all switch on in the same iteration."""
    from types import SimpleNamespace

    rng = np.random.default_rng(seed)
    verts, tets = [], []
    for i in range(k):
        for j in range(k):
            base = np.array([i * pitch, j * pitch, z0 * (1.0 + tilt * rng.uniform(-0.5, 0.5))])
            tets.append(_CUBE_TETS + 8 * (i * k + j))
            verts.append(base + size * _CUBE_CORNERS)
    verts, tets = np.concatenate(verts), np.concatenate(tets)
    nb = verts.shape[0]
    g = k + 2
    ax = (np.arange(g) - 1.0) * pitch + 0.5 * (size - pitch)      # floor vertices between the cubes
    fx, fy = np.meshgrid(ax, ax, indexing="ij")
    floor = np.stack([fx.ravel(), fy.ravel(), np.zeros(g * g)], axis=1)
    ftris, fedges = _grid_mesh(g)
    positions = np.concatenate([verts, floor])
    btris, bedges = tet_boundary(tets)
    tris = np.concatenate([btris, ftris + nb])
    edges = np.concatenate([bedges, fedges + nb])
    # lumped masses: a quarter of each tet's mass to each of its vertices (mesh.py:295-305)
    p = positions[tets]
    vol = np.abs(np.einsum("ij,ij->i", np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), p[:, 3] - p[:, 0])) / 6.0
    masses = np.zeros(positions.shape[0])
    np.add.at(masses, tets.ravel(), np.repeat(0.25 * density * vol, 4))
    fixed = np.zeros(positions.shape[0], dtype=bool)
    fixed[nb:] = True
    lo, hi = positions.min(axis=0), positions.max(axis=0)
    v0 = np.zeros_like(positions)
    v0[:nb, 2] = -0.25
    return SimpleNamespace(positions=positions, rest_positions=positions.copy(), masses=masses, fixed=fixed, tets=tets,
                           surf_tris=tris, surf_edges=edges, surf_verts=np.unique(tris),
                           gravity=np.array([0.0, 0.0, -9.81]), bbox_diagonal=float(np.linalg.norm(hi - lo)),
                           d_hat=d_hat, kappa=kappa, dt=dt, v0=v0, name=f"cube-drop-{k}x{k}")
