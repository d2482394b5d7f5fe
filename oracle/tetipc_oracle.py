"""CPU oracle for the GIPC barrier hot path -- TEST INFRASTRUCTURE ONLY.

A batched NumPy restatement of the reference ``tetipc`` algorithm for the path
SURVEY.md section 8 names.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this module;
the product package ``paper_2308_09400_b200`` never does (it fails loudly when
its CUDA library is missing).

Parity status: PINNED.  ``tests/golden/make_golden.py`` imports the real
reference (``/root/reference/pkg/src``, both its ``_numpy`` backend and its
Cython ``_core`` backend built in /tmp) in the build container, runs it on seeded
inputs and freezes the outputs under ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks this restatement against those files and
against the reference tests' own known-answer values.

Every function cites the reference file:line it follows (paths relative to
``/root/reference/pkg/src/tetipc``).  Nothing here is copied: the reference
evaluates one stencil per Python call through objects; this file evaluates
whole SoA stencil tables at once.  Floating point: all arithmetic is elementwise
NumPy mul/add/div/sqrt (never einsum/BLAS) in the scalar left-to-right order of
``kernels/_core.pyx`` so that, on an x86-64 host without FMA contraction, the
discrete outputs (region codes, active tests, promotion) are bit-exact with the
reference's compiled backend.

Stencil table (SoA) used by the oracle and by the CUDA path alike:

    kind   uint8 (n,)   code = rank of StencilKind.value in string order, which is
                        the reference list order (proximity.py:27-34, :82-83):
                        0 EE, 1 EE-par, 2 PE, 3 PE-par, 4 PP, 5 PP-par, 6 PT
    verts  int32 (n,4)  global vertex ids, -1 padded (PE: 3, PP: 2)
    sub    uint8 (n,)   parallel kinds: local indices of the reduced stencil, two
                        bits each, entry k at bits [2k, 2k+2)   (proximity.py:57-60)
    eps_x  f64   (n,)   parallel tolerance, 0 for non-parallel kinds
"""

import numpy as np

EE, EEP, PE, PEP, PP, PPP, PT = range(7)
KIND_NAMES = (
    "edge-edge",
    "edge-edge-parallel",
    "point-edge",
    "point-edge-parallel",
    "point-point",
    "point-point-parallel",
    "point-triangle",
)
#: vertices per stencil kind (proximity.py:67-75)
KIND_SIZE = np.array([4, 4, 3, 4, 2, 4, 4], dtype=np.int64)
#: number of entries of ``sub`` per parallel kind
SUB_LEN = np.array([0, 4, 0, 3, 0, 2, 0], dtype=np.int64)
IS_PARALLEL = np.array([0, 1, 0, 1, 0, 1, 0], dtype=bool)

STATUS_ACTIVE, STATUS_INACTIVE, STATUS_PENETRATION = 0, 1, 2

# region code -> (reduced kind, local vertex selection); proximity.py:100-127
PT_LOCAL = {
    0: (PT, (0, 1, 2, 3)),
    1: (PP, (0, 1)),
    2: (PP, (0, 2)),
    3: (PP, (0, 3)),
    4: (PE, (0, 1, 2)),
    5: (PE, (0, 2, 3)),
    6: (PE, (0, 3, 1)),
}
EE_LOCAL = {
    8: (EE, (0, 1, 2, 3)),
    2: (PE, (0, 2, 3)),
    5: (PE, (1, 2, 3)),
    6: (PE, (2, 0, 1)),
    7: (PE, (3, 0, 1)),
    0: (PP, (0, 2)),
    1: (PP, (0, 3)),
    3: (PP, (1, 2)),
    4: (PP, (1, 3)),
}
PARALLEL_OF = {EE: EEP, PE: PEP, PP: PPP}


def pack_sub(local):
    """Pack a tuple of local indices (each 0..3) two bits per entry."""
    out = 0
    for k, loc in enumerate(local):
        out |= (int(loc) & 3) << (2 * k)
    return out


def unpack_sub(byte, length):
    return tuple((int(byte) >> (2 * k)) & 3 for k in range(length))


# ----------------------------------------------------------------------------
# small vector helpers, scalar left-to-right order (kernels/_core.pyx:22-35)
# ----------------------------------------------------------------------------

def _dot(a, b):
    return a[..., 0] * b[..., 0] + a[..., 1] * b[..., 1] + a[..., 2] * b[..., 2]


def _two_prod_err(a, b, p):
    """Exact a*b - p (Dekker/Veltkamp split); a, b, p float64 arrays."""
    split = 134217729.0  # 2**27 + 1
    ca, cb = split * a, split * b
    ah = ca - (ca - a)
    bh = cb - (cb - b)
    al, bl = a - ah, b - bh
    return ((ah * bh - p) + ah * bl + al * bh) + al * bl


def _fma(a, b, c):
    """round(a*b + c) via error-free transformations.

    Exact except for double-rounding ties (probability ~2^-53 per operation);
    used only to mirror BLAS ddot on 3-vectors, see ``_dot_blas``.
    """
    p = a * b
    e = _two_prod_err(a, b, p)
    s = p + c
    bb = s - p
    t = (p - (s - bb)) + (c - bb)  # p + c == s + t exactly
    return s + (t + e)


def _dot_blas(a, b):
    """3-vector dot as the reference's ``np.dot`` evaluates it.

    proximity.py:172-176 (_point_edge_eval), :189 (point-point), :218 and :257-259
    (edge_parallel_eps) call np.dot on length-3 vectors, which goes to OpenBLAS ddot
    (0.3.30, Haswell/Zen kernels): a sequential tail loop compiled with FMA
    contraction, i.e. fma(a2,b2, fma(a1,b1, a0*b0)).  Verified bit-for-bit against
    np.dot on 20000 random vectors in the build container.  The kernels.* functions
    (_core.pyx) do NOT contract; they use ``_dot``.
    """
    d = a[..., 0] * b[..., 0]
    d = _fma(a[..., 1], b[..., 1], d)
    return _fma(a[..., 2], b[..., 2], d)


def _cross(a, b):
    return np.stack(
        [
            a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
            a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
            a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0],
        ],
        axis=-1,
    )


def _clamp01(v):
    return np.where(v < 0.0, 0.0, np.where(v > 1.0, 1.0, v))


def _f64(a):
    return np.atleast_2d(np.asarray(a, dtype=np.float64))


# ----------------------------------------------------------------------------
# a4-a7: narrow-phase primitives
# ----------------------------------------------------------------------------

def pt_classify_batch(p, t1, t2, t3):
    """Point-triangle closest feature (kernels/_core.pyx:46-106; _numpy.py:26-99).

    Returns (codes i64 (n,), d2 (n,), grad (n,4,3), w (n,2)).
    """
    p, t1, t2, t3 = _f64(p), _f64(t1), _f64(t2), _f64(t3)
    n = p.shape[0]
    ab, ac, ap = t2 - t1, t3 - t1, p - t1
    d1, d2_ = _dot(ab, ap), _dot(ac, ap)
    bp = p - t2
    d3, d4 = _dot(ab, bp), _dot(ac, bp)
    cp = p - t3
    d5, d6 = _dot(ab, cp), _dot(ac, cp)
    vc = d1 * d4 - d3 * d2_
    vb = d5 * d2_ - d1 * d6
    va = d3 * d6 - d5 * d4

    # priority-ordered region tests, first hit wins (_core.pyx:72-92)
    tests = [
        (1, (d1 <= 0.0) & (d2_ <= 0.0)),
        (2, (d3 >= 0.0) & (d4 <= d3)),
        (4, (vc <= 0.0) & (d1 >= 0.0) & (d3 <= 0.0)),
        (3, (d6 >= 0.0) & (d5 <= d6)),
        (6, (vb <= 0.0) & (d2_ >= 0.0) & (d6 <= 0.0)),
        (5, (va <= 0.0) & (d4 - d3 >= 0.0) & (d5 - d6 >= 0.0)),
    ]
    codes = np.zeros(n, dtype=np.int64)
    open_ = np.ones(n, dtype=bool)
    for code, hit in tests:
        take = open_ & hit
        codes[take] = code
        open_ &= ~take

    w1 = np.zeros(n)
    w2 = np.zeros(n)
    with np.errstate(divide="ignore", invalid="ignore"):
        w1 = np.where(codes == 2, 1.0, w1)
        w1 = np.where(codes == 4, d1 / (d1 - d3), w1)
        w2 = np.where(codes == 3, 1.0, w2)
        w2 = np.where(codes == 6, d2_ / (d2_ - d6), w2)
        t = (d4 - d3) / ((d4 - d3) + (d5 - d6))
        w1 = np.where(codes == 5, 1.0 - t, w1)
        w2 = np.where(codes == 5, t, w2)
        denom = va + vb + vc
        w1 = np.where(codes == 0, vb / denom, w1)
        w2 = np.where(codes == 0, vc / denom, w2)

    w0 = 1.0 - w1 - w2
    closest = w0[:, None] * t1 + w1[:, None] * t2 + w2[:, None] * t3
    r = p - closest
    d2 = _dot(r, r)
    grad = np.empty((n, 4, 3))
    grad[:, 0] = 2.0 * r
    grad[:, 1] = (-2.0 * w0)[:, None] * r
    grad[:, 2] = (-2.0 * w1)[:, None] * r
    grad[:, 3] = (-2.0 * w2)[:, None] * r
    return codes, d2, grad, np.stack([w1, w2], axis=1)


def ee_classify_batch(a1, a2, b1, b2):
    """Clamped segment-segment closest pair (kernels/_core.pyx:109-150).

    Returns (codes = 3*ra+rb, d2, grad (n,4,3), (s,t)).
    """
    a1, a2, b1, b2 = _f64(a1), _f64(a2), _f64(b1), _f64(b2)
    n = a1.shape[0]
    da, db, r = a2 - a1, b2 - b1, a1 - b1
    a, e = _dot(da, da), _dot(db, db)
    f = _dot(db, r)
    b = _dot(da, db)
    c = _dot(da, r)
    denom = a * e - b * b
    with np.errstate(divide="ignore", invalid="ignore"):
        pos = denom > 0.0
        s = np.where(pos, _clamp01((b * f - c * e) / np.where(pos, denom, 1.0)), 0.0)
        t = (b * s + f) / e
        low, high = t < 0.0, t > 1.0
        s = np.where(low, _clamp01(-c / a), s)
        s = np.where(high, _clamp01((b - c) / a), s)
        t = np.where(low, 0.0, np.where(high, 1.0, t))
    ra = np.where(s <= 0.0, 0, np.where(s >= 1.0, 1, 2))
    rb = np.where(t <= 0.0, 0, np.where(t >= 1.0, 1, 2))
    codes = (3 * ra + rb).astype(np.int64)
    rvec = (a1 + s[:, None] * da) - (b1 + t[:, None] * db)
    d2 = _dot(rvec, rvec)
    grad = np.empty((n, 4, 3))
    grad[:, 0] = (2.0 * (1.0 - s))[:, None] * rvec
    grad[:, 1] = (2.0 * s)[:, None] * rvec
    grad[:, 2] = (-2.0 * (1.0 - t))[:, None] * rvec
    grad[:, 3] = (-2.0 * t)[:, None] * rvec
    return codes, d2, grad, np.stack([s, t], axis=1)


def cross_sq_batch(a1, a2, b1, b2):
    """c = |(a2-a1) x (b2-b1)|^2 and its gradient (kernels/_core.pyx:195-219)."""
    a1, a2, b1, b2 = _f64(a1), _f64(a2), _f64(b1), _f64(b2)
    u, v = a2 - a1, b2 - b1
    w = _cross(u, v)
    c = _dot(w, w)
    gu, gv = _cross(v, w), _cross(w, u)
    grad = np.stack([-2.0 * gu, 2.0 * gu, -2.0 * gv, 2.0 * gv], axis=1)
    return c, grad


def point_edge_batch(p, e1, e2):
    """Point-segment distance, gradient over (p,e1,e2) (proximity.py:170-180)."""
    p, e1, e2 = _f64(p), _f64(e1), _f64(e2)
    e = e2 - e1
    ee = _dot_blas(e, e)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = _clamp01(_dot_blas(p - e1, e) / ee)
    r = p - e1 - t[:, None] * e
    d2 = _dot_blas(r, r)
    grad = np.stack([2.0 * r, (-2.0 * (1.0 - t))[:, None] * r, (-2.0 * t)[:, None] * r], axis=1)
    return d2, grad, t


# ----------------------------------------------------------------------------
# a8/a9: per-stencil distance and parallel measure on a table
# ----------------------------------------------------------------------------

def _gather(positions, verts):
    """positions[(n,4) ids] with -1 padding mapped to vertex 0 (unused rows)."""
    idx = np.where(verts < 0, 0, verts)
    return positions[idx]


def stencil_distance_batch(kind, verts, sub, positions):
    """d2 (n,) and grad_d2 padded to (n,4,3) for every table row.

    Follows proximity.py:183-222: PP direct, PE a7, PT/EE full re-classification
    (zero rows off the active branch), parallel kinds evaluated on x[sub] and
    scattered back to the four-vertex layout.
    """
    kind = np.asarray(kind)
    n = kind.shape[0]
    x = _gather(np.asarray(positions, dtype=np.float64), np.asarray(verts))
    d2 = np.zeros(n)
    grad = np.zeros((n, 4, 3))

    def rows(k):
        return np.flatnonzero(kind == k)

    i = rows(PP)
    if i.size:
        r = x[i, 0] - x[i, 1]
        d2[i] = _dot_blas(r, r)
        grad[i, 0], grad[i, 1] = 2.0 * r, -2.0 * r
    i = rows(PE)
    if i.size:
        d2[i], g, _ = point_edge_batch(x[i, 0], x[i, 1], x[i, 2])
        grad[i, :3] = g
    i = rows(PT)
    if i.size:
        _, d2[i], grad[i], _ = pt_classify_batch(x[i, 0], x[i, 1], x[i, 2], x[i, 3])
    i = rows(EE)
    if i.size:
        _, d2[i], grad[i], _ = ee_classify_batch(x[i, 0], x[i, 1], x[i, 2], x[i, 3])

    sub = np.asarray(sub)
    loc = np.stack([(sub >> (2 * k)) & 3 for k in range(4)], axis=1).astype(np.int64)
    i = rows(EEP)
    if i.size:
        xs = np.take_along_axis(x[i], loc[i][:, :, None], axis=1)
        _, d2[i], g, _ = ee_classify_batch(xs[:, 0], xs[:, 1], xs[:, 2], xs[:, 3])
        full = np.zeros((i.size, 4, 3))
        for row in range(4):
            full[np.arange(i.size), loc[i, row]] = g[:, row]
        grad[i] = full
    i = rows(PEP)
    if i.size:
        xs = np.take_along_axis(x[i], loc[i][:, :, None], axis=1)
        d2[i], g, _ = point_edge_batch(xs[:, 0], xs[:, 1], xs[:, 2])
        full = np.zeros((i.size, 4, 3))
        for row in range(3):
            full[np.arange(i.size), loc[i, row]] = g[:, row]
        grad[i] = full
    i = rows(PPP)
    if i.size:
        xs = np.take_along_axis(x[i], loc[i][:, :, None], axis=1)
        r = xs[:, 0] - xs[:, 1]
        d2[i] = _dot_blas(r, r)
        full = np.zeros((i.size, 4, 3))
        full[np.arange(i.size), loc[i, 0]] = 2.0 * r
        full[np.arange(i.size), loc[i, 1]] = -2.0 * r
        grad[i] = full
    return d2, grad


def parallel_measure_batch(verts, positions):
    """(c, grad_c (n,4,3)) on the four stencil vertices (proximity.py:225-229)."""
    x = _gather(np.asarray(positions, dtype=np.float64), np.asarray(verts))
    return cross_sq_batch(x[:, 0], x[:, 1], x[:, 2], x[:, 3])


# ----------------------------------------------------------------------------
# a13/a14: barrier scalars (qlog production form and the log diagnostic form)
# ----------------------------------------------------------------------------

def barrier_scalars(g, scale, form="qlog"):
    """(b, b', b'') at gap g with S = kappa*d_hat^4 (barrier.py:76-101)."""
    g = np.asarray(g, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        lg = np.log(g)
        om = 1.0 - g
        if form == "qlog":
            b = scale * om**2 * lg * lg
            bg = scale * (-2.0 * om * lg * lg + 2.0 * om**2 * lg / g)
            bgg = scale * (2.0 * lg * lg - 8.0 * om * lg / g + 2.0 * om**2 * (1.0 - lg) / g**2)
        elif form == "log":
            b = -scale * om**2 * lg
            bg = scale * (2.0 * om * lg - om**2 / g)
            bgg = scale * (-2.0 * lg + om * (3.0 * g + 1.0) / g**2)
        else:
            raise ValueError(f"unknown barrier form {form!r}")
    return b, bg, bgg


def lambda1(g, scale, form="qlog"):
    """4 g b'' + 2 b' (barrier.py:104-106)."""
    _, bg, bgg = barrier_scalars(g, scale, form)
    return 4.0 * np.asarray(g) * bgg + 2.0 * bg


def filtered_lambda1(g, scale, eps_g, use_filter=True, form="qlog"):
    """lambda1 frozen at lambda1(eps_g) below the proximal limit (barrier.py:114-120)."""
    lam = lambda1(g, scale, form)
    if not use_filter:
        return lam
    return np.where(np.asarray(g) >= eps_g, lam, lambda1(eps_g, scale, form))


# ----------------------------------------------------------------------------
# a16-a18: mollifier and the coupled 2x2 eigen system
# ----------------------------------------------------------------------------

def mollifier(c, eps_x):
    """(e, e', e'') of the parallel-edge mollifier (mollifier.py:55-67)."""
    c = np.asarray(c, dtype=np.float64)
    eps_x = np.asarray(eps_x, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        inside = c < eps_x
        e = np.where(inside, -(c * c) / (eps_x * eps_x) + 2.0 * c / eps_x, 1.0)
        de = np.where(inside, -2.0 * c / (eps_x * eps_x) + 2.0 / eps_x, 0.0)
        d2e = np.where(inside, -2.0 / (eps_x * eps_x), 0.0)
    return e, de, d2e


def mollified_eigensystem(g, c, eps_x, scale, form="qlog"):
    """Closed-form retained eigenpair (lambda8', q_gamma, q_f) (mollifier.py:106-144).

    Also returns the intermediates (lam_gamma1, lam_g1, t, p, lambda7') used by
    the golden checks.
    """
    g = np.asarray(g, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    b, bg, bgg = barrier_scalars(g, scale, form)
    e, de, d2e = mollifier(c, eps_x)
    b_gamma, b_gamma2 = de * b, d2e * b
    b_g, b_g2, b_gamma_g = e * bg, e * bgg, de * bg
    lam_gamma1 = 2.0 * (b_gamma + 2.0 * c * b_gamma2)
    lam_g1 = 2.0 * (b_g + 2.0 * g * b_g2)
    t = b_gamma_g * np.sqrt(c) * np.sqrt(g)
    p = 0.5 * np.sqrt((lam_gamma1 - lam_g1) ** 2 + 64.0 * t * t)
    mean = 0.5 * (lam_gamma1 + lam_g1)
    lam7, lam8 = mean - p, mean + p
    decoupled = (np.abs(8.0 * t) < 1e-12 * (np.abs(lam_gamma1) + np.abs(lam_g1))) | (t == 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        k2 = (lam_gamma1 - lam_g1 + 2.0 * p) / (8.0 * t)
        nrm = np.sqrt(k2 * k2 + 1.0)
        q_gamma = np.where(decoupled, np.where(lam_gamma1 >= lam_g1, 1.0, 0.0), k2 / nrm)
        q_f = np.where(decoupled, np.where(lam_gamma1 >= lam_g1, 0.0, 1.0), 1.0 / nrm)
    return {
        "lam_gamma1": lam_gamma1,
        "lam_g1": lam_g1,
        "t": t,
        "p": p,
        "lambda7p": lam7,
        "lambda8p": lam8,
        "q_gamma": q_gamma,
        "q_f": q_f,
        "b_gamma": b_gamma,
        "b_g": b_g,
    }


def mollified_eigensystem_extended(g, c, eps_x, scale, decoupled=None, ulps=0.0):
    """mollifier.py:106-144 evaluated in x87 extended precision (64-bit mantissa) from the SAME fp64
    inputs (g, c, eps_x): the arbiter for rows where k2 = (dl + 2p)/(8t) cancels (DESIGN.md section 2,
    "conditioning of k2").  ``decoupled`` = the fp64 evaluation's branch decision (the reference's),
    reused so that both evaluations describe the same branch.  ``ulps`` != 0 perturbs the two channel
    eigenvalues by that many fp64 ulps in opposite directions and k2 by the same many ulps of its
    numerator's terms (|dl| + 2p)/|8t|: the change it causes is the first-order noise an fp64 evaluation
    of the reference formula carries (inputs that differ in the last bits of ``log``, and the rounding of
    dl + 2p where it cancels).
    Returns (lambda8', q_gamma, q_f) as longdouble arrays.  qlog form only.
    """
    ld = np.longdouble
    g, c, eps_x = (np.asarray(a, dtype=np.float64).astype(ld) for a in (g, c, eps_x))
    scale = ld(scale)
    with np.errstate(divide="ignore", invalid="ignore"):
        lg, om = np.log(g), ld(1.0) - g
        b = scale * om**2 * lg * lg
        bg = scale * (-2 * om * lg * lg + 2 * om**2 * lg / g)
        bgg = scale * (2 * lg * lg - 8 * om * lg / g + 2 * om**2 * (1 - lg) / g**2)
        inside = c < eps_x
        e = np.where(inside, -(c * c) / (eps_x * eps_x) + 2 * c / eps_x, ld(1.0))
        de = np.where(inside, -2 * c / (eps_x * eps_x) + 2 / eps_x, ld(0.0))
        d2e = np.where(inside, -2 / (eps_x * eps_x), ld(0.0))
        lam_gamma1 = 2 * (de * b + 2 * c * (d2e * b))
        lam_g1 = 2 * (e * bg + 2 * g * (e * bgg))
        if ulps:
            du = ld(ulps) * ld(2.0) ** -52
            lam_gamma1 = lam_gamma1 * (1 + du)
            lam_g1 = lam_g1 * (1 - du)
        t = de * bg * np.sqrt(c) * np.sqrt(g)
        p = np.sqrt((lam_gamma1 - lam_g1) ** 2 + 64 * t * t) / 2
        lam8 = (lam_gamma1 + lam_g1) / 2 + p
        if decoupled is None:
            decoupled = (np.abs(8 * t) < ld(1e-12) * (np.abs(lam_gamma1) + np.abs(lam_g1))) | (t == 0)
        k2 = (lam_gamma1 - lam_g1 + 2 * p) / (8 * t)
        if ulps:   # rounding of the numerator dl + 2p in fp64: the part that explodes when it cancels
            k2 = k2 + du * (np.abs(lam_gamma1 - lam_g1) + 2 * p) / np.abs(8 * t)
        nrm = np.sqrt(k2 * k2 + 1)
        q_gamma = np.where(decoupled, np.where(lam_gamma1 >= lam_g1, ld(1.0), ld(0.0)), k2 / nrm)
        q_f = np.where(decoupled, np.where(lam_gamma1 >= lam_g1, ld(0.0), ld(1.0)), 1 / nrm)
    return lam8, q_gamma, q_f


def mollified_blocks_arbiter(kind, verts, sub, eps_x, positions, d_hat, kappa, dt2=1.0, ulps=8.0):
    """Extended-precision mollified blocks of the parallel rows of a table + the per-row fp64 noise bound.

    For every row (parallel kinds only, others get NaN / 0): ``hess`` (n,12,12) fp64-rounded block
    lam8 w w^T with (lam8, q) from ``mollified_eigensystem_extended``, and ``noise`` (n,) = the largest
    block-entry change, relative to the block's max-abs, when the two channel eigenvalues move by
    ``ulps`` fp64 ulps -- what two correct fp64 evaluations of mollifier.py:113-127 may differ by.
    Geometry (f, grad f, sqrt c, grad sqrt c) is the fp64 one (bit-identical on every side).
    """
    kind = np.asarray(kind)
    n = kind.shape[0]
    par = np.flatnonzero(IS_PARALLEL[kind])
    hess = np.full((n, 12, 12), np.nan)
    noise = np.zeros(n)
    if par.size == 0:
        return hess, noise
    verts = np.asarray(verts)
    d2, grad_d2 = stencil_distance_batch(kind[par], verts[par], np.asarray(sub)[par], positions)
    c, grad_c = parallel_measure_batch(verts[par], positions)
    scale = kappa * d_hat**4
    with np.errstate(divide="ignore", invalid="ignore"):
        d = np.sqrt(d2)
        f = d / d_hat
        u_f = (grad_d2 / (2.0 * d * d_hat)[:, None, None]).reshape(-1, 12)
        sqrt_c = np.sqrt(c)
        safe = np.where(sqrt_c > 0.0, sqrt_c, 1.0)
        u_c = np.where((sqrt_c > 0.0)[:, None], grad_c.reshape(-1, 12) / (2.0 * safe)[:, None], 0.0)
        g, cc = f * f, sqrt_c * sqrt_c
        ref = mollified_eigensystem(g, cc, np.asarray(eps_x)[par], scale)
        dec = (np.abs(8.0 * ref["t"]) < 1e-12 * (np.abs(ref["lam_gamma1"]) + np.abs(ref["lam_g1"]))) | (ref["t"] == 0.0)
        blocks = []
        for u in (0.0, ulps, -ulps):
            lam8, qg, qf = mollified_eigensystem_extended(g, cc, np.asarray(eps_x)[par], scale, dec, u)
            w = qg[:, None] * u_c.astype(np.longdouble) + qf[:, None] * u_f.astype(np.longdouble)
            blocks.append(np.longdouble(dt2) * np.maximum(lam8, 0)[:, None, None] * (w[:, :, None] * w[:, None, :]))
        top = np.abs(blocks[0]).reshape(len(par), -1).max(axis=1)
        top = np.where(top > 0, top, 1)
        dev = np.maximum(np.abs(blocks[1] - blocks[0]), np.abs(blocks[2] - blocks[0])).reshape(len(par), -1).max(axis=1)
    live = (d2 > 0.0) & (d2 < d_hat * d_hat)
    hess[par] = np.where(live[:, None, None], blocks[0].astype(np.float64), 0.0)
    noise[par] = np.where(live, (dev / top).astype(np.float64), 0.0)
    return hess, noise


# ----------------------------------------------------------------------------
# a12, a15, a17, a19-a22: per-stencil energy, gradient and PSD block
# ----------------------------------------------------------------------------

def local_quadratics_batch(kind, verts, sub, eps_x, positions, d_hat, kappa,
                           d_thr_ratio=0.1, use_filter=True, form="qlog", dt2=1.0):
    """Energy, gradient and rank-1 PSD block of every table row.

    Returns a dict with
      status (n,) u8   0 active, 1 inactive (d2 >= d_hat^2), 2 d2 <= 0
      energy (n,)      a20: b(g) or e(c) b(g) with g = d2/d_hat**2; NOT dt2 scaled
                       (solver.py:127-146); 0 for inactive rows
      grad   (n,12)    dt2-scaled gradient, padded with zeros beyond 3*s
      hess   (n,12,12) dt2-scaled PSD block, padded
      f, lam           diagnostics
    Follows gap.py:56-82 (f, grad f, sqrt c, grad sqrt c), barrier.py:163-177
    (plain kinds) and mollifier.py:89-103, :191-210 (parallel kinds); the dt2
    scaling and the inactive skip are solver.py:202-209.
    """
    kind = np.asarray(kind)
    verts = np.asarray(verts)
    n = kind.shape[0]
    eps_x = np.asarray(eps_x, dtype=np.float64)
    scale = kappa * d_hat**4
    eps_g = d_thr_ratio * d_thr_ratio
    d2, grad_d2 = stencil_distance_batch(kind, verts, sub, positions)
    status = np.where(d2 <= 0.0, STATUS_PENETRATION,
                      np.where(d2 >= d_hat**2, STATUS_INACTIVE, STATUS_ACTIVE)).astype(np.uint8)
    active = status == STATUS_ACTIVE
    par = IS_PARALLEL[kind]

    with np.errstate(divide="ignore", invalid="ignore"):
        d = np.sqrt(d2)
        f = d / d_hat
        u_f = (grad_d2 / (2.0 * d * d_hat)[:, None, None]).reshape(n, 12)
        g = f * f
        b, bg, bgg = barrier_scalars(g, scale, form)

        # plain kinds (barrier.py:172-176)
        coef = 2.0 * f * bg
        grad = coef[:, None] * u_f
        lam = np.maximum(filtered_lambda1(g, scale, eps_g, use_filter, form), 0.0)
        w = u_f.copy()

        # energy uses g = d2/d_hat^2, not f*f (solver.py:141-145)
        g_e = d2 / d_hat**2
        energy = barrier_scalars(g_e, scale, form)[0]

        if np.any(par):
            i = np.flatnonzero(par)
            c, grad_c = parallel_measure_batch(verts[i], positions)
            sqrt_c = np.sqrt(c)
            safe = np.where(sqrt_c > 0.0, sqrt_c, 1.0)
            u_c = np.where((sqrt_c > 0.0)[:, None], grad_c.reshape(-1, 12) / (2.0 * safe)[:, None], 0.0)
            cc = sqrt_c * sqrt_c
            sys = mollified_eigensystem(g[i], cc, eps_x[i], scale, form)
            grad[i] = (sys["b_gamma"] * 2.0 * sqrt_c)[:, None] * u_c + (sys["b_g"] * 2.0 * f[i])[:, None] * u_f[i]
            w[i] = sys["q_gamma"][:, None] * u_c + sys["q_f"][:, None] * u_f[i]
            lam[i] = np.maximum(sys["lambda8p"], 0.0)
            energy[i] = mollifier(c, eps_x[i])[0] * energy[i]

    hess = lam[:, None, None] * (w[:, :, None] * w[:, None, :])
    grad = dt2 * grad
    hess = dt2 * hess
    dead = ~active
    grad[dead] = 0.0
    hess[dead] = 0.0
    energy = np.where(active, energy, 0.0)
    lam = np.where(active, lam, 0.0)
    return {"status": status, "energy": energy, "grad": grad, "hess": hess, "f": f, "lam": lam,
            "d2": d2}


def barrier_energy(kind, verts, sub, eps_x, positions, d_hat, kappa, form="qlog"):
    """Total barrier energy; raises on d2 <= 0 like solver.py:132-133."""
    out = local_quadratics_batch(kind, verts, sub, eps_x, positions, d_hat, kappa, form=form)
    if np.any(out["status"] == STATUS_PENETRATION):
        raise ValueError("nonpositive distance on a stencil")
    return float(np.sum(out["energy"]))


def family_views(kind, verts, out):
    """Split a padded batch result into the size families of ``group_blocks``.

    solver.py:237-248 stacks blocks by stencil size (2, 3, 4 ascending) keeping
    list order and skipping inactive rows (solver.py:204-205).  Returns
    ``[(s, rows, vids (nb,s) i64, grad (nb,3s), hess (nb,3s,3s))]``.
    """
    size = KIND_SIZE[np.asarray(kind)]
    active = out["status"] == STATUS_ACTIVE
    fams = []
    for s in (2, 3, 4):
        rows = np.flatnonzero((size == s) & active)
        if rows.size == 0:
            continue
        fams.append((
            s,
            rows,
            np.asarray(verts)[rows, :s].astype(np.int64),
            np.ascontiguousarray(out["grad"][rows, : 3 * s]),
            np.ascontiguousarray(out["hess"][rows, : 3 * s, : 3 * s]),
        ))
    return fams


# ----------------------------------------------------------------------------
# a23-a29: gradient scatter, matvec, block-Jacobi, PCG, assembled matrix
# ----------------------------------------------------------------------------

def scatter_gradient(masses, fixed, x, x_tilde, families):
    """m (x - x~) + sum scatter(grad); fixed rows zero (solver.py:218-226)."""
    n = x.shape[0]
    g3 = masses[:, None] * (x - x_tilde)
    for _, _, vids, grad, _ in families:
        np.add.at(g3, vids, grad.reshape(vids.shape[0], vids.shape[1], 3))
    g3[fixed] = 0.0
    return g3.reshape(3 * n)


def matvec_blocks(hess, vids, x, out):
    """out += scatter(H_b gather(x)), serial block order (kernels/_core.pyx:222-247)."""
    nb = hess.shape[0]
    if nb == 0:
        return
    s = vids.shape[1]
    xg = x.reshape(-1, 3)[vids].reshape(nb, 3 * s)
    y = (hess * xg[:, None, :]).sum(axis=2)
    np.add.at(out.reshape(-1, 3), vids, y.reshape(nb, s, 3))


def matvec_matrix_free(grouped, masses, fixed, v):
    """A v with Dirichlet rows/cols as identity (solver.py:251-262)."""
    n = masses.shape[0]
    vin = v.copy()
    vin.reshape(n, 3)[fixed] = 0.0
    out = (masses[:, None] * vin.reshape(n, 3)).reshape(-1).copy()
    for hess, vids in grouped:
        matvec_blocks(hess, vids, vin, out)
    out.reshape(n, 3)[fixed] = v.reshape(n, 3)[fixed]
    return out


def block_jacobi(grouped, masses, fixed):
    """Inverse 3x3 diagonal blocks (solver.py:265-276)."""
    n = masses.shape[0]
    diag = np.zeros((n, 3, 3))
    diag[:] = np.eye(3)[None] * masses[:, None, None]
    for hess, vids in grouped:
        for k in range(vids.shape[1]):
            np.add.at(diag, vids[:, k], hess[:, 3 * k:3 * k + 3, 3 * k:3 * k + 3])
    diag[fixed] = np.eye(3)
    return np.linalg.inv(diag)


def pcg_solve(grouped, masses, fixed, rhs, rel_tol, max_iters, matvec=None):
    """Block-Jacobi PCG (solver.py:279-315). Returns (d, iters, converged)."""
    n = masses.shape[0]
    pinv = block_jacobi(grouped, masses, fixed)
    if matvec is None:
        def matvec(c):
            return matvec_matrix_free(grouped, masses, fixed, c)

    def prec(r):
        return (pinv * r.reshape(n, 1, 3)).sum(axis=2).reshape(-1)

    d = np.zeros_like(rhs)
    r = rhs.copy()
    r.reshape(n, 3)[fixed] = 0.0
    s = prec(r)
    delta_new = float(r @ s)
    delta0 = delta_new
    if delta0 <= 0.0:
        return d, 0, True
    c = s.copy()
    iters = 0
    while iters < max_iters and delta_new > rel_tol * delta0:
        q = matvec(c)
        denom = float(c @ q)
        if denom <= 0.0:
            break
        alpha = delta_new / denom
        d += alpha * c
        r -= alpha * q
        s = prec(r)
        delta_old = delta_new
        delta_new = float(r @ s)
        c = s + (delta_new / delta_old) * c
        iters += 1
    return d, iters, delta_new <= rel_tol * delta0


def assemble_dense(grouped, masses, fixed):
    """The assembled global matrix (tests/test_solver.py:71-84 of the reference)."""
    n = masses.shape[0]
    a = np.zeros((3 * n, 3 * n))
    for v in range(n):
        a[3 * v:3 * v + 3, 3 * v:3 * v + 3] = masses[v] * np.eye(3)
    for hess, vids in grouped:
        for blk, ids in zip(hess, vids):
            idx = (3 * ids[:, None] + np.arange(3)[None]).reshape(-1)
            a[np.ix_(idx, idx)] += blk
    fd = np.repeat(fixed, 3)
    a[fd, :] = 0.0
    a[:, fd] = 0.0
    a[fd, fd] = 1.0
    return a


def assemble_bsr(grouped, masses, fixed):
    """3x3-block CSR of the same matrix: (rowptr i32 (N+1), colidx i32, vals (nnzb,3,3)).

    Sparsity pattern := {(i,j): i,j in some block's vert_ids} U {(i,i)}, fixed
    rows/cols reduced to the identity diagonal.  Column indices
    ascend within a row.  Contributions are summed in block (list) order.
    """
    n = masses.shape[0]
    rows = [np.arange(n, dtype=np.int64)]
    cols = [np.arange(n, dtype=np.int64)]
    vals = [np.eye(3)[None] * masses[:, None, None]]
    for hess, vids in grouped:
        nb, s = vids.shape
        sub = hess.reshape(nb, s, 3, s, 3).transpose(0, 1, 3, 2, 4)  # (nb, a, b, 3, 3)
        ra = np.broadcast_to(vids[:, :, None], (nb, s, s))
        cb = np.broadcast_to(vids[:, None, :], (nb, s, s))
        rows.append(ra.reshape(-1))
        cols.append(cb.reshape(-1))
        vals.append(sub.reshape(-1, 3, 3))
    rows, cols, vals = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    keep = ~(fixed[rows] | fixed[cols]) | (rows == cols)
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    key = rows * n + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    uniq, first = np.unique(key, return_index=True)
    out = np.add.reduceat(vals, first, axis=0)
    r, c = uniq // n, uniq % n
    fx = fixed[r]
    out[fx] = np.eye(3)
    rowptr = np.zeros(n + 1, dtype=np.int32)
    np.add.at(rowptr, r + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.int32)
    return rowptr, c.astype(np.int32), out


def bsr_pattern(vids_list, n, fixed):
    """(rowptr, colidx) of ``assemble_bsr`` from the families' vertex ids alone -- the sparsity pattern
    {(i,j): i,j in one block} U {(i,i)} with fixed rows/cols reduced to the diagonal (SURVEY.md a29,
    tests/test_solver.py:71-84 of the reference) -- cheap enough for a million contacts."""
    keys = [np.arange(n, dtype=np.int64) * (n + 1)]
    for vids in vids_list:
        vids = np.asarray(vids, dtype=np.int64)
        r = np.repeat(vids, vids.shape[1], axis=1).reshape(-1)
        c = np.tile(vids, (1, vids.shape[1])).reshape(-1)
        keep = ~(fixed[r] | fixed[c]) | (r == c)
        keys.append(r[keep] * n + c[keep])
    uniq = np.unique(np.concatenate(keys))
    r = uniq // n
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, r + 1, 1)
    return np.cumsum(rowptr).astype(np.int32), (uniq % n).astype(np.int32)


def bsr_rows_dense(grouped, masses, fixed, rows):
    """Block rows ``rows`` of the assembled matrix as {row: {col: 3x3}} summed in list order -- the value
    check of a million-contact matrix on a sample of rows without building the whole thing."""
    want = np.zeros(masses.shape[0], dtype=bool)
    want[rows] = True
    out = {int(r): {int(r): (np.eye(3) if fixed[r] else masses[r] * np.eye(3))} for r in rows}
    for hess, vids in grouped:
        nb, s = vids.shape
        hit = np.argwhere(want[vids])
        for b, a in hit:
            i = int(vids[b, a])
            if fixed[i]:
                continue
            for cc in range(s):
                j = int(vids[b, cc])
                if fixed[j]:
                    continue
                blk = hess[b, 3 * a:3 * a + 3, 3 * cc:3 * cc + 3]
                out[i][j] = out[i].get(j, 0.0) + blk
    return out


def bsr_matvec(rowptr, colidx, vals, x):
    n = rowptr.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    y = np.zeros((n, 3))
    np.add.at(y, rows, (vals * x.reshape(n, 3)[colidx][:, None, :]).sum(axis=2))
    return y.reshape(-1)


# ----------------------------------------------------------------------------
# a10/a11: narrow phase -> ordered contact list
# ----------------------------------------------------------------------------

def edge_parallel_eps(rest_positions, ea, eb):
    """1e-3 |la|^2 |lb|^2 from rest positions (proximity.py:251-259).

    The reference uses np.dot on 3-vectors: see ``_dot_blas``.
    """
    la = rest_positions[ea[:, 1]] - rest_positions[ea[:, 0]]
    lb = rest_positions[eb[:, 1]] - rest_positions[eb[:, 0]]
    return 1e-3 * _dot_blas(la, la) * _dot_blas(lb, lb)


_PT_KIND = np.array([PT_LOCAL[c][0] for c in range(7)], dtype=np.uint8)
_PT_SEL = np.array([PT_LOCAL[c][1] + (0,) * (4 - len(PT_LOCAL[c][1])) for c in range(7)], dtype=np.int64)
_EE_KIND = np.array([EE_LOCAL[c][0] for c in range(9)], dtype=np.uint8)
_EE_SEL = np.array([EE_LOCAL[c][1] + (0,) * (4 - len(EE_LOCAL[c][1])) for c in range(9)], dtype=np.int64)
_EE_SUB = np.array([pack_sub(EE_LOCAL[c][1]) for c in range(9)], dtype=np.uint8)


def aabb_candidates(positions, surf_verts, tris, edges, d_hat):
    """The reference's broad phase, all pairs (proximity.py:232-248, :275-287, :303-317).

    Returns (vt (m,4), ee (k,4)): every (surface vertex, triangle) whose boxes
    [p - d_hat, p + d_hat] and AABB(triangle) overlap with the vertex not a corner, and every
    edge pair i < j whose AABBs inflated by d_hat/2 overlap and that share no endpoint -- rows in
    the reference's order (by first box, then second).  O(n^2) memory: small scenes only.
    """
    x = np.asarray(positions, dtype=np.float64)
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    verts = np.asarray(surf_verts, dtype=np.int64)

    def overlap(lo_a, hi_a, lo_b, hi_b):
        ok = np.ones((lo_a.shape[0], lo_b.shape[0]), dtype=bool)
        for k in range(3):
            ok &= lo_a[:, k:k + 1] <= hi_b[None, :, k]
            ok &= lo_b[None, :, k] <= hi_a[:, k:k + 1]
        return np.argwhere(ok)

    vt = np.zeros((0, 4), np.int64)
    if verts.size and tris.size:
        p = x[verts]
        tx = x[tris]
        pairs = overlap(p - d_hat, p + d_hat, tx.min(axis=1), tx.max(axis=1))
        vid, tv = verts[pairs[:, 0]], tris[pairs[:, 1]]
        keep = (vid != tv[:, 0]) & (vid != tv[:, 1]) & (vid != tv[:, 2])
        vt = np.concatenate([vid[keep, None], tv[keep]], axis=1)
    ee = np.zeros((0, 4), np.int64)
    if edges.shape[0] > 1:
        e1, e2 = x[edges[:, 0]], x[edges[:, 1]]
        lo_e = np.minimum(e1, e2) - d_hat * 0.5
        hi_e = np.maximum(e1, e2) + d_hat * 0.5
        pairs = overlap(lo_e, hi_e, lo_e, hi_e)
        pairs = pairs[pairs[:, 0] < pairs[:, 1]]
        ea, eb = edges[pairs[:, 0]], edges[pairs[:, 1]]
        keep = (ea[:, 0] != eb[:, 0]) & (ea[:, 0] != eb[:, 1]) & (ea[:, 1] != eb[:, 0]) & (ea[:, 1] != eb[:, 1])
        ee = np.concatenate([ea[keep], eb[keep]], axis=1)
    return vt, ee


def narrow_phase(positions, rest_positions, vt_pairs, ee_pairs, d_hat, promote_parallel=True):
    """Candidate queries -> the reference's ordered contact list as a table.

    ``vt_pairs`` (m,4) = (vertex, t1, t2, t3), ``ee_pairs`` (k,4) = (a1,a2,b1,b2),
    any duplicate-free superset of the near queries (incident/adjacent pairs
    already removed).  Follows proximity.py:284-358: keep d2 < d_hat*d_hat, reduce
    to the active branch, promote EE queries with c < eps_x, sort by
    (kind.value, verts, origin).  Returns dict(kind, verts, sub, eps_x,
    origin_type (1 "ee", 2 "vt"), origin (n,4)).
    """
    positions = np.asarray(positions, dtype=np.float64)
    ks, vs, subs, epss, ots, ors = [], [], [], [], [], []
    vt_pairs = np.asarray(vt_pairs, dtype=np.int64).reshape(-1, 4)
    ee_pairs = np.asarray(ee_pairs, dtype=np.int64).reshape(-1, 4)
    if vt_pairs.shape[0]:
        x = positions[vt_pairs]
        codes, d2, _, _ = pt_classify_batch(x[:, 0], x[:, 1], x[:, 2], x[:, 3])
        near = np.flatnonzero(d2 < d_hat * d_hat)
        k = _PT_KIND[codes[near]]
        sel = _PT_SEL[codes[near]]
        v = np.take_along_axis(vt_pairs[near], sel, axis=1)
        size = KIND_SIZE[k]
        v[np.arange(4)[None, :] >= size[:, None]] = -1
        ks.append(k); vs.append(v); subs.append(np.zeros(near.size, np.uint8))
        epss.append(np.zeros(near.size)); ots.append(np.full(near.size, 2, np.uint8))
        ors.append(vt_pairs[near])
    if ee_pairs.shape[0]:
        x = positions[ee_pairs]
        codes, d2, _, _ = ee_classify_batch(x[:, 0], x[:, 1], x[:, 2], x[:, 3])
        cval, _ = cross_sq_batch(x[:, 0], x[:, 1], x[:, 2], x[:, 3])
        near = np.flatnonzero(d2 < d_hat * d_hat)
        q = ee_pairs[near]
        eps = edge_parallel_eps(np.asarray(rest_positions, dtype=np.float64), q[:, 0:2], q[:, 2:4])
        k = _EE_KIND[codes[near]]
        prom = (cval[near] < eps) if promote_parallel else np.zeros(near.size, bool)
        sel = _EE_SEL[codes[near]]
        v = np.take_along_axis(q, sel, axis=1)
        size = KIND_SIZE[k]
        v[np.arange(4)[None, :] >= size[:, None]] = -1
        v = np.where(prom[:, None], q, v)
        k = np.where(prom, k + 1, k).astype(np.uint8)  # EE->EEP, PE->PEP, PP->PPP
        ks.append(k); vs.append(v)
        subs.append(np.where(prom, _EE_SUB[codes[near]], 0).astype(np.uint8))
        epss.append(np.where(prom, eps, 0.0)); ots.append(np.full(near.size, 1, np.uint8))
        ors.append(q)
    if not ks:
        z4 = np.zeros((0, 4), np.int32)
        return {"kind": np.zeros(0, np.uint8), "verts": z4, "sub": np.zeros(0, np.uint8),
                "eps_x": np.zeros(0), "origin_type": np.zeros(0, np.uint8), "origin": z4.copy()}
    kind = np.concatenate(ks); verts = np.concatenate(vs); sub = np.concatenate(subs)
    eps_x = np.concatenate(epss); ot = np.concatenate(ots); origin = np.concatenate(ors)
    # tuple comparison: shorter tuples only meet within one kind, so -1 padding is inert
    order = np.lexsort((origin[:, 3], origin[:, 2], origin[:, 1], origin[:, 0], ot,
                        verts[:, 3], verts[:, 2], verts[:, 1], verts[:, 0], kind))
    return {"kind": kind[order], "verts": verts[order].astype(np.int32), "sub": sub[order],
            "eps_x": eps_x[order], "origin_type": ot[order], "origin": origin[order].astype(np.int32)}


# ---------------------------------------------------------------------------------------------
# additive CCD: kernels/_core.pyx:250-325, proximity.py:388-432
# ---------------------------------------------------------------------------------------------
PAIR_PT, PAIR_EE, PAIR_PE, PAIR_PP = 0, 1, 2, 3
_PAIR_SIZE = {PAIR_PT: 4, PAIR_EE: 4, PAIR_PE: 3, PAIR_PP: 2}


def _pair_dist2(x, pair_kind):
    """_pair_dist2_c (_core.pyx:250-269) on a batch: x (n,s,3) -> d2 (n,)."""
    if pair_kind == PAIR_PT:
        return pt_classify_batch(x[:, 0], x[:, 1], x[:, 2], x[:, 3])[1]
    if pair_kind == PAIR_EE:
        return ee_classify_batch(x[:, 0], x[:, 1], x[:, 2], x[:, 3])[1]
    if pair_kind == PAIR_PE:
        e = x[:, 2] - x[:, 1]
        ee = _dot(e, e)
        r = x[:, 0] - x[:, 1]
        t = _clamp01(_dot(r, e) / ee)
        r = r - t[:, None] * e
        return _dot(r, r)
    r = x[:, 0] - x[:, 1]
    return _dot(r, r)


def accd_max_step_batch(x, dx, pair_kind, slack, max_iter=512):
    """accd_max_step (_core.pyx:272-325) for n pairs of one kind at once: x, dx (n,s,3).

    Every pair runs the reference's scalar loop; pairs that left the loop are masked out, so each
    row sees exactly the operations of a lone call.  Returns (step (n,), bad (n,) bool) where bad
    marks a non-positive initial distance (the reference raises ValueError, :307-308).
    """
    x = np.asarray(x, dtype=np.float64)
    dx = np.asarray(dx, dtype=np.float64)
    n, s = x.shape[0], x.shape[1]
    mean = np.zeros((n, 3))
    for v in range(s):
        mean = mean + dx[:, v]
    mean = mean / s
    q = dx - mean[:, None, :]
    norms = np.sqrt(q[..., 0] * q[..., 0] + q[..., 1] * q[..., 1] + q[..., 2] * q[..., 2])
    if pair_kind == PAIR_PT:
        lp = norms[:, 0] + np.maximum(norms[:, 1], np.maximum(norms[:, 2], norms[:, 3]))
    elif pair_kind == PAIR_EE:
        lp = np.maximum(norms[:, 0], norms[:, 1]) + np.maximum(norms[:, 2], norms[:, 3])
    elif pair_kind == PAIR_PE:
        lp = norms[:, 0] + np.maximum(norms[:, 1], norms[:, 2])
    else:
        lp = norms[:, 0] + norms[:, 1]
    out = np.ones(n)
    live = lp != 0.0
    d0 = np.zeros(n)
    if live.any():
        d0[live] = np.sqrt(_pair_dist2(x[live], pair_kind))
    bad = live & ~(d0 > 0.0)
    live &= ~bad
    out[bad] = 0.0
    gap = (1.0 - slack) * d0
    t = np.zeros(n)
    idx = np.flatnonzero(live)
    for _ in range(max_iter):
        if idx.size == 0:
            break
        xt = x[idx] + t[idx, None, None] * q[idx]
        d = np.sqrt(_pair_dist2(xt, pair_kind))
        step = (d - gap[idx]) / lp[idx]
        stop = step <= 0.0                      # break: returns t
        full = ~stop & (t[idx] + step >= 1.0)   # return 1.0
        go = ~stop & ~full
        out[idx[stop]] = t[idx[stop]]
        out[idx[full]] = 1.0
        t[idx[go]] = t[idx[go]] + step[go]
        tiny = go & (step < 1e-14)              # break after the update
        out[idx[tiny]] = t[idx[tiny]]
        idx = idx[go & ~tiny]
    out[idx] = t[idx]                           # iteration cap
    return out, bad


def sweep_candidates(positions, directions, surf_verts, tris, edges, d_hat):
    """sweep_candidates (proximity.py:388-421), all pairs: (vt (m,4), ee (k,4)) in the reference's order."""
    x0 = np.asarray(positions, dtype=np.float64)
    x1 = x0 + np.asarray(directions, dtype=np.float64)
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    verts = np.asarray(surf_verts, dtype=np.int64)
    margin = 1e-3 * d_hat

    def overlap(lo_a, hi_a, lo_b, hi_b):
        ok = np.ones((lo_a.shape[0], lo_b.shape[0]), dtype=bool)
        for k in range(3):
            ok &= lo_a[:, k:k + 1] <= hi_b[None, :, k]
            ok &= lo_b[None, :, k] <= hi_a[:, k:k + 1]
        return np.argwhere(ok)

    vt = np.zeros((0, 4), np.int64)
    if verts.size and tris.size:
        lo_v = np.minimum(x0[verts], x1[verts]) - margin
        hi_v = np.maximum(x0[verts], x1[verts]) + margin
        lo_t = np.minimum(x0[tris].min(axis=1), x1[tris].min(axis=1)) - margin
        hi_t = np.maximum(x0[tris].max(axis=1), x1[tris].max(axis=1)) + margin
        pairs = overlap(lo_v, hi_v, lo_t, hi_t)
        vid, tv = verts[pairs[:, 0]], tris[pairs[:, 1]]
        keep = (vid != tv[:, 0]) & (vid != tv[:, 1]) & (vid != tv[:, 2])
        vt = np.concatenate([vid[keep, None], tv[keep]], axis=1)
    ee = np.zeros((0, 4), np.int64)
    if edges.shape[0] > 1:
        lo_e = np.minimum(x0[edges].min(axis=1), x1[edges].min(axis=1)) - margin
        hi_e = np.maximum(x0[edges].max(axis=1), x1[edges].max(axis=1)) + margin
        pairs = overlap(lo_e, hi_e, lo_e, hi_e)
        pairs = pairs[pairs[:, 0] < pairs[:, 1]]
        ea, eb = edges[pairs[:, 0]], edges[pairs[:, 1]]
        keep = (ea[:, 0] != eb[:, 0]) & (ea[:, 0] != eb[:, 1]) & (ea[:, 1] != eb[:, 0]) & (ea[:, 1] != eb[:, 1])
        ee = np.concatenate([ea[keep], eb[keep]], axis=1)
    return vt, ee


def global_ccd_filter(positions, directions, vt, ee, slack=0.9, max_iter=512):
    """global_ccd_filter (proximity.py:424-432) over PT candidates vt and EE candidates ee."""
    x = np.asarray(positions, dtype=np.float64)
    d = np.asarray(directions, dtype=np.float64)
    alpha = 1.0
    for ids, kind in ((np.asarray(vt, dtype=np.int64).reshape(-1, 4), PAIR_PT),
                      (np.asarray(ee, dtype=np.int64).reshape(-1, 4), PAIR_EE)):
        if ids.shape[0]:
            step, bad = accd_max_step_batch(x[ids], d[ids], kind, slack, max_iter)
            if bad.any():
                raise ValueError("additive CCD requires a strictly positive initial distance")
            alpha = min(alpha, float(step.min()))
    return alpha


# ---------------------------------------------------------------------------------------------
# lagged smooth Coulomb friction: friction.py
# ---------------------------------------------------------------------------------------------
def stencil_witness_batch(kind, verts, sub, positions):
    """Branch witness (n,2) of every table row as DistanceResult.witness holds it
    (proximity.py:183-222): PT (w1,w2), EE (s,t), PE (t,-), PP (-,-); parallel kinds on x[sub]."""
    kind = np.asarray(kind)
    n = kind.shape[0]
    x = _gather(np.asarray(positions, dtype=np.float64), np.asarray(verts))
    wit = np.zeros((n, 2))
    sub = np.asarray(sub)
    loc = np.stack([(sub >> (2 * k)) & 3 for k in range(4)], axis=1).astype(np.int64)
    i = np.flatnonzero(kind == PE)
    if i.size:
        wit[i, 0] = point_edge_batch(x[i, 0], x[i, 1], x[i, 2])[2]
    i = np.flatnonzero(kind == PT)
    if i.size:
        wit[i] = pt_classify_batch(x[i, 0], x[i, 1], x[i, 2], x[i, 3])[3]
    i = np.flatnonzero(kind == EE)
    if i.size:
        wit[i] = ee_classify_batch(x[i, 0], x[i, 1], x[i, 2], x[i, 3])[3]
    i = np.flatnonzero(kind == EEP)
    if i.size:
        xs = np.take_along_axis(x[i], loc[i][:, :, None], axis=1)
        wit[i] = ee_classify_batch(xs[:, 0], xs[:, 1], xs[:, 2], xs[:, 3])[3]
    i = np.flatnonzero(kind == PEP)
    if i.size:
        xs = np.take_along_axis(x[i], loc[i][:, :, None], axis=1)
        wit[i, 0] = point_edge_batch(xs[:, 0], xs[:, 1], xs[:, 2])[2]
    return wit


def friction_state(kind, verts, sub, positions, raw_grad):
    """update_friction_state (friction.py:148-171) for every table row.

    raw_grad (n,12): the raw (not dt^2-scaled) barrier gradient of each stencil, zero padded.
    Returns dict(status (n,) u8: 0 datum / 1 skipped (d2 <= 0 or lambda_n <= 0) / 3 undefined normal,
    lambda_n (n,), cn (n,4) = coeffs/|coeffs|, t1 (n,3), t2 (n,3)); the basis of row i is
    T[3v:3v+3, k] = cn[i,v] * t_k[i] (build_basis, friction.py:128-145).
    """
    kind = np.asarray(kind)
    n = kind.shape[0]
    sub = np.asarray(sub)
    d2, grad_d2 = stencil_distance_batch(kind, verts, sub, positions)
    wit = stencil_witness_batch(kind, verts, sub, positions)
    w0, w1 = wit[:, 0], wit[:, 1]
    loc = np.stack([(sub >> (2 * k)) & 3 for k in range(4)], axis=1).astype(np.int64)
    co = np.zeros((n, 4))
    side = np.zeros((n, 4), dtype=bool)
    # _witness_coefficients (friction.py:85-117)
    i = kind == PP
    co[i, 0], co[i, 1] = 1.0, -1.0
    side[i, 0] = True
    i = kind == PE
    co[i, 0], co[i, 1], co[i, 2] = 1.0, -(1.0 - w0[i]), -w0[i]
    side[i, 0] = True
    i = kind == PT
    co[i, 0], co[i, 1], co[i, 2], co[i, 3] = 1.0, -(1.0 - w0[i] - w1[i]), -w0[i], -w1[i]
    side[i, 0] = True
    i = kind == EE
    co[i, 0], co[i, 1], co[i, 2], co[i, 3] = 1.0 - w0[i], w0[i], -(1.0 - w1[i]), -w1[i]
    side[i, 0] = side[i, 1] = True
    for k, nl in ((EEP, 4), (PEP, 3), (PPP, 2)):
        rows = np.flatnonzero(kind == k)
        if not rows.size:
            continue
        if k == EEP:
            local = np.stack([1.0 - w0[rows], w0[rows], -(1.0 - w1[rows]), -w1[rows]], axis=1)
        elif k == PEP:
            local = np.stack([np.ones(rows.size), -(1.0 - w0[rows]), -w0[rows]], axis=1)
        else:
            local = np.stack([np.ones(rows.size), -np.ones(rows.size)], axis=1)
        for r in range(nl):
            co[rows, loc[rows, r]] = local[:, r]
            pos = local[:, r] > 0.0
            side[rows[pos], loc[rows[pos], r]] = True
    status = np.zeros(n, np.uint8)
    status[~(d2 > 0.0)] = 1
    with np.errstate(divide="ignore", invalid="ignore"):
        one = np.sum(np.where(side[:, :, None], grad_d2, 0.0), axis=1)
        d = np.sqrt(d2)
        normal = one / (2.0 * d)[:, None]
        nn = np.sqrt(np.sum(normal * normal, axis=1))
        status[(status == 0) & (nn == 0.0)] = 3
        normal = normal / nn[:, None]
        m = np.argmin(np.abs(normal), axis=1)          # first minimum on ties, like np.argmin in the reference
        ref = np.zeros((n, 3))
        ref[np.arange(n), m] = 1.0
        t1 = np.cross(normal, ref)
        t1 = t1 / np.sqrt(np.sum(t1 * t1, axis=1))[:, None]
        t2 = np.cross(normal, t1)
        gs = np.sum(np.where(side[:, :, None], np.asarray(raw_grad, dtype=np.float64).reshape(n, 4, 3), 0.0), axis=1)
        lam = np.sqrt(np.sum(gs * gs, axis=1))
        status[(status == 0) & ~(lam > 0.0)] = 1
        cn = co / np.sqrt(np.sum(co * co, axis=1))[:, None]
    ok = status == 0
    return {"status": status, "lambda_n": np.where(ok, lam, 0.0), "cn": np.where(ok[:, None], cn, 0.0),
            "t1": np.where(ok[:, None], t1, 0.0), "t2": np.where(ok[:, None], t2, 0.0)}


def friction_basis(cn, t1, t2, s):
    """basis_T (3s,2) of one datum from its frame."""
    basis = np.zeros((3 * s, 2))
    for v in range(s):
        basis[3 * v:3 * v + 3, 0] = cn[v] * t1
        basis[3 * v:3 * v + 3, 1] = cn[v] * t2
    return basis


def f0_f1(un, eps_v, dt):
    """f0_f1 (friction.py:33-46), vectorised."""
    un = np.asarray(un, dtype=np.float64)
    h = dt * eps_v
    f1 = -un * un / (h * h) + 2.0 * un / h
    f1p = -2.0 * un / (h * h) + 2.0 / h
    f0 = -un**3 / (3.0 * h * h) + un * un / h + h / 3.0
    slide = un >= h
    return np.where(slide, un, f0), np.where(slide, 1.0, f1), np.where(slide, 0.0, f1p)


def friction_blocks(verts, size, lambda_n, cn, t1, t2, x, x_start, mu, eps_v, dt):
    """Per datum: potential (not dt^2-scaled), grad = -dt^2 friction_force, hess = dt^2
    friction_hessian_psd, padded to 12 (friction.py:49-82, :174-178; solver.py:147-152, :210-214)."""
    verts = np.asarray(verts)
    n = verts.shape[0]
    rel = _gather(np.asarray(x, dtype=np.float64), verts) - _gather(np.asarray(x_start, dtype=np.float64), verts)
    live = (np.arange(4)[None, :] < np.asarray(size)[:, None])
    cnl = np.where(live, cn, 0.0)
    u0 = np.sum(cnl * np.einsum("nvk,nk->nv", rel, t1), axis=1)
    u1 = np.sum(cnl * np.einsum("nvk,nk->nv", rel, t2), axis=1)
    un = np.sqrt(u0 * u0 + u1 * u1)
    f0, f1, f1p = f0_f1(un, eps_v, dt)
    ml = mu * lambda_n
    energy = ml * f0
    # T as (n,12,2)
    T = np.zeros((n, 12, 2))
    for v in range(4):
        T[:, 3 * v:3 * v + 3, 0] = cnl[:, v:v + 1] * t1
        T[:, 3 * v:3 * v + 3, 1] = cnl[:, v:v + 1] * t2
    u = np.stack([u0, u1], axis=1)
    zero = un == 0.0
    safe = np.where(zero, 1.0, un)
    force = -(ml * f1 / safe)[:, None] * np.einsum("nrk,nk->nr", T, u)
    force[zero] = 0.0
    uhat = u / safe[:, None]
    outer = uhat[:, :, None] * uhat[:, None, :]
    eye = np.eye(2)[None]
    core = np.maximum(f1p, 0.0)[:, None, None] * outer + np.maximum(f1 / safe, 0.0)[:, None, None] * (eye - outer)
    core[zero] = (2.0 / (eps_v * dt)) * np.eye(2)
    hess = ml[:, None, None] * np.einsum("nrk,nkl,ncl->nrc", T, core, T)
    dt2 = dt * dt
    return {"energy": energy, "grad": -dt2 * force, "hess": dt2 * hess, "u": u}


# ---------------------------------------------------------------------------------------------
# stable neo-Hookean tetrahedra: elasticity.py
# ---------------------------------------------------------------------------------------------
def elastic_rest(rest_positions, tets):
    """rest_data (elasticity.py:39-56) without the explicit 9x12 maps: (rest_inv (t,3,3), vols (t,))."""
    v = np.asarray(rest_positions, dtype=np.float64)
    tets = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    dm = np.stack([v[tets[:, 1]] - v[tets[:, 0]], v[tets[:, 2]] - v[tets[:, 0]], v[tets[:, 3]] - v[tets[:, 0]]], axis=2)
    return np.linalg.inv(dm), np.linalg.det(dm) / 6.0


def elastic_blocks(positions, tets, rest_inv, vols, mu, lam, project=True):
    """batch_grad_hess (elasticity.py:128-137): (energy (t,), grad (t,12), hess (t,12,12)), volume-scaled."""
    v = np.asarray(positions, dtype=np.float64)
    tets = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    t = tets.shape[0]
    ds = np.stack([v[tets[:, 1]] - v[tets[:, 0]], v[tets[:, 2]] - v[tets[:, 0]], v[tets[:, 3]] - v[tets[:, 0]]], axis=2)
    f = ds @ rest_inv
    j = np.linalg.det(f)
    alpha = 1.0 + mu / lam
    f0, f1, f2 = f[:, :, 0], f[:, :, 1], f[:, :, 2]
    gj_m = np.stack([np.cross(f1, f2), np.cross(f2, f0), np.cross(f0, f1)], axis=2)
    vec = lambda m: np.swapaxes(m, -1, -2).reshape(t, 9)  # noqa: E731  column-major
    energy = (0.5 * mu * (np.einsum("tij,tij->t", f, f) - 3.0) + 0.5 * lam * (j - alpha) ** 2) * vols
    p = vec(mu[:, None, None] * f + (lam * (j - alpha))[:, None, None] * gj_m)
    g = np.zeros((t, 9, 12))
    for c in range(3):
        for vtx in range(4):
            w = -rest_inv[:, :, c].sum(axis=1) if vtx == 0 else rest_inv[:, vtx - 1, c]
            for i in range(3):
                g[:, 3 * c + i, 3 * vtx + i] = w
    grad = vols[:, None] * np.einsum("tki,tk->ti", g, p)
    gj = vec(gj_m)
    h = mu[:, None, None] * np.eye(9)[None] + lam[:, None, None] * np.einsum("ti,tj->tij", gj, gj)

    def skew(u):
        s_ = np.zeros((t, 3, 3))
        s_[:, 0, 1], s_[:, 0, 2], s_[:, 1, 0] = -u[:, 2], u[:, 1], u[:, 2]
        s_[:, 1, 2], s_[:, 2, 0], s_[:, 2, 1] = -u[:, 0], -u[:, 1], u[:, 0]
        return s_

    hj = np.zeros((t, 9, 9))
    hj[:, 0:3, 3:6], hj[:, 0:3, 6:9] = -skew(f2), skew(f1)
    hj[:, 3:6, 0:3], hj[:, 3:6, 6:9] = skew(f2), -skew(f0)
    hj[:, 6:9, 0:3], hj[:, 6:9, 3:6] = -skew(f1), skew(f0)
    h = h + (lam * (j - alpha))[:, None, None] * hj
    if project:
        w_, q = np.linalg.eigh(h)
        h = np.einsum("tik,tk,tjk->tij", q, np.maximum(w_, 0.0), q)
    hess = vols[:, None, None] * np.einsum("tki,tkl,tlj->tij", g, h, g)
    return energy, grad, hess


# ----------------------------------------------------------------------------
# N4 (second half): multilevel additive Schwarz preconditioner
# ----------------------------------------------------------------------------
# NOT in /root/reference (the package has block-Jacobi only, solver.py:265-276).  PAPER.md:683-685 names the
# method -- the MAS preconditioner of Wu, Wang and Wang, "A GPU-Based Multilevel Additive Schwarz Preconditioner
# for Cloth and Deformable Body Simulation", ACM TOG 41(4), 2022 -- and this is a restatement of its published
# structure: Morton-ordered vertices, domains of 32, piecewise-constant coarse spaces, additive combination of
# exact domain solves.  PARITY UNPINNED for the operator itself (no reference implementation to compare with);
# what IS pinned is the solve: the direction a MAS-driven PCG returns must satisfy the reference's own stopping
# rule (solver.py:302) on the reference's own matrix, which the tests evaluate with `assemble_dense` /
# `block_jacobi` above.

MAS_DOMAIN = 32


def mas_order(positions, n=None):
    """rank (n,) int32: position of every vertex in the domain order.  Morton order of the positions quantised
    isotropically to 10 bits per axis over the largest extent (ties keep index order); None -> index order."""
    if positions is None:
        return np.arange(n, dtype=np.int32)
    p = np.asarray(positions, dtype=np.float64)
    lo = p.min(axis=0)
    ext = (p.max(axis=0) - lo).max()
    code = np.zeros(p.shape[0], dtype=np.uint32)
    if ext > 0.0:
        q = ((p - lo) / ext * 1023.0).astype(np.uint32)
        for k in range(3):
            v = q[:, k].astype(np.uint32)
            s = np.zeros_like(v)
            for b in range(10):
                s |= ((v >> np.uint32(b)) & np.uint32(1)) << np.uint32(3 * b)
            code |= s << np.uint32(k)
    order = np.argsort(code, kind="stable")
    rank = np.empty(p.shape[0], dtype=np.int32)
    rank[order] = np.arange(p.shape[0], dtype=np.int32)
    return rank


def mas_setup(rowptr, colidx, vals, rank, levels=1, fixed=None):
    """Per level: (node of every vertex, stored domain inverses (ndom, 96, 96) -- fp64 inverse, symmetrised,
    rounded to fp32 as the device stores them).  Level-l nodes are runs of 32**l vertices of the domain order.
    Dirichlet vertices (``fixed``) are left out of the coarse spaces (node -1 above level 0): the corrections
    leave them exactly at rest; a coarse node without free vertices gets the identity."""
    n = rowptr.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    out = []
    for l in range(levels):
        node = rank.astype(np.int64) >> (5 * l)
        if l > 0 and fixed is not None:
            node = np.where(np.asarray(fixed, bool), -1, node)
        nnode = (n + MAS_DOMAIN ** l - 1) // MAS_DOMAIN ** l
        ndom = (nnode + MAS_DOMAIN - 1) // MAS_DOMAIN
        if l > 0 and (n + MAS_DOMAIN - 1) // MAS_DOMAIN < 2:
            break
        a = np.zeros((ndom, 3 * MAS_DOMAIN, 3 * MAS_DOMAIN))
        gi, gj = node[rows], node[colidx]
        same = ((gi >> 5) == (gj >> 5)) & (gi >= 0) & (gj >= 0)
        d_, ki, kj = (gi >> 5)[same], (gi & 31)[same], (gj & 31)[same]
        for r_ in range(3):
            for c_ in range(3):
                np.add.at(a, (d_, 3 * ki + r_, 3 * kj + c_), vals[same, r_, c_])
        pad = np.arange(nnode, ndom * MAS_DOMAIN)              # padding nodes: identity
        empty = np.setdiff1d(np.arange(nnode), node[node >= 0]) if l > 0 else np.zeros(0, np.int64)
        for g in np.concatenate([pad, empty]).astype(np.int64):
            k = g & 31
            a[g >> 5, 3 * k:3 * k + 3, 3 * k:3 * k + 3] = np.eye(3)
        inv = np.linalg.inv(a)
        inv = (0.5 * (inv + np.swapaxes(inv, 1, 2))).astype(np.float32).astype(np.float64)
        out.append((node, inv))
    return out


def mas_apply(levels, r):
    """z = sum_l P_l D_l^-1 P_l^T r."""
    n = r.shape[0] // 3
    z = np.zeros_like(r)
    for node, inv in levels:
        ndom = inv.shape[0]
        rc = np.zeros((ndom * MAS_DOMAIN, 3))
        inside = node >= 0
        np.add.at(rc, node[inside], r.reshape(n, 3)[inside])
        yc = np.einsum("dij,dj->di", inv, rc.reshape(ndom, 3 * MAS_DOMAIN)).reshape(-1, 3)
        z.reshape(n, 3)[inside] += yc[node[inside]]
    return z


def pcg_solve_mas(rowptr, colidx, vals, pinv, fixed, rhs, rel_tol, max_iters, levels):
    """pcg_solve (solver.py:279-315) driven by the MAS operator; stops on the reference's rule measured with the
    block-Jacobi inverses ``pinv``.  Returns (d, iters, converged)."""
    n = rowptr.shape[0] - 1

    def bj(r_):
        return np.einsum("nij,nj->ni", pinv, r_.reshape(n, 3)).reshape(-1)

    d = np.zeros_like(rhs)
    r = rhs.copy()
    r.reshape(n, 3)[fixed] = 0.0
    s = mas_apply(levels, r)
    delta_new = float(r @ s)
    bj0 = bj_new = float(r @ bj(r))
    if bj0 <= 0.0 or delta_new <= 0.0:
        return d, 0, bj0 <= 0.0
    c = s.copy()
    iters = 0
    while iters < max_iters and bj_new > rel_tol * bj0:
        q = bsr_matvec(rowptr, colidx, vals, c)
        denom = float(c @ q)
        if denom <= 0.0:
            break
        alpha = delta_new / denom
        d += alpha * c
        r -= alpha * q
        s = mas_apply(levels, r)
        delta_old = delta_new
        delta_new = float(r @ s)
        bj_new = float(r @ bj(r))
        c = s + (delta_new / delta_old) * c
        iters += 1
    return d, iters, bj_new <= rel_tol * bj0
