"""Lagged smooth Coulomb friction on the GPU.

Mirror of ``/root/reference/pkg/src/tetipc/friction.py``: the same names, arguments and results for
the per-datum functions (``f0_f1``, ``potential``, ``friction_force``, ``friction_hessian_psd``,
``tangential_displacement``, ``update_friction_state``, ``FrictionDatum``), each an n = 1 shim over
the batched kernels behind ``include/b200ipc.h``; and the batched, device-resident forms the solver
path uses: ``update_state`` (once per time step) and ``evaluate`` (once per Newton iteration), whose
``FrictionBatch.families`` feed ``solver.NewtonSystem`` next to the barrier families.
"""

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib, device
from .barrier import LocalQuadratic
from .proximity import KIND_CODE, KIND_SIZE, StencilKind, StencilTable
from .stencils import BarrierBatch, DeviceStencilTable, Family, FAMILY_KINDS


@dataclass
class FrictionDatum:
    """Per-contact lagged friction state (friction.py:17-30); ``basis_T`` is (3s, 2)."""

    stencil: object
    lambda_n: float
    basis_T: np.ndarray
    mu: float
    eps_v: float
    dt: float


@dataclass
class FrictionState:
    """Device-resident friction data of one time step: a kind-sorted table of the kept stencils and
    their frames (cn[4], t1[3], t2[3], lambda_n, 0); T[3v:3v+3, k] = cn_v t_k."""

    table: DeviceStencilTable
    frame: object          # (n,12) device
    rows_dev: object       # rows of the source table that became data (device int64)
    mu: float
    eps_v: float
    dt: float

    @property
    def n(self):
        return self.table.n

    @property
    def rows(self):
        """Rows of the source table that became data, as a host array."""
        return device.to_host(self.rows_dev)


@dataclass
class FrictionBatch:
    state: FrictionState
    energy: object                                  # (n,) device, not dt^2-scaled
    families: dict = field(default_factory=dict)    # s -> Family(vids, grad, hess)

    def total_energy(self):
        return float(self.energy.sum().item()) if self.state.n else 0.0

    def grouped(self):
        return [(self.families[s].hess, self.families[s].vids) for s in sorted(self.families)]


def _koff(kind_off):
    return (C.c_int64 * 8)(*[int(v) for v in kind_off])


def update_state(table, positions, mu, eps_v, dt, barrier_batch=None, params=None):
    """``update_friction_state`` (friction.py:148-171) for a whole contact table.

    ``barrier_batch``: a ``stencils.evaluate(table, positions, params, dt=1.0)`` result whose gradient
    families are the RAW barrier gradients (evaluated here when omitted; then ``params`` is needed).
    Raises ValueError when a contact normal is undefined (friction.py:138-139).
    """
    from . import stencils

    if isinstance(table, StencilTable):
        table = DeviceStencilTable.from_host(table)
    pos = device.to_device(positions, np.float64)
    n = table.n
    if mu <= 0.0 or n == 0:
        empty = DeviceStencilTable(0, np.zeros(8, np.int64), device.empty((0, 4), np.int32), device.empty((0,), np.uint8),
                                   device.empty((0,)))
        return FrictionState(empty, device.empty((0, 12)), device.empty((0,), np.int64), float(mu), float(eps_v), float(dt))
    if barrier_batch is None:
        barrier_batch = stencils.evaluate(table, pos, params, dt=1.0, want_energy=False, want_hess=False)
    if not isinstance(barrier_batch, BarrierBatch):
        raise TypeError("barrier_batch must come from stencils.evaluate(..., dt=1.0)")

    def g(s):
        fam = barrier_batch.families.get(s)
        return device.ptr(None if fam is None else fam.grad)

    frame = device.empty((n, 12))
    status = device.empty((n,), np.uint8)
    _lib.check(_lib.lib().b200ipc_friction_state(n, _koff(table.kind_off), device.ptr(table.verts), device.ptr(table.sub),
                                                 device.ptr(pos), g(2), g(3), g(4), device.ptr(frame),
                                                 device.ptr(status), device.stream()), "friction_state")
    # compaction of the kept rows on the device (the reference skips d2 <= 0 and lambda_n <= 0 stencils);
    # only eight counters and one flag cross PCIe
    t = device.torch()
    ok = status == 0
    # kept rows per kind = differences of the running count of kept rows at the kind boundaries (the table is
    # kind-sorted and the compaction keeps its order)
    running = t.cat([t.zeros(1, dtype=t.int64, device=ok.device), t.cumsum(ok, 0, dtype=t.int64)])
    at = running[t.as_tensor(np.asarray(table.kind_off, dtype=np.int64), device=ok.device)]
    host = t.cat([at[1:] - at[:-1], (status == 3).any().to(t.int64).reshape(1)]).cpu().numpy()
    if host[7]:
        raise ValueError("undefined contact normal for friction basis")
    keep = t.nonzero(ok).squeeze(1)
    koff = np.concatenate([[0], np.cumsum(host[:7])]).astype(np.int64)
    # whole rows by index (torch's 2-D index_select / advanced indexing: 0.55 ms each for the (n,12) frames and the
    # (n,4) vertex rows of 1 M contacts)
    sub = DeviceStencilTable(int(keep.shape[0]), koff, device.gather_rows(table.verts, keep), table.sub.index_select(0, keep),
                             device.gather_rows(table.eps_x, keep))
    return FrictionState(sub, device.gather_rows(frame, keep), keep, float(mu), float(eps_v), float(dt))


def evaluate(state, positions, positions_start, want_energy=True, want_grad=True, want_hess=True):
    """Friction blocks of one Newton iteration (solver.py:210-214): grad = -dt^2 friction_force,
    hess = dt^2 friction_hessian_psd per datum, in ``group_blocks`` family order; energy (n,) is the
    un-scaled potential of ``_friction_energy`` (solver.py:147-152)."""
    x = device.to_device(positions, np.float64)
    xs = device.to_device(positions_start, np.float64)
    table = state.table
    n = table.n
    fams = {}
    for s in (2, 3, 4):
        nb = table.family_count(s)
        if nb:
            fams[s] = Family(s, table.family_vids(s), device.empty((nb, 3 * s)) if want_grad else None,
                             device.empty((nb, 3 * s, 3 * s)) if want_hess else None)
    energy = device.empty((n,)) if want_energy else None

    def p(s, name):
        fam = fams.get(s)
        return device.ptr(None if fam is None else getattr(fam, name))

    if n:
        _lib.check(_lib.lib().b200ipc_friction_blocks(
            n, _koff(table.kind_off), device.ptr(table.verts), device.ptr(state.frame), device.ptr(x), device.ptr(xs),
            state.mu, state.eps_v, state.dt, device.ptr(energy), p(2, "grad"), p(2, "hess"), p(3, "grad"),
            p(3, "hess"), p(4, "grad"), p(4, "hess"), device.stream()), "friction_blocks")
    return FrictionBatch(state, energy, fams)


# ---- the reference's per-datum entry points (n = 1 shims) ---------------------------------------

def _explicit(datum, u, want):
    basis = np.ascontiguousarray(datum.basis_T, dtype=np.float64)
    s = basis.shape[0] // 3
    d_basis = device.to_device(basis.reshape(1, 3 * s, 2))
    d_u = device.to_device(np.asarray(u, dtype=np.float64).reshape(1, 2))
    d_lam = device.to_device(np.array([datum.lambda_n], dtype=np.float64))
    pot = device.empty((1,)) if want == "potential" else None
    force = device.empty((1, 3 * s)) if want == "force" else None
    hess = device.empty((1, 3 * s, 3 * s)) if want == "hess" else None
    _lib.check(_lib.lib().b200ipc_friction_explicit(1, s, device.ptr(d_basis), device.ptr(d_u), device.ptr(d_lam),
                                                    float(datum.mu), float(datum.eps_v), float(datum.dt),
                                                    device.ptr(pot), device.ptr(force), device.ptr(hess),
                                                    device.stream()), "friction_explicit")
    return device.to_host(pot if pot is not None else (force if force is not None else hess))[0]


def f0_f1(u_norm, eps_v, dt):
    """Smoothing pair (friction.py:33-46) -> (f0, f1, f1')."""
    lam = device.to_device(np.array([1.0]))
    basis = device.to_device(np.array([[[1.0, 0.0], [0.0, 1.0], [0.0, 0.0], [0.0, 0.0], [0.0, 0.0], [0.0, 0.0]]]))
    un = float(u_norm)
    d_u = device.to_device(np.array([[un, 0.0]]))
    pot, force, hess = device.empty((1,)), device.empty((1, 6)), device.empty((1, 6, 6))
    _lib.check(_lib.lib().b200ipc_friction_explicit(1, 2, device.ptr(basis), device.ptr(d_u), device.ptr(lam), 1.0,
                                                    float(eps_v), float(dt), device.ptr(pot), device.ptr(force),
                                                    device.ptr(hess), device.stream()), "friction_explicit")
    f0 = float(device.to_host(pot)[0])
    if un >= dt * eps_v:
        return f0, 1.0, 0.0
    f1 = -float(device.to_host(force)[0, 0])          # force = -f1/|u| T u = -f1 e_1
    return f0, f1, float(device.to_host(hess)[0, 0, 0])   # core eigenvalue along u = max(f1', 0) = f1' below h


def potential(datum, u):
    return float(_explicit(datum, u, "potential"))


def friction_force(datum, u):
    return _explicit(datum, u, "force")


def friction_hessian_psd(datum, u):
    hess = _explicit(datum, u, "hess")
    return LocalQuadratic(vert_ids=np.asarray(datum.stencil.verts, dtype=np.int64), grad=np.zeros(hess.shape[0]),
                          hess=hess)


def tangential_displacement(datum, positions, positions_start):
    """u = T^T (x - x_start) over the stencil vertices (friction.py:174-178)."""
    ids = list(datum.stencil.verts)
    rel = (np.asarray(positions)[ids] - np.asarray(positions_start)[ids]).reshape(-1)
    return np.asarray(datum.basis_T).T @ rel


def update_friction_state(stencils, barrier_gradients, positions, mu, eps_v, dt):
    """Twin of friction.py:148-171: list of ``FrictionDatum`` from the end-of-step contact set and the
    raw barrier gradients of its stencils."""
    given = list(stencils)
    if mu <= 0.0 or not given:
        return []
    # the reference takes the stencils in any order with a positionally matched gradient list; the device table
    # wants kind-sorted rows: sort with a (stable) permutation and hand the data back in the caller's order
    order = sorted(range(len(given)), key=lambda i: KIND_CODE[StencilKind(given[i].kind.value)])
    stencils = [given[i] for i in order]
    table = StencilTable.from_stencils(stencils)
    dev = DeviceStencilTable.from_host(table)
    fams = {}
    off = table.kind_offsets()
    for s in (2, 3, 4):
        rows = np.concatenate([np.arange(off[k], off[k + 1]) for k in FAMILY_KINDS[s]]).astype(np.int64)
        if rows.size:
            g = np.stack([np.asarray(barrier_gradients[order[r]], dtype=np.float64).reshape(3 * s) for r in rows])
            fams[s] = Family(s, None, device.to_device(g), None)
    batch = BarrierBatch(dev, None, None, fams)
    state = update_state(dev, positions, mu, eps_v, dt, barrier_batch=batch)
    frames = device.to_host(state.frame)
    out = []
    for fr, r in zip(frames, state.rows):
        s = int(KIND_SIZE[table.kind[r]])
        basis = np.zeros((3 * s, 2))
        for v in range(s):
            basis[3 * v:3 * v + 3, 0] = fr[v] * fr[4:7]
            basis[3 * v:3 * v + 3, 1] = fr[v] * fr[7:10]
        out.append((order[r], FrictionDatum(stencil=stencils[r], lambda_n=float(fr[10]), basis_T=basis, mu=mu,
                                            eps_v=eps_v, dt=dt)))
    return [d for _, d in sorted(out, key=lambda t: t[0])]
