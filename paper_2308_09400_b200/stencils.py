"""Batched contact-stencil evaluation on the GPU: energy, gradient, PSD blocks.

The batched twin of the reference's per-stencil loop in
``SimState.assemble_local_quadratics`` / ``_barrier_energy`` (solver.py:127-146, :190-216):
one call evaluates a whole kind-sorted ``StencilTable`` through ``b200ipc_barrier_stencils``
and leaves the results in HBM, grouped in the size families ``group_blocks`` produces
(solver.py:237-248), ready for assembly / matvec without a host round trip.
"""

from dataclasses import dataclass, field

import numpy as np

import ctypes as C

from . import _lib, device
from .barrier import BarrierParams, LocalQuadratic, c_params
from .gap import InterpenetrationError
from .proximity import EE, EEP, FAMILY4_KINDS, PE, PEP, PP, PPP, PT, StencilTable

FAMILY_KINDS = {2: (PP,), 3: (PE,), 4: FAMILY4_KINDS}


@dataclass
class DeviceStencilTable:
    """A ``StencilTable`` resident in HBM (verts int32 (n,4), sub u8, eps_x f64)."""

    n: int
    kind_off: np.ndarray  # host (8,) int64
    verts: object
    sub: object
    eps_x: object
    host: StencilTable = None

    @classmethod
    def from_host(cls, table):
        return cls(len(table), table.kind_offsets(), device.to_device(table.verts), device.to_device(table.sub),
                   device.to_device(table.eps_x), table)

    def family_count(self, s):
        off = self.kind_off
        return int(sum(off[k + 1] - off[k] for k in FAMILY_KINDS[s]))

    def family_vids(self, s, dtype=np.int64):
        """(nb,s) vertex ids of a size family, in group_blocks order (device tensor)."""
        t = device.torch()
        off = self.kind_off
        parts = [self.verts[int(off[k]):int(off[k + 1]), :s] for k in FAMILY_KINDS[s] if off[k + 1] > off[k]]
        if not parts:
            return device.empty((0, s), dtype)
        out = parts[0] if len(parts) == 1 else t.cat(parts, dim=0)
        return out.to(device._dtype(dtype)).contiguous()


@dataclass
class Family:
    """One size family: the (hess, vids) pair of ``group_blocks`` plus the gradients."""

    s: int
    vids: object   # (nb,s) int64 device
    grad: object   # (nb,3s) device or None
    hess: object   # (nb,3s,3s) device or None; (nb,s,s,3,3) when ``tiled``
    fac: object = None   # (nb,3s) device or None: rank-1 factor z, hess == z z^T
    tiled: bool = False  # hess is sub-block-major (the assembly's internal layout), not the reference's

    def dense_hess(self):
        """The reference's (nb,3s,3s) blocks whatever the device layout (a permuted copy when ``tiled``)."""
        if self.hess is None or not self.tiled:
            return self.hess
        nb, s = self.hess.shape[0], self.s
        return self.hess.permute(0, 1, 3, 2, 4).reshape(nb, 3 * s, 3 * s).contiguous()


@dataclass
class BarrierBatch:
    """Device-resident result of one stencil evaluation."""

    table: DeviceStencilTable
    energy: object            # (n,) per-stencil energy, table order (or None)
    status: object            # (n,) u8
    families: dict = field(default_factory=dict)   # s -> Family
    _summary: tuple = None

    def summary(self):
        """(total energy, n_inactive, n_penetrating): one deterministic device reduction + D2H."""
        if self._summary is None:
            res = device.zeros((1,))
            cnt = device.zeros((2,), np.int64)
            ws = device.empty((_lib_ws_doubles(),))
            _lib.check(_lib.lib().b200ipc_reduce_energy(self.table.n, device.ptr(self.energy), device.ptr(self.status),
                                                        device.ptr(res), device.ptr(cnt), device.ptr(ws),
                                                        device.stream()), "reduce_energy")
            c = device.to_host(cnt)
            self._summary = (float(device.to_host(res)[0]), int(c[0]), int(c[1]))
        return self._summary

    def raise_on_penetration(self):
        """The reference raises InterpenetrationError on d2 <= 0 (gap.py:61, solver.py:132)."""
        if self._summary is None and self.energy is None:   # evaluated without energies: count the flags alone
            penetrating = int((self.status == 2).sum().item())
        else:
            penetrating = self.summary()[2]
        if penetrating:
            bad = np.flatnonzero(device.to_host(self.status) == 2)
            raise InterpenetrationError(f"nonpositive squared distance on {bad.size} stencil(s), first row {bad[0]}")

    def grouped(self):
        """``[(hess, vids)]`` by ascending stencil size, as ``group_blocks`` returns (device tensors)."""
        return [(self.families[s].dense_hess(), self.families[s].vids) for s in sorted(self.families)]

    def to_local_quadratics(self, keep_inactive=False):
        """Host ``LocalQuadratic`` list in the reference's block order, inactive rows dropped
        (solver.py:202-209) unless ``keep_inactive`` (then one entry per table row, zeros for inactive rows:
        the positional list ``barrier_gradient_blocks`` returns, solver.py:186-188).  Outputs that were not
        requested from ``evaluate`` come back as ``None`` fields."""
        status = device.to_host(self.status)
        out = [None] * self.table.n
        off = self.table.kind_off
        for s, fam in self.families.items():
            rows = np.concatenate([np.arange(off[k], off[k + 1]) for k in FAMILY_KINDS[s]])
            vids = device.to_host(fam.vids)
            grad = device.to_host(fam.grad) if fam.grad is not None else None
            hess = device.to_host(fam.dense_hess()) if fam.hess is not None else None
            for j, r in enumerate(rows):
                if status[r] == 0 or keep_inactive:
                    out[r] = LocalQuadratic(vert_ids=vids[j].copy(), grad=None if grad is None else grad[j].copy(),
                                            hess=None if hess is None else hess[j].copy())
        return [b for b in out if b is not None]


def _lib_ws_doubles():
    return 16384 // 8


def evaluate(table, positions, params, dt=1.0, want_energy=True, want_grad=True, want_hess=True,
             want_factors=False, out=None, hess_layout="dense"):
    """Evaluate every stencil of ``table`` at ``positions``.

    ``table``: ``StencilTable`` or ``DeviceStencilTable``; ``positions``: (N,3) host array or
    device tensor; ``params``: ``BarrierParams``; ``dt``: time step (grad/hess are scaled by
    dt**2, energy is not, like solver.py:207-208).  ``out``: a previous ``BarrierBatch`` for the
    same table whose buffers are reused.  ``want_factors`` adds the rank-1 factors z (hess = z z^T);
    with ``want_hess=False`` the dense blocks are skipped and ``NewtonSystem.assemble_from_factors``
    builds the matrix from z alone.  ``hess_layout="subblock"`` leaves the dense blocks on the device as
    (nb,s,s,3,3) -- the layout ``NewtonSystem.set_pattern(..., tiled=...)`` + ``assemble`` gather fastest; ``Family.dense_hess()``
    and everything host-facing still give the reference's (nb,3s,3s).  Returns a ``BarrierBatch`` (asynchronous).
    """
    if hess_layout not in ("dense", "subblock"):
        raise ValueError("hess_layout must be 'dense' or 'subblock'")
    tiled = hess_layout == "subblock"
    if isinstance(table, StencilTable):
        table = DeviceStencilTable.from_host(table)
    if not isinstance(params, BarrierParams):
        raise TypeError("params must be BarrierParams")
    pos = device.to_device(positions, np.float64)
    if pos.dim() != 2 or pos.shape[1] != 3:
        raise ValueError("positions must be (N, 3)")
    n = table.n
    if out is None:
        fams = {}
        for s in (2, 3, 4):
            nb = table.family_count(s)
            if nb == 0:
                continue
            fams[s] = Family(s, table.family_vids(s),
                             device.empty((nb, 3 * s)) if want_grad else None,
                             device.empty((nb, s, s, 3, 3) if tiled else (nb, 3 * s, 3 * s)) if want_hess else None,
                             device.empty((nb, 3 * s)) if want_factors else None, tiled)
        out = BarrierBatch(table, device.empty((n,)) if want_energy else None, device.empty((n,), np.uint8), fams)
    elif any(f.tiled != tiled for f in out.families.values()):
        raise ValueError("out was evaluated with another hess_layout")
    out._summary = None
    prm = c_params(params, dt)
    koff = (C.c_int64 * 8)(*[int(v) for v in table.kind_off])

    def fam_ptr(s, name):
        fam = out.families.get(s)
        return device.ptr(getattr(fam, name) if fam is not None else None)

    _lib.check(_lib.lib().b200ipc_barrier_stencils_layout(
        prm, pos.shape[0], device.ptr(pos), n, koff, device.ptr(table.verts), device.ptr(table.sub),
        device.ptr(table.eps_x), device.ptr(out.energy), device.ptr(out.status),
        fam_ptr(2, "grad"), fam_ptr(2, "hess"), fam_ptr(3, "grad"), fam_ptr(3, "hess"),
        fam_ptr(4, "grad"), fam_ptr(4, "hess"), fam_ptr(2, "fac"), fam_ptr(3, "fac"), fam_ptr(4, "fac"),
        1 if tiled else 0, device.stream()), "barrier_stencils")
    return out


def barrier_energy(table, positions, params):
    """Total barrier energy of a contact list (SimState._barrier_energy, solver.py:127-146).

    Raises InterpenetrationError when any stencil has d2 <= 0.
    """
    batch = evaluate(table, positions, params, want_grad=False, want_hess=False)
    batch.raise_on_penetration()
    return batch.summary()[0]


__all__ = ["BarrierBatch", "DeviceStencilTable", "Family", "barrier_energy", "evaluate",
           "EE", "EEP", "PE", "PEP", "PP", "PPP", "PT"]
