"""Contact-list construction on the GPU: grid broad phase + narrow phase.

``find_contact_pairs`` keeps the reference's signature and result
(``/root/reference/pkg/src/tetipc/proximity.py:262-358``): a list of ``ContactStencil`` sorted by
(kind.value, verts, origin).  The O(n^2) AABB sweep is replaced by a uniform-grid join
(``BroadPhase`` -> ``b200ipc_broad_phase_*``) that evaluates the reference's own overlap predicate,
so the candidate sets are identical; classification, the d2 < d_hat^2 filter, parallel promotion,
eps_x and the sort run in ``b200ipc_narrow_phase``.  ``BroadPhase.query`` and
``narrow_phase_device`` are the batched, device-resident forms: positions in, stencil table out,
nothing crosses PCIe in between.
"""

import ctypes as C
from types import SimpleNamespace

import numpy as np

from . import _lib, device
from .proximity import StencilTable
from .stencils import DeviceStencilTable


class BroadPhase:
    """Device-resident broad phase of one scene: surface arrays uploaded once, one query per detect.

    ``surf_verts (nv,)``, ``tris (nt,3)``, ``edges (ne,2)``: the reference ``Scene``'s surface arrays.
    ``cell`` defaults to max(2 d_hat, median edge length at ``positions``) -- speed only.
    """

    def __init__(self, surf_verts, tris, edges, d_hat, positions=None, cell=None):
        self.d_hat = float(d_hat)
        tris = np.asarray(tris).reshape(-1, 3)
        edges = np.asarray(edges).reshape(-1, 2)
        if surf_verts is None:
            surf_verts = np.unique(tris)
        self.surf_verts = device.to_device(np.asarray(surf_verts).reshape(-1), np.int32)
        self.tris = device.to_device(tris, np.int32)
        self.edges = device.to_device(edges, np.int32)
        if cell is None:
            cell = 2.0 * self.d_hat
            if positions is not None and len(edges):
                x = np.asarray(positions, dtype=np.float64)
                cell = max(cell, float(np.median(np.linalg.norm(x[edges[:, 1]] - x[edges[:, 0]], axis=1))))
        self.cell = float(cell)
        self._h = C.c_void_p()
        _lib.check(_lib.lib().b200ipc_broad_create(C.byref(self._h)), "broad_create")

    def close(self):
        if getattr(self, "_h", None) is not None and self._h:
            _lib.lib().b200ipc_broad_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()

    def query(self, positions):
        """positions (N,3) host array or device tensor -> (vt (m,4), ee (k,4)) int32 device tensors."""
        pos = device.to_device(positions, np.float64)
        lo = pos.amin(dim=0).cpu().numpy() - 2.0 * self.cell
        origin = (C.c_double * 3)(*[float(v) for v in lo])
        n_vt, n_ee = C.c_int64(0), C.c_int64(0)
        L = _lib.lib()
        _lib.check(L.b200ipc_broad_phase_count(
            self._h, pos.shape[0], device.ptr(pos), self.surf_verts.shape[0], device.ptr(self.surf_verts),
            self.tris.shape[0], device.ptr(self.tris), self.edges.shape[0], device.ptr(self.edges), self.d_hat,
            self.cell, origin, C.byref(n_vt), C.byref(n_ee), device.stream()), "broad_phase_count")
        vt = device.empty((max(int(n_vt.value), 1), 4), np.int32)
        ee = device.empty((max(int(n_ee.value), 1), 4), np.int32)
        _lib.check(L.b200ipc_broad_phase_fill(self._h, device.ptr(vt), device.ptr(ee), device.stream()),
                   "broad_phase_fill")
        return vt[:int(n_vt.value)], ee[:int(n_ee.value)]


def narrow_phase_device(positions, rest_positions, vt, ee, d_hat, promote_parallel=True, want_origin=True):
    """Queries -> ``DeviceStencilTable`` (plus origin tensors when ``want_origin``).

    positions / rest_positions: (N,3); vt (m,4), ee (k,4) integer arrays or device tensors.
    """
    pos = device.to_device(positions, np.float64)
    rest = device.to_device(rest_positions, np.float64)
    d_vt = device.to_device(np.asarray(vt).reshape(-1, 4) if not hasattr(vt, "data_ptr") else vt, np.int32)
    d_ee = device.to_device(np.asarray(ee).reshape(-1, 4) if not hasattr(ee, "data_ptr") else ee, np.int32)
    n_vt, n_ee = int(d_vt.shape[0]), int(d_ee.shape[0])
    cap = max(n_vt + n_ee, 1)
    kind = device.empty((cap,), np.uint8)
    verts = device.empty((cap, 4), np.int32)
    sub = device.empty((cap,), np.uint8)
    eps = device.empty((cap,))
    otype = device.empty((cap,), np.uint8) if want_origin else None
    origin = device.empty((cap, 4), np.int32) if want_origin else None
    n_out = C.c_int64(0)
    koff = (C.c_int64 * 8)()
    d_hat = float(d_hat)
    _lib.check(_lib.lib().b200ipc_narrow_phase(
        pos.shape[0], device.ptr(pos), device.ptr(rest), n_vt, device.ptr(d_vt), n_ee, device.ptr(d_ee),
        d_hat * d_hat, 1 if promote_parallel else 0, device.ptr(kind), device.ptr(verts), device.ptr(sub),
        device.ptr(eps), device.ptr(otype), device.ptr(origin), C.byref(n_out), koff, device.stream()),
        "narrow_phase")
    n = int(n_out.value)
    table = DeviceStencilTable(n, np.array(list(koff), dtype=np.int64), verts[:n], sub[:n], eps[:n], None)
    extra = SimpleNamespace(kind=kind[:n], origin_type=None if otype is None else otype[:n],
                            origin=None if origin is None else origin[:n])
    return table, extra


def narrow_phase(positions, rest_positions, vt, ee, d_hat, promote_parallel=True):
    """Host ``StencilTable`` of the ordered contact list for the given candidate queries."""
    table, extra = narrow_phase_device(positions, rest_positions, vt, ee, d_hat, promote_parallel)
    host = StencilTable(device.to_host(extra.kind), device.to_host(table.verts), device.to_host(table.sub),
                        device.to_host(table.eps_x), device.to_host(extra.origin_type), device.to_host(extra.origin))
    table.host = host
    return host


def find_contact_pairs(scene, positions, d_hat, promote_parallel=True):
    """All contact stencils closer than ``d_hat`` (proximity.py:262-358).

    ``scene`` needs ``surf_tris``, ``surf_edges`` and ``rest_positions`` (the reference's
    ``Scene`` works as is).
    """
    positions = np.asarray(positions, dtype=np.float64)
    bp = BroadPhase(getattr(scene, "surf_verts", None), scene.surf_tris, scene.surf_edges, d_hat, positions)
    try:
        vt, ee = bp.query(positions)
        return narrow_phase(positions, scene.rest_positions, vt, ee, d_hat, promote_parallel).to_stencils()
    finally:
        bp.close()
