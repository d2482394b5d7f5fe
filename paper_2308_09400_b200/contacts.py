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
        # a scene with edges much longer than a cell (cloth on a coarse collider): the long boxes get a grid of their
        # own, or every vertex would probe the cells a LONG box could start in (speed only)
        self.coarse_cell = 0.0
        if positions is not None and len(edges):
            x = np.asarray(positions, dtype=np.float64)
            longest = float(np.linalg.norm(x[edges[:, 1]] - x[edges[:, 0]], axis=1).max())
            if longest + self.d_hat > 2.0 * self.cell:
                self.coarse_cell = 1.25 * longest + 2.0 * self.d_hat
        _lib.check(_lib.lib().b200ipc_broad_set_coarse_cell(self._h, self.coarse_cell), "broad_set_coarse_cell")

    def close(self):
        if getattr(self, "_h", None) is not None and self._h:
            _lib.lib().b200ipc_broad_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: module globals may already be gone
            pass

    def _grid(self, span, margin):
        """Grid origin (two cells below the lowest coordinate) and the cell-count hint for the key width."""
        lo = span[0] - 2.0 * self.cell - margin
        cells = np.ceil((span[1] - lo + margin + 2.0 * self.cell) / self.cell).astype(np.int64) + 1
        cells = np.minimum(np.maximum(cells, 1), 1 << 21)
        _lib.check(_lib.lib().b200ipc_broad_set_grid_cells(self._h, int(cells[0]), int(cells[1]), int(cells[2])),
                   "broad_set_grid_cells")
        return (C.c_double * 3)(*[float(v) for v in lo])

    def query(self, positions):
        """positions (N,3) host array or device tensor -> (vt (m,4), ee (k,4)) int32 device tensors.
        The rows are a deterministic SET in no particular order (the narrow phase sorts its output)."""
        pos = device.to_device(positions, np.float64)
        t = device.torch()
        origin = self._grid(t.stack(t.aminmax(pos, dim=0)).cpu().numpy(), 0.0)
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

    def sweep(self, positions, directions, margin=None):
        """sweep_candidates (proximity.py:388-421) on the device: pairs whose swept AABBs (pose at
        ``positions`` and at ``positions + directions``, grown by 1e-3 d_hat) overlap ->
        (vt (m,4) PAIR_PT ids, ee (k,4) PAIR_EE ids) int32 device tensors."""
        pos = device.to_device(positions, np.float64)
        dirs = device.to_device(directions, np.float64)
        margin = 1e-3 * self.d_hat if margin is None else float(margin)
        t = device.torch()
        span = t.stack(t.aminmax(t.cat([pos, pos + dirs]), dim=0)).cpu().numpy()   # over both poses
        origin = self._grid(span, margin)
        n_vt, n_ee = C.c_int64(0), C.c_int64(0)
        L = _lib.lib()
        _lib.check(L.b200ipc_sweep_candidates_count(
            self._h, pos.shape[0], device.ptr(pos), device.ptr(dirs), self.surf_verts.shape[0],
            device.ptr(self.surf_verts), self.tris.shape[0], device.ptr(self.tris), self.edges.shape[0],
            device.ptr(self.edges), margin, self.cell, origin, C.byref(n_vt), C.byref(n_ee), device.stream()),
            "sweep_candidates_count")
        vt = device.empty((max(int(n_vt.value), 1), 4), np.int32)
        ee = device.empty((max(int(n_ee.value), 1), 4), np.int32)
        _lib.check(L.b200ipc_broad_phase_fill(self._h, device.ptr(vt), device.ptr(ee), device.stream()),
                   "broad_phase_fill")
        return vt[:int(n_vt.value)], ee[:int(n_ee.value)]

    def ccd_step_bound(self, positions, directions, slack=0.9, max_iter=512):
        """sweep_candidates + global_ccd_filter (solver.py:337-340) without leaving the device:
        the largest step fraction along ``directions`` every swept candidate pair verifies."""
        pos = device.to_device(positions, np.float64)
        dirs = device.to_device(directions, np.float64)
        vt, ee = self.sweep(pos, dirs)
        return ccd_filter_device(vt, ee, pos, dirs, slack, max_iter)


def ccd_filter_device(vt, ee, positions, directions, slack=0.9, max_iter=512):
    """min(1, min over candidate pairs of accd_max_step) -> float; raises like the reference when a
    pair's current distance is not positive."""
    if not 0.0 < slack < 1.0:
        raise ValueError("slack must lie in (0, 1)")
    out = device.empty((2,))  # [alpha, n_invalid (int64 bits)]
    _lib.check(_lib.lib().b200ipc_ccd_filter(
        int(vt.shape[0]), device.ptr(vt), int(ee.shape[0]), device.ptr(ee), device.ptr(positions),
        device.ptr(directions), float(slack), int(max_iter), C.c_void_p(out.data_ptr()),
        C.c_void_p(out.data_ptr() + 8), device.stream()), "ccd_filter")
    host = device.to_host(out)
    if int(host[1:2].view(np.int64)[0]) != 0:
        raise ValueError("additive CCD requires a strictly positive initial distance")  # _core.pyx:307-308
    return float(host[0])


_PAIR_OF_KIND = {"point-triangle": 0, "edge-edge": 1, "edge-edge-parallel": 1, "point-edge-parallel": 1,
                 "point-point-parallel": 1, "point-edge": 2, "point-point": 3}  # proximity.py:361-369


def ccd_filter_superset_device(vt, ee, positions, directions, sweep_margin, slack=0.9, max_iter=512):
    """``ccd_filter_device`` over any SUPERSET of ``sweep_candidates``' lists: each pair is first put to the
    reference's swept-box test at ``sweep_margin`` (the reference: 1e-3 d_hat), the survivors go through ACCD --
    the same bound as over the reference's own list (min is order-free).  One swept join with a margin of d_hat/2
    can thus serve the CCD filter AND every line-search detection along the step."""
    if not 0.0 < slack < 1.0:
        raise ValueError("slack must lie in (0, 1)")
    out = device.empty((2,))  # [alpha, n_invalid (int64 bits)]
    scratch = device.empty((2 * (int(vt.shape[0]) + int(ee.shape[0])) + 2,))   # 16 bytes per pair + the two counts
    _lib.check(_lib.lib().b200ipc_ccd_filter_swept(
        int(vt.shape[0]), device.ptr(vt), int(ee.shape[0]), device.ptr(ee), device.ptr(positions),
        device.ptr(directions), float(sweep_margin), float(slack), int(max_iter), device.ptr(scratch),
        C.c_void_p(out.data_ptr()), C.c_void_p(out.data_ptr() + 8), device.stream()), "ccd_filter_swept")
    host = device.to_host(out)
    if int(host[1:2].view(np.int64)[0]) != 0:
        raise ValueError("additive CCD requires a strictly positive initial distance")  # _core.pyx:307-308
    return float(host[0])


def accd_step_bound(stencil, positions, directions, slack=0.9, max_iter=512):
    """Twin of proximity.py:372-385: ACCD bound of one stencil along ``directions``."""
    from . import kernels

    if not 0.0 < slack < 1.0:
        raise ValueError("slack must lie in (0, 1)")
    ids = list(stencil.verts)
    return kernels.accd_max_step(np.asarray(positions)[ids], np.asarray(directions)[ids],
                                 _PAIR_OF_KIND[stencil.kind.value], slack, max_iter)


def sweep_candidates(scene, positions, directions, d_hat):
    """Twin of proximity.py:388-421: list of (pair_kind, (ids...)) whose swept AABBs overlap: PT
    candidates, then EE candidates, each sorted by vertex ids (the device list is an unordered set)."""
    from . import kernels

    bp = BroadPhase(getattr(scene, "surf_verts", None), scene.surf_tris, scene.surf_edges, d_hat, positions)
    try:
        vt, ee = bp.sweep(positions, directions)
        vt, ee = device.to_host(vt), device.to_host(ee)
    finally:
        bp.close()
    vt, ee = vt[np.lexsort(vt.T[::-1])], ee[np.lexsort(ee.T[::-1])]
    return ([(kernels.PAIR_PT, tuple(int(v) for v in row)) for row in vt]
            + [(kernels.PAIR_EE, tuple(int(v) for v in row)) for row in ee])


def global_ccd_filter(scene, positions, directions, candidates, slack=0.9, max_iter=512):
    """Twin of proximity.py:424-432: min of the per-pair ACCD bounds over ``candidates``."""
    from . import kernels

    if not candidates:
        return 1.0
    ids = np.zeros((len(candidates), 4), np.int32)
    kinds = np.zeros(len(candidates), np.uint8)
    for k, (pair, verts) in enumerate(candidates):
        kinds[k] = pair
        ids[k, :len(verts)] = verts
    step, status = kernels.accd_max_step_device(device.to_device(ids), device.to_device(kinds),
                                                device.to_device(positions, np.float64),
                                                device.to_device(directions, np.float64), slack, max_iter)
    if int(device.to_host(status).max()) != 0:
        raise ValueError("additive CCD requires a strictly positive initial distance")
    return float(min(1.0, device.to_host(step).min()))


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
