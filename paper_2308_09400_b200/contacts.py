"""Contact-list construction: host broad phase + GPU narrow phase.

``find_contact_pairs`` keeps the reference's signature and result
(``/root/reference/pkg/src/tetipc/proximity.py:262-358``): a list of ``ContactStencil`` sorted by
(kind.value, verts, origin).  The O(n^2) AABB sweep is replaced by a conservative uniform-grid
join on the host (any duplicate-free superset of the near queries gives the identical list);
classification, the d2 < d_hat^2 filter, parallel promotion, eps_x and the sort run on the GPU
(``b200ipc_narrow_phase``).  ``narrow_phase_device`` is the batched, device-resident form.
"""

import ctypes as C
from types import SimpleNamespace

import numpy as np

from . import _lib, device
from .proximity import StencilTable
from .stencils import DeviceStencilTable
from .workloads import broad_phase


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
    view = SimpleNamespace(positions=positions, tris=np.asarray(scene.surf_tris), edges=np.asarray(scene.surf_edges),
                           d_hat=float(d_hat))
    surf_verts = getattr(scene, "surf_verts", None)
    vt, ee = broad_phase(view, surf_verts=surf_verts)
    return narrow_phase(positions, scene.rest_positions, vt, ee, d_hat, promote_parallel).to_stencils()
