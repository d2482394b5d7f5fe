"""Stable neo-Hookean tetrahedra on the GPU.

Mirror of ``/root/reference/pkg/src/tetipc/elasticity.py``: ``ElasticMaterial``, ``rest_data``,
``batch_grad_hess``, ``tet_energy_grad_hess``, ``tet_local_quadratic`` keep their names, arguments and
results; ``TetMesh`` is the device-resident form (rest data uploaded once, one ``evaluate`` per Newton
iteration) whose (hess, vids) family goes to ``solver.NewtonSystem`` next to the barrier families.
The 9x9 dPsi/dF^2 is projected PSD analytically (closed-form twist / flip / scaling eigenpairs from a
3x3 SVD of F, in registers; the reference calls LAPACK ``eigh`` -- the projection is unique).
"""

from dataclasses import dataclass, field

import numpy as np

from . import _lib, device
from .barrier import LocalQuadratic
from .stencils import Family


def lame_parameters(youngs_E, poisson_nu):
    """(mu, lambda) of an isotropic material; E > 0 and 0 < nu < 1/2 or ValueError (elasticity.py:24-30)."""
    if not (youngs_E > 0.0 and 0.0 < poisson_nu < 0.5):
        raise ValueError("need E > 0 and nu in (0, 0.5)")
    shear = 0.5 * youngs_E / (1.0 + poisson_nu)
    return shear, 2.0 * shear * poisson_nu / (1.0 - 2.0 * poisson_nu)


@dataclass
class ElasticMaterial:
    """Field-compatible with the reference's material record (elasticity.py:18-30)."""

    youngs_E: float
    poisson_nu: float
    lame_mu: float = field(init=False, default=0.0)
    lame_lambda: float = field(init=False, default=0.0)

    def __post_init__(self):
        self.lame_mu, self.lame_lambda = lame_parameters(self.youngs_E, self.poisson_nu)


def dvec_f_dx(rest_inv):
    """(t,9,12) maps x -> vec(F) implied by rest_inv: row 3c+i, column 3v+i holds w_vc with
    w_0c = -sum_r rest_inv[r,c] and w_vc = rest_inv[v-1,c]; pure indexing, kept for API parity."""
    rest_inv = np.asarray(rest_inv, dtype=np.float64)
    t = rest_inv.shape[0]
    w = np.concatenate([-rest_inv.sum(axis=1, keepdims=True), rest_inv], axis=1)      # (t, 4 vertices, 3 columns c)
    maps = np.zeros((t, 3, 3, 4, 3))                                                    # [t, c, i, v, i']
    for i in range(3):
        maps[:, :, i, :, i] = np.swapaxes(w, 1, 2)
    return maps.reshape(t, 9, 12)


class TetMesh:
    """Device-resident tet set: ``tets (t,4)``, rest data computed once (``rest_data``)."""

    def __init__(self, rest_positions, tets, mu, lam):
        tets = np.asarray(tets).reshape(-1, 4)
        self.t = int(tets.shape[0])
        self.tets = device.to_device(tets, np.int32)
        self.vids = device.to_device(tets, np.int64)
        self.mu = device.to_device(np.broadcast_to(np.asarray(mu, dtype=np.float64), (self.t,)).copy())
        self.lam = device.to_device(np.broadcast_to(np.asarray(lam, dtype=np.float64), (self.t,)).copy())
        self.rest_inv = device.empty((self.t, 3, 3))
        self.vols = device.empty((self.t,))
        rest = device.to_device(rest_positions, np.float64)
        _lib.check(_lib.lib().b200ipc_elastic_rest(self.t, device.ptr(self.tets), device.ptr(rest),
                                                   device.ptr(self.rest_inv), device.ptr(self.vols), device.stream()),
                   "elastic_rest")

    def evaluate(self, positions, dt=1.0, project=True, want_energy=True, want_grad=True, want_hess=True):
        """(energy (t,), Family(s=4, vids, grad (t,12), hess (t,12,12))): grad / hess scaled by dt**2
        (solver.py:196-200), energy volume-scaled but not dt-scaled (``_elastic_energy``, :154-159)."""
        pos = device.to_device(positions, np.float64)
        energy = device.empty((self.t,)) if want_energy else None
        grad = device.empty((self.t, 12)) if want_grad else None
        hess = device.empty((self.t, 12, 12)) if want_hess else None
        _lib.check(_lib.lib().b200ipc_elastic_blocks(
            self.t, device.ptr(self.tets), device.ptr(pos), device.ptr(self.rest_inv), device.ptr(self.vols),
            device.ptr(self.mu), device.ptr(self.lam), float(dt) ** 2, 1 if project else 0, device.ptr(energy),
            device.ptr(grad), device.ptr(hess), device.stream()), "elastic_blocks")
        return energy, Family(4, self.vids, grad, hess)


def rest_data(rest_positions, tets):
    """Twin of elasticity.py:39-56: (rest_inv (t,3,3), vols (t,), g (t,9,12))."""
    tets = np.asarray(tets).reshape(-1, 4)
    mesh = TetMesh(rest_positions, tets, 1.0, 1.0)
    rest_inv, vols = device.to_host(mesh.rest_inv), device.to_host(mesh.vols)
    return rest_inv, vols, dvec_f_dx(rest_inv)


def batch_grad_hess(positions, tets, rest_inv, vols, g_maps, mu, lam, project=True):
    """Twin of elasticity.py:128-137 (``g_maps`` is implied by ``rest_inv`` and ignored)."""
    tets = np.asarray(tets).reshape(-1, 4)
    t = tets.shape[0]
    d_tets = device.to_device(tets, np.int32)
    args = [device.to_device(np.ascontiguousarray(a, dtype=np.float64)) for a in (positions, rest_inv, vols)]
    d_mu = device.to_device(np.broadcast_to(np.asarray(mu, dtype=np.float64), (t,)).copy())
    d_lam = device.to_device(np.broadcast_to(np.asarray(lam, dtype=np.float64), (t,)).copy())
    e, g, h = device.empty((t,)), device.empty((t, 12)), device.empty((t, 12, 12))
    _lib.check(_lib.lib().b200ipc_elastic_blocks(t, device.ptr(d_tets), *[device.ptr(a) for a in args], device.ptr(d_mu),
                                                 device.ptr(d_lam), 1.0, 1 if project else 0, device.ptr(e), device.ptr(g),
                                                 device.ptr(h), device.stream()), "elastic_blocks")
    return device.to_host(e), device.to_host(g), device.to_host(h)


def tet_energy_grad_hess(rest_inv, positions, material, project=True):
    """Twin of elasticity.py:140-159: one tet, rest volume recovered from ``rest_inv``."""
    rest_inv = np.asarray(rest_inv, dtype=np.float64).reshape(1, 3, 3)
    vol = np.array([1.0 / (6.0 * np.linalg.det(rest_inv[0]))])
    e, g, h = batch_grad_hess(np.asarray(positions, dtype=np.float64), np.array([[0, 1, 2, 3]]), rest_inv, vol, None,
                              np.array([material.lame_mu]), np.array([material.lame_lambda]), project=project)
    return float(e[0]), g[0], h[0]


def tet_local_quadratic(vert_ids, grad, hess):
    return LocalQuadratic(vert_ids=np.asarray(vert_ids, dtype=np.int64), grad=grad, hess=hess)
