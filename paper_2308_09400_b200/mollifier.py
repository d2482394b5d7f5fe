"""Mollified near-parallel edge-edge entry points with the reference's signatures
(mollifier.py:55-144, :191-210), evaluated by ``b200ipc_mollified_eigensystem`` and
``b200ipc_blocks_from_jacobian``."""

from dataclasses import dataclass

import numpy as np

from . import _lib, device
from .barrier import _blocks_from_jac, c_params
from .proximity import PARALLEL_KINDS, StencilKind


_IDX_G1 = 4   # slot (2,2) of the 3x3 J-space layout: gamma channel diagonal (mollifier.py:21)
_IDX_F1 = 8   # slot (3,3): gap channel diagonal (mollifier.py:22)


@dataclass
class MollifiedEigenSystem:
    """The reference's record, field for field (mollifier.py:35-52): ``lambda_gamma`` / ``lambda_g`` hold
    (primary, twist, twist) of the two channels, ``lambda7p <= lambda8p`` the eigenvalues of the 2x2 coupling
    block and ``q8p`` its normalised eigenmatrix (9-vector, entries at slots (2,2) and (3,3)); ``q_gamma2`` /
    ``q_gamma3`` are the constant twist directions.  After them, what the kernel computes besides: the two
    entries of ``q8p`` as scalars, the channel derivatives and the mollifier value / slope."""

    lambda_gamma: tuple
    lambda_g: tuple
    t: float
    p: float
    lambda7p: float
    lambda8p: float
    q_gamma2: np.ndarray
    q_gamma3: np.ndarray
    q8p: np.ndarray
    q_gamma: float = 0.0
    q_f: float = 0.0
    b_gamma: float = 0.0
    b_g: float = 0.0
    e_k: float = 0.0
    de_dgamma: float = 0.0


def mollified_eigensystem_batch(g, c, eps_x, params):
    """(n,12) host array: lam_gamma1, lam_g1, t, p, lambda7', lambda8', q_gamma, q_f, b_gamma, b_g, e, e'."""
    g = np.ascontiguousarray(np.atleast_1d(g), dtype=np.float64)
    c = np.ascontiguousarray(np.broadcast_to(np.asarray(c, dtype=np.float64), g.shape))
    eps = np.ascontiguousarray(np.broadcast_to(np.asarray(eps_x, dtype=np.float64), g.shape))
    if np.any(eps <= 0.0):
        raise ValueError("eps_x must be positive")
    if np.any(c < 0.0):
        raise ValueError("parallelness measure must be nonnegative")
    out = device.empty((g.shape[0], 12))
    d_g, d_c, d_eps = device.to_device(g), device.to_device(c), device.to_device(eps)  # keep alive until launch
    _lib.check(_lib.lib().b200ipc_mollified_eigensystem(
        c_params(params), g.shape[0], device.ptr(d_g), device.ptr(d_c), device.ptr(d_eps), device.ptr(out),
        device.stream()), "mollified_eigensystem")
    return device.to_host(out)


def mollified_eigensystem(g, c, params, eps_x):
    """Closed-form eigensystem of the mollified J-space Hessian (mollifier.py:106-144)."""
    lam_gamma1, lam_g1, t, p, lam7p, lam8p, q_gamma, q_f, b_gamma, b_g, e_k, de = (
        float(v) for v in mollified_eigensystem_batch(g, c, eps_x, params)[0])
    q8p = np.zeros(9)
    q8p[_IDX_G1], q8p[_IDX_F1] = q_gamma, q_f
    q_gamma2 = np.zeros(9)
    q_gamma2[5] = -1.0     # twist onto slot (3,2) (mollifier.py:129-130)
    q_gamma3 = np.zeros(9)
    q_gamma3[3] = 1.0      # twist onto slot (1,2) (mollifier.py:131-132)
    lam_gamma23, lam_g23 = 2.0 * b_gamma, 2.0 * b_g           # mollifier.py:110, :112
    return MollifiedEigenSystem(lambda_gamma=(lam_gamma1, lam_gamma23, lam_gamma23), lambda_g=(lam_g1, lam_g23, lam_g23),
                                t=t, p=p, lambda7p=lam7p, lambda8p=lam8p, q_gamma2=q_gamma2, q_gamma3=q_gamma3, q8p=q8p,
                                q_gamma=q_gamma, q_f=q_f, b_gamma=b_gamma, b_g=b_g, e_k=e_k, de_dgamma=de)


def mollified_barrier_value(g, c, params, eps_x):
    """e_k(c) * b(g) (mollifier.py:70-71)."""
    from .barrier import barrier_value

    return float(mollified_eigensystem_batch(g, c, eps_x, params)[0, 10]) * barrier_value(g, params)


def mollified_gradient(stencil, jac, params):
    """Stacked per-vertex gradient of the mollified barrier (mollifier.py:89-103)."""
    if StencilKind(stencil.kind.value) not in PARALLEL_KINDS:
        raise ValueError("mollified gradient applies to parallel stencils")
    return _blocks_from_jac(stencil, jac, params, parallel=True).grad


def build_mollified_local_quadratic(stencil, jac, params):
    """Gradient and PSD block of a parallel stencil (mollifier.py:191-210)."""
    if StencilKind(stencil.kind.value) not in PARALLEL_KINDS:
        raise ValueError("mollified block applies to parallel stencils")
    return _blocks_from_jac(stencil, jac, params, parallel=True)
