"""Mollified near-parallel edge-edge entry points with the reference's signatures
(mollifier.py:55-144, :191-210), evaluated by ``b200ipc_mollified_eigensystem`` and
``b200ipc_blocks_from_jacobian``."""

from dataclasses import dataclass

import numpy as np

from . import _lib, device
from .barrier import _blocks_from_jac, c_params
from .proximity import PARALLEL_KINDS, StencilKind


@dataclass
class MollifiedEigenSystem:
    """Channel eigenvalues and the retained coupled pair (mollifier.py:35-52)."""

    lambda_gamma1: float
    lambda_g1: float
    t: float
    p: float
    lambda7p: float
    lambda8p: float
    q_gamma: float
    q_f: float
    b_gamma: float
    b_g: float
    e_k: float
    de_dgamma: float


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
    return MollifiedEigenSystem(*[float(v) for v in mollified_eigensystem_batch(g, c, eps_x, params)[0]])


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
