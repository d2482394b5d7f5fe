"""Barrier parameters, block type and scalar entry points with the reference's signatures.

Mirrors ``/root/reference/pkg/src/tetipc/barrier.py:24-120,163-177``.  The scalar functions
broadcast over ``g`` like the reference's but evaluate on the GPU
(``b200ipc_barrier_scalars``); ``build_local_quadratic`` is the n = 1 view of the batched
block kernel.
"""

from dataclasses import dataclass

import numpy as np

from . import _lib, device
from .proximity import IS_PARALLEL, KIND_CODE, KIND_SIZE, PARALLEL_KINDS, StencilKind

FORM_QLOG = "qlog"
FORM_LOG = "log"


@dataclass
class BarrierParams:
    """Barrier stiffness and activation thresholds (barrier.py:24-53)."""

    d_hat: float
    kappa: float = 1e5
    d_thr_ratio: float = 0.1
    use_filter: bool = True
    form: str = FORM_QLOG

    def __post_init__(self):
        if not 0.0 < self.d_thr_ratio < 1.0:
            raise ValueError("d_thr_ratio must lie in (0, 1)")
        if self.d_hat <= 0.0 or self.kappa <= 0.0:
            raise ValueError("d_hat and kappa must be positive")
        if self.form not in (FORM_QLOG, FORM_LOG):
            raise ValueError(f"unknown barrier form {self.form!r}")

    @property
    def d_thr(self):
        return self.d_thr_ratio * self.d_hat

    @property
    def eps_g(self):
        return self.d_thr_ratio * self.d_thr_ratio


@dataclass
class LocalQuadratic:
    """Per-stencil PSD block with its gradient (barrier.py:63-73)."""

    vert_ids: np.ndarray
    grad: np.ndarray
    hess: np.ndarray


def c_params(params, dt=1.0):
    """``struct b200ipc_params`` with every derived constant evaluated the way the reference's
    Python expressions evaluate it (barrier.py:79, :51-53; gap.py:63; solver.py:134, :192)."""
    d_hat = float(params.d_hat)
    return _lib.Params(
        d_hat=d_hat,
        d_hat_sq=d_hat * d_hat,
        d_hat_pow2=d_hat**2,
        scale=float(params.kappa) * d_hat**4,
        eps_g=float(params.eps_g),
        dt2=float(dt) ** 2,
        use_filter=1 if params.use_filter else 0,
        form=0 if params.form == FORM_QLOG else 1,
    )


def _scalars(g, params):
    g_arr = np.asarray(g, dtype=np.float64)
    flat = np.ascontiguousarray(g_arr.reshape(-1))
    out = device.empty((flat.shape[0], 6))
    prm = c_params(params)
    d_g = device.to_device(flat)
    _lib.check(_lib.lib().b200ipc_barrier_scalars(prm, flat.shape[0], device.ptr(d_g), device.ptr(out),
                                                  device.stream()), "barrier_scalars")
    return device.to_host(out), g_arr.shape


def _col(g, params, k):
    out, shape = _scalars(g, params)
    res = out[:, k].reshape(shape)
    return res if res.ndim else np.float64(res)


def barrier_value(g, params):
    """b(g) (barrier.py:76-83)."""
    return _col(g, params, 0)


def barrier_dg(g, params):
    """b'(g) (barrier.py:86-92)."""
    return _col(g, params, 1)


def barrier_d2g(g, params):
    """b''(g) (barrier.py:95-101)."""
    return _col(g, params, 2)


def lambda1(g, params):
    """4 g b'' + 2 b' (barrier.py:104-106)."""
    return _col(g, params, 3)


def lambda23(g, params):
    """2 b' (barrier.py:109-111)."""
    return _col(g, params, 4)


def filtered_lambda1(g, params):
    """lambda1 frozen below eps_g (barrier.py:114-120)."""
    return _col(g, params, 5)


def _blocks_from_jac(stencil, jac, params, parallel):
    code = KIND_CODE[StencilKind(stencil.kind.value)]
    if bool(IS_PARALLEL[code]) != parallel:
        raise ValueError("parallel stencils take the mollified path" if not parallel
                         else "mollified block applies to parallel stencils")
    s = int(KIND_SIZE[code])
    gf = np.zeros((1, 12))
    gf[0, : 3 * s] = np.asarray(jac.grad_f, dtype=np.float64).reshape(-1)
    kind = device.to_device(np.array([code], np.uint8))
    f = device.to_device(np.array([jac.f], np.float64))
    sc = gsc = eps = None
    if parallel:
        sc = device.to_device(np.array([jac.sqrt_c], np.float64))
        gsc = device.to_device(np.asarray(jac.grad_sqrt_c, dtype=np.float64).reshape(1, 12))
        eps = device.to_device(np.array([stencil.eps_x], np.float64))
    grad, hess = device.empty((1, 12)), device.empty((1, 12, 12))
    prm = c_params(params)
    d_gf = device.to_device(gf)
    _lib.check(_lib.lib().b200ipc_blocks_from_jacobian(
        prm, 1, device.ptr(kind), device.ptr(f), device.ptr(d_gf), device.ptr(sc),
        device.ptr(gsc), device.ptr(eps), device.ptr(grad), device.ptr(hess), device.stream()),
        "blocks_from_jacobian")
    g, h = device.to_host(grad)[0, : 3 * s], device.to_host(hess)[0, : 3 * s, : 3 * s]
    return LocalQuadratic(vert_ids=np.asarray(stencil.verts, dtype=np.int64), grad=g.copy(), hess=h.copy())


def build_local_quadratic(stencil, jac, params):
    """Gradient and rank-1 PSD block of a non-parallel stencil (barrier.py:163-177)."""
    if StencilKind(stencil.kind.value) in PARALLEL_KINDS:
        raise ValueError("parallel stencils take the mollified path")
    return _blocks_from_jac(stencil, jac, params, parallel=False)
