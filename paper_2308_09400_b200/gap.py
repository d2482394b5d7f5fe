"""Diagonal constraint Jacobian with the reference's signatures (gap.py:23-88), evaluated by
``b200ipc_diagonal_jacobian``; ``stencil_distance`` / ``parallel_measure`` are views of the
same kernel's outputs (proximity.py:183-229)."""

from dataclasses import dataclass

import numpy as np

from . import _lib, device
from .barrier import BarrierParams, c_params
from .proximity import (IS_PARALLEL, KIND_SIZE, SIMPLEX_DIM, DistanceResult, StencilKind, StencilTable)


class GapError(ValueError):
    pass


class BarrierInactiveError(GapError):
    """Distance at or beyond d_hat: the stencil should have been culled."""


class InterpenetrationError(GapError):
    """Zero or negative squared distance: the state is already invalid."""


@dataclass
class DiagonalJacobian:
    m: int
    f: float
    grad_f: np.ndarray
    sqrt_c: float = None
    grad_sqrt_c: np.ndarray = None


@dataclass
class GapValue:
    g: float
    gamma: float = None


def diagonal_jacobian_batch(table, positions, d_hat):
    """All Jacobian quantities for every table row, as host arrays padded to four vertex rows.

    Returns dict(d2, grad_d2 (n,4,3), witness (n,2), f, grad_f (n,4,3), c, grad_c, sqrt_c,
    grad_sqrt_c, status).  Parallel-only outputs are NaN on other rows.
    """
    n = len(table)
    pos = device.to_device(positions, np.float64)
    prm = c_params(BarrierParams(d_hat=d_hat, kappa=1.0))
    names = ("d2", "grad_d2", "witness", "f", "grad_f", "c", "grad_c", "sqrt_c", "grad_sqrt_c")
    shapes = {"d2": (n,), "grad_d2": (n, 4, 3), "witness": (n, 2), "f": (n,), "grad_f": (n, 4, 3), "c": (n,),
              "grad_c": (n, 4, 3), "sqrt_c": (n,), "grad_sqrt_c": (n, 4, 3)}
    t = device.torch()
    bufs = {k: t.full(shapes[k], float("nan"), dtype=t.float64, device="cuda") for k in names}
    status = device.empty((n,), np.uint8)
    d_kind, d_verts, d_sub = (device.to_device(table.kind), device.to_device(table.verts),
                              device.to_device(table.sub))  # named: temporaries would alias before the launch
    _lib.check(_lib.lib().b200ipc_diagonal_jacobian(
        prm, pos.shape[0], device.ptr(pos), n, device.ptr(d_kind), device.ptr(d_verts), device.ptr(d_sub),
        *[device.ptr(bufs[k]) for k in names], device.ptr(status), device.stream()), "diagonal_jacobian")
    out = {k: device.to_host(v) for k, v in bufs.items()}
    out["status"] = device.to_host(status)
    return out


def _single(stencil, positions, d_hat):
    table = StencilTable.from_stencils([stencil])
    out = diagonal_jacobian_batch(table, np.asarray(positions, dtype=np.float64), d_hat)
    code = int(table.kind[0])
    return code, {k: v[0] for k, v in out.items()}


def stencil_distance(stencil, positions):
    """Exact pair distance of one stencil (proximity.py:183-222)."""
    code, r = _single(stencil, positions, 1.0)
    rows = 4 if IS_PARALLEL[code] else int(KIND_SIZE[code])
    kind = StencilKind(stencil.kind.value)
    if kind in (StencilKind.POINT_POINT, StencilKind.POINT_POINT_PARALLEL):
        wit = np.zeros(0)
    elif kind in (StencilKind.POINT_EDGE, StencilKind.POINT_EDGE_PARALLEL):
        wit = r["witness"][:1].copy()
    else:
        wit = r["witness"].copy()
    return DistanceResult(d2=float(r["d2"]), grad_d2=r["grad_d2"][:rows].copy(), witness=wit)


def parallel_measure(stencil, positions):
    """Parallelness measure c and its gradient (proximity.py:225-229)."""
    code, r = _single(stencil, positions, 1.0)
    if not IS_PARALLEL[code]:
        raise ValueError("parallel_measure applies to parallel stencils")
    return float(r["c"]), r["grad_c"].copy()


def build_diagonal_jacobian(stencil, positions, d_hat, dist=None):
    """f, sqrt(c) and their gradients for an active stencil (gap.py:56-82).

    ``dist`` is accepted for signature compatibility; the kernel always re-evaluates it.
    """
    code, r = _single(stencil, positions, d_hat)
    if r["status"] == 2:
        raise InterpenetrationError(f"nonpositive squared distance on stencil {stencil.verts}")
    if r["status"] == 1:
        raise BarrierInactiveError(f"stencil {stencil.verts} is farther than d_hat")
    rows = 4 if IS_PARALLEL[code] else int(KIND_SIZE[code])
    sqrt_c = grad_sqrt_c = None
    if IS_PARALLEL[code]:
        sqrt_c, grad_sqrt_c = float(r["sqrt_c"]), r["grad_sqrt_c"].copy()
    return DiagonalJacobian(m=SIMPLEX_DIM[StencilKind(stencil.kind.value)], f=float(r["f"]),
                            grad_f=r["grad_f"][:rows].copy(), sqrt_c=sqrt_c, grad_sqrt_c=grad_sqrt_c)


def gap_function(jac):
    """g = f^2, gamma = c when present (gap.py:85-88)."""
    gamma = None if jac.sqrt_c is None else jac.sqrt_c * jac.sqrt_c
    return GapValue(g=jac.f * jac.f, gamma=gamma)
