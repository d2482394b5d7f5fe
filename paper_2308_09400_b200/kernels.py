"""``tetipc.kernels``-shaped backend running on the B200 (the reference's plugin seam).

Same names, arguments and return values as the reference's backend modules
(``/root/reference/pkg/src/tetipc/kernels/__init__.py:21-32``): host arrays in, fresh host
NumPy arrays out, ``matvec_blocks`` accumulating in place into ``out``.  Each call copies
its inputs to the GPU, runs the sm_100a kernel behind the C ABI (``include/b200ipc.h``) and
copies the results back.  The ``*_device`` variants take and return device tensors.

``accd_max_step`` is the n = 1 shim of the batched
``accd_max_step_device`` / ``contacts.global_ccd_filter``.
"""

import numpy as np

from . import _lib, device

BACKEND = "b200"

PAIR_PT = 0
PAIR_EE = 1
PAIR_PE = 2
PAIR_PP = 3


def _in4(a, b, c, d):
    arrs = [np.ascontiguousarray(np.atleast_2d(v), dtype=np.float64) for v in (a, b, c, d)]
    n = arrs[0].shape[0]
    for v in arrs:
        if v.shape != (n, 3):
            raise ValueError("expected four (n, 3) arrays")
    return n, [device.to_device(v) for v in arrs]


def classify_device(op, pts, want_grad=True):
    """Run pt/ee classify on four (n,3) device tensors -> (codes, d2, grad, w) tensors."""
    n = pts[0].shape[0]
    codes = device.empty((n,), np.int64)
    d2 = device.empty((n,))
    grad = device.empty((n, 4, 3)) if want_grad else None
    w = device.empty((n, 2))
    fn = _lib.lib().b200ipc_pt_classify if op == "pt" else _lib.lib().b200ipc_ee_classify
    _lib.check(fn(n, *[device.ptr(p) for p in pts], device.ptr(codes), device.ptr(d2), device.ptr(grad),
                  device.ptr(w), device.stream()), f"{op}_classify")
    return codes, d2, grad, w


def cross_sq_device(pts, want_grad=True):
    n = pts[0].shape[0]
    c = device.empty((n,))
    grad = device.empty((n, 4, 3)) if want_grad else None
    _lib.check(_lib.lib().b200ipc_cross_sq(n, *[device.ptr(p) for p in pts], device.ptr(c), device.ptr(grad),
                                           device.stream()), "cross_sq")
    return c, grad


def pt_classify_batch(p, t1, t2, t3):
    """Twin of kernels/_core.pyx:153-171: (codes i64, d2, grad (n,4,3), w (n,2))."""
    _, pts = _in4(p, t1, t2, t3)
    return tuple(device.to_host(t) for t in classify_device("pt", pts))


def ee_classify_batch(a1, a2, b1, b2):
    """Twin of kernels/_core.pyx:174-192: codes = 3*ra+rb, w = (s, t)."""
    _, pts = _in4(a1, a2, b1, b2)
    return tuple(device.to_host(t) for t in classify_device("ee", pts))


def cross_sq_batch(a1, a2, b1, b2):
    """Twin of kernels/_core.pyx:195-219: (c, grad (n,4,3))."""
    _, pts = _in4(a1, a2, b1, b2)
    return tuple(device.to_host(t) for t in cross_sq_device(pts))


def matvec_blocks_device(hess, vids, x, out):
    nb, s = vids.shape
    _lib.check(_lib.lib().b200ipc_matvec_blocks(nb, s, device.ptr(hess), device.ptr(vids), device.ptr(x),
                                                device.ptr(out), device.stream()), "matvec_blocks")


def matvec_blocks(hess, vids, x, out):
    """Twin of kernels/_core.pyx:222-247: ``out += scatter(H_b @ gather(x))`` in place."""
    hess = np.ascontiguousarray(hess, dtype=np.float64)
    vids = np.ascontiguousarray(vids, dtype=np.int64)
    if hess.shape[0] == 0:
        return
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.c_contiguous):
        raise ValueError("out must be a C-contiguous float64 array")  # _core.pyx:226 typed memoryview
    d_out = device.to_device(out)
    d_hess, d_vids, d_x = device.to_device(hess), device.to_device(vids), device.to_device(x, np.float64)
    matvec_blocks_device(d_hess, d_vids, d_x, d_out)
    out[...] = device.to_host(d_out).reshape(out.shape)


def accd_max_step_device(ids, pair_kind, positions, directions, slack, max_iter=512, want_status=True):
    """Batched ACCD: ids (n,4) int32 device tensor, pair_kind an int (uniform) or a (n,) uint8 tensor,
    positions / directions (N,3) device tensors -> (step (n,), status (n,) or None) device tensors."""
    n = int(ids.shape[0])
    step = device.empty((max(n, 1),))
    status = device.empty((max(n, 1),), np.uint8) if want_status else None
    uniform = isinstance(pair_kind, (int, np.integer))
    kinds = None if uniform else pair_kind
    _lib.check(_lib.lib().b200ipc_accd_max_step(n, device.ptr(ids), device.ptr(kinds), int(pair_kind) if uniform else 0,
                                                device.ptr(positions), device.ptr(directions), float(slack),
                                                int(max_iter), device.ptr(step), device.ptr(status), device.stream()),
               "accd_max_step")
    return step[:n], None if status is None else status[:n]


def accd_max_step(x, dx, pair_kind, slack, max_iter=512):
    """Twin of kernels/_core.pyx:272-325: x, dx (s,3) of ONE pair -> step fraction (float)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    dx = np.ascontiguousarray(dx, dtype=np.float64)
    s = x.shape[0]
    ids = np.full((1, 4), 0, np.int32)
    ids[0, :s] = np.arange(s)
    step, status = accd_max_step_device(device.to_device(ids), int(pair_kind), device.to_device(x),
                                        device.to_device(dx), slack, max_iter)
    if int(device.to_host(status)[0]) != 0:
        raise ValueError("additive CCD requires a strictly positive initial distance")  # _core.pyx:307-308
    return float(device.to_host(step)[0])


def get_backend(name):
    if name == "b200":
        import sys

        return sys.modules[__name__]
    raise ValueError(f"unknown kernel backend {name!r}")
