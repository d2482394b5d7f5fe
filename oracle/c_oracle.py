"""ctypes wrapper of oracle/_build/liboracle_c.so (the plain-C restatement, oracle_c.c).

TEST / BASELINE INFRASTRUCTURE ONLY -- see oracle/tetipc_oracle.py.  Built by ``make -C oracle``
(``__graft_entry__.build()`` runs it).  ``reference_core()`` returns the reference's own compiled
kernel module from oracle/_ref/ (binary built from /root/reference by oracle/build_ref.sh) or None.
"""

import ctypes as C
import importlib.util
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle_c.so")


class Params(C.Structure):
    _fields_ = [("d_hat", C.c_double), ("d_hat_sq", C.c_double), ("d_hat_pow2", C.c_double), ("scale", C.c_double),
                ("eps_g", C.c_double), ("dt2", C.c_double), ("use_filter", C.c_int32), ("form", C.c_int32)]


_lib = None


def available():
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB)
        _lib.oracle_barrier_stencils.restype = C.c_int
        _lib.oracle_num_threads.restype = C.c_int
    return _lib


def set_threads(n):
    lib().oracle_set_threads(C.c_int(int(n)))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def make_params(d_hat, kappa, d_thr_ratio=0.1, use_filter=True, form="qlog", dt=1.0):
    return Params(d_hat, d_hat * d_hat, d_hat**2, kappa * d_hat**4, d_thr_ratio * d_thr_ratio, dt**2,
                  1 if use_filter else 0, 0 if form == "qlog" else 1)


def classify(op, a, b, c, d):
    pts = [np.ascontiguousarray(np.atleast_2d(v), dtype=np.float64) for v in (a, b, c, d)]
    n = pts[0].shape[0]
    codes, d2 = np.empty(n, np.int64), np.empty(n)
    grad, w = np.empty((n, 4, 3)), np.empty((n, 2))
    fn = lib().oracle_pt_classify if op == "pt" else lib().oracle_ee_classify
    fn(C.c_int64(n), *[_p(v) for v in pts], _p(codes), _p(d2), _p(grad), _p(w))
    return codes, d2, grad, w


def family_counts(kind_off):
    n2 = int(kind_off[5] - kind_off[4])
    n3 = int(kind_off[3] - kind_off[2])
    n4 = int(kind_off[7] - kind_off[0]) - n2 - n3
    return n2, n3, n4


def barrier_stencils(prm, positions, kind_off, verts, sub, eps_x, out=None, want_blocks=True):
    """Same contract as b200ipc_barrier_stencils on host arrays. Returns a dict of outputs."""
    positions = np.ascontiguousarray(positions, dtype=np.float64)
    verts = np.ascontiguousarray(verts, dtype=np.int32)
    sub = np.ascontiguousarray(sub, dtype=np.uint8)
    eps_x = np.ascontiguousarray(eps_x, dtype=np.float64)
    koff = np.ascontiguousarray(kind_off, dtype=np.int64)
    n = int(koff[7])
    if out is None:
        n2, n3, n4 = family_counts(koff)
        out = {"energy": np.empty(n), "status": np.empty(n, np.uint8)}
        if want_blocks:
            out.update(grad2=np.empty((n2, 6)), hess2=np.empty((n2, 6, 6)), grad3=np.empty((n3, 9)),
                       hess3=np.empty((n3, 9, 9)), grad4=np.empty((n4, 12)), hess4=np.empty((n4, 12, 12)))
    lib().oracle_barrier_stencils(C.byref(prm), _p(positions), C.c_int64(n), _p(koff), _p(verts), _p(sub), _p(eps_x),
                                  _p(out["energy"]), _p(out["status"]), _p(out.get("grad2")), _p(out.get("hess2")),
                                  _p(out.get("grad3")), _p(out.get("hess3")), _p(out.get("grad4")),
                                  _p(out.get("hess4")))
    return out


def matvec_blocks(hess, vids, x, out):
    hess = np.ascontiguousarray(hess, dtype=np.float64)
    vids = np.ascontiguousarray(vids, dtype=np.int64)
    lib().oracle_matvec_blocks(C.c_int64(hess.shape[0]), C.c_int32(vids.shape[1]), _p(hess), _p(vids), _p(x), _p(out))


def reference_core():
    """The reference's own compiled kernels (oracle/_ref/_core*.so), or None if not built."""
    ref_dir = os.path.join(HERE, "_ref")
    if not os.path.isdir(ref_dir):
        return None
    for f in os.listdir(ref_dir):
        if f.startswith("_core") and f.endswith(".so"):
            spec = importlib.util.spec_from_file_location("_core", os.path.join(ref_dir, f))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    return None
