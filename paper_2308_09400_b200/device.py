"""Device-memory plumbing: torch owns HBM and streams, the kernels get raw pointers."""

import ctypes as C

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        if not _t.cuda.is_available():
            raise RuntimeError("paper_2308_09400_b200 needs a CUDA device (sm_100a); there is no CPU path")
        _torch = _t
    return _torch


_NP2T = None


def _dtype(np_dtype):
    global _NP2T
    t = torch()
    if _NP2T is None:
        _NP2T = {np.dtype(np.float64): t.float64, np.dtype(np.int64): t.int64, np.dtype(np.int32): t.int32,
                 np.dtype(np.uint8): t.uint8, np.dtype(np.bool_): t.bool}
    return _NP2T[np.dtype(np_dtype)]


def empty(shape, dtype=np.float64):
    return torch().empty(shape, dtype=_dtype(dtype), device="cuda")


def zeros(shape, dtype=np.float64):
    return torch().zeros(shape, dtype=_dtype(dtype), device="cuda")


def to_device(a, dtype=None):
    """Host array (or device tensor) -> contiguous device tensor of ``dtype``."""
    t = torch()
    if isinstance(a, t.Tensor):
        out = a if dtype is None else a.to(_dtype(dtype))
        return out.cuda().contiguous()
    arr = np.ascontiguousarray(a, dtype=dtype)
    if not arr.flags.writeable:
        arr = arr.copy()
    return t.from_numpy(arr).cuda()


def to_host(x):
    return x.detach().cpu().numpy()


def ptr(x):
    """Raw device pointer of a tensor (None -> NULL).

    The caller must keep ``x`` referenced until the kernel is launched: a temporary created
    inside the argument list can be recycled by the caching allocator for the next temporary.
    """
    return C.c_void_p(None) if x is None else C.c_void_p(x.data_ptr())


def stream():
    return C.c_void_p(torch().cuda.current_stream().cuda_stream)


def gather_rows(src, idx):
    """``src[idx]`` along dim 0 for a contiguous device tensor (rows of any width), by ``b200ipc_gather_rows``."""
    from . import _lib

    t = torch()
    src = src.contiguous()
    idx = idx.to(t.int64).contiguous()
    out = t.empty((idx.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    row_bytes = src.element_size() * (int(src.numel() // src.shape[0]) if src.shape[0] else 1)
    if row_bytes % 4 or idx.shape[0] == 0 or src.shape[0] == 0:
        return src.index_select(0, idx)          # byte-wide rows (the u8 columns): torch's 1-D path is fine there
    _lib.check(_lib.lib().b200ipc_gather_rows(idx.shape[0], row_bytes, ptr(src), ptr(idx), ptr(out), stream()),
               "gather_rows")
    return out
