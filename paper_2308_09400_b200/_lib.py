"""ctypes binding of libb200ipc.so -- the C-ABI drop-in boundary (include/b200ipc.h).

There is no CPU fallback: importing this module without the built library raises, and
every entry point needs a CUDA device.
"""

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("B200IPC_LIB") or os.path.join(HERE, "libb200ipc.so")  # override: tuning builds only


class B200IpcError(RuntimeError):
    """Non-zero return code from a b200ipc_* entry point."""


class Params(C.Structure):
    """struct b200ipc_params."""

    _fields_ = [
        ("d_hat", C.c_double),
        ("d_hat_sq", C.c_double),
        ("d_hat_pow2", C.c_double),
        ("scale", C.c_double),
        ("eps_g", C.c_double),
        ("dt2", C.c_double),
        ("use_filter", C.c_int32),
        ("form", C.c_int32),
    ]


class PcgResult(C.Structure):
    """struct b200ipc_pcg_result."""

    _fields_ = [
        ("iters", C.c_int32),
        ("converged", C.c_int32),
        ("delta0", C.c_double),
        ("delta_new", C.c_double),
    ]


_vp, _i64, _i32, _dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double

# name -> argtypes; every function returns int unless listed in _RESTYPE
SIGNATURES = {
    "b200ipc_abi_version": [],
    "b200ipc_build_info": [],
    "b200ipc_launch_count": [],
    "b200ipc_gather_rows": [_i64, _i64, _vp, _vp, _vp, _vp],
    "b200ipc_fp64_probe": [C.POINTER(_dbl), _vp],
    "b200ipc_pt_classify": [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_ee_classify": [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_cross_sq": [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_matvec_blocks": [_i64, _i32, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_matvec_begin": [_i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_matvec_end": [_i64, _vp, _vp, _vp, _vp],
    "b200ipc_barrier_stencils": [C.POINTER(Params), _i64, _vp, _i64, C.POINTER(_i64), _vp, _vp, _vp,
                                 _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_barrier_stencils_ex": [C.POINTER(Params), _i64, _vp, _i64, C.POINTER(_i64), _vp, _vp, _vp,
                                    _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_barrier_stencils_layout": [C.POINTER(Params), _i64, _vp, _i64, C.POINTER(_i64), _vp, _vp, _vp,
                                        _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp],
    "b200ipc_reduce_energy": [_i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_diagonal_jacobian": [C.POINTER(Params), _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_blocks_from_jacobian": [C.POINTER(Params), _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_barrier_scalars": [C.POINTER(Params), _i64, _vp, _vp, _vp],
    "b200ipc_mollified_eigensystem": [C.POINTER(Params), _i64, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_narrow_phase": [_i64, _vp, _vp, _i64, _vp, _i64, _vp, _dbl, _i32, _vp, _vp, _vp, _vp, _vp, _vp,
                             C.POINTER(_i64), C.POINTER(_i64), _vp],
    "b200ipc_broad_create": [C.POINTER(_vp)],
    "b200ipc_broad_destroy": [_vp],
    "b200ipc_broad_set_grid_cells": [_vp, C.c_int32, C.c_int32, C.c_int32],
    "b200ipc_broad_set_coarse_cell": [_vp, _dbl],
    "b200ipc_broad_phase_count": [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _dbl, _dbl, C.POINTER(_dbl),
                                  C.POINTER(_i64), C.POINTER(_i64), _vp],
    "b200ipc_broad_phase_fill": [_vp, _vp, _vp, _vp],
    "b200ipc_sweep_candidates_count": [_vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _dbl, _dbl,
                                       C.POINTER(_dbl), C.POINTER(_i64), C.POINTER(_i64), _vp],
    "b200ipc_accd_max_step": [_i64, _vp, _vp, _i32, _vp, _vp, _dbl, _i32, _vp, _vp, _vp],
    "b200ipc_ccd_filter": [_i64, _vp, _i64, _vp, _vp, _vp, _dbl, _i32, _vp, _vp, _vp],
    "b200ipc_ccd_filter_swept": [_i64, _vp, _i64, _vp, _vp, _vp, _dbl, _dbl, _i32, _vp, _vp, _vp, _vp],
    "b200ipc_friction_state": [_i64, C.POINTER(_i64), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_friction_blocks": [_i64, C.POINTER(_i64), _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _vp, _vp, _vp, _vp, _vp,
                                _vp, _vp, _vp],
    "b200ipc_friction_explicit": [_i64, _i32, _vp, _vp, _vp, _dbl, _dbl, _dbl, _vp, _vp, _vp, _vp],
    "b200ipc_elastic_rest": [_i64, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_elastic_blocks": [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _i32, _vp, _vp, _vp, _vp],
    "b200ipc_assembly_create": [C.POINTER(_vp)],
    "b200ipc_assembly_destroy": [_vp],
    "b200ipc_assembly_set_variant": [_vp, _i32],
    "b200ipc_assembly_set_symbolic": [_vp, _i32],
    "b200ipc_assembly_set_layout": [_vp, C.c_uint32],
    "b200ipc_assembly_stats": [_vp, C.POINTER(_i64)],
    "b200ipc_assemble_symbolic": [_vp, _i64, _vp, _i32, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_vp),
                                  C.POINTER(_i64), _vp],
    "b200ipc_assembly_pattern": [_vp, _vp, _vp, _vp],
    "b200ipc_assemble_numeric": [_vp, _vp, C.POINTER(_vp), _vp, _vp],
    "b200ipc_assemble_numeric_factors": [_vp, _vp, C.POINTER(_vp), _vp, _vp],
    "b200ipc_scatter_gradient": [_vp, _vp, _vp, _vp, C.POINTER(_vp), _vp, _vp],
    "b200ipc_bsr_spmv": [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_block_jacobi": [_i64, _vp, _vp, _vp, _vp, _vp],
    "b200ipc_pcg_workspace_bytes": [_i64],
    "b200ipc_pcg": [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _i32, _vp, _i64, C.POINTER(PcgResult),
                    _vp],
    "b200ipc_mas_create": [C.POINTER(_vp)],
    "b200ipc_mas_destroy": [_vp],
    "b200ipc_mas_order": [_vp, _i64, _vp, _vp],
    "b200ipc_mas_get_order": [_vp, _vp, _vp],
    "b200ipc_mas_setup": [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _i32, _vp],
    "b200ipc_mas_apply": [_vp, _vp, _vp, _vp],
    "b200ipc_pcg_mas_workspace_bytes": [_i64],
    "b200ipc_pcg_mas": [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _i32, _vp, _i64,
                        C.POINTER(PcgResult), _vp],
}
_RESTYPE = {"b200ipc_build_info": C.c_char_p, "b200ipc_launch_count": _i64,
            "b200ipc_pcg_workspace_bytes": _i64, "b200ipc_pcg_mas_workspace_bytes": _i64}

_lib = None


def lib():
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise B200IpcError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2308_09400_b200._build` "
                "(there is no CPU fallback)"
            )
        handle = C.CDLL(LIB_PATH)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(handle, name)  # AttributeError if the header and the library disagree
            fn.argtypes = argtypes
            fn.restype = _RESTYPE.get(name, C.c_int)
        _lib = handle
    return _lib


def check(rc, what):
    if rc != 0:
        if rc < 0:
            raise B200IpcError(f"{what}: CUDA error {-rc}")
        raise B200IpcError(f"{what}: argument/state error {rc}")
