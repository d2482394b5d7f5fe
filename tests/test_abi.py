"""The C-ABI library loads on a CPU-only box and exports every symbol include/b200ipc.h declares
(no compute calls without a GPU)."""

import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "b200ipc.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(?:int|int64_t|const char\*)\s+(b200ipc_\w+)\s*\(([^;]*?)\)\s*;", text, flags=re.S):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    return out


def test_header_declares_the_expected_surface():
    fns = declared_functions()
    for name in ("b200ipc_pt_classify", "b200ipc_ee_classify", "b200ipc_cross_sq", "b200ipc_matvec_blocks",
                 "b200ipc_barrier_stencils", "b200ipc_reduce_energy", "b200ipc_narrow_phase",
                 "b200ipc_assemble_symbolic", "b200ipc_assemble_numeric", "b200ipc_scatter_gradient",
                 "b200ipc_bsr_spmv", "b200ipc_block_jacobi", "b200ipc_pcg", "b200ipc_diagonal_jacobian",
                 "b200ipc_blocks_from_jacobian", "b200ipc_barrier_scalars", "b200ipc_mollified_eigensystem"):
        assert name in fns, name


def test_library_exports_every_declared_symbol():
    from paper_2308_09400_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libb200ipc.so is not built: run `python -m paper_2308_09400_b200._build`")
    handle = _lib.lib()
    fns = declared_functions()
    assert len(fns) >= 25
    for name, nargs in fns.items():
        assert hasattr(handle, name), f"{name} declared in b200ipc.h but not exported"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
        assert len(_lib.SIGNATURES[name]) == nargs, f"{name}: header has {nargs} parameters"
    for name in _lib.SIGNATURES:
        assert name in fns, f"{name} bound in _lib.py but not declared in b200ipc.h"
    assert handle.b200ipc_abi_version() == 1
    assert b"sm_100a" in handle.b200ipc_build_info()
    assert handle.b200ipc_launch_count() >= 0


def test_broad_phase_handle_and_grid_hint_without_a_device():
    """Handle life cycle and the grid-cell hint are host-only calls: valid handle -> 0, NULL -> EINVAL."""
    import ctypes as C

    from paper_2308_09400_b200 import _lib

    L = _lib.lib()
    h = C.c_void_p()
    assert L.b200ipc_broad_create(C.byref(h)) == 0 and h
    assert L.b200ipc_broad_set_grid_cells(h, 140, 140, 6) == 0
    assert L.b200ipc_broad_set_grid_cells(h, 0, -5, 1 << 30) == 0      # out-of-range hints fall back / clamp
    assert L.b200ipc_broad_set_grid_cells(None, 1, 1, 1) != 0
    assert L.b200ipc_broad_destroy(h) == 0


def test_struct_layouts_match_header():
    import ctypes as C

    from paper_2308_09400_b200 import _lib

    assert C.sizeof(_lib.Params) == 6 * 8 + 2 * 4
    assert C.sizeof(_lib.PcgResult) == 2 * 4 + 2 * 8
    from oracle import c_oracle

    assert C.sizeof(c_oracle.Params) == C.sizeof(_lib.Params)


def test_product_never_imports_the_oracle():
    """A product path routed through the oracle (or any CPU fallback) would void parity."""
    pkg = os.path.join(ROOT, "paper_2308_09400_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f
                assert "tetipc_oracle" not in src and "c_oracle" not in src, f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2308_09400_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(_lib.B200IpcError, match="no CPU fallback"):
        _lib.lib()
