"""The streamed SpMV / PCG through the C ABI on synthetic BSR matrices that exercise its edges:
rows longer than a shared-memory stage (global fallback inside the same kernel), odd and even block
counts (end-of-array patches of the 16-byte-aligned bulk copies), row counts that are not multiples of
the chunk size, single-row and diagonal-only matrices, and chunk-size overrides."""

import ctypes as C
import os
import zlib

import numpy as np
import pytest

from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2308_09400_b200 import _lib, device

    return _lib, device


def random_bsr(rng, n, row_len, symmetric=False, heavy_rows=()):
    """Random block pattern with the diagonal always present; values O(1), diagonal dominant if symmetric."""
    cols = []
    for r in range(n):
        k = row_len(r)
        c = set(rng.integers(0, n, size=max(k - 1, 0)).tolist()) | {r}
        if r in heavy_rows:
            c |= set(range(min(n, heavy_rows[r])))
        cols.append(c)
    if symmetric:
        for r in range(n):
            for c in list(cols[r]):
                cols[c].add(r)
    rowptr = np.zeros(n + 1, np.int32)
    colidx, vals = [], []
    for r in range(n):
        cs = sorted(cols[r])
        rowptr[r + 1] = rowptr[r] + len(cs)
        colidx.extend(cs)
    colidx = np.asarray(colidx, np.int32)
    vals = rng.normal(size=(len(colidx), 3, 3)) * 0.1
    if symmetric:
        pos = {}
        rows = np.repeat(np.arange(n), np.diff(rowptr))
        for k, (r, c) in enumerate(zip(rows, colidx)):
            pos[(r, c)] = k
        for (r, c), k in pos.items():
            if r < c:
                vals[pos[(c, r)]] = vals[k].T
            elif r == c:
                deg = rowptr[r + 1] - rowptr[r]
                vals[k] = 0.5 * (vals[k] + vals[k].T) + (1.0 + 0.35 * deg) * np.eye(3)
    return rowptr, colidx, vals


def gpu_spmv(L, rowptr, colidx, vals, x):
    _lib, device = L
    n = len(rowptr) - 1
    d = [device.to_device(a) for a in (rowptr, colidx, vals, x)]
    y = device.empty((3 * n,))
    _lib.check(_lib.lib().b200ipc_bsr_spmv(n, len(colidx), *[device.ptr(t) for t in d], device.ptr(y), device.stream()),
               "bsr_spmv")
    return device.to_host(y)


CASES = [
    ("tiny-1-row", 1, lambda r: 1, {}),
    ("diag-only-odd", 33, lambda r: 1, {}),
    ("short-rows-even", 100, lambda r: 2, {}),
    ("ragged", 257, lambda r: 1 + (7 * r) % 23, {}),
    ("one-heavy-row", 900, lambda r: 5, {417: 900}),          # 900 blocks > one stage: global fallback for its chunk
    ("two-heavy-rows", 1500, lambda r: 9, {3: 1400, 1499: 700}),
    ("cloth-like", 4000, lambda r: 17 + (r % 5), {}),
]


@pytest.mark.parametrize("name,n,row_len,heavy", CASES, ids=[c[0] for c in CASES])
def test_streamed_spmv_matches_oracle(L, name, n, row_len, heavy):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    rowptr, colidx, vals = random_bsr(rng, n, row_len, heavy_rows=heavy)
    x = rng.normal(size=3 * n)
    ref = o.bsr_matvec(rowptr, colidx, vals, x)
    scale = np.abs(ref).max()
    for env in (None, "3", "12", "120"):            # default chunking and forced chunk sizes
        if env is None:
            os.environ.pop("B200IPC_SPMV_ROWS_PER_CHUNK", None)
        else:
            os.environ["B200IPC_SPMV_ROWS_PER_CHUNK"] = env
        got = gpu_spmv(L, rowptr, colidx, vals, x)
        assert np.abs(got - ref).max() <= 1e-12 * scale, (name, env)
    os.environ.pop("B200IPC_SPMV_ROWS_PER_CHUNK", None)
    os.environ["B200IPC_SPMV_MODE"] = "legacy"       # the direct-load kernels agree too
    try:
        got = gpu_spmv(L, rowptr, colidx, vals, x)
    finally:
        os.environ.pop("B200IPC_SPMV_MODE", None)
    assert np.abs(got - ref).max() <= 1e-12 * scale


@pytest.mark.parametrize("n,heavy", [(50, {}), (777, {}), (1200, {5: 1000})], ids=["small", "odd", "heavy-row"])
def test_streamed_pcg_on_synthetic_spd(L, n, heavy):
    _lib, device = L
    rng = np.random.default_rng(n)
    rowptr, colidx, vals = random_bsr(rng, n, lambda r: 6, symmetric=True, heavy_rows=heavy)
    nnzb = len(colidx)
    dense = np.zeros((3 * n, 3 * n))
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    for r, c, blk in zip(rows, colidx, vals):
        dense[3 * r:3 * r + 3, 3 * c:3 * c + 3] = blk
    assert np.allclose(dense, dense.T) and np.linalg.eigvalsh(dense).min() > 0
    rhs = rng.normal(size=3 * n)
    d_rowptr, d_colidx, d_vals = device.to_device(rowptr), device.to_device(colidx), device.to_device(vals)
    pinv = device.empty((n, 3, 3))
    _lib.check(_lib.lib().b200ipc_block_jacobi(n, device.ptr(d_rowptr), device.ptr(d_colidx), device.ptr(d_vals),
                                               device.ptr(pinv), device.stream()), "block_jacobi")
    fixed = device.to_device(np.zeros(n, np.uint8))
    nbytes = int(_lib.lib().b200ipc_pcg_workspace_bytes(n))
    ws = device.empty(((nbytes + 7) // 8,))
    d = device.empty((3 * n,))
    res = _lib.PcgResult()
    _lib.check(_lib.lib().b200ipc_pcg(n, nnzb, device.ptr(d_rowptr), device.ptr(d_colidx), device.ptr(d_vals),
                                      device.ptr(pinv), device.ptr(fixed), device.ptr(device.to_device(rhs)), device.ptr(d),
                                      1e-20, 500, device.ptr(ws), nbytes, C.byref(res), device.stream()), "pcg")
    sol = np.linalg.solve(dense, rhs)
    got = device.to_host(d)
    assert res.converged and res.iters > 3
    assert np.abs(got - sol).max() <= 1e-8 * np.abs(sol).max()
