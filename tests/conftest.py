"""Shared fixtures. GPU tests carry @pytest.mark.gpu and need a B200 + the built library."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run with -m gpu on the B200 box)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def rel_err(got, ref, floor=0.0):
    """max |got-ref| / max(|ref|, floor*max|ref|) over all entries."""
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    scale = np.maximum(np.abs(ref), floor * (np.abs(ref).max() if ref.size else 1.0))
    scale = np.where(scale == 0.0, 1.0, scale)
    return float(np.max(np.abs(got - ref) / scale)) if ref.size else 0.0


def block_rel_err(got, ref):
    """Per-entry error relative to each block's (row's) max-abs, as BASELINE.md states:
    entries that are analytically zero are measured against the block scale."""
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return 0.0
    n = ref.shape[0]
    scale = np.abs(ref.reshape(n, -1)).max(axis=1)
    scale = np.where(scale == 0.0, 1.0, scale).reshape((n,) + (1,) * (ref.ndim - 1))
    return float(np.max(np.abs(got - ref) / scale))


def row_rel_err(got, ref):
    """block_rel_err per row: (n,) array of max |got-ref| over the block / the block's max-abs."""
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    n = ref.shape[0]
    scale = np.abs(ref.reshape(n, -1)).max(axis=1)
    scale = np.where(scale == 0.0, 1.0, scale)
    return np.abs(got - ref).reshape(n, -1).max(axis=1) / scale


def entry_rel_err(got, ref, floor=1e-6):
    """True per-entry relative error: |got-ref| / |ref| for every entry with |ref| > floor * (its block's
    max-abs); entries below that (the analytically-zero ones and their round-off)
    are measured against floor * block max-abs, i.e. they must be < tol * floor of the block scale."""
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return 0.0
    n = ref.shape[0]
    top = np.abs(ref.reshape(n, -1)).max(axis=1)
    top = np.where(top == 0.0, 1.0, top).reshape((n,) + (1,) * (ref.ndim - 1))
    scale = np.maximum(np.abs(ref), floor * top)
    return float(np.max(np.abs(got - ref) / scale))
