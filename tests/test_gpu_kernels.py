"""GPU parity: tetipc.kernels twins (pt/ee classify, cross_sq, matvec_blocks) through the C ABI.

Bit-exact against the reference's compiled backend (golden, frozen from the real `_core`) and
against the oracle on fresh seeded inputs.
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2308_09400_b200 import kernels

    return kernels


def test_backend_name(K):
    assert K.BACKEND == "b200"
    assert (K.PAIR_PT, K.PAIR_EE, K.PAIR_PE, K.PAIR_PP) == (0, 1, 2, 3)


def test_classify_golden_bit_exact(K):
    z = load_golden("classify")
    pts = [z[f"in{j}"] for j in range(4)]
    for name, fn in (("pt", K.pt_classify_batch), ("ee", K.ee_classify_batch)):
        codes, d2, grad, w = fn(*pts)
        assert codes.dtype == np.int64 and grad.shape == (pts[0].shape[0], 4, 3) and w.shape[1] == 2
        np.testing.assert_array_equal(codes, z[f"{name}_core_codes"])
        np.testing.assert_array_equal(d2, z[f"{name}_core_d2"])
        np.testing.assert_array_equal(grad, z[f"{name}_core_grad"])
        np.testing.assert_array_equal(w, z[f"{name}_core_w"])
    c, g = K.cross_sq_batch(*pts)
    np.testing.assert_array_equal(c, z["cs_core_c"])
    np.testing.assert_array_equal(g, z["cs_core_grad"])


@pytest.mark.parametrize("n", [1, 127, 128, 129, 100003])
def test_classify_random_vs_oracle_bit_exact(K, n):
    rng = np.random.default_rng(n)
    pts = [rng.normal(size=(n, 3)) for _ in range(4)]
    for gpu, ref in ((K.pt_classify_batch, o.pt_classify_batch), (K.ee_classify_batch, o.ee_classify_batch)):
        got, exp = gpu(*pts), ref(*pts)
        for a, b in zip(got, exp):
            np.testing.assert_array_equal(a, b)
    got, exp = K.cross_sq_batch(*pts), o.cross_sq_batch(*pts)
    np.testing.assert_array_equal(got[0], exp[0])
    np.testing.assert_array_equal(got[1], exp[1])


def test_classify_empty_and_shape_errors(K):
    e = np.zeros((0, 3))
    codes, d2, grad, w = K.pt_classify_batch(e, e, e, e)
    assert codes.shape == (0,) and grad.shape == (0, 4, 3)
    with pytest.raises(ValueError):
        K.ee_classify_batch(np.zeros((2, 3)), np.zeros((3, 3)), np.zeros((2, 3)), np.zeros((2, 3)))
    # 1-D inputs are promoted like np.atleast_2d in the reference
    p = np.array([0.1, 0.05, 0.5])
    codes, d2, _, _ = K.pt_classify_batch(p, [1, 0, 0], [-1, 1, 0], [-1, -1, 0])
    assert codes[0] == 0 and d2[0] == pytest.approx(0.25)


def test_degenerate_parallel_edges(K):
    """Exactly parallel segments: denom == 0 branch of _ee_one, c == 0."""
    from paper_2308_09400_b200 import workloads as wl

    rng = np.random.default_rng(4)
    x = wl.gen_exact_parallel_edge_edge(rng, 64, rng.integers(13, 58, 64))
    pts = [x[:, j] for j in range(4)]
    got, exp = K.ee_classify_batch(*pts), o.ee_classify_batch(*pts)
    for a, b in zip(got, exp):
        np.testing.assert_array_equal(a, b)
    c, _ = K.cross_sq_batch(*pts)
    assert np.all(c == 0.0)


@pytest.mark.parametrize("s", [2, 3, 4])
def test_matvec_blocks_parity(K, rng, s):
    """test_kernels.py:42-54 of the reference, against the oracle (serial order) to 1e-13."""
    nb, n = 40, 30
    hess = rng.normal(size=(nb, 3 * s, 3 * s))
    hess = hess + hess.transpose(0, 2, 1)
    vids = np.stack([rng.choice(n, size=s, replace=False) for _ in range(nb)]).astype(np.int64)
    x = rng.normal(size=3 * n)
    out_a = rng.normal(size=3 * n)
    out_b = out_a.copy()
    K.matvec_blocks(hess, vids, x, out_a)
    o.matvec_blocks(hess, vids, x, out_b)
    np.testing.assert_allclose(out_a, out_b, rtol=1e-12, atol=1e-12)


def test_matvec_blocks_golden_and_large(K, rng):
    z = load_golden("classify")
    out = np.zeros(90)
    K.matvec_blocks(z["mv_hess"], z["mv_vids"], z["mv_x"], out)
    np.testing.assert_allclose(out, z["mv_core_out"], rtol=1e-12, atol=1e-12)
    nb, n = 50000, 20000
    hess = rng.normal(size=(nb, 12, 12))
    vids = rng.integers(0, n, size=(nb, 4)).astype(np.int64)
    x = rng.normal(size=3 * n)
    a, b = np.zeros(3 * n), np.zeros(3 * n)
    K.matvec_blocks(hess, vids, x, a)
    o.matvec_blocks(hess, vids, x, b)
    assert np.max(np.abs(a - b)) <= 1e-11 * np.max(np.abs(b))
    K.matvec_blocks(np.zeros((0, 12, 12)), np.zeros((0, 4), np.int64), x, a)  # empty family: no-op
