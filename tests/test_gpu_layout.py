"""Sub-block-major dense blocks -- the internal device layout (nb,s,s,3,3) between the stencil kernel and the
BSR assembly (include/b200ipc.h: b200ipc_barrier_stencils_layout, b200ipc_assembly_set_layout).  It must be the
reference's LocalQuadratic.hess (solver.py:202-209) in another order, bit for bit, and the matrix assembled from
it must be bitwise the matrix assembled from the reference layout, with both symbolic phases and both walkers,
also when only SOME families are sub-block-major (elastic / friction blocks stay row-major)."""

import numpy as np
import pytest

from oracle import tetipc_oracle as o

pytestmark = pytest.mark.gpu


def tile(h):
    """(nb,3s,3s) -> (nb,s,s,3,3)"""
    nb, d, _ = h.shape
    s = d // 3
    return np.ascontiguousarray(h.reshape(nb, s, 3, s, 3).transpose(0, 1, 3, 2, 4))


@pytest.mark.parametrize("config", ["mixed", "parallel"])
def test_stencil_kernel_layouts_hold_the_same_numbers(config):
    from paper_2308_09400_b200 import barrier, device, proximity, stencils, workloads

    qb = workloads.config1_batch(n_pt=3000, n_ee=3000) if config == "mixed" else workloads.config2_batch(n=5000)
    tab = o.narrow_phase(qb.positions, qb.rest_positions, qb.vt, qb.ee, qb.d_hat)
    table = proximity.StencilTable(tab["kind"], tab["verts"], tab["sub"], tab["eps_x"])
    params = barrier.BarrierParams(d_hat=qb.d_hat, kappa=qb.kappa)
    dense = stencils.evaluate(table, qb.positions, params, dt=0.01)
    tiled = stencils.evaluate(table, qb.positions, params, dt=0.01, hess_layout="subblock")
    assert set(dense.families) == set(tiled.families) and len(dense.families) >= 1
    for s, fam in tiled.families.items():
        assert fam.tiled and tuple(fam.hess.shape[1:]) == (s, s, 3, 3)
        ref = device.to_host(dense.families[s].hess)
        assert np.array_equal(device.to_host(fam.hess), tile(ref))
        assert np.array_equal(device.to_host(fam.dense_hess()), ref)
        assert np.array_equal(device.to_host(fam.grad), device.to_host(dense.families[s].grad))
    assert np.array_equal(device.to_host(tiled.energy), device.to_host(dense.energy))
    # the host-facing views are the reference's whatever the device layout
    for (ha, va), (hb, vb) in zip(dense.grouped(), tiled.grouped()):
        assert np.array_equal(device.to_host(ha), device.to_host(hb)) and np.array_equal(device.to_host(va), device.to_host(vb))
    qa, qt = dense.to_local_quadratics(), tiled.to_local_quadratics()
    assert len(qa) == len(qt) and all(np.array_equal(x.hess, y.hess) for x, y in zip(qa[:200], qt[:200]))
    # buffers of one layout are not silently reused for the other
    with pytest.raises(ValueError):
        stencils.evaluate(table, qb.positions, params, out=dense, hess_layout="subblock")
    with pytest.raises(ValueError):
        stencils.evaluate(table, qb.positions, params, hess_layout="rows")


def random_families(rng, n, counts):
    grouped = []
    for s, nb in counts:
        vids = np.stack([rng.choice(n, size=s, replace=False) for _ in range(nb)]).astype(np.int64)
        z = rng.normal(size=(nb, 3 * s))
        grouped.append((z[:, :, None] * z[:, None, :] + 0.01 * rng.normal(size=(nb, 3 * s, 3 * s)), vids))
    return grouped


@pytest.mark.parametrize("mode", [0, 1], ids=["rows", "sort"])
@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("flags", [(True, True, True), (False, True, False), (True, False, True)])
def test_assembly_is_bitwise_layout_independent(mode, variant, flags):
    from paper_2308_09400_b200 import device, solver

    rng = np.random.default_rng(7 + 10 * mode + variant)
    n = 1500
    grouped = random_families(rng, n, [(2, 2500), (3, 3000), (4, 8000)])
    masses = rng.uniform(0.5, 2.0, size=n)
    fixed = rng.uniform(size=n) < 0.05
    fams = [(v.shape[1], v) for _, v in grouped]

    ref = solver.NewtonSystem(masses, fixed)
    ref.set_symbolic_mode(mode)
    ref.set_numeric_variant(variant)
    ref.set_pattern(fams)
    vals_ref = device.to_host(ref.assemble([h for h, _ in grouped]))
    sysm = solver.NewtonSystem(masses, fixed)
    sysm.set_symbolic_mode(mode)
    sysm.set_numeric_variant(variant)
    sysm.set_pattern(fams, tiled=flags)
    vals = device.to_host(sysm.assemble([tile(h) if t else h for (h, _), t in zip(grouped, flags)]))
    assert np.array_equal(device.to_host(sysm.colidx), device.to_host(ref.colidx))
    assert np.array_equal(vals, vals_ref)
    # and against the oracle's dense assembly of the reference-layout blocks
    _, _, o_vals = o.assemble_bsr(grouped, masses, fixed)
    assert np.abs(vals - o_vals).max() <= 1e-12 * np.abs(o_vals).max()
    # the layout belongs to the pattern: going back to row-major needs no new handle
    sysm.set_pattern(fams)
    assert np.array_equal(device.to_host(sysm.assemble([h for h, _ in grouped])), vals_ref)
    # the row-wise numeric kernel reads whole rows of row-major blocks: typed error, not a wrong matrix
    sysm.set_pattern(fams, tiled=flags)
    sysm.set_numeric_variant(4)
    with pytest.raises(Exception):
        sysm.assemble([tile(h) if t else h for (h, _), t in zip(grouped, flags)])
    with pytest.raises(ValueError):
        sysm.set_pattern(fams, tiled=[True])
    ref.close()
    sysm.close()


def test_empty_family_keeps_the_flags_aligned():
    from paper_2308_09400_b200 import device, solver

    rng = np.random.default_rng(3)
    n = 400
    grouped = random_families(rng, n, [(2, 300), (4, 900)])
    masses = rng.uniform(0.5, 2.0, size=n)
    fixed = np.zeros(n, bool)
    fams = [(2, grouped[0][1]), (3, np.zeros((0, 3), np.int64)), (4, grouped[1][1])]
    sysm = solver.NewtonSystem(masses, fixed)
    sysm.set_pattern(fams, tiled=[False, True, True])          # the middle (empty) family is dropped
    vals = device.to_host(sysm.assemble([grouped[0][0], tile(grouped[1][0])]))
    ref = solver.NewtonSystem(masses, fixed)
    ref.set_pattern(fams)
    assert np.array_equal(vals, device.to_host(ref.assemble([grouped[0][0], grouped[1][0]])))
    sysm.close()
    ref.close()
