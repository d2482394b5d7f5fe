import sys, numpy as np
sys.path.insert(0, ".")
from oracle import tetipc_oracle as o
from paper_2308_09400_b200 import device, solver
rng = np.random.default_rng(12345)
bad = 0
for case in range(150):
    n = int(rng.integers(2, 4000))
    fams = []
    for s in (2, 3, 4):
        if n < s: continue
        nb = int(rng.integers(0, 6 * n))
        if nb == 0: continue
        # clustered vertex choices so that rows get long / share many columns
        centre = rng.integers(0, n, size=nb)
        width = max(s, int(rng.integers(s, max(s + 1, n // int(rng.integers(1, 40)) + s))))
        vids = np.stack([(c + rng.choice(width, size=s, replace=False)) % n for c in centre]).astype(np.int64)
        # distinct vertices per block
        ok = np.array([len(set(v)) == s for v in vids])
        vids = vids[ok]
        if len(vids) == 0: continue
        z = rng.normal(size=(len(vids), 3 * s))
        fams.append((z[:, :, None] * z[:, None, :], vids))
    masses = rng.uniform(0.5, 2.0, size=n)
    fixed = rng.uniform(size=n) < rng.choice([0.0, 0.02, 0.3])
    res = {}
    for mode in (0, 1):
        sysm = solver.NewtonSystem(masses, fixed)
        sysm.set_symbolic_mode(mode)
        sysm.set_pattern([(v.shape[1], v) for _, v in fams])
        sysm.assemble([h for h, _ in fams])
        res[mode] = sysm.to_scipy_like() + (sysm.stats()["symbolic"], sysm.stats()["sources"])
        sysm.close()
    ra, ca, va, pa, sa = res[0]; rb, cb, vb, pb, sb = res[1]
    orow, ocol, oval = o.assemble_bsr(fams, masses, fixed)
    good = ((sa == sb or pa == 'sort') and np.array_equal(ra, rb) and np.array_equal(ca, cb) and np.array_equal(va, vb)
            and np.array_equal(ra, orow) and np.array_equal(ca, ocol)
            and np.abs(va - oval).max() <= 1e-12 * max(np.abs(oval).max(), 1.0))
    if not good:
        bad += 1
        print("MISMATCH case", case, n, [len(v) for _, v in fams], pa, "fixed", int(fixed.sum()))
        print("  rowptr rows==sort", np.array_equal(ra, rb), "colidx", np.array_equal(ca, cb), "vals bitwise", np.array_equal(va, vb))
        print("  rowptr rows==oracle", np.array_equal(ra, orow), "colidx", np.array_equal(ca, ocol), "nnzb", len(ca), len(cb), len(ocol))
        if va.shape == oval.shape:
            print("  max|va-oval|", np.abs(va - oval).max(), "scale", np.abs(oval).max(), " max|vb-oval|", np.abs(vb - oval).max())
        if va.shape == vb.shape and not np.array_equal(va, vb):
            d = np.abs(va - vb).reshape(len(va), -1).max(axis=1)
            blk = np.flatnonzero(d > 0)
            rows_of = np.searchsorted(ra, blk, side="right") - 1
            print("  differing blocks", len(blk), "first", blk[:5], "rows", rows_of[:5], "cols", ca[blk[:5]], "row lengths", np.diff(ra)[rows_of[:5]], "max diff", d.max())
print("cases 150, mismatches", bad)
