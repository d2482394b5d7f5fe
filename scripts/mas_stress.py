"""Scratch: randomised stress of the MAS-preconditioned PCG against dense solves (sizes around the domain and
coarse-domain boundaries, 0 - 30 % Dirichlet vertices, both level counts, Morton and index order)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import tetipc_oracle as o
from paper_2308_09400_b200 import device, solver
rng = np.random.default_rng(777)
sizes = [1, 2, 31, 32, 33, 63, 64, 65, 100, 1023, 1024, 1025, 1056, 1057, 2047, 2049, 3000]
bad = 0
for case, n in enumerate(sizes * 2):
    fams = []
    for s in (2, 3, 4):
        if n < s:
            continue
        nb = int(rng.integers(1, 4 * n + 2))
        centre = rng.integers(0, n, size=nb)
        width = max(s, min(n, int(rng.integers(s, 40))))
        vids = np.stack([(c + rng.choice(width, size=s, replace=False)) % n for c in centre]).astype(np.int64)
        vids = vids[np.array([len(set(v)) == s for v in vids])]
        if len(vids):
            z = rng.normal(size=(len(vids), 3 * s)) * rng.choice([1.0, 30.0])
            fams.append((z[:, :, None] * z[:, None, :], vids))
    masses = rng.uniform(0.5, 2.0, size=n)
    fixed = rng.uniform(size=n) < rng.choice([0.0, 0.05, 0.3])
    pos = rng.normal(size=(n, 3)) * np.array([1.0, 1.0, rng.choice([1.0, 1e-3])])
    a = o.assemble_dense(fams, masses, fixed)
    rhs = rng.normal(size=3 * n)
    b = rhs.copy(); b.reshape(n, 3)[fixed] = 0.0
    sol = np.linalg.solve(a, b)
    sysm = solver.NewtonSystem(masses, fixed)
    sysm.set_pattern([(v.shape[1], v) for _, v in fams])
    sysm.assemble([h for h, _ in fams])
    for order in ("morton", "index"):
        sysm.mas_order(pos if order == "morton" else None)
        for levels in (1, 2):
            d, iters, ok, d0, dn = sysm.pcg(rhs, 1e-22, 5000, preconditioner="mas", mas_levels=levels)
            d = device.to_host(d)
            err = np.abs(d - sol).max() / max(np.abs(sol).max(), 1e-300)
            zero_fixed = not d.reshape(n, 3)[fixed].any()
            if not (ok and err <= 1e-7 and zero_fixed):
                bad += 1
                print("FAIL n", n, order, "levels", levels, "ok", ok, "iters", iters, "err", err, "fixed zero", zero_fixed)
    sysm.close()
print("cases", 2 * len(sizes) * 4, "failures", bad)
