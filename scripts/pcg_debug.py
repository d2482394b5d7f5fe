"""Scratch: PCG on the golden scene in legacy / stream SpMV modes."""
import os, sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import load_golden
from paper_2308_09400_b200 import solver
z = load_golden("scene")
grouped = [(z[f"fam{s}_hess"], z[f"fam{s}_vids"]) for s in (2, 3, 4) if f"fam{s}_hess" in z]
rhs = -z["ref_gradient"]; a = z["ref_dense"]; n = z["masses"].shape[0]
r0 = rhs.copy(); r0.reshape(n, 3)[z["fixed"]] = 0.0
prec = lambda r: np.einsum("nij,nj->ni", z["ref_pinv"], r.reshape(n, 3)).reshape(-1)
delta0 = r0 @ prec(r0)
print("n", n, "ref iters", int(z["ref_pcg_iters"]), int(z["ref_pcg12_iters"]))
for mode in ("legacy", "stream"):
    os.environ["B200IPC_SPMV_MODE"] = mode
    for tol in (1e-4, 1e-12):
        for rep in range(2):
            d, iters, ok = solver.pcg_solve(grouped, z["masses"], z["fixed"], rhs, tol, 5000)
            res = r0 - a @ d
            ref = z["ref_pcg_d"] if tol == 1e-4 else z["ref_pcg12_d"]
            diff = d - ref
            print(mode, tol, "iters", iters, ok, "true crit", (res @ prec(res)) / delta0,
                  "energy diff rel", np.sqrt(diff @ a @ diff) / np.sqrt(ref @ a @ ref), flush=True)
