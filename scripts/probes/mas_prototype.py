"""CPU prototype of the multilevel additive Schwarz preconditioner on the bench matrix (cloth stack 4x140x140):
iteration counts of block-Jacobi PCG vs MAS variants, before any CUDA is written.  scipy only; not product."""
import os, sys, time
import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench
from oracle import c_oracle, tetipc_oracle as o
from paper_2308_09400_b200 import workloads

def build(scene):
    cache = f"/tmp/mas_{scene.name}.npz"
    if os.path.exists(cache):
        z = np.load(cache)
        return sp.csr_matrix((z["data"], z["indices"], z["indptr"])), z["rhs"]
    tab = bench.host_scene_table(scene)
    koff = np.searchsorted(tab["kind"], np.arange(8)).astype(np.int64)
    prm = c_oracle.make_params(scene.d_hat, scene.kappa, dt=scene.dt)
    out = c_oracle.barrier_stencils(prm, scene.positions, koff, tab["verts"], tab["sub"], tab["eps_x"])
    verts = tab["verts"]
    fam_rows = {2: np.arange(koff[4], koff[5]), 3: np.arange(koff[2], koff[3]),
                4: np.concatenate([np.arange(koff[k], koff[k + 1]) for k in (0, 1, 3, 5, 6)])}
    n = scene.masses.shape[0]
    rows, cols, vals = [], [], []
    g = np.zeros(3 * n)
    for s_ in (2, 3, 4):
        r_ = fam_rows[s_]
        if not len(r_): continue
        vids = verts[r_, :s_].astype(np.int64)
        idx = (3 * vids[:, :, None] + np.arange(3)[None, None]).reshape(len(r_), 3 * s_)
        rows.append(np.repeat(idx, 3 * s_, axis=1).reshape(-1)); cols.append(np.tile(idx, (1, 3 * s_)).reshape(-1))
        vals.append(out[f"hess{s_}"].reshape(-1))
        np.add.at(g, idx.reshape(-1), out[f"grad{s_}"].reshape(-1))
    rows.append(np.arange(3 * n)); cols.append(np.arange(3 * n)); vals.append(np.repeat(scene.masses, 3))
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(3 * n, 3 * n)).tocsr()
    fixed = np.asarray(scene.fixed, bool)
    keep = np.repeat(~fixed, 3).astype(float)
    D = sp.diags(keep)
    A = (D @ A @ D + sp.diags(1.0 - keep)).tocsr()
    x_tilde = scene.positions + 1e-4 * np.random.default_rng(1).normal(size=scene.positions.shape)
    g += (scene.masses[:, None] * (scene.positions - x_tilde)).reshape(-1)
    rhs = -g * keep
    np.savez(cache, data=A.data, indices=A.indices, indptr=A.indptr, rhs=rhs)
    return A, rhs

def pcg(A, rhs, prec, stop_prec, tol=1e-4, cap=2000):
    """PCG with preconditioner `prec`; stops on the REFERENCE's rule measured with `stop_prec` (block-Jacobi)."""
    d = np.zeros_like(rhs); r = rhs.copy(); s = prec(r)
    delta = r @ s
    ref0 = r @ stop_prec(r)
    c = s.copy(); it = 0
    while it < cap and r @ stop_prec(r) > tol * ref0:
        q = A @ c; den = c @ q
        if den <= 0: break
        a = delta / den; d += a * c; r -= a * q; s = prec(r)
        dn = r @ s; c = s + (dn / delta) * c; delta = dn; it += 1
    return d, it

def block_jacobi(A):
    n = A.shape[0] // 3
    B = sp.bsr_matrix(A, blocksize=(3, 3))
    diag = np.zeros((n, 3, 3))
    for i in range(n):
        pass
    # diagonal blocks
    Bc = B.tocsr()
    idx = np.arange(n)
    for a in range(3):
        for b in range(3):
            diag[:, a, b] = np.asarray(Bc[3 * idx + a, 3 * idx + b]).reshape(-1)
    pinv = np.linalg.inv(diag)
    return lambda r: np.einsum("nij,nj->ni", pinv, r.reshape(n, 3)).reshape(-1)

def morton(pos, bits=10):
    lo, hi = pos.min(0), pos.max(0)
    q = ((pos - lo) / np.maximum(hi - lo, 1e-300) * ((1 << bits) - 1)).astype(np.uint64)
    def spread(v):
        out = np.zeros_like(v)
        for b in range(bits):
            out |= ((v >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b)
        return out
    return spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))

def mas(A, order, levels, group=32, ratio=32):
    """Additive multilevel Schwarz: level l nodes = runs of ratio**l fine nodes (in `order`), domains = `group`
    consecutive level-l nodes; M^-1 = sum_l P_l blockdiag(inv(P_l^T A P_l restricted to domains)) P_l^T."""
    n = A.shape[0] // 3
    rank = np.empty(n, np.int64); rank[order] = np.arange(n)
    ops = []
    for l in range(levels):
        node = rank // (ratio ** l)            # level-l node of each fine vertex
        nn = int(node.max()) + 1
        P = sp.csr_matrix((np.ones(3 * n), ((3 * np.arange(n)[:, None] + np.arange(3)).reshape(-1),
                                            (3 * node[:, None] + np.arange(3)).reshape(-1))), shape=(3 * n, 3 * nn))
        Ac = (P.T @ A @ P).tocsr()
        nd = (nn + group - 1) // group
        inv = []
        for d_ in range(nd):
            a0, a1 = 3 * group * d_, min(3 * group * (d_ + 1), 3 * nn)
            inv.append(np.linalg.inv(Ac[a0:a1, a0:a1].toarray()))
        ops.append((P, sp.block_diag(inv).tocsr()))
        if nd == 1: break
    def apply(r):
        z = np.zeros_like(r)
        for P, Dinv in ops:
            z += P @ (Dinv @ (P.T @ r))
        return z
    return apply, len(ops)

if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "stack"
    scene = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2) if which == "stack" else workloads.cloth_on_sphere()
    t0 = time.time(); A, rhs = build(scene); print("built", A.shape, A.nnz, f"{time.time()-t0:.1f}s")
    n = A.shape[0] // 3
    bj = block_jacobi(A)
    t0 = time.time(); d, it = pcg(A, rhs, bj, bj); print("block-jacobi iters", it, f"{time.time()-t0:.1f}s")
    orders = {"index": np.arange(n), "morton": np.argsort(morton(scene.positions), kind="stable")}
    for name, order in orders.items():
        for levels in (1, 2, 3, 4):
            apply, nl = mas(A, order, levels)
            d2, it2 = pcg(A, rhs, apply, bj)
            print(f"MAS order={name} levels={nl}: iters {it2}  |d-d_bj|/|d| = {np.linalg.norm(d2-d)/np.linalg.norm(d):.2e}", flush=True)
