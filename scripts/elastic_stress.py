"""Scratch: 60 k random tets -- rest shapes from fat to sliver, deformations from mild to inverted, flattened,
nearly rank-one and rotated -- against the oracle's eigh projection (oracle.elastic_blocks, pinned to the reference)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import tetipc_oracle as o
from paper_2308_09400_b200 import device, elasticity
rng = np.random.default_rng(99)
nt = 60_000
rest = rng.normal(size=(nt, 4, 3))
rest[: nt // 4, 3] = rest[: nt // 4, :3].mean(axis=1) + 0.02 * rng.normal(size=(nt // 4, 3))     # slivers
F = np.tile(np.eye(3), (nt, 1, 1)) + rng.normal(size=(nt, 3, 3)) * rng.choice([0.01, 0.3, 1.0, 3.0], size=(nt, 1, 1))
q, _ = np.linalg.qr(rng.normal(size=(nt, 3, 3)))
kind = rng.integers(0, 5, size=nt)
F[kind == 1] *= -1.0                                   # inverted
F[kind == 2, :, 2] *= 1e-4                             # flattened
F[kind == 3] = (rng.normal(size=(int((kind == 3).sum()), 3, 1)) * rng.normal(size=(int((kind == 3).sum()), 1, 3))
                + 1e-6 * rng.normal(size=(int((kind == 3).sum()), 3, 3)))                       # nearly rank one
F = q @ F
x = np.einsum("tij,tvj->tvi", F, rest).reshape(-1, 3)
restf = rest.reshape(-1, 3)
tets = np.arange(4 * nt).reshape(nt, 4)
rest_inv, vols = o.elastic_rest(restf, tets)[:2]
good = np.abs(vols) > 1e-6
mu, lam = np.full(nt, 3.7e4), np.full(nt, 8.6e4)
e_ref, g_ref, h_ref = o.elastic_blocks(x, tets[good], rest_inv[good], vols[good], mu[good], lam[good])
mesh = elasticity.TetMesh(restf, tets[good], mu[good], lam[good])
energy, fam = mesh.evaluate(x)
h = device.to_host(fam.hess)
g = device.to_host(fam.grad)
scale = np.abs(h_ref).reshape(len(h), -1).max(axis=1)
err = np.abs(h - h_ref).reshape(len(h), -1).max(axis=1) / np.maximum(scale, 1e-300)
gs = np.maximum(np.abs(g_ref).max(axis=1), 1e-6 * np.abs(g_ref).max())
gerr = (np.abs(g - g_ref).max(axis=1) / gs)
print("tets", len(h), "hess err max %.3e  p99.9 %.3e   grad err max %.3e" % (err.max(), np.percentile(err, 99.9), gerr.max()))
w = np.flatnonzero(err > 1e-9)
print("rows over 1e-9:", len(w), "kinds", np.bincount(kind[good][w], minlength=5) if len(w) else "-")
ev = np.linalg.eigvalsh(0.5 * (h + np.swapaxes(h, 1, 2)))
# block = vol * G^T P G with P the projected F-space Hessian (elasticity.py:114-137): PSD for a positively oriented
# REST tet; the random rest shapes here are negatively oriented half of the time (mesh loading rejects those), and
# both the reference and this kernel then return the same negative-semidefinite block
pos = vols[good] > 0
rel_min = ev.min(axis=1) / np.maximum(scale, 1e-300)
rel_max = ev.max(axis=1) / np.maximum(scale, 1e-300)
print("positively oriented rest tets: %d, min eig / block scale worst %.3e;  negatively oriented: %d, max eig / block scale worst %.3e;  finite %s"
      % (int(pos.sum()), rel_min[pos].min(), int((~pos).sum()), rel_max[~pos].max(), bool(np.isfinite(h).all())))
