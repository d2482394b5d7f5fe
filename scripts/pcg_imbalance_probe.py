"""Scratch (B200IPC_PCG_TIMING build): per-CTA product time of pcg_stream_kernel -- is the imbalance systematic?"""
import sys
import numpy as np
sys.path.insert(0, ".")
exec(open("scripts/mas_probe.py").read().split("def wall")[0])
sysm.block_jacobi()
sysm.pcg(rhs, 1e-30, 5)
d, iters, ok, _, _ = sysm.pcg(rhs, 1e-30, 200)
ws = device.to_host(sysm._pcg_ws)
part = ws[21 * sysm.n:]
prod = part[1024:1024 + 148] / iters / 1e3
wait1 = part[1024 + 512:1024 + 512 + 148] / iters / 1e3
nchunks = (sysm.n + 26) // 27
mine = np.array([(nchunks - b + 147) // 148 for b in range(148)])
order = np.argsort(prod)
print("product us/iter per CTA: min %.1f  p25 %.1f  median %.1f  p75 %.1f  max %.1f" % tuple(np.percentile(prod, [0, 25, 50, 75, 100])))
print("fastest CTAs:", [(int(b), round(float(prod[b]), 1), int(mine[b])) for b in order[:8]])
print("slowest CTAs:", [(int(b), round(float(prod[b]), 1), int(mine[b])) for b in order[-8:]])
print("corr(product time, chunks owned) = %.2f" % np.corrcoef(prod, mine)[0, 1])
rowptr = device.to_host(sysm.rowptr)
blocks = np.array([sum(int(rowptr[min((b + 148 * k + 1) * 27, sysm.n)] - rowptr[min((b + 148 * k) * 27, sysm.n)]) for k in range(mine[b])) for b in range(148)])
print("corr(product time, blocks owned) = %.2f; blocks min/max %d/%d" % (np.corrcoef(prod, blocks)[0, 1], blocks.min(), blocks.max()))

smid = part[3600:3600 + 148].astype(int)
by_sm = sorted(zip(smid.tolist(), prod.tolist(), range(148)))
print("SM id -> product us (CTA):")
for k in range(0, 148, 8):
    print("  " + "  ".join(f"{sm:3d}:{t:5.1f}({b:3d})" for sm, t, b in by_sm[k:k + 8]))
