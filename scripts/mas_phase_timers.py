"""Scratch: per-phase timers of pcg_mas_kernel and pcg_stream_kernel (library built with B200IPC_PCG_TIMING=1)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
exec(open("scripts/mas_probe.py").read().split("def wall")[0])
import torch
sysm.mas_order(pos); sysm.mas_setup(1); sysm._mas_stale = False
names = ("product+blocksum", "sync1+sumparts", "update+blocksum", "sync2+sumparts")
for prec in ("mas", "block_jacobi"):
    sysm.pcg(rhs, 1e-30, 5, preconditioner=prec)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d, iters, ok, _, _ = sysm.pcg(rhs, 1e-30, 60, preconditioner=prec)
    torch.cuda.synchronize(); print(prec, "us/iter", (time.perf_counter() - t0) * 1e6 / iters)
    ws = device.to_host(sysm._pcg_ws)
    if prec == "mas":
        part = ws[33 * sysm.n + 3 * 4096:]
        for k, name in enumerate(names):
            t = part[512 * k: 512 * k + 148] / iters / 1e3
            print("  ", name, "us/iter: min %.2f mean %.2f max %.2f" % (t.min(), t.mean(), t.max()))
    else:
        part = ws[21 * sysm.n:]
        for k, name in enumerate(names):
            t = part[1024 + 512 * k: 1024 + 512 * k + 148] / iters / 1e3
            print("  ", name, "us/iter: min %.2f mean %.2f max %.2f" % (t.min(), t.mean(), t.max()))
