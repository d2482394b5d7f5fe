python - <<'PY'
import sys, time, os
import numpy as np
sys.path.insert(0, ".")
exec(open("scripts/mas_probe.py").read().split("def wall")[0])
import torch
def wall(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best, out
sysm.mas_order(pos); sysm.mas_setup(1); sysm._mas_stale = False
for dbg in ("0", "1"):
    os.environ["B200IPC_MAS_DEBUG"] = dbg
    t, out = wall(lambda: sysm.pcg(rhs, 1e-30, 60, preconditioner="mas", mas_levels=1))
    print("debug", dbg, f"{t:.3f} ms for {out[1]} iters: {t/out[1]*1e3:.1f} us/iter")
t, out = wall(lambda: sysm.pcg(rhs, 1e-30, 60))
print("block-jacobi", f"{t:.3f} ms for {out[1]} iters: {t/out[1]*1e3:.1f} us/iter")
PY
