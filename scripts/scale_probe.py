"""bench.py's Newton section on a cloth stack 4 x (default) the bench scale: how the fractions move when the matrix
(~400 MB) no longer comes near the L2.   python scripts/scale_probe.py [layers n]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2308_09400_b200 import _lib, barrier, contacts, device, solver, stencils, workloads

layers, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8, 180)
peak, src = bench.measured_peak()
pkg = (workloads, contacts, stencils, solver, barrier, device, _lib)
scene = workloads.cloth_stack(layers=layers, n=n, seed=3, d_hat_rel=0.2)
out = bench.newton_section(torch, pkg, 20, 3, peak, scene, extras=False, cpu_leg=False)
out["peak"] = [peak, src]
print(json.dumps(out))
