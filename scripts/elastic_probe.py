"""Scratch: the bench's elastic workload (400k private tets), CUDA-event time of energy + gradient + projected block."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2308_09400_b200 import device, elasticity
rng_e = np.random.default_rng(11)
n_tet = 400_000
rest_t = rng_e.normal(size=(4 * n_tet, 3))
mesh_t = elasticity.TetMesh(rest_t, np.arange(4 * n_tet).reshape(n_tet, 4), 3.7e4, 8.6e4)
x_t = device.to_device(rest_t + 0.1 * rng_e.normal(size=rest_t.shape))
for _ in range(3): mesh_t.evaluate(x_t, dt=0.01)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): mesh_t.evaluate(x_t, dt=0.01)
b.record(); torch.cuda.synchronize()
print("elastic blocks: %.1f us per call (incl. output allocation)" % (a.elapsed_time(b) * 100))
