"""Scratch: time the elastic block kernel (400 k random tets)."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2308_09400_b200 import elasticity, device
import bench
rng = np.random.default_rng(11); n = 400_000
rest = rng.normal(size=(4 * n, 3)); tets = np.arange(4 * n).reshape(n, 4)
mesh = elasticity.TetMesh(rest, tets, 3.7e4, 8.6e4)
x = device.to_device(rest + 0.3 * rng.normal(size=rest.shape))
mesh.evaluate(x, dt=0.01)
print("elastic ms", bench.time_steps(torch, lambda: mesh.evaluate(x, dt=0.01), 20, 3, lambda: None) / 20)
