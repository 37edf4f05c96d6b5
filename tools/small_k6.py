"""K6 kernels (surface diagonal, wrap correction) of a clamped 128^2 plate, 5 mat-vecs (for an ncu launch list)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2301_11828_b200 import FastForce, build_kernel
n = 128
h = 1.0 / n
dl = 3.015 * h
ff = FastForce((n, n), 3, build_kernel(2, h, dl, 3, 1.0, 1.0), device=0)
ff.set_geometry(h, [0.0, 0.0], dl, 1.0)
ff.add_constraint([-9, -9], [9, dl], 3, 0, 0.0)
u = torch.empty((2, n * n), dtype=torch.float64, device="cuda").uniform_(-1, 1)
f = torch.empty_like(u)
s = torch.cuda.Stream()
for _ in range(5):
    ff.matvec_device(u, f, 1, s)
torch.cuda.synchronize()
print("ok")
