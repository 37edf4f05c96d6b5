"""Config-1 (128^2 clamped plate) CG iterations, for ncu of the small-lattice kernels."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_11828_b200 import FastForce, build_kernel  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
h = 1.0 / n
dl = 3.015 * h
ff = FastForce((n, n), 3, build_kernel(2, h, dl, 3, 1.0, 1.0), device=0)
ff.set_geometry(h, [0, 0], dl, 1.0)
for ax in range(2):
    lo, hi = [-9, -9], [9, 9]
    hi[ax] = dl
    ff.add_constraint(lo, hi, 3, 0, 0.0)
    lo, hi = [-9, -9], [9, 9]
    lo[ax] = 1 - dl
    ff.add_constraint(lo, hi, 3, 0, 0.0)
b = torch.empty((2, n * n), dtype=torch.float64, device="cuda").uniform_(-1, 1)
x = torch.empty_like(b)
ff.cg_solve_device(b, x, tol=1e-30, maxit=int(sys.argv[2]) if len(sys.argv) > 2 else 3)
torch.cuda.synchronize()
print("ok")
