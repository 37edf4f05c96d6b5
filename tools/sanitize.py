"""Small cases of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck):  compute-sanitizer --tool racecheck python tools/sanitize.py
  64^2 clamped plate: K1/K3/K5 + wrap + surface, CG, VV with breaking
  16^3 clamped cube: K1..K5 3D + wrap (+x strip), CG
  4096 x 16 periodic rows: K1 TMA-store / K5 TMA-gather row kernels
  64 x 2048: the TMEM-parked K3 (2048-point periodic columns)
  96 x 80 (padded embedding): padded row/column kernels"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_11828_b200 import FastForce, build_kernel  # noqa: E402


def plate(dims, clamp=True, crack=False):
    dim = len(dims)
    h = 1.0 / dims[0]
    dl = 3.015 * h
    ff = FastForce(dims, 3, build_kernel(dim, h, dl, 3, 1.0, 1.0), device=0)
    ff.set_geometry(h, [0.0] * dim, dl, 1.0)
    if clamp:
        for ax in range(dim):
            lo, hi = [-9.0] * dim, [9.0] * dim
            hi[ax] = dl
            ff.add_constraint(lo, hi, (1 << dim) - 1, 0, 0.0)
    if crack and dim == 2:
        ff.seed_segment((0.0, 0.5), (0.3, 0.5))
    return ff


def matvec(ff, batch=1):
    n = ff.n
    u = torch.empty((batch, ff.dim, n), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    f = torch.empty_like(u)
    ff.matvec_device(u, f, batch)
    torch.cuda.synchronize()
    return float(f.abs().max())


def main():
    ff = plate((64, 64), crack=True)
    matvec(ff, 2)
    b = torch.empty((2, 64 * 64), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    x = torch.empty_like(b)
    ff.cg_solve_device(b, x, tol=1e-8, maxit=50)
    ff.close()
    ff = plate((64, 64), clamp=False, crack=True)
    dl = 3.015 / 64
    ff.add_constraint((0.0, 1.0 - dl), (1.0, 1.0), 0b10, 1, 0.05)
    ff.add_constraint((0.0, 0.0), (1.0, dl), 0b10, 1, -0.05)
    ff.sim_init(1e-3)
    print("vv breaks", ff.sim_step(20, 1e-3))
    ff.close()
    ff = plate((16, 16, 16))
    matvec(ff)
    b = torch.empty((3, 16 ** 3), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    x = torch.empty_like(b)
    ff.cg_solve_device(b, x, tol=1e-8, maxit=20)
    ff.close()
    for dims in ((4096, 16), (64, 2048), (96, 80)):
        ff = plate(dims, clamp=False)
        print(dims, matvec(ff, 1))
        ff.close()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
