"""Per-iteration CG cost vs one mat-vec (configs 1, 3, 4 geometry)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2301_11828_b200 import FastForce, build_kernel
M = 3
for dims in [(128, 128), (1024, 1024), (128, 128, 128)]:
    dim = len(dims)
    n = 1
    for d in dims:
        n *= d
    h = 1.0 / dims[0]
    dl = 3.015 * h
    ff = FastForce(dims, M, build_kernel(dim, h, dl, M, 1.0, 1.0), device=0)
    ff.set_geometry(h, [0.0] * dim, dl, 1.0)
    big = 10.0
    for ax in range(dim):
        lo, hi = [-big] * dim, [big] * dim
        hi[ax] = dl
        ff.add_constraint(lo, hi, (1 << dim) - 1, 0, 0.0)
        lo, hi = [-big] * dim, [big] * dim
        lo[ax] = 1.0 - dl
        ff.add_constraint(lo, hi, (1 << dim) - 1, 0, 0.0)
    s = torch.cuda.Stream()
    b = torch.empty((dim, n), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    x = torch.empty_like(b)
    f = torch.empty_like(b)
    for _ in range(3):
        ff.matvec_device(b, f, 1, s)
    ff.cg_solve_device(b, x, tol=1e-30, maxit=20, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        ff.matvec_device(b, f, 1, s)
    e1.record(s)
    torch.cuda.synchronize()
    mv = e0.elapsed_time(e1) / 20
    e0.record(s)
    it, rel = ff.cg_solve_device(b, x, tol=1e-30, maxit=100, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{dims}: matvec {mv:.4f} ms, CG {e0.elapsed_time(e1) / it:.4f} ms/iter ({it} its)")
    ff.timing(True)
    ff.timing_read()
    ff.cg_solve_device(b, x, tol=1e-30, maxit=20, stream=s)
    torch.cuda.synchronize()
    print("   cg passes (20 its):", {k: round(v[0] / 20, 4) for k, v in ff.timing_read().items()})
    ff.close()
