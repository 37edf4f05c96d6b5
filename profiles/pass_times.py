"""Per-pass device times (CUDA events on the launching stream) of one K.u
configuration:  python profiles/pass_times.py 256 256 256 --batch 1 --reps 10"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dims", type=int, nargs="+")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    from paper_2301_11828_b200 import FastForce, build_kernel
    dims = tuple(a.dims)
    dim = len(dims)
    h = 1.0 / dims[0]
    ff = FastForce(dims, 3, build_kernel(dim, h, 3.015 * h, 3, 1.0, 1.0))
    n = 1
    for d in dims:
        n *= d
    u = torch.empty((a.batch, dim, n), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    f = torch.empty_like(u)
    s = torch.cuda.Stream()
    for _ in range(3):
        ff.matvec_device(u, f, a.batch, s)
    torch.cuda.synchronize()
    ff.timing_read()
    ff.timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        ff.matvec_device(u, f, a.batch, s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    passes = {k: round(v[0] / a.reps, 4) for k, v in ff.timing_read().items()}
    dof = a.batch * dim * n
    print(f"dims={dims} batch={a.batch}: {ms:.4f} ms/matvec, {dof / ms / 1e6:.3e} DOF-matvecs/s, passes(ms)={passes}")


if __name__ == "__main__":
    main()
