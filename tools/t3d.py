"""256^3 K.u time with per-pass timing on and off (bench 3D roofline check)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_11828_b200 import FastForce, build_kernel
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
h = 1.0 / n
ff = FastForce((n, n, n), 3, build_kernel(3, h, 3.015 * h, 3, 1.0, 1.0))
ff.set_geometry(h, [0, 0, 0], 3.015 * h, 1.0)
u = torch.empty((3, n ** 3), dtype=torch.float64, device="cuda").uniform_(-1, 1)
f = torch.empty_like(u)
s = torch.cuda.Stream()
for _ in range(3):
    ff.matvec_device(u, f, 1, s)
torch.cuda.synchronize()
for on in (False, True, True, False):
    ff.timing_read()
    ff.timing(on)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(10):
        ff.matvec_device(u, f, 1, s)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"timing={on}: {e0.elapsed_time(e1) / 10:.4f} ms/matvec device, host {(time.perf_counter() - t0) * 100:.3f} ms",
          {k: round(v[0] / 10, 4) for k, v in ff.timing_read().items()})
