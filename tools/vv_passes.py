"""Per-pass device time of the config-5 VV step (2048^2, notch, velocity BCs)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2301_11828_b200 import FastForce, build_kernel
M = 3
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
h = 1.0 / n
dl = 3.015 * h
K = build_kernel(2, h, dl, M, 1.0, 1.0)
lam = max(sum(2.0 * np.abs(K[0 if (a, b) == (0, 0) else (1 if a != b else 2)]).sum() for b in range(2)) for a in range(2))
dt = 0.8 * 2.0 * (1.0 / lam) ** 0.5
ff = FastForce((n, n), M, K)
ff.set_geometry(h, [0.0, 0.0], dl, 1.0)
ff.add_constraint((0.0, 1.0 - dl), (1.0, 1.0), 0b10, 1, 1e-4)
ff.add_constraint((0.0, 0.0), (1.0, dl), 0b10, 1, -1e-4)
ff.seed_segment((0.0, 0.5), (0.25, 0.5))
ff.sim_init(dt)
ff.sim_step(10, 1e-3)
ff.timing_read()
ff.timing(True)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
ff.sim_step(100, 1e-3)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 100 * 1e3
p = ff.timing_read()
ff.timing(False)
print(f"wall ms/step {wall:.3f}")
for k, (ms, c) in p.items():
    print(f"  {k:12s} {ms / 100:.4f} ms/step  launches/step {c / 100:.1f}")
t0 = time.perf_counter()
ff.sim_step(100, 1e-3)
torch.cuda.synchronize()
print(f"wall ms/step (timing off) {(time.perf_counter() - t0) / 100 * 1e3:.3f}")
t0 = time.perf_counter()
ff.sim_step(100, -1.0)
torch.cuda.synchronize()
print(f"wall ms/step without stretch test {(time.perf_counter() - t0) / 100 * 1e3:.3f}")
