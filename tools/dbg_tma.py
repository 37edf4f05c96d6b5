import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2301_11828_b200.engine import FastForce, build_kernel
for n in (256, 1024):
    h = 1 / n
    K = build_kernel(2, h, 3.015 * h, 3, 1.0, 1.0)
    ff = FastForce((n, n), 3, K)
    u = np.random.default_rng(0).uniform(-1, 1, (2, 2, n * n))
    os.environ["PDGPU_NO_TMA"] = "1"
    f0 = ff.matvec(u)
    del os.environ["PDGPU_NO_TMA"]
    f1 = ff.matvec(u)
    d = np.abs(f1 - f0).reshape(2, 2, n, n)
    print(n, "max diff", d.max(), "rel", np.linalg.norm(f1 - f0) / np.linalg.norm(f0))
    bad = np.argwhere(d > 1e-9 * np.abs(f0).max())
    print("  bad count", len(bad), "first", bad[:5].tolist(), "rows with errors", np.unique(bad[:, 2])[:10], "cols", np.unique(bad[:, 3])[:10])
    ff.close()
