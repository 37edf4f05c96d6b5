"""The all-to-all distributed-FFT arm (pdgpu_set_transpose; SURVEY.md 8e,
north_star's transpose scheme) against the single-engine K.u and the
oracle: G = 1 (the engine's own path, transposes as copies) and G = 2, 3, 4
engines of one process (pdgpu_group_matvec_transpose: device copies for the
NCCL all-to-all), balanced and uneven row / column splits, batch 2, with
the global faces' y aliases taken from the opposite end's rows."""
import numpy as np
import pytest
import torch

from oracle.oracle import Oracle, Rng, random_field

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _engines(nx, ny, G, row_bounds=None, col_bounds=None):
    from paper_2301_11828_b200 import FastForce, build_kernel
    from paper_2301_11828_b200.engine import transpose_splits
    h = 1.0 / nx
    K = build_kernel(2, h, 3.015 * h, 3, 1.0, 1.0)
    rb, cb = transpose_splits(nx, ny, G)
    rb = rb if row_bounds is None else row_bounds
    cb = cb if col_bounds is None else col_bounds
    out = []
    for r in range(G):
        e = FastForce((nx, rb[r + 1] - rb[r]), 3, K)
        e.set_geometry(h, [0.0, rb[r] * h], 3.015 * h, 1.0)
        e.set_transpose(G, r, ny, rb, cb)
        out.append(e)
    return out, rb, K, h


@pytest.mark.parametrize("G,rows,cols", [(2, None, None), (3, None, None), (4, None, None),
                                         (3, [0, 40, 100, 128], [0, 10, 50, 65])])
def test_group_transpose_matches_single_engine(G, rows, cols):
    from paper_2301_11828_b200 import FastForce
    from paper_2301_11828_b200.engine import group_matvec_transpose
    nx = ny = 128
    engines, rb, K, h = _engines(nx, ny, G, rows, cols)
    single = FastForce((nx, ny), 3, K)
    single.set_geometry(h, [0.0, 0.0], 3.015 * h, 1.0)
    batch = 2
    u = torch.empty((batch, 2, ny, nx), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    f = torch.empty_like(u)
    single.matvec_device(u.reshape(batch, 2, -1), f.reshape(batch, 2, -1), batch)
    us = [u[:, :, rb[r]:rb[r + 1], :].contiguous().reshape(batch, 2, -1) for r in range(G)]
    fs = [torch.empty_like(x) for x in us]
    group_matvec_transpose(engines, us, fs, batch)
    torch.cuda.synchronize()
    got = torch.cat([fs[r].reshape(batch, 2, rb[r + 1] - rb[r], nx) for r in range(G)], dim=2)
    assert rel(got.cpu().numpy(), f.cpu().numpy()) <= 1e-12
    for e in engines + [single]:
        e.close()


def test_one_rank_transpose_matches_oracle():
    n = 64
    engines, rb, K, h = _engines(n, n, 1)
    o = Oracle((n, n), h=h, delta=3.015 * h, M=3, E=1.0, thickness=1.0)
    u = random_field(Rng(8800), 2, o.n)
    assert rel(engines[0].matvec(u), o.matvec(u)) <= 1e-11
    assert rel(engines[0].apply(u), o.apply(u)) <= 1e-11
    engines[0].close()
