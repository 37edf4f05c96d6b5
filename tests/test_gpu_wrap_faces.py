"""The 3D wrap correction's tiled face passes (k_wrap_face, lattices with
every axis periodic and at least 192 nodes per axis) against the oracle and
against the per-state kernel (PDGPU_WRAP_NOFACE=1): plain K.u (apply, D^e
separate), the corrected mat-vec with D^e folded into the passes, constrained
rows (the wrap mask and the surface mask differ in matvec), and a batch of 2."""
import numpy as np
import pytest

from oracle.oracle import Oracle, Rng, random_field

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _pair(dims, clamp):
    from paper_2301_11828_b200 import FastForce
    h = 1.0 / dims[0]
    dl = 3.015 * h
    o = Oracle(dims, h=h, delta=dl, M=3, E=1.0, thickness=1.0)
    ff = FastForce(dims, 3, o.kernel())
    ff.set_geometry(h, None, dl, 1.0)
    if clamp:
        for obj in (o, ff):
            lo, hi = [0.0, 0.0, 0.0], [1.0, 1.0, 1.0]
            hi[2] = dl
            obj.add_constraint(lo, hi, 7)
            lo, hi = [0.0, 0.0, 0.0], [1.0, 1.0, 1.0]
            lo[0] = 1.0 - dl
            obj.add_constraint(lo, hi, 0b010)
    return o, ff


@pytest.mark.parametrize("clamp", [False, True])
def test_face_passes_match_oracle(clamp):
    dims = (192, 192, 192)
    o, ff = _pair(dims, clamp)
    u = random_field(Rng(5100), 3, o.n)
    assert rel(ff.matvec(u), o.matvec(u)) <= 1e-11   # D^e folded into the passes
    assert rel(ff.apply(u), o.apply(u)) <= 1e-11     # wrap only, D^e separate
    ff.close()


def test_face_passes_equal_per_state_kernel(monkeypatch):
    import torch
    from paper_2301_11828_b200 import FastForce, build_kernel
    dims = (256, 256, 256)
    h = 1.0 / 256
    K = build_kernel(3, h, 3.015 * h, 3, 1.0, 1.0)
    u = torch.empty((2, 3, 256 ** 3), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    out = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("PDGPU_WRAP_NOFACE", env)
        ff = FastForce(dims, 3, K)
        ff.set_geometry(h, None, 3.015 * h, 1.0)
        f = torch.empty_like(u)
        ff.matvec_device(u, f, 2)
        torch.cuda.synchronize()
        out.append(f.cpu().numpy())
        ff.close()
    assert rel(out[0], out[1]) <= 1e-13
