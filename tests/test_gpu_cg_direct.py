"""CG with the direct-stencil operator (pdgpu_set_cg_operator(h, 1)): the
same K as MSBFM summed directly (csrc/direct.cu, with the constraint mask)
plus the same corrections.  Graded like the MSBFM CG: the first
iterates against the oracle's, and the solution through the oracle mat-vec,
on config 1 (clamped 128^2), the config-3 geometry with its crack and
prescribed layers (256^2), and a clamped 24^3 cube."""
import numpy as np
import pytest

from oracle.oracle import Oracle, Rng, random_field

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _pair(dims):
    from paper_2301_11828_b200 import FastForce
    h = 1.0 / dims[0]
    o = Oracle(dims, h=h, delta=3.015 * h, M=3, E=1.0, thickness=1.0)
    ff = FastForce(dims, 3, o.kernel())
    ff.set_geometry(h, None, 3.015 * h, 1.0)
    return o, ff, h


def _clamp(objs, dim, dl):
    for ax in range(dim):
        for lo_side in (True, False):
            lo, hi = [0.0] * dim, [1.0] * dim
            if lo_side:
                hi[ax] = dl
            else:
                lo[ax] = 1.0 - dl
            for obj in objs:
                obj.add_constraint(lo, hi, (1 << dim) - 1)


@pytest.mark.parametrize("dims", [(128, 128), (24, 24, 24)])
def test_cg_direct_clamped(dims):
    o, ff, h = _pair(dims)
    _clamp((o, ff), len(dims), 3.015 * h)
    ff.cg_operator("direct")
    b = random_field(Rng(1001), len(dims), o.n)
    x, it, relres, _ = ff.cg_solve(b, tol=1e-10, maxit=20000)
    assert relres <= 1e-10
    assert o.static_residual(b, x) <= 1e-10 * (1 + 1e-3)
    xo, _, _, _ = o.cg(b, tol=1e-10, maxit=5)
    x5, it5, _, _ = ff.cg_solve(b, tol=1e-10, maxit=5)
    assert it5 == 5 and rel(x5, xo) <= 1e-11
    ff.close()


def test_cg_direct_crack_and_prescribed_layers():
    n = 256
    o, ff, h = _pair((n, n))
    dl = 3.015 * h
    for obj in (o, ff):
        obj.add_constraint((0.0, 1.0 - dl), (1.0, 1.0), 0b01)
        obj.add_constraint((0.0, 1.0 - dl), (1.0, 1.0), 0b10, 0, 1e-3)
        obj.add_constraint((0.0, 0.0), (1.0, dl), 0b01)
        obj.add_constraint((0.0, 0.0), (1.0, dl), 0b10, 0, -1e-3)
        obj.seed_segment((0.25, 0.5), (0.75, 0.5))
    ff.cg_operator("direct")
    b = np.zeros((2, o.n))
    x, it, relres, _ = ff.cg_solve(b, tol=1e-10, maxit=50000)
    assert relres <= 1e-10
    assert o.static_residual(b, x) <= 1e-10 * (1 + 1e-3)
    ff.cg_operator("msbfm")
    xm, itm, _, _ = ff.cg_solve(b, tol=1e-10, maxit=50000)
    assert rel(x, xm) <= 1e-8  # both converged to the same solution
    ff.close()
