"""GPU parity of the spectral product and the corrected mat-vec against the
CPU oracle (oracle/oracle.c) -- the reference's own shapes and BASELINE
config 1.  Tolerance: relative L2 <= 1e-11 (BASELINE.json north_star)."""
import numpy as np
import pytest

from oracle.oracle import Oracle, Rng, random_field

pytestmark = pytest.mark.gpu
TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def engine_for(o: Oracle):
    from paper_2301_11828_b200 import FastForce
    return FastForce(o.dims, o.M, o.kernel())


# tests/test_convolution.cpp:129-155 shapes, random (non-even) stencils
@pytest.mark.parametrize("dims,M", [((16, 12), 2), ((32, 32), 3), ((40, 20), 4), ((9, 7), 2),
                                    ((8, 8, 8), 2), ((12, 10, 8), 3), ((16, 16, 16), 4)])
def test_random_stencil_full_stack(dims, M):
    rng = Rng(37 + len(dims))
    o = Oracle(dims, h=0.5, M=M)
    o.random_kernel(rng)
    u = random_field(rng, len(dims), o.n)
    ff = engine_for(o)
    assert not ff.symbol_is_real()
    f = ff.apply(u)
    assert rel(f, o.apply(u)) <= TOL


@pytest.mark.parametrize("dims", [(128, 128), (64, 48), (33, 17), (16, 16, 16), (24, 20, 12)])
def test_physical_kernel_matvec(dims):
    h = 1.0 / dims[0]
    o = Oracle(dims, h=h, delta=3.015 * h, M=3, E=1.0, thickness=1.0)
    ff = engine_for(o)
    assert ff.symbol_is_real()
    u = random_field(Rng(1000), len(dims), o.n)
    assert rel(ff.apply(u), o.apply(u)) <= TOL
    assert rel(ff.matvec(u), o.matvec(u)) <= TOL


def test_config1_constrained_with_bonds():
    n = 128
    h = 1.0 / n
    d = 3.015 * h
    o = Oracle((n, n), h=h, delta=d, M=3)
    from paper_2301_11828_b200 import FastForce
    ff = FastForce((n, n), 3, o.kernel())
    ff.set_geometry(h, [0, 0], d, 1.0)
    for lo, hi in [((0, 0), (1, d)), ((0, 1 - d), (1, 1)), ((0, 0), (d, 1)), ((1 - d, 0), (1, 1))]:
        o.add_constraint(lo, hi, 3)
        ff.add_constraint(lo, hi, 3)
    rng = Rng(7)
    o.random_ledger(rng, 50)
    ff.break_bonds(o.ledger_pairs())
    assert np.array_equal(ff.ledger_pairs(), o.ledger_pairs())
    u = random_field(Rng(1000), 2, o.n)
    assert rel(ff.matvec(u), o.matvec(u)) <= TOL


def test_batched_apply_matches_single():
    n = 64
    o = Oracle((n, n), h=1 / n, delta=3.015 / n, M=3)
    ff = engine_for(o)
    u = np.stack([random_field(Rng(2000 + i), 2, o.n) for i in range(3)])
    fb = ff.matvec(u)
    for i in range(3):
        assert rel(fb[i], o.matvec(u[i])) <= TOL


@pytest.mark.parametrize("dims", [(96, 80), (24, 20, 16)])
def test_separable_symbol_mode(dims, monkeypatch):
    """PDGPU_SYMBOL=separable: per-column symbol coefficients instead of the
    O(N) table -- same K.u to 1e-11."""
    monkeypatch.setenv("PDGPU_SYMBOL", "separable")
    h = 1.0 / dims[0]
    o = Oracle(dims, h=h, delta=3.015 * h, M=3, E=1.0, thickness=1.0)
    ff = engine_for(o)
    assert ff.symbol_mode() == "separable"
    u = random_field(Rng(31), len(dims), o.n)
    assert rel(ff.matvec(u), o.matvec(u)) <= TOL
