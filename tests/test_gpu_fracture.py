"""GPU update_bonds / ledger / error contract against the oracle and the
reference's own fracture and error tests (tests/test_fracture.cpp,
tests/test_convolution.cpp:72-75,120-126, tests/test_corrections.cpp:383-394)."""
import numpy as np
import pytest

from oracle.oracle import Oracle, Rng, random_field

pytestmark = pytest.mark.gpu
STEEL_E = 2e11


def engine(o, h):
    from paper_2301_11828_b200 import FastForce
    ff = FastForce(o.dims, o.M, o.kernel())
    ff.set_geometry(h, None, o.M * h, 1.0)
    return ff


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def test_threshold_inclusive_and_monotone():
    n, h = 12, 0.0025
    o = Oracle((n, n), h=h, M=3, E=STEEL_E, thickness=0.0025)
    ff = engine(o, h)
    s0 = 0.015625  # exact power of two (test_fracture.cpp:147-155)
    u = np.zeros((2, n * n))
    u[0, 1] = s0 * h
    new = ff.update_bonds(dev(u), s0)
    assert [0, 1] in new.tolist()
    assert len(ff.update_bonds(dev(np.zeros_like(u)), s0)) == 0  # monotone (:157-169)


@pytest.mark.parametrize("dims,M", [((20, 16), 3), ((10, 9, 8), 2)])
def test_random_stretch_matches_oracle(dims, M):
    h = 0.01
    o = Oracle(dims, h=h, M=M, E=STEEL_E, thickness=0.0025)
    ff = engine(o, h)
    u = 0.02 * h * random_field(Rng(5), len(dims), o.n)
    for s0 in (0.01, 0.004, 0.001):
        new_o = o.update_bonds(u, s0)
        new_g = ff.update_bonds(dev(u), s0)
        assert np.array_equal(new_o, new_g)  # same pairs in the same visiting order
        assert np.array_equal(o.ledger_pairs(), ff.ledger_pairs())


def test_watch_box():
    n, h = 20, 0.01
    o = Oracle((n, n), h=h, M=2, E=STEEL_E, thickness=0.0025)
    ff = engine(o, h)
    s0 = 0.005
    u = np.zeros((2, n * n))
    u[0, 1 * n + 1] = 10 * s0 * h
    u[0, 10 * n + 10] = 10 * s0 * h
    watch = (np.array([0.0, 0.0]), np.array([0.05, 0.05]))
    new_o = o.update_bonds(u, s0, watch)
    new_g = ff.update_bonds(dev(u), s0, watch)
    assert len(new_g) > 0 and np.array_equal(new_o, new_g)
    assert all(p not in (10 * n + 10,) and q not in (10 * n + 10,) for p, q in new_g)


def test_errors():
    from paper_2301_11828_b200 import FastForce, HorizonTooLargeForGrid, LedgerOutOfBand, ShapeMismatch, build_kernel
    K = build_kernel(2, 0.5, 2.0, 4, 1.0, 1.0)
    with pytest.raises(HorizonTooLargeForGrid):  # convolution.hpp:61-62
        FastForce((4, 4), 4, K)
    ff = FastForce((5, 5), 4, K)  # M+1 nodes suffice
    with pytest.raises(ShapeMismatch):  # convolution.hpp:120-121
        ff.apply(np.zeros((2, 26)))
    K2 = build_kernel(2, 0.0025, 0.005, 2, 2e11, 0.0025)
    ff2 = FastForce((14, 14), 2, K2)
    with pytest.raises(LedgerOutOfBand):  # corrections.hpp:99-100
        ff2.break_bonds([[0, 5]])


def test_empty_ledger_and_zero_field():
    n = 16
    o = Oracle((n, n), h=0.01, M=3)
    ff = engine(o, 0.01)
    assert len(ff.ledger_pairs()) == 0
    f = ff.matvec(np.zeros((2, n * n)))
    assert np.all(f == 0.0)


def test_rigid_translation_force_free():
    # tests/test_corrections.cpp:340-361 / criterion 4
    n, h = 18, 0.0025
    o = Oracle((n, 14), h=h, M=3, E=STEEL_E, thickness=0.0025)
    o.random_ledger(Rng(555), 30)
    ff = engine(o, h)
    ff.break_bonds(o.ledger_pairs())
    u = np.zeros((2, o.n))
    u[0] = 2.5e-4
    u[1] = -1.25e-4
    f = ff.matvec(u)
    row = np.abs(o.kernel()[0]).sum() - abs(o.kernel()[0][(o.kernel().shape[1] - 1) // 2])
    assert np.abs(f).max() <= 1e-12 * row * 2.5e-4


def test_linearity():
    n = 32
    o = Oracle((n, 24), h=0.0025, M=3, E=STEEL_E, thickness=0.0025)
    ff = engine(o, 0.0025)
    u = random_field(Rng(91), 2, o.n)
    v = random_field(Rng(92), 2, o.n)
    fu, fv, fc = ff.apply(u), ff.apply(v), ff.apply(1.7 * u - 0.35 * v)
    assert np.abs(fc - (1.7 * fu - 0.35 * fv)).max() <= 1e-12 * np.abs(fc).max()
