"""On-device set-up: D^e / near-surface rows
(corrections.hpp:24-42) and crack seeding (fracture.hpp:164-198) run as
kernels; PDGPU_HOST_ASSEMBLY=1 selects the host restatement (assembly.cpp).
Both must give bit-identical ledgers and K.u, including segments with width,
segments along lattice lines (the orientation predicates' zero band), 3D
notches with and without width, and cracks that leave the lattice."""
import numpy as np
import pytest

from oracle.oracle import Oracle, Rng, random_field

pytestmark = pytest.mark.gpu

SEGMENTS = [((0.25, 0.5), (0.75, 0.5), 0.0), ((0.0, 0.5), (0.25, 0.5), 0.0), ((0.1, 0.13), (0.83, 0.71), 0.0),
            ((0.2, 0.3), (0.7, 0.35), 0.05), ((-0.5, 0.40625), (1.5, 0.40625), 0.0), ((0.3, 0.3), (0.3, 0.9), 0.02)]
NOTCHES = [(2, 0.5, 0.0, (0.2, 0.2, 0.0), (0.8, 0.7, 1.0)), (0, 0.37, 0.06, (0.0, 0.1, 0.2), (1.0, 0.6, 0.9)),
           (1, 0.5, 0.0, (-1.0, -1.0, -1.0), (2.0, 2.0, 2.0))]


def _engine(dims, monkeypatch, host):
    from paper_2301_11828_b200 import FastForce, build_kernel
    if host:
        monkeypatch.setenv("PDGPU_HOST_ASSEMBLY", "1")
    else:
        monkeypatch.delenv("PDGPU_HOST_ASSEMBLY", raising=False)
    dim = len(dims)
    h = 1.0 / dims[0]
    ff = FastForce(dims, 3, build_kernel(dim, h, 3.015 * h, 3, 1.0, 1.0), device=0)
    ff.set_geometry(h, [0.0] * dim, 3.015 * h, 1.0)
    return ff


@pytest.mark.parametrize("dims", [(64, 48), (96, 96)])
def test_segments_device_equals_host(dims, monkeypatch):
    ffs = [_engine(dims, monkeypatch, host) for host in (False, True)]
    for a, b, w in SEGMENTS:
        added = [ff.seed_segment(a, b, w) for ff in ffs]
        assert added[0] == added[1]
    pd, ph = ffs[0].ledger_pairs(), ffs[1].ledger_pairs()
    assert len(pd) > 0 and np.array_equal(pd, ph)
    u = random_field(Rng(77), 2, int(np.prod(dims)))
    fd, fh = ffs[0].matvec(u), ffs[1].matvec(u)
    assert np.array_equal(fd, fh)  # D^e rows and the bond correction bit-identical
    for ff in ffs:
        ff.close()


def test_notches_device_equals_host(monkeypatch):
    dims = (24, 20, 16)
    ffs = [_engine(dims, monkeypatch, host) for host in (False, True)]
    for ax, plane, w, lo, hi in NOTCHES:
        added = [ff.seed_notch(ax, plane, w, lo, hi) for ff in ffs]
        assert added[0] == added[1] and added[0] > 0
    assert np.array_equal(ffs[0].ledger_pairs(), ffs[1].ledger_pairs())
    u = random_field(Rng(78), 3, int(np.prod(dims)))
    assert np.array_equal(ffs[0].matvec(u), ffs[1].matvec(u))
    for ff in ffs:
        ff.close()


def test_device_seed_matches_oracle(monkeypatch):
    """the config-3 crack on a small plate: the oracle's seeding (pinned to the reference's 9,210-bond ledger)"""
    n = 128
    h = 1.0 / n
    o = Oracle((n, n), h=h, delta=3.015 * h, M=3, E=1.0, thickness=1.0)
    o.seed_segment((0.25, 0.5), (0.75, 0.5))
    ff = _engine((n, n), monkeypatch, False)
    ff.seed_segment((0.25, 0.5), (0.75, 0.5))
    assert np.array_equal(ff.ledger_pairs(), o.ledger_pairs())
    ff.close()


@pytest.mark.parametrize("dims", [(64, 64), (20, 24, 16), (7, 9)])
def test_surface_rows_device_equals_host(dims, monkeypatch):
    ffs = [_engine(dims, monkeypatch, host) for host in (False, True)]
    u = random_field(Rng(79), len(dims), int(np.prod(dims)))
    assert np.array_equal(ffs[0].matvec(u), ffs[1].matvec(u))
    for ff in ffs:
        ff.close()
