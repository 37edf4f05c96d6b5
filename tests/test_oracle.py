"""Pin the CPU oracle (oracle/oracle.c) before trusting it.

Known answers are the reference's own (tests/test_material_kernel.cpp,
tests/test_fracture.cpp, tests/test_grid.cpp); golden vectors were produced
by the reference itself (oracle/gen_golden.py, oracle/_ref).  Inputs are
regenerated here with the oracle's restatement of std::mt19937 +
uniform_real_distribution, and the fixtures' input checksums pin that
restatement too.  CPU only.
"""
import ctypes as C
import math
import os

import numpy as np
import pytest

from oracle.oracle import Oracle, Rng, _d, olib, random_field

G = os.path.join(os.path.dirname(__file__), "golden")
STEEL_E = 2e11


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def csum(a):
    a = np.asarray(a, dtype=np.float64)
    return np.array([a.sum(), (a * a).sum()])


# ----------------------------------------------------------- known answers --
def test_alpha_known_answers():
    L = olib()
    # tests/test_material_kernel.cpp:11-15
    assert L.orc_alpha(2e11, 0.03, 2, 0.0025) == pytest.approx(8.488263631567753e18, rel=1e-14)
    assert L.orc_alpha(math.pi, 1.0, 3, 0.0) == pytest.approx(12.0, rel=1e-14)
    assert L.orc_alpha(2e11, 0.003, 3, 0.0) == pytest.approx(9.431404035075278e21, rel=1e-14)


def test_critical_stretch_known_answers():
    L = olib()
    # tests/test_material_kernel.cpp:21-24
    assert L.orc_critical_stretch(100.0, 2e11, 0.03, 0) == pytest.approx(0.00015254853881062816, rel=1e-14)
    assert L.orc_critical_stretch(100.0, 2e11, 0.03, 1) == pytest.approx(0.00014770448757545966, rel=1e-14)


def test_kernel_entries_and_row_sums():
    # tests/test_material_kernel.cpp:57-115: 16x16 grid, h = 0.0025, M = 3, steel
    o = Oracle((16, 16), h=0.0025, M=3, E=STEEL_E, thickness=0.0025)
    K = o.kernel().reshape(3, 7, 7)  # [pair][oy][ox]
    assert np.count_nonzero(K[0]) - 1 == 22  # 22 nonzero K^xx off centre (:97)
    for p in range(3):
        off = K[p].copy()
        off[3, 3] = 0.0
        s = 0.0
        # centre is -(sum in for_each_offset order), kernel.hpp:119-125
        for ox in range(-3, 4):
            for oy in range(-3, 4):
                if 0 < ox * ox + oy * oy <= 9:
                    s += K[p, oy + 3, ox + 3]
        assert K[p, 3, 3] == -s
    assert np.array_equal(K[0], K[0][::-1, ::-1])  # parity under negation (:108-115)
    assert np.array_equal(K[1], K[1][::-1, ::-1])
    assert K[0, 3, 6] != 0.0 and K[0, 3 + 1, 6] == 0.0  # rim vs just outside (:83-86)
    assert K[1, 3, 4] == 0.0  # axis bond has no shear coupling (:85)


def test_bond_stretch_known_answers():
    L = olib()
    h = 0.01
    xp = np.array([0.0, 0.0])
    xq = np.array([h, 0.0])
    z = np.zeros(2)

    def s(uq):
        return L.orc_bond_stretch(2, _d(xp), _d(xq), _d(z), _d(np.asarray(uq, dtype=np.float64)))

    # tests/test_fracture.cpp:10-19
    assert s([0.0, 0.0]) == 0.0
    assert s([0.01 * h, 0.0]) == pytest.approx(0.01, rel=1e-12)
    assert s([0.0, h]) == pytest.approx(0.41421356237309515, rel=1e-14)
    assert s([-0.25 * h, 0.0]) < 0.0


def test_threshold_inclusive_and_monotone():
    # tests/test_fracture.cpp:147-169: s == s0 breaks; relaxing does not heal
    n = 12
    o = Oracle((n, n), h=0.0025, M=3, E=STEEL_E, thickness=0.0025)
    s0 = 0.015625
    u = np.zeros((2, n * n))
    u[0, 1] = s0 * 0.0025
    o.update_bonds(u, s0)
    pairs = {tuple(p) for p in o.ledger_pairs()}
    assert (0, 1) in pairs
    before = len(pairs)
    assert len(o.update_bonds(np.zeros_like(u), s0)) == 0
    assert len(o.ledger_pairs()) == before


def test_rng_is_mt19937():
    # std::mt19937 default-seed (5489) 10000th output is 4123659995 (C++ [rand.predef])
    r = Rng(5489)
    v = 0
    for _ in range(10000):
        v = r.next()
    assert v == 4123659995


def test_near_surface_count():
    # tests/test_grid.cpp:98-104: interior count (Nx-2M)(Ny-2M)
    o = Oracle((20, 14), h=1.0, M=3)
    ns, _ = o.regions()
    assert int((ns == 0).sum()) == (20 - 6) * (14 - 6)


# ------------------------------------------------------------ golden vectors --
def test_conv_golden():
    d = np.load(os.path.join(G, "conv_random.npz"))
    for dim, ncase in ((2, 4), (3, 3)):
        rng = Rng(37 + dim)
        for k in range(ncase):
            tag = f"d{dim}_{k}"
            dims = tuple(int(x) for x in d[tag + "_dims"])
            M = int(d[tag + "_M"])
            o = Oracle(dims, h=0.5, M=M)
            o.random_kernel(rng)
            u = random_field(rng, dim, o.n)
            np.testing.assert_allclose(csum(o.kernel()), d[tag + "_K_csum"], rtol=1e-14)
            np.testing.assert_allclose(csum(u), d[tag + "_u_csum"], rtol=1e-14)
            f = o.apply(u)
            assert rel(f, d[tag + "_f"]) <= 1e-12, tag          # reference FFT path
            assert rel(f, d[tag + "_fdirect"]) <= 1e-14, tag    # reference direct oracle
            assert float(d[tag + "_resid"]) <= 1e-10


def test_corrections_golden():
    d = np.load(os.path.join(G, "corrections.npz"))
    rng = Rng(1234)
    for k in range(3):
        tag = f"c{k}"
        dims = tuple(int(x) for x in d[tag + "_dims"])
        M = int(d[tag + "_M"])
        h = 0.0025
        o = Oracle(dims, h=h, M=M, E=STEEL_E, thickness=0.0025)
        box = d[tag + "_box"]
        o.add_constraint(box[:2], box[2:], 0b01)
        o.random_ledger(rng, 40)
        u = random_field(rng, 2, o.n)
        np.testing.assert_allclose(csum(u), d[tag + "_u_csum"], rtol=1e-14)
        assert np.array_equal(o.ledger_pairs(), d[tag + "_ledger"])
        assert rel(o.matvec(u), d[tag + "_f"]) <= 1e-12
        assert rel(o.dense(u), d[tag + "_fdense"]) <= 1e-14


def test_acceptance_golden():
    d = np.load(os.path.join(G, "acceptance.npz"))
    for dim, shapes in ((2, [(16, 12), (32, 32), (40, 20)]), (3, [(8, 8, 8), (12, 10, 8), (16, 16, 16)])):
        rng = Rng(2024 + dim)
        k = 0
        for dims in shapes:
            for M in (2, 3, 4):
                tag = f"d{dim}_{k}"
                h = 0.01
                o = Oracle(dims, h=h, M=M, E=STEEL_E, thickness=0.0025)
                axis = rng.next() % dim
                depth = (1 + rng.next() % M) * h
                lo = [0.0] * dim
                hi = [dims[i] * h for i in range(dim)]
                if rng.next() % 2:
                    hi[axis] = lo[axis] + depth
                else:
                    lo[axis] = hi[axis] - depth
                mask = 1 + rng.next() % ((1 << dim) - 1)
                assert mask == int(d[tag + "_mask"])
                np.testing.assert_array_equal(np.array(lo + hi), d[tag + "_box"])
                o.add_constraint(lo, hi, mask)
                o.random_ledger(rng, rng.next() % 51)
                u = random_field(rng, dim, o.n)
                np.testing.assert_allclose(csum(u), d[tag + "_u_csum"], rtol=1e-14)
                assert np.array_equal(o.ledger_pairs(), d[tag + "_ledger"]), tag
                assert rel(o.matvec(u), d[tag + "_f"]) <= 1e-12, tag
                assert rel(o.dense(u), d[tag + "_fdense"]) <= 1e-14, tag
                k += 1


def clamp_boxes(dim, dl):
    out = []
    for ax in range(dim):
        lo0, hi0 = [0.0] * dim, [1.0] * dim
        hi0[ax] = dl
        lo1, hi1 = [0.0] * dim, [1.0] * dim
        lo1[ax] = 1.0 - dl
        out += [(lo0, hi0), (lo1, hi1)]
    return out


def config_oracle(dims):
    dim = len(dims)
    h = 1.0 / dims[0]
    o = Oracle(dims, h=h, delta=3.015 * h, M=3, E=1.0, thickness=1.0)
    for lo, hi in clamp_boxes(dim, 3.015 * h):
        o.add_constraint(lo, hi, (1 << dim) - 1)
    return o


def test_configs_golden():
    d = np.load(os.path.join(G, "configs.npz"))
    o = config_oracle((128, 128))
    u = random_field(Rng(1000), 2, o.n)
    np.testing.assert_allclose(csum(u), d["c1_u_csum"], rtol=1e-14)
    assert rel(o.matvec(u), d["c1_f"]) <= 1e-12
    b = random_field(Rng(1001), 2, o.n)
    x, it, relres, hist = o.cg(b, tol=1e-10, maxit=20000, nhist=20)
    assert relres <= 1e-10
    assert abs(it - int(d["c1_cg_iters"])) <= 2
    assert rel(hist[19], d["c1_cg_x20"]) <= 1e-11  # first iterates agree
    assert o.static_residual(b, d["c1_cg_x"]) <= 1e-10 * 1.001  # reference solution solves ours (ii)
    o3 = config_oracle((24, 24, 24))
    u3 = random_field(Rng(4000), 3, o3.n)
    np.testing.assert_allclose(csum(u3), d["c4_u_csum"], rtol=1e-14)
    assert rel(o3.matvec(u3), d["c4_f"]) <= 1e-12


def test_seeds_golden():
    import hashlib
    d = np.load(os.path.join(G, "seeds.npz"))
    for tag, n, a, b in (("c3", 1024, (0.25, 0.5), (0.75, 0.5)), ("c5", 2048, (0.0, 0.5), (0.25, 0.5))):
        h = 1.0 / n
        o = Oracle((n, n), h=h, delta=3.015 * h, M=3)
        o.seed_segment(a, b)
        p = o.ledger_pairs()
        assert len(p) == int(d[tag + "_count"])
        assert hashlib.sha256(np.ascontiguousarray(p, dtype=np.int64).tobytes()).hexdigest() == str(d[tag + "_hash"])


def precracked_oracle():
    h = 0.05 / 100.0
    delta = 3 * h
    o = Oracle((100, 100), h=h, delta=delta, M=3, E=2e11, thickness=0.0025, rho=7850.0)
    o.add_constraint((0.0, 0.05 - delta), (0.05, 0.05), 0b10, 1, 20.0)
    o.add_constraint((0.0, 0.0), (0.05, delta), 0b10, 1, -20.0)
    o.seed_segment((0.02, 0.025), (0.03, 0.025))
    return o


@pytest.mark.parametrize("tag,s0", [("s0_1e-2", 0.01), ("s0_5e-3", 5e-3)])
def test_vv_golden(tag, s0):
    """acceptance_main.cpp:197-219 criterion 5: trajectory <= 1e-8, ledgers identical."""
    d = np.load(os.path.join(G, "vv_precracked.npz"))
    o = precracked_oracle()
    o.sim_init(1.3367e-8)
    per = [o.sim_step(1, s0=s0) for _ in range(200)]
    u, v, f, t = o.sim_get()
    assert t == float(d[tag + "_t"])
    assert per == list(d[tag + "_broken_per_step"])
    assert np.array_equal(o.ledger_pairs(), d[tag + "_ledger"])
    assert np.abs(u - d[tag + "_u"]).max() <= 1e-8 * np.abs(d[tag + "_u"]).max()


def _adr_oracle(dims):
    from oracle.gen_golden import adr_problem
    return adr_problem(dims, ref=False)


@pytest.mark.parametrize("tag,dims,fixed,steps", [("p2", (64, 64), None, 300), ("p2_fixed", (64, 64), 0.05, 200),
                                                  ("p3", (16, 16, 16), None, 100)])
def test_adr_golden(tag, dims, fixed, steps):
    """AdrIntegrator (timestepping.hpp:79-162) restated in oracle.c against the
    reference's own ADR trajectory (oracle/gen_golden.py gen_adr): u and the
    adaptive damping trace."""
    d = np.load(os.path.join(G, "adr.npz"))
    o = _adr_oracle(dims)
    o.sim_init_adr(1.0, fixed_damping=fixed)
    trace = []
    for _ in range(steps // 25):
        o.sim_step(25)
        trace.append(o.adr_damping())
    u, v, f, t = o.sim_get()
    assert t == float(d[tag + "_t"])
    # the reference's own FFT-vs-dense ADR criterion (tests/test_timestepping.cpp:168-176):
    # max |du| <= 1e-8 max |u| after the run (adaptive damping amplifies round-off)
    assert np.abs(u - d[tag + "_u"]).max() <= 1e-8 * np.abs(d[tag + "_u"]).max()
    assert np.allclose(trace, d[tag + "_damping"], rtol=1e-6, atol=0)
