"""Periodic embedding (P = N + wrap correction, engine.h Plan) against the
padded one (P = 2N, the reference's PadTransform, convolution.hpp:58-71) and
against the CPU oracle.  Both must give the reference's linear correlation:
relative L2 <= 1e-11 on every row, constrained ones included, for arbitrary
(complex-symbol) stencils, the physical ones, mixed periodic/padded axes,
the constraint-mask / body-force epilogue and CG."""
import numpy as np
import pytest

from oracle.oracle import Oracle, Rng, random_field

pytestmark = pytest.mark.gpu
TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def make(o, embed, monkeypatch):
    from paper_2301_11828_b200 import FastForce
    if embed == "padded":
        monkeypatch.setenv("PDGPU_EMBED", "padded")
    else:
        monkeypatch.delenv("PDGPU_EMBED", raising=False)
    return FastForce(o.dims, o.M, o.kernel())


@pytest.mark.parametrize("dims,M,bits", [((64, 64), 3, 3), ((64, 48), 3, 1), ((48, 64), 3, 2), ((16, 16), 3, 3),
                                         ((32, 32, 32), 3, 7), ((32, 24, 16), 3, 5), ((24, 20, 12), 3, 0),
                                         ((16, 16), 8, 0), ((32, 16), 8, 1)])
def test_embedding_choice(dims, M, bits, monkeypatch):
    o = Oracle(dims, h=1.0 / dims[0], delta=3.015 / dims[0], M=M)
    assert make(o, "periodic", monkeypatch).embedding() == bits
    assert make(o, "padded", monkeypatch).embedding() == 0


@pytest.mark.parametrize("dims,M", [((64, 64), 3), ((32, 128), 2), ((128, 40), 4), ((40, 64), 3), ((16, 16), 7),
                                    ((16, 16, 16), 3), ((32, 16, 16), 2), ((16, 24, 32), 3), ((32, 32, 12), 2),
                                    ((512, 37), 3), ((256, 20, 8), 2), ((4096, 24), 3), ((2048, 20), 2),
                                    ((8192, 16), 2)])
def test_random_stencil_both_embeddings(dims, M, monkeypatch):
    rng = Rng(91 + M)
    o = Oracle(dims, h=0.5, M=M)
    o.random_kernel(rng)
    u = np.stack([random_field(rng, len(dims), o.n) for _ in range(2)])
    want = np.stack([o.apply(u[i]) for i in range(2)])
    fp = make(o, "periodic", monkeypatch)
    assert fp.embedding() != 0
    got_p = fp.apply(u)
    got_z = make(o, "padded", monkeypatch).apply(u)
    assert rel(got_p, want) <= TOL
    assert rel(got_z, want) <= TOL
    assert rel(got_p, got_z) <= TOL


def test_longest_periodic_rows(monkeypatch):
    """16384-node rows: the periodic embedding's longest x transform (2 x 4096-point
    halves through the unpipelined K1, whose staging would not fit); the padded
    embedding of the same lattice is refused (NOT_SUPPORTED) at create time."""
    from paper_2301_11828_b200 import FastForce
    rng = Rng(97)
    o = Oracle((16384, 16), h=0.5, M=2)
    o.random_kernel(rng)
    u = random_field(rng, 2, o.n)
    ff = make(o, "periodic", monkeypatch)
    assert ff.embedding() == 3
    assert rel(ff.apply(u), o.apply(u)) <= TOL
    monkeypatch.setenv("PDGPU_EMBED", "padded")
    with pytest.raises(NotImplementedError):
        FastForce(o.dims, o.M, o.kernel())


@pytest.mark.parametrize("dims", [(128, 128), (256, 64), (32, 32, 32)])
def test_physical_corrected_matvec_with_bonds(dims, monkeypatch):
    d = len(dims)
    h = 1.0 / dims[0]
    o = Oracle(dims, h=h, delta=3.015 * h, M=3)
    ff = make(o, "periodic", monkeypatch)
    assert ff.embedding() == (1 << d) - 1
    o.random_ledger(Rng(5), 40)
    ff.break_bonds(o.ledger_pairs())
    u = random_field(Rng(1000 + d), d, o.n)
    assert rel(ff.matvec(u), o.matvec(u)) <= TOL


@pytest.mark.parametrize("dims", [(128, 128), (64, 32, 32)])
def test_constrained_epilogue_and_cg(dims, monkeypatch):
    """Constraint mask + body force in the K5 epilogue, then the wrap
    correction must leave constrained rows at zero (timestepping.hpp:306-309);
    CG (scale -1, masked operand) must meet the oracle's residual."""
    torch = pytest.importorskip("torch")
    d = len(dims)
    h = 1.0 / dims[0]
    dl = 3.015 * h
    o = Oracle(dims, h=h, delta=dl, M=3)
    ff = make(o, "periodic", monkeypatch)
    ff.set_geometry(h, [0.0] * d, dl, 1.0)
    ext = [dims[a] * h for a in range(d)]
    for ax in range(d):
        for side in (0, 1):
            lo = [0.0] * d
            hi = list(ext)
            if side == 0:
                hi[ax] = dl
            else:
                lo[ax] = ext[ax] - dl
            o.add_constraint(lo, hi, (1 << d) - 1)
            ff.add_constraint(lo, hi, (1 << d) - 1)
    body = random_field(Rng(77), d, o.n)
    o.set_body(body)
    ff.set_body(body)
    u = random_field(Rng(78), d, o.n)
    ud = torch.tensor(u, device="cuda")
    fd = torch.empty_like(ud)
    ff.evaluate_force_device(ud, fd)
    torch.cuda.synchronize()
    f = fd.cpu().numpy()
    want = o.evaluate_force(u)
    assert rel(f, want) <= TOL
    cm = o.regions()[1] if isinstance(o.regions(), tuple) else None
    if cm is not None:
        for a in range(d):
            assert np.all(f[a][(cm >> a) & 1 == 1] == 0.0)
    b = random_field(Rng(79), d, o.n)
    x, it, relres, _ = ff.cg_solve(b, tol=1e-10, maxit=20000)
    assert relres <= 1e-10
    assert o.static_residual(b, x) <= 1.001e-10


@pytest.mark.parametrize("dims", [(64, 64), (32, 32, 32)])
def test_separable_symbol_periodic(dims, monkeypatch):
    monkeypatch.setenv("PDGPU_SYMBOL", "separable")
    h = 1.0 / dims[0]
    o = Oracle(dims, h=h, delta=3.015 * h, M=3)
    ff = make(o, "periodic", monkeypatch)
    assert ff.symbol_mode() == "separable" and ff.embedding() == (1 << len(dims)) - 1
    u = random_field(Rng(31), len(dims), o.n)
    assert rel(ff.matvec(u), o.matvec(u)) <= TOL


def test_cg_after_workspace_growth(monkeypatch):
    """A CG solve, then a larger-batch mat-vec (the workspace is reallocated),
    then CG again: the captured CG iteration must not keep the old buffers."""
    torch = pytest.importorskip("torch")
    n = 64
    h = 1.0 / n
    o = Oracle((n, n), h=h, delta=3.015 * h, M=3)
    ff = make(o, "periodic", monkeypatch)
    ff.set_geometry(h, [0.0, 0.0], 3.015 * h, 1.0)
    for lo, hi in [((0, 0), (1, 3.015 * h)), ((0, 1 - 3.015 * h), (1, 1))]:
        o.add_constraint(lo, hi, 3)
        ff.add_constraint(lo, hi, 3)
    b = random_field(Rng(5), 2, o.n)
    x1, it1, rel1, _ = ff.cg_solve(b, tol=1e-10, maxit=5000)
    u = np.stack([random_field(Rng(6 + i), 2, o.n) for i in range(8)])
    fb = ff.matvec(u)  # batch 8 > the CG's batch-1 workspace
    assert rel(fb[3], o.matvec(u[3])) <= TOL
    x2, it2, rel2, _ = ff.cg_solve(b, tol=1e-10, maxit=5000)
    assert it1 == it2 and rel2 <= 1e-10
    assert np.array_equal(x1, x2)


@pytest.mark.parametrize("dims,M,a,b", [((64, 48), 3, 0, 0), ((64, 48), 3, 0, 1), ((33, 17), 2, 1, 1),
                                        ((16, 12, 20), 2, 0, 2), ((16, 16, 16), 3, 1, 1)])
def test_convolver_single_pair(dims, M, a, b):
    """Convolver<Dim> (convolution.hpp:210-230): one stencil pair, one scalar
    field, against a direct correlation f[p] = sum_o K_ab(o) u[p+o] (zero
    outside the lattice), as tests/test_convolution.cpp:104-118 checks it."""
    from paper_2301_11828_b200 import Convolver, pair_index
    rng = Rng(211 + M)
    o = Oracle(dims, h=0.5, M=M)
    o.random_kernel(rng)
    K = o.kernel()
    dim = len(dims)
    u = random_field(rng, 1, o.n)[0]
    cv = Convolver(dims, M, K, a, b)
    f = cv.apply(u)
    side = 2 * M + 1
    Kp = K.reshape(dim * (dim + 1) // 2, *([side] * dim))[pair_index(dim, a, b)]  # [o_{d-1}]...[o_0]
    U = u.reshape(tuple(reversed(dims)))  # [.., y, x]
    pad = np.pad(U, M)
    want = np.zeros_like(U)
    for idx in np.ndindex(*([side] * dim)):
        kv = Kp[idx]
        if kv == 0.0:
            continue
        sl = tuple(slice(i, i + n) for i, n in zip(idx, reversed(dims)))
        want += kv * pad[sl]
    assert rel(f, want.reshape(-1)) <= TOL
    cv.close()
