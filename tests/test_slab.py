"""Halo slab decomposition (paper_2301_11828_b200/slab.py).

CPU (gloo, world size 2 and 3): SlabForce's ghost-row exchange, slab origin
and D^e bookkeeping and its all-reduced CG, with a test double for the
per-rank engine built on the C oracle (the oracle's FFT convolution on the
extended slab + the global lattice's D^e rows) -- the gathered owned rows must
equal the oracle's single-lattice K.u and CG solution.

GPU: the libpdgpu engine behind the same class -- several slabs of one
lattice on one device (ghost rows filled from the global field instead of by
P2P, since gpurun has one GPU) must reproduce the single-engine K.u.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

N = 32
M = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _geom(n):
    h = 1.0 / n
    return h, 3.015 * h


def _clamp(add, n, dim=2):
    """Config-1 style clamp: the four delta-deep face layers, all directions."""
    h, delta = _geom(n)
    big = 10.0
    for ax in range(dim):
        lo = [-big] * dim
        hi = [big] * dim
        hi[ax] = delta
        add(lo, hi, (1 << dim) - 1, 0, 0.0)
        lo = [-big] * dim
        hi = [big] * dim
        lo[ax] = 1.0 - delta
        add(lo, hi, (1 << dim) - 1, 0, 0.0)


class OracleSlabEngine:
    """Test double of the per-rank engine: C-oracle FFT convolution on the
    extended slab (zero outside it) plus D^e taken from the global lattice."""

    def __init__(self, ext_dims, global_dims, K, de_global):
        self.ext, self.gdims, self.K, self.de_g = tuple(ext_dims), tuple(global_dims), K, de_global
        self.dim = len(ext_dims)
        self.plane = int(np.prod(ext_dims[:-1]))
        self.n = int(np.prod(ext_dims))
        self.cons = []
        self.h, self.origin = 1.0, np.zeros(self.dim)
        self._o = None

    def _oracle(self):
        from oracle.oracle import Oracle
        if self._o is None:
            self._o = Oracle(self.ext, h=self.h, delta=3.015 * self.h, M=M, origin=self.origin)
            self._o.set_kernel(self.K)
            for c in self.cons:
                self._o.add_constraint(*c)
        return self._o

    def set_slab(self, rows, off):
        self.rows, self.off = rows, off
        self.de = self.de_g[:, off * self.plane:off * self.plane + self.n]
        self.ghosts = None

    def set_ghosts(self, g):
        """pdgpu_set_ghosts contract: g (batch, dim, 2, M, plane), side 0 = rows before the slab."""
        self.ghosts = g

    def _apply_with_ghosts(self, ub, g):
        """The engine's ghost-mode result: the oracle on [ghost_lo; slab; ghost_hi], owned rows."""
        from oracle.oracle import Oracle
        lo_int, hi_int = self.off > 0, self.off + self.ext[-1] < self.rows
        gl, gh = (M if lo_int else 0), (M if hi_int else 0)
        parts = ([g[:, 0].numpy()] if gl else []) + [ub.reshape(self.dim, self.ext[-1], self.plane)] + \
                ([g[:, 1].numpy()] if gh else [])
        ue = np.concatenate(parts, axis=1).reshape(self.dim, -1)
        org = self.origin.copy()
        org[-1] -= gl * self.h
        o = Oracle(self.ext[:-1] + (self.ext[-1] + gl + gh,), h=self.h, delta=3.015 * self.h, M=M, origin=org)
        o.set_kernel(self.K)
        fe = o.apply(ue).reshape(self.dim, -1, self.plane)
        return np.ascontiguousarray(fe[:, gl:gl + self.ext[-1]].reshape(self.dim, -1))

    def set_geometry(self, h, origin, delta, rho):
        """pdgpu_set_geometry contract for slabs: the global origin; this engine's
        first row sits at row `off` of the global lattice."""
        org = np.array(origin, dtype=np.float64)
        org[-1] += self.off * h
        self.h, self.origin, self._o = h, org, None

    def add_constraint(self, lo, hi, mask, kind=0, value=0.0):
        self.cons.append((lo, hi, mask, kind, value))
        self._o = None

    def constraint_values(self):
        o = self._oracle()
        _, cm = o.regions()
        uc = np.zeros((self.dim, self.n))  # only zero-valued displacement constraints here
        return cm, uc

    def matvec_device(self, u, f, batch, stream=None):
        from paper_2301_11828_b200.engine import pair_index
        o = self._oracle()
        for b in range(batch):
            ub = u[b].numpy()
            fb = o.apply(ub) if self.ghosts is None else self._apply_with_ghosts(ub, self.ghosts[b])
            for a in range(self.dim):
                for c in range(self.dim):
                    fb[a] += self.de[pair_index(self.dim, a, c)] * ub[c]
            f[b].copy_(torch.from_numpy(fb))


def _global_oracle(n, clamp):
    from oracle.oracle import Oracle
    h, delta = _geom(n)
    o = Oracle((n, n), h=h, delta=delta, M=M)
    if clamp:
        _clamp(o.add_constraint, n)
    return o


def _worker(rank, world, port, q, halo="ghost"):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    from oracle.oracle import Rng, random_field
    from paper_2301_11828_b200 import dist as D
    from paper_2301_11828_b200.slab import SlabForce
    r, w, _ = D.init("gloo")
    g = _global_oracle(N, clamp=False)
    K, de = g.kernel(), g.de()
    h, delta = _geom(N)
    sf = SlabForce((N, N), M, K, rank=r, world=w,
                   engine=lambda ext: OracleSlabEngine(ext, (N, N), K, de), halo=halo)
    sf.set_geometry(h, None, delta, 1.0)
    u = random_field(Rng(4100), 2, N * N)
    ub = torch.from_numpy(np.stack([sf.owned(u), sf.owned(-0.5 * u)]))
    f = sf.matvec(ub)
    # CG on the clamped problem
    sfc = SlabForce((N, N), M, K, rank=r, world=w,
                    engine=lambda ext: OracleSlabEngine(ext, (N, N), K, de), halo=halo)
    sfc.set_geometry(h, None, delta, 1.0)
    _clamp(sfc.add_constraint, N)
    b = random_field(Rng(4101), 2, N * N)
    x, it, rel = sfc.cg_solve(torch.from_numpy(np.ascontiguousarray(sfc.owned(b))), tol=1e-10, maxit=2000)
    parts = [None] * w
    import torch.distributed as dist
    dist.all_gather_object(parts, (sf.r0, sf.r1, f.numpy(), x.numpy(), it, rel))
    if r == 0:
        q.put(parts)
    D.finalize()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,halo", [(2, "ghost"), (3, "ghost"), (2, "embedded"), (3, "embedded")])
def test_slab_halo_gloo(world, halo):
    from oracle.oracle import Rng, random_field
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, halo)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=500)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _global_oracle(N, clamp=False)
    u = random_field(Rng(4100), 2, N * N)
    f_ref = np.stack([g.matvec(u), g.matvec(-0.5 * u)])
    f = np.zeros_like(f_ref)
    x = np.zeros((2, N * N))
    for r0, r1, fr, xr, it, rel in parts:
        f[:, :, r0 * N:r1 * N] = fr
        x[:, r0 * N:r1 * N] = xr
        assert rel <= 1e-10
    err = np.linalg.norm(f - f_ref) / np.linalg.norm(f_ref)
    assert err <= 1e-12, err
    gc = _global_oracle(N, clamp=True)
    b = random_field(Rng(4101), 2, N * N)
    x_ref, it_ref, rel_ref, _ = gc.cg(b, tol=1e-10, maxit=2000)
    assert abs(parts[0][4] - it_ref) <= 2
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-7
    # the GPU-free CG answer satisfies the oracle's own static residual
    assert gc.static_residual(b, x) <= 1e-10 * (1 + 1e-3)


def test_slab_rows_partition():
    from paper_2301_11828_b200.slab import slab_rows
    for n, w in [(4096, 8), (100, 3), (7, 7)]:
        spans = [slab_rows(n, r, w) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))


def _emulated_slabs(dims, K, world, u, dev, constraints=(), halo="ghost"):
    """All slabs of one lattice on one GPU; ghost rows copied from the global
    field (what the P2P exchange delivers)."""
    from paper_2301_11828_b200.slab import SlabForce
    plane = int(np.prod(dims[:-1]))
    h = 1.0 / dims[0]
    out = torch.zeros_like(u)
    for r in range(world):
        sf = SlabForce(dims, M, K, rank=r, world=world, device=dev, halo=halo)
        sf.set_geometry(h, None, 3.015 * h, 1.0)
        for c in constraints:
            sf.add_constraint(*c)
        lo = (sf.r0 - sf.gl) * plane
        hi = (sf.r1 + sf.gh) * plane

        def fill(ext, lo=lo, hi=hi):
            ext.copy_(u[:, :, lo:hi])

        def fill_ghosts(u3, g, sf=sf):
            if sf.gl:
                g[:, :, 0].copy_(u[:, :, (sf.r0 - M) * plane:sf.r0 * plane].reshape(g.shape[0], sf.dim, M, plane))
            if sf.gh:
                g[:, :, 1].copy_(u[:, :, sf.r1 * plane:(sf.r1 + M) * plane].reshape(g.shape[0], sf.dim, M, plane))

        sf.exchange = fill
        sf.exchange_ghosts = fill_ghosts
        out[:, :, sf.r0 * plane:sf.r1 * plane] = sf.matvec(sf.owned(u).contiguous())
        sf.eng.close()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("halo", ["ghost", "embedded"])
@pytest.mark.parametrize("dims,world", [((256, 256), 4), ((96, 80), 3), ((24, 20, 32), 4), ((32, 32, 64), 2),
                                        ((512, 512), 8), ((256, 256, 64), 4), ((256, 192, 32), 2)])
def test_slab_engine_gpu(dims, world, halo):
    # (256, 256, 64) / 4 and (256, 192, 32) / 2: 16-plane slabs of 256-wide planes -- the
    # first runs the tiled wrap face passes with ghost planes in the z pass
    from oracle.oracle import Rng, random_field
    from paper_2301_11828_b200.engine import FastForce, build_kernel
    dev = torch.device("cuda:0")
    dim = len(dims)
    n = int(np.prod(dims))
    h = 1.0 / dims[0]
    K = build_kernel(dim, h, 3.015 * h, M, 1.0, 1.0 if dim == 2 else 0.0)
    u = torch.from_numpy(np.stack([random_field(Rng(4200 + i), dim, n) for i in range(2)])).to(dev)
    full = FastForce(dims, M, K)
    full.set_geometry(h, None, 3.015 * h, 1.0)
    f_ref = torch.zeros_like(u)
    full.matvec_device(u, f_ref, 2, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    f = _emulated_slabs(dims, K, world, u, dev, halo=halo)
    torch.cuda.synchronize()
    err = float(torch.linalg.norm(f - f_ref) / torch.linalg.norm(f_ref))
    assert err <= 1e-12, err
    full.close()


def _engine(dims, dev_index=0):
    from paper_2301_11828_b200.engine import FastForce, build_kernel
    dim = len(dims)
    h = 1.0 / dims[0]
    K = build_kernel(dim, h, 3.015 * h, M, 1.0, 1.0 if dim == 2 else 0.0)
    ff = FastForce(dims, M, K, device=dev_index)
    ff.set_geometry(h, None, 3.015 * h, 1.0)
    return ff, K, h


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(128, 128), (32, 32, 32)])
def test_comm_one_rank_matches_plain_engine(dims):
    """An engine with an NCCL communicator of one rank runs the multi-rank code
    path (split CG update, ncclAllReduce of every dot product inside the
    captured iteration, all-reduced ADR damping sums); all-reducing over one
    rank is the identity, so every result equals the plain engine's bit for bit."""
    from oracle.oracle import Rng, random_field
    dim = len(dims)
    n = int(np.prod(dims))
    plain, K, h = _engine(dims)
    comm, _, _ = _engine(dims)
    comm.comm_init(1, 0, comm.comm_unique_id())
    dl = 3.015 * h
    for ff in (plain, comm):
        for ax in range(dim):
            lo, hi = [0.0] * dim, [1.0] * dim
            hi[ax] = dl
            ff.add_constraint(lo, hi, (1 << dim) - 1, 0, 0.0)
        top_lo = [0.0] * dim
        top_lo[-1] = 1.0 - dl
        ff.add_constraint(top_lo, [1.0] * dim, 1 << (dim - 1), 0, 1e-3)  # prescribed layer: the any_uc branch
    u = torch.from_numpy(random_field(Rng(77), dim, n)).cuda()
    f0, f1 = torch.empty_like(u), torch.empty_like(u)
    plain.matvec_device(u, f0)
    comm.matvec_device(u, f1)
    torch.cuda.synchronize()
    assert torch.equal(f0, f1)
    b = torch.from_numpy(random_field(Rng(78), dim, n)).cuda()
    x0, x1 = torch.empty_like(b), torch.empty_like(b)
    it0, r0 = plain.cg_solve_device(b, x0, tol=1e-9, maxit=5000)
    it1, r1 = comm.cg_solve_device(b, x1, tol=1e-9, maxit=5000)
    assert it0 == it1 and r0 == r1 and r1 <= 1e-9
    assert torch.equal(x0, x1)
    # ADR: damping sums all-reduced before c is formed
    for ff in (plain, comm):
        ff.set_body(np.full((dim, n), 1e-3))
        ff.sim_init_adr(1.0)
        ff.sim_step(20)
    ua = plain.sim_get()[0]
    ub = comm.sim_get()[0]
    assert np.array_equal(ua, ub) and plain.adr_damping() == comm.adr_damping()


@pytest.mark.gpu
@pytest.mark.parametrize("dims,world", [((256, 256), 4), ((64, 48, 32), 4), ((512, 512), 8)])
def test_packed_halo_slabs_gpu(dims, world):
    """The NCCL exchange's data layout on one GPU: every slab packs its first /
    last M rows with pdgpu_halo_pack, the neighbours' packed rows are placed
    in a receive buffer [2][batch][dim][M][plane] exactly as ncclRecv leaves
    them, and the engine reads them through pdgpu_set_ghosts_strided; the
    gathered owned rows must equal the single engine's K.u."""
    from oracle.oracle import Rng, random_field
    from paper_2301_11828_b200.slab import slab_rows
    dim = len(dims)
    n = int(np.prod(dims))
    plane = n // dims[-1]
    batch = 2
    full, K, h = _engine(dims)
    u = torch.from_numpy(np.stack([random_field(Rng(4300 + i), dim, n) for i in range(batch)])).cuda()
    f_ref = torch.empty_like(u)
    full.matvec_device(u, f_ref, batch)
    engines, sends = [], []
    from paper_2301_11828_b200.engine import FastForce
    for r in range(world):
        r0, r1 = slab_rows(dims[-1], r, world)
        ff = FastForce(dims[:-1] + (r1 - r0,), M, K)
        org = [0.0] * dim
        org[-1] = r0 * h
        ff.set_geometry(h, org, 3.015 * h, 1.0)
        ff.set_slab(dims[-1], r0)
        uo = u[:, :, r0 * plane:r1 * plane].contiguous()
        send = torch.zeros((2, batch, dim, M, plane), dtype=torch.float64, device="cuda")
        ff.halo_pack(uo, send, batch)
        engines.append((ff, r0, r1, uo))
        sends.append(send)
    f = torch.zeros_like(u)
    side = batch * dim * M * plane
    for r, (ff, r0, r1, uo) in enumerate(engines):
        recv = torch.zeros((2, batch, dim, M, plane), dtype=torch.float64, device="cuda")
        if r > 0:
            recv[0].copy_(sends[r - 1][1])  # what ncclRecv from rank - 1 delivers
        if r < world - 1:
            recv[1].copy_(sends[r + 1][0])
        ff.set_ghosts_strided(recv, M * plane, side)
        fo = torch.empty_like(uo)
        ff.matvec_device(uo, fo, batch)
        torch.cuda.synchronize()
        f[:, :, r0 * plane:r1 * plane] = fo
    err = float(torch.linalg.norm(f - f_ref) / torch.linalg.norm(f_ref))
    assert err <= 1e-12, err


def _vv_engines(dims, world, dt_scale=0.8, rate_per_step=1e-4):
    """Config-5 geometry (notch (0,0.5)-(0.25,0.5), velocity-driven top/bottom
    delta-layers) on the whole lattice and on `world` row slabs."""
    from paper_2301_11828_b200.engine import FastForce, build_kernel
    from paper_2301_11828_b200.slab import slab_rows
    n = dims[0]
    h = 1.0 / n
    dl = 3.015 * h
    K = build_kernel(2, h, dl, M, 1.0, 1.0)
    lam = max(sum(2.0 * np.abs(K[0 if (a, b) == (0, 0) else (1 if a != b else 2)]).sum() for b in range(2))
              for a in range(2))
    dt = dt_scale * 2.0 * (1.0 / lam) ** 0.5
    rate = rate_per_step / dt

    def setup(ff):
        ff.set_geometry(h, [0.0, 0.0], dl, 1.0)
        ff.add_constraint((0.0, 1.0 - dl), (1.0, 1.0), 0b10, 1, rate)
        ff.add_constraint((0.0, 0.0), (1.0, dl), 0b10, 1, -rate)

    full = FastForce(dims, M, K)
    setup(full)
    slabs = []
    for r in range(world):
        r0, r1 = slab_rows(dims[1], r, world)
        ff = FastForce((dims[0], r1 - r0), M, K)
        ff.set_slab(dims[1], r0)
        setup(ff)
        slabs.append(ff)
    return full, slabs, dt


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_fracture_across_slabs_gpu(world):
    """Velocity Verlet with bond breaking over row slabs (pdgpu_group_sim_step,
    the single-process form of the NCCL slab path): the notch and the torn
    layers' bonds cross slab faces; per-step breaks, the ledger (union of the
    slabs' pairs, global ids) and u must equal the single engine's."""
    from paper_2301_11828_b200.engine import group_sim_step
    dims = (256, 256)
    full, slabs, dt = _vv_engines(dims, world)
    a = full.seed_segment((0.0, 0.5), (0.25, 0.5))
    b = sum(s.seed_segment((0.0, 0.5), (0.25, 0.5)) for s in slabs)
    assert a == b > 0

    def union():
        return np.concatenate([s.ledger_pairs() for s in slabs])

    def rows(x):
        return x[np.lexsort((x[:, 1], x[:, 0]))]

    assert np.array_equal(rows(union()), full.ledger_pairs())
    full.sim_init(dt)
    for s in slabs:
        s.sim_init(dt)
    total = 0
    for blk in range(8):
        pf = [full.sim_step(1, s0=1e-3) for _ in range(10)]
        pg = [group_sim_step(slabs, 1, s0=1e-3) for _ in range(10)]
        assert pf == pg, blk
        total += sum(pf)
        assert np.array_equal(rows(union()), full.ledger_pairs()), blk
    assert total > 100
    uf = full.sim_get()[0]
    plane = dims[0]
    ug = np.concatenate([s.sim_get()[0] for s in slabs], axis=1)
    assert np.linalg.norm(ug - uf) / np.linalg.norm(uf) <= 1e-10
    for s in slabs:
        s.close()
    full.close()
