"""Halo (overlap-save) slab decomposition of the MSBFM operator over ranks.

SURVEY.md sec.8e.  The FFT convolution couples every node, but the stencil
reaches only M rows, so the operator on a block of rows needs the rows
themselves plus M rows on either side.  Rank r owns rows [r0, r1) of the
slowest axis (rows j in 2D, planes k in 3D; node p = (k*Ny + j)*Nx + i,
grid.hpp:30-36) and runs its own FFT convolution (one libpdgpu engine).
Two halo modes: "ghost" (default) -- the engine's lattice is exactly the owned
rows (a power-of-two count keeps every axis on the periodic embedding, so a
rank does 1/G of the single-GPU transform work) and the M rows beyond each
interior face arrive in a side buffer whose stencil terms the engine's wrap
correction adds; "embedded" -- the ghost rows are part of the engine's
lattice (R + 2M rows, zero-padded transforms).

Two transports for the ghost rows (2*M*plane*dim*8 bytes per rank per
vector, 393 KB at 4096^2, against the two full all-to-all transposes of a
distributed FFT):
  "engine" (default on CUDA + NCCL, ghost mode): the library's own NCCL
      exchange (pdgpu_comm_init, csrc/comm.cpp): packed rows go out on a side
      stream while the spectral passes run, and CG runs entirely on the
      device (one captured iteration, its two dot products all-reduced by
      ncclAllReduce inside the graph, no per-iteration host read).
  "torch": torch.distributed point-to-point of the same packed rows -- the
      gloo CPU tests drive the host logic through this with a test-double
      engine; CG is then the restated loop below with all-reduced dots.

Exactness: for an owned row every in-band neighbour lies in the owned or ghost
rows, the engine's zero padding only replaces rows outside the global lattice
(where the reference pads with zeros too, convolution.hpp:183-195), and
pdgpu_set_slab rebuilds D^e / near-surface flags against the global faces
(grid.hpp:181-189, corrections.hpp:24-42).  Ghost-row outputs are discarded.
Fracture across slab faces: see FastForce.sim_* with a communicator
(DESIGN.md sec.6).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def slab_rows(n_rows: int, rank: int, world: int):
    """Owned rows [r0, r1) of `rank` (balanced contiguous split)."""
    return n_rows * rank // world, n_rows * (rank + 1) // world


class SlabForce:
    """One rank's share of K.u on a row slab with M ghost rows per interior face.

    dims/M/stencils as FastForce.  engine(ext_dims) -> engine object (default:
    FastForce on `device`); it must offer set_slab, set_geometry,
    add_constraint, constraint_values and matvec_device(u, f, batch, stream).
    Fields are torch tensors (batch, dim, R*plane) of the owned rows.
    """

    def __init__(self, dims, M: int, stencils, rank: int = 0, world: int = 1, device=None, engine=None,
                 group=None, halo: str = "ghost", transport: str = "auto"):
        self.dims = tuple(int(d) for d in dims)
        self.dim = len(self.dims)
        self.M = int(M)
        self.rank, self.world, self.group = int(rank), int(world), group
        self.plane = int(np.prod(self.dims[:-1]))
        self.rows = self.dims[-1]
        self.r0, self.r1 = slab_rows(self.rows, self.rank, self.world)
        self.R = self.r1 - self.r0
        if self.world > 1 and self.R < self.M:
            raise ValueError(f"slab of {self.R} rows is thinner than the horizon M = {self.M}")
        self.gl = self.M if self.r0 > 0 else 0
        self.gh = self.M if self.r1 < self.rows else 0
        if halo not in ("ghost", "embedded"):
            raise ValueError("halo must be 'ghost' or 'embedded'")
        # "ghost": the engine's lattice is the owned rows (periodic along the
        # slowest axis when R is a power of two) and the neighbours' rows
        # arrive in a side buffer read by the wrap correction
        # (pdgpu_set_ghosts); "embedded": the ghost rows are part of the
        # engine's lattice (zero-padded transforms of R + 2M rows).
        self.halo = halo
        self.L = self.R if halo == "ghost" else self.R + self.gl + self.gh
        self.off = self.r0 if halo == "ghost" else self.r0 - self.gl
        self.ext_dims = self.dims[:-1] + (self.L,)
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        if engine is None:
            from .engine import FastForce

            if self.device.type != "cuda":
                raise RuntimeError("SlabForce needs a CUDA device (libpdgpu engine)")
            engine = lambda ext: FastForce(ext, self.M, stencils, device=self.device.index or 0)  # noqa: E731
        self.eng = engine(self.ext_dims)
        self.eng.set_slab(self.rows, self.off)
        self._bufs = {}
        if transport == "auto":
            nccl = dist.is_available() and dist.is_initialized() and dist.get_backend(group) == "nccl"
            transport = "engine" if (self.device.type == "cuda" and halo == "ghost" and
                                     (nccl or self.world == 1) and hasattr(self.eng, "comm_init")) else "torch"
        if transport not in ("engine", "torch"):
            raise ValueError("transport must be 'engine', 'torch' or 'auto'")
        if transport == "engine" and halo != "ghost":
            raise ValueError("the engine transport fills ghost-mode side buffers")
        self.transport = transport
        if transport == "engine":
            uid = [self.eng.comm_unique_id() if self.rank == 0 else None]
            if self.world > 1:
                dist.broadcast_object_list(uid, src=0, group=group)
            self.eng.comm_init(self.world, self.rank, uid[0])

    # ------------------------------------------------------------ set-up
    def set_geometry(self, h: float, origin=None, delta: float = 0.0, rho: float = 1.0):
        """Global geometry: the engine keeps the global origin and places its
        rows at [off, off + L) of the global lattice (pdgpu_set_slab), so node
        positions are the reference's own (grid.hpp:53-57) bit for bit."""
        org = np.zeros(self.dim) if origin is None else np.array(origin, dtype=np.float64)
        self.eng.set_geometry(h, org, delta, rho)

    def add_constraint(self, lo, hi, dir_mask: int, kind: int = 0, value: float = 0.0):
        self.eng.add_constraint(lo, hi, dir_mask, kind, value)

    @property
    def n_owned(self) -> int:
        return self.R * self.plane

    def owned(self, x):
        """Owned rows of a global field (..., N) -> (..., R*plane)."""
        return x[..., self.r0 * self.plane:self.r1 * self.plane]

    # ------------------------------------------------------------ halo
    def _buf(self, batch: int):
        if batch not in self._bufs:
            z = lambda: torch.zeros((batch, self.dim, self.L * self.plane), dtype=torch.float64,  # noqa: E731
                                    device=self.device)
            g = torch.zeros((batch, self.dim, 2, self.M, self.plane), dtype=torch.float64, device=self.device)
            self._bufs[batch] = (z(), z(), g)
        return self._bufs[batch]

    def exchange_ghosts(self, u3, g):
        """Ghost mode: g (batch, dim, 2, M, plane) <- the M rows before / after
        this slab from the neighbours (zeros at global faces); u3 the owned
        rows (batch, dim, R*plane)."""
        if self.world == 1:
            return
        b = u3.shape[0]
        e = u3.reshape(b, self.dim, self.R, self.plane)
        M = self.M
        ops, recvs = [], []
        if self.gl:
            peer = self.rank - 1
            ops.append(dist.P2POp(dist.isend, e[:, :, :M].contiguous(), peer, self.group))
            buf = torch.empty((b, self.dim, M, self.plane), dtype=u3.dtype, device=u3.device)
            ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
            recvs.append((buf, 0))
        if self.gh:
            peer = self.rank + 1
            ops.append(dist.P2POp(dist.isend, e[:, :, self.R - M:].contiguous(), peer, self.group))
            buf = torch.empty((b, self.dim, M, self.plane), dtype=u3.dtype, device=u3.device)
            ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
            recvs.append((buf, 1))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        for buf, side in recvs:
            g[:, :, side].copy_(buf)

    def exchange(self, ext):
        """Fill the ghost rows of ext (batch, dim, L*plane) from the neighbours."""
        if self.world == 1:
            return
        b = ext.shape[0]
        e = ext.view(b, self.dim, self.L, self.plane)
        M, gl, R = self.M, self.gl, self.R
        ops, recvs = [], []
        if self.gl:
            peer = self.rank - 1
            ops.append(dist.P2POp(dist.isend, e[:, :, gl:gl + M].contiguous(), peer, self.group))
            buf = torch.empty((b, self.dim, M, self.plane), dtype=ext.dtype, device=ext.device)
            ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
            recvs.append((buf, 0))
        if self.gh:
            peer = self.rank + 1
            ops.append(dist.P2POp(dist.isend, e[:, :, gl + R - M:gl + R].contiguous(), peer, self.group))
            buf = torch.empty((b, self.dim, M, self.plane), dtype=ext.dtype, device=ext.device)
            ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
            recvs.append((buf, gl + R))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        for buf, row in recvs:
            e[:, :, row:row + M].copy_(buf)

    def _stream(self):
        return torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None

    # ------------------------------------------------------------ K.u
    def matvec(self, u, f=None):
        """f = A u (FastForce::apply + apply_corrections) on the owned rows;
        u, f: (batch, dim, R*plane) or (dim, R*plane)."""
        squeeze = u.dim() == 2
        u3 = u.unsqueeze(0) if squeeze else u
        b = u3.shape[0]
        ext, fext, g = self._buf(b)
        if self.transport == "engine":
            # the library exchanges the halo rows itself (NCCL, overlapped)
            uc = u3 if u3.is_contiguous() else u3.contiguous()
            if f is not None:
                f3 = f.unsqueeze(0) if squeeze else f
                if f3.is_contiguous():
                    self.eng.matvec_device(uc, f3, b, stream=self._stream())
                    return f
            self.eng.matvec_device(uc, fext, b, stream=self._stream())
            out = fext
        elif self.halo == "ghost":
            # the engine reads the owned rows in place and writes f directly
            uc = u3 if u3.is_contiguous() else u3.contiguous()
            self.exchange_ghosts(uc, g)
            self.eng.set_ghosts(g if self.world > 1 else None)
            if f is not None:
                f3 = f.unsqueeze(0) if squeeze else f
                if f3.is_contiguous():
                    self.eng.matvec_device(uc, f3, b, stream=self._stream())
                    return f
            self.eng.matvec_device(uc, fext, b, stream=self._stream())
            out = fext
        else:
            own = slice(self.gl * self.plane, (self.gl + self.R) * self.plane)
            ext[:, :, own].copy_(u3)
            self.exchange(ext)
            self.eng.matvec_device(ext, fext, b, stream=self._stream())
            out = fext[:, :, own]
        if f is None:
            f = out.clone()
        else:
            (f.unsqueeze(0) if squeeze else f).copy_(out)
            return f
        return f[0] if squeeze else f

    # ------------------------------------------------------------ CG
    def _allsum(self, t):
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t

    def dot(self, a, b):
        return self._allsum(torch.sum(a * b).reshape(1))

    def constraint_values(self):
        """(free[dim, R*plane] fp64 0/1 mask, uc[dim, R*plane]) on the owned rows."""
        mask, uc = self.eng.constraint_values()
        g0 = 0 if self.halo == "ghost" else self.gl
        own = slice(g0 * self.plane, (g0 + self.R) * self.plane)
        mask = np.asarray(mask)[own]
        free = np.stack([((mask >> a) & 1) == 0 for a in range(self.dim)]).astype(np.float64)
        uc = np.asarray(uc).reshape(self.dim, -1)[:, own]
        to = lambda x: torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=self.device)  # noqa: E731
        return to(free), to(uc)

    def cg_solve(self, b, tol: float = 1e-10, maxit: int = 10000):
        """Solve K_ff x_f = b_f over all ranks (K := -A on free DOFs, x = u_c on
        constrained ones); b, x: (dim, R*plane) owned rows.  Returns
        (x, iterations, relative residual).  Engine transport: the device CG
        of pdgpu_cg_solve with NCCL-all-reduced dots."""
        if self.transport == "engine":
            bc = b.contiguous()
            x = torch.empty_like(bc)
            it, rel = self.eng.cg_solve_device(bc, x, tol=tol, maxit=maxit, stream=self._stream())
            return x, it, rel
        free, uc = self.constraint_values()
        any_uc = bool(self._allsum(torch.tensor([float(torch.count_nonzero(uc))], dtype=torch.float64,
                                                device=self.device)).item() > 0)
        if any_uc:
            r = free * (b + self.matvec(uc))
        else:
            r = free * b
        x = torch.zeros_like(r)
        p = r.clone()
        rr = self.dot(r, r)
        bnorm = float(rr.sqrt().item())
        k, rel = 0, (1.0 if bnorm > 0 else 0.0)
        while bnorm > 0 and k < maxit:
            q = -free * self.matvec(p)
            alpha = rr / self.dot(p, q)
            x.add_(alpha * p)
            r.sub_(alpha * q)
            rr_new = self.dot(r, r)
            k += 1
            rel = float(rr_new.sqrt().item()) / bnorm
            if rel <= tol:
                break
            p.mul_(rr_new / rr).add_(r)
            rr = rr_new
        if any_uc:
            x.add_(uc)
        return x, k, rel
