"""Python host mirror of the reference `pdfast` operator API over libpdgpu.

Names, argument meaning and error behaviour follow the reference
(proj/include/pdfast/*.hpp); all compute goes through the C ABI
(include/pdgpu.h) into the sm_100a kernels.  Host arrays are numpy fp64 in
the reference layout (component-major SoA, node p = (k*Ny + j)*Nx + i);
device arrays are torch CUDA tensors of the same layout (batched
[batch][dim][N]).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


class Error(RuntimeError):
    """pdfast::Error (errors.hpp:8-10)."""


class HorizonTooLargeForGrid(Error):
    """errors.hpp:21-23; raised by the engine ctor (convolution.hpp:61-62)."""


class ShapeMismatch(Error):
    """errors.hpp:24-26; field length != lattice size (convolution.hpp:120-121)."""


class LedgerOutOfBand(Error):
    """errors.hpp:27-29; broken bond outside the band (corrections.hpp:99-100)."""


class CudaError(Error):
    pass


class IoError(Error):
    """pdfast::IoError (errors.hpp:33-35)"""


_CODES = {1: HorizonTooLargeForGrid, 2: ShapeMismatch, 3: LedgerOutOfBand, 4: ValueError, 5: CudaError,
          6: MemoryError, 7: NotImplementedError, 8: IoError}


def _check(rc: int):
    if rc != 0:
        lib = _lib.load()
        msg = lib.pdgpu_last_error().decode()
        raise _CODES.get(rc, Error)(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_lib.c_double_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def n_pairs(dim: int) -> int:
    """kernel.hpp:14-15"""
    return dim * (dim + 1) // 2


def pair_index(dim: int, a: int, b: int) -> int:
    """kernel.hpp:19-28"""
    if a > b:
        a, b = b, a
    if dim == 2:
        return a + b
    return (0, 3, 5)[a] + b - a


def band_offsets(dim: int, M: int) -> np.ndarray:
    """In-band off-centre offsets in KernelStack::for_each_offset order (kernel.hpp:71-89)."""
    out = []
    zr = M if dim == 3 else 0
    for a in range(-M, M + 1):
        for b in range(-M, M + 1):
            for c in range(-zr, zr + 1):
                n2 = a * a + b * b + c * c
                if 0 < n2 <= M * M:
                    out.append((a, b, c))
    return np.array(out, dtype=np.int64).reshape(-1, 3)


def build_kernel(dim: int, h: float, delta: float, M: int, E: float, thickness: float = 0.0) -> np.ndarray:
    """build_kernel (kernel.hpp:99-127) -> (n_pairs, (2M+1)^dim) stencils, KernelStack storage order."""
    lib = _lib.load()
    out = np.zeros((n_pairs(dim), (2 * M + 1) ** dim))
    _check(lib.pdgpu_build_kernel(dim, h, delta, M, E, thickness, _dp(out)))
    return out


def near_surface(dims, M: int) -> np.ndarray:
    """Regions near-surface flags (grid.hpp:181-189)."""
    lib = _lib.load()
    dims_a = (C.c_int * len(dims))(*dims)
    out = np.zeros(int(np.prod(dims)), dtype=np.uint8)
    _check(lib.pdgpu_near_surface(len(dims), dims_a, M, out.ctypes.data_as(_lib.c_uint8_p)))
    return out


class FastForce:
    """GPU counterpart of pdfast::FastForce<Dim> (convolution.hpp:237-274),
    extended with the correction, fracture and solver state the reference
    keeps in Simulation (timestepping.hpp:167-351).

    FastForce(dims, M, stencils) mirrors FastForce(grid, hz, K): dims =
    Grid::dims, M = Horizon::M, stencils = KernelStack components.
    """

    def __init__(self, dims, M: int, stencils: np.ndarray, device: int = 0):
        self._lib = _lib.load()
        self.dims = tuple(int(d) for d in dims)
        self.dim = len(self.dims)
        self.M = int(M)
        self.n = int(np.prod(self.dims))
        st = _f64(stencils).reshape(-1)
        if st.size != n_pairs(self.dim) * (2 * M + 1) ** self.dim:
            raise ValueError("stencils must be n_pairs x (2M+1)^dim")
        dims_a = (C.c_int * self.dim)(*self.dims)
        h = C.c_void_p()
        _check(self._lib.pdgpu_create(self.dim, dims_a, self.M, _dp(st), device, C.byref(h)))
        self._h = h
        self._geom = (1.0, np.zeros(self.dim))

    # ------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._lib.pdgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    # ---------------------------------------------------------- geometry
    def set_geometry(self, h: float, origin=None, delta: float = 0.0, rho: float = 1.0):
        org = _f64(origin if origin is not None else np.zeros(self.dim))
        self._geom = (float(h), org.copy())
        _check(self._lib.pdgpu_set_geometry(self._h, h, _dp(org), delta, rho))

    # ------------------------------------------------------ spectral apply
    def apply(self, u: np.ndarray) -> np.ndarray:
        """FastForce::apply (convolution.hpp:249-259) on host fields (dim, N) or (B, dim, N)."""
        u = _f64(u)
        n_nodes = u.shape[-1]
        batch = max(u.size // max(self.dim * n_nodes, 1), 1)
        f = np.empty_like(u)
        _check(self._lib.pdgpu_apply_host(self._h, _dp(u), _dp(f), n_nodes, batch))
        return f

    def apply_device(self, u, f, batch: int = 1, stream=None):
        """Device pointers / torch tensors, layout [batch][dim][N]."""
        _check(self._lib.pdgpu_apply(self._h, _ptr(u), _ptr(f), batch, _stream(stream, u, f)))

    def apply_direct_device(self, u, f, batch: int = 1, stream=None):
        """FastForce::apply by direct stencil summation on the device (cross-check
        of apply_device; the reference oracle's tbt_apply_all)."""
        _check(self._lib.pdgpu_apply_direct(self._h, _ptr(u), _ptr(f), batch, _stream(stream, u, f)))

    def last_imag_residue(self) -> float:
        """FastForce::last_imag_residue (convolution.hpp:261).  Always 0.0: the
        R2C/C2R transforms never form an imaginary part of the output."""
        return self._lib.pdgpu_last_imag_residue(self._h)

    def footprint_bytes(self) -> int:
        return self._lib.pdgpu_footprint_bytes(self._h)

    PASSES = ("K1_rfft_x", "K2_fft_y", "K3_spectral", "K4_ifft_y", "K5_irfft_x", "K6_surface_wrap", "K6_bonds", "vec",
              "halo_exchange")

    def timing(self, on: bool = True):
        _check(self._lib.pdgpu_timing_enable(self._h, 1 if on else 0))

    def timing_read(self):
        """{pass name: (total ms, launches)} since the last read (CUDA events on the launching stream)."""
        npass = len(self.PASSES)
        ms = np.zeros(npass)
        cnt = np.zeros(npass, dtype=np.int64)
        _check(self._lib.pdgpu_timing_read(self._h, _dp(ms), cnt.ctypes.data_as(_lib.c_int64_p), npass))
        return {n: (float(ms[i]), int(cnt[i])) for i, n in enumerate(self.PASSES) if cnt[i]}

    def launch_count(self) -> int:
        return int(self._lib.pdgpu_launch_count(self._h))

    def symbol_is_real(self) -> bool:
        return bool(self._lib.pdgpu_symbol_is_real(self._h))

    def embedding(self) -> int:
        """Bit d set: axis d uses the periodic embedding (P = N + wrap correction)."""
        return int(self._lib.pdgpu_embedding(self._h))

    def symbol_mode(self) -> str:
        """'complex-table' | 'real-table' | 'separable' (per-column coefficients)."""
        return ("complex-table", "real-table", "separable")[self._lib.pdgpu_symbol_mode(self._h)]

    def symbol_stream_bytes(self) -> int:
        """Bytes of symbol table the 2D spectral pass reads per launch (the full
        table, or the mirror planes over ky in [0, Pl/2])."""
        return int(self._lib.pdgpu_symbol_stream_bytes(self._h))

    # --------------------------------------------------------- corrections
    def set_regions(self, near_surface=None, constraint_mask=None):
        ns = None if near_surface is None else np.ascontiguousarray(near_surface, dtype=np.uint8)
        cm = None if constraint_mask is None else np.ascontiguousarray(constraint_mask, dtype=np.uint8)
        _check(self._lib.pdgpu_set_regions(self._h, None if ns is None else ns.ctypes.data_as(_lib.c_uint8_p),
                                           None if cm is None else cm.ctypes.data_as(_lib.c_uint8_p)))

    def set_slab(self, global_rows: int, row_offset: int):
        """This lattice is rows [row_offset, row_offset + dims[-1]) of one with
        `global_rows` rows along the slowest axis (halo slab decomposition):
        near-surface flags and D^e follow the global faces."""
        _check(self._lib.pdgpu_set_slab(self._h, int(global_rows), int(row_offset)))

    def set_ghosts(self, ghosts):
        """Ghost rows of the interior slab faces (device tensor [batch][dim][2][M][plane]) or None."""
        _check(self._lib.pdgpu_set_ghosts(self._h, None if ghosts is None else _ptr(ghosts)))
        self._ghosts = ghosts  # keep the buffer alive while the engine may read it

    def set_ghosts_strided(self, ghosts, vec_comp_stride: int, side_stride: int):
        """Ghost rows with an explicit layout (pdgpu_set_ghosts_strided), e.g. the
        receive buffer of a halo exchange [2][batch][dim][M][plane]."""
        _check(self._lib.pdgpu_set_ghosts_strided(self._h, None if ghosts is None else _ptr(ghosts),
                                                  int(vec_comp_stride), int(side_stride)))
        self._ghosts = ghosts

    def halo_pack(self, u, send, batch: int = 1, stream=None):
        """send[2][batch][dim][M][plane] <- the first / last M owned rows of u (pdgpu_halo_pack)."""
        _check(self._lib.pdgpu_halo_pack(self._h, _ptr(u), batch, _ptr(send), _stream(stream, u, send)))

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        """Attach an NCCL communicator (pdgpu_comm_init): from then on every K.u
        exchanges the halo rows with rank -+ 1 and CG all-reduces its dots."""
        buf = C.create_string_buffer(bytes(uid), 128)
        _check(self._lib.pdgpu_comm_init(self._h, int(nranks), int(rank), buf))

    @staticmethod
    def comm_unique_id() -> bytes:
        """ncclGetUniqueId (pdgpu_comm_unique_id): 128 bytes to broadcast to every rank."""
        lib = _lib.load()
        buf = C.create_string_buffer(128)
        _check(lib.pdgpu_comm_unique_id(buf))
        return buf.raw

    def constraint_values(self):
        """(mask[N] uint8 constrained-direction bits, uc[dim, N] prescribed
        displacements) -- what cg_solve masks with and shifts by."""
        mask = np.zeros(self.n, dtype=np.uint8)
        uc = np.zeros((self.dim, self.n))
        _check(self._lib.pdgpu_constraint_values(self._h, mask.ctypes.data_as(_lib.c_uint8_p), _dp(uc)))
        return mask, uc

    def set_surface_diag(self, de: np.ndarray):
        de = _f64(de)
        _check(self._lib.pdgpu_set_surface_diag(self._h, _dp(de)))

    def set_ledger(self, row_start: np.ndarray, partners: np.ndarray):
        rs = np.ascontiguousarray(row_start, dtype=np.int64)
        pt = np.ascontiguousarray(partners, dtype=np.int64)
        if pt.size == 0:
            pt = np.zeros(1, dtype=np.int64)
        _check(self._lib.pdgpu_set_ledger(self._h, rs.ctypes.data_as(_lib.c_int64_p), pt.ctypes.data_as(_lib.c_int64_p)))

    def break_bonds(self, pairs):
        pr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
        _check(self._lib.pdgpu_break_bonds(self._h, pr.ctypes.data_as(_lib.c_int64_p), pr.shape[0]))

    def ledger_pairs(self) -> np.ndarray:
        cnt = C.c_int64()
        _check(self._lib.pdgpu_ledger_pairs(self._h, None, 0, C.byref(cnt)))
        out = np.zeros((max(cnt.value, 1), 2), dtype=np.int64)
        _check(self._lib.pdgpu_ledger_pairs(self._h, out.ctypes.data_as(_lib.c_int64_p), cnt.value, C.byref(cnt)))
        return out[: cnt.value]

    def matvec(self, u: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """FastForce::apply + apply_corrections (corrections.hpp:76-110) on host fields."""
        u = _f64(u)
        batch = max(u.size // max(self.dim * u.shape[-1], 1), 1)
        f = np.empty_like(u) if out is None else out
        if f.dtype != np.float64 or not f.flags.c_contiguous or f.shape != u.shape:
            raise ValueError("out must be a C-contiguous float64 array shaped like u")
        _check(self._lib.pdgpu_matvec_host(self._h, _dp(u), _dp(f), u.shape[-1], batch))
        return f

    def matvec_device(self, u, f, batch: int = 1, stream=None):
        _check(self._lib.pdgpu_matvec(self._h, _ptr(u), _ptr(f), batch, _stream(stream, u, f)))

    def apply_corrections_device(self, u, f, batch: int = 1, stream=None):
        _check(self._lib.pdgpu_apply_corrections(self._h, _ptr(u), _ptr(f), batch, _stream(stream, u, f)))

    def evaluate_force_device(self, u, f, stream=None):
        _check(self._lib.pdgpu_evaluate_force(self._h, _ptr(u), _ptr(f), _stream(stream, u, f)))

    # ------------------------------------------------------------- problem
    def add_constraint(self, lo, hi, dir_mask: int, kind: int = 0, value: float = 0.0):
        _check(self._lib.pdgpu_add_constraint(self._h, _dp(_f64(lo)), _dp(_f64(hi)), int(dir_mask), int(kind),
                                              float(value)))

    def add_load(self, lo, hi, value):
        _check(self._lib.pdgpu_add_load(self._h, _dp(_f64(lo)), _dp(_f64(hi)), _dp(_f64(value))))

    def set_body(self, body: np.ndarray):
        _check(self._lib.pdgpu_set_body(self._h, _dp(_f64(body))))

    def seed_segment(self, a, b, width: float = 0.0) -> int:
        seg = _f64([a[0], a[1], b[0], b[1], width])
        added = C.c_int64()
        _check(self._lib.pdgpu_seed_segment(self._h, _dp(seg), C.byref(added)))
        return added.value

    def seed_notch(self, axis: int, plane: float, width: float, lo, hi) -> int:
        nt = _f64([axis, plane, width, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]])
        added = C.c_int64()
        _check(self._lib.pdgpu_seed_notch(self._h, _dp(nt), C.byref(added)))
        return added.value

    # ------------------------------------------------------------ fracture
    def update_bonds(self, u, s0: float, watch=None, cap: int = 1 << 20) -> np.ndarray:
        """update_bonds (fracture.hpp:204-231); u is a device tensor [dim][N]."""
        w = None if watch is None else _f64(np.concatenate([np.asarray(watch[0]), np.asarray(watch[1])]))
        out = np.zeros((cap, 2), dtype=np.int64)
        cnt = C.c_int64()
        if getattr(u, "is_cuda", False):  # the sweep runs on the engine stream: order it after u's producers
            import torch
            torch.cuda.current_stream(u.device).synchronize()
        _check(self._lib.pdgpu_update_bonds(self._h, _ptr(u), float(s0), None if w is None else _dp(w),
                                            out.ctypes.data_as(_lib.c_int64_p), cap, C.byref(cnt)))
        return out[: min(cnt.value, cap)]

    # ------------------------------------------------------------------ CG
    def cg_solve(self, b: np.ndarray, tol: float = 1e-10, maxit: int = 10000, nhist: int = 0):
        b = _f64(b)
        x = np.empty_like(b)
        it = C.c_int()
        rel = C.c_double()
        hist = np.zeros((max(nhist, 1),) + b.shape) if nhist else None
        _check(self._lib.pdgpu_cg_solve_host(self._h, _dp(b), _dp(x), tol, maxit, C.byref(it), C.byref(rel),
                                             None if hist is None else _dp(hist), nhist))
        return x, it.value, rel.value, hist

    def set_transpose(self, nranks: int, rank: int, global_rows: int, row_bounds=None, col_bounds=None):
        """Distributed-FFT arm (pdgpu_set_transpose): this engine holds rows
        row_bounds[rank]..row_bounds[rank+1] of an Nx x global_rows lattice and
        the half-spectrum columns col_bounds[rank]..; balanced splits by default."""
        rb, cb = transpose_splits(self.dims[0], global_rows, nranks)
        rb = rb if row_bounds is None else [int(x) for x in row_bounds]
        cb = cb if col_bounds is None else [int(x) for x in col_bounds]
        _check(self._lib.pdgpu_set_transpose(self._h, int(nranks), int(rank), int(global_rows),
                                             (C.c_int * len(rb))(*rb), (C.c_int * len(cb))(*cb)))

    def cg_operator(self, kind: str = "msbfm"):
        """CG's operator: "msbfm" (default) or "direct" (the direct stencil sum of the same K)."""
        if kind not in ("msbfm", "direct"):
            raise ValueError(kind)
        _check(self._lib.pdgpu_set_cg_operator(self._h, 1 if kind == "direct" else 0))

    def cg_solve_device(self, b, x, tol: float = 1e-10, maxit: int = 10000, stream=None):
        it = C.c_int()
        rel = C.c_double()
        _check(self._lib.pdgpu_cg_solve(self._h, _ptr(b), _ptr(x), tol, maxit, C.byref(it), C.byref(rel),
                                        _stream(stream, b, x)))
        return it.value, rel.value

    # ------------------------------------------------------------------ VV
    def sim_init(self, dt: float, v0=None):
        _check(self._lib.pdgpu_sim_init(self._h, dt, None if v0 is None else _dp(_f64(v0))))

    def sim_init_adr(self, dt: float, fixed_damping=None):
        """Simulation with Integrator::Adr (timestepping.hpp:79-162); None = adaptive damping."""
        _check(self._lib.pdgpu_sim_init_adr(self._h, dt, float("nan") if fixed_damping is None else float(fixed_damping)))

    def adr_damping(self) -> float:
        """Simulation::adr_damping(): damping of the last ADR step."""
        c = C.c_double()
        _check(self._lib.pdgpu_sim_adr_damping(self._h, C.byref(c)))
        return c.value

    def sim_step(self, n_steps: int = 1, s0: float = -1.0, watch=None) -> int:
        w = None if watch is None else _f64(np.concatenate([np.asarray(watch[0]), np.asarray(watch[1])]))
        nb = C.c_int64()
        _check(self._lib.pdgpu_sim_step(self._h, n_steps, s0, None if w is None else _dp(w), C.byref(nb)))
        return nb.value

    def sim_newly_broken(self) -> np.ndarray:
        """Simulation::newly_broken() (timestepping.hpp:273): pairs broken in the last step."""
        cnt = C.c_int64()
        _check(self._lib.pdgpu_sim_newly_broken(self._h, None, 0, C.byref(cnt)))
        out = np.zeros((max(cnt.value, 1), 2), dtype=np.int64)
        _check(self._lib.pdgpu_sim_newly_broken(self._h, out.ctypes.data_as(_lib.c_int64_p), cnt.value, C.byref(cnt)))
        return out[: cnt.value]

    def sim_finite(self) -> bool:
        """Simulation::finite() (timestepping.hpp:256-261), evaluated on the device."""
        ok = C.c_int()
        _check(self._lib.pdgpu_sim_finite(self._h, C.byref(ok)))
        return bool(ok.value)

    def sim_monitor(self, nodes):
        """Record u at `nodes` after every sim_step step on the device (MonitorWriter rows)."""
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        _check(self._lib.pdgpu_sim_monitor(self._h, nodes.ctypes.data_as(_lib.c_int64_p), len(nodes)))
        self._mon_n = len(nodes)

    def sim_monitor_read(self):
        """Drain the recorded rows: (steps[k], t[k], values[k, node, dim])."""
        cnt = C.c_int64()
        _check(self._lib.pdgpu_sim_monitor_read(self._h, None, None, None, 0, C.byref(cnt)))
        k = cnt.value
        steps = np.zeros(max(k, 1), dtype=np.int64)
        t = np.zeros(max(k, 1))
        vals = np.zeros((max(k, 1), getattr(self, "_mon_n", 0), self.dim))
        _check(self._lib.pdgpu_sim_monitor_read(self._h, steps.ctypes.data_as(_lib.c_int64_p), _dp(t), _dp(vals), k,
                                                C.byref(cnt)))
        return steps[:k], t[:k], vals[:k]

    def write_snapshot(self, directory: str, u: np.ndarray, step: int, t: float, damage=None) -> str:
        """write_snapshot_dat (output.hpp:76-102) of host field u (dim, N) on this lattice/geometry."""
        return write_snapshot(directory, self.dims, self._geom[0], self._geom[1], u, step, t, damage)

    def sim_get(self):
        u = np.zeros((self.dim, self.n))
        v = np.zeros_like(u)
        f = np.zeros_like(u)
        t = C.c_double()
        _check(self._lib.pdgpu_sim_get(self._h, _dp(u), _dp(v), _dp(f), C.byref(t)))
        return u, v, f, t.value


def transpose_splits(nx: int, global_rows: int, nranks: int):
    """Balanced row and half-spectrum column splits of the distributed-FFT arm."""
    hx = nx // 2 + 1
    return ([global_rows * g // nranks for g in range(nranks + 1)], [hx * g // nranks for g in range(nranks + 1)])


def group_matvec_transpose(engines, us, fs, batch: int = 1):
    """One K.u over n engines of one process (pdgpu_group_matvec_transpose);
    us / fs: per-engine device tensors [batch][dim][own rows * Nx]."""
    lib = _lib.load()
    n = len(engines)
    hs = (C.c_void_p * n)(*[e.handle for e in engines])
    up = (C.c_void_p * n)(*[_ptr(u) for u in us])
    fp = (C.c_void_p * n)(*[_ptr(f) for f in fs])
    _check(lib.pdgpu_group_matvec_transpose(hs, n, up, fp, int(batch)))


def group_sim_step(engines, n_steps: int = 1, s0: float = -1.0, watch=None) -> int:
    """pdgpu_group_sim_step: n engines holding consecutive row slabs of one
    lattice (set_slab), stepped together in one process -- halo rows and the
    face ledgers move by device copies (the single-process counterpart of the
    NCCL slab path).  Returns the bonds broken over all slabs."""
    lib = _lib.load()
    hs = (C.c_void_p * len(engines))(*[e.handle for e in engines])
    dim = engines[0].dim
    w = None if watch is None else _f64(np.concatenate([np.asarray(watch[0]), np.asarray(watch[1])]))
    nb = C.c_int64()
    _check(lib.pdgpu_group_sim_step(hs, len(engines), int(n_steps), float(s0), None if w is None else _dp(w),
                                    C.byref(nb)))
    del dim
    return nb.value


def write_snapshot(directory: str, dims, h: float, origin, u: np.ndarray, step: int, t: float, damage=None) -> str:
    """write_snapshot_dat (output.hpp:76-102): directory/snap_%07d.dat, %.17g values; returns the path."""
    lib = _lib.load()
    dim = len(dims)
    n = int(np.prod(dims))
    u = _f64(u).reshape(dim, n)
    org = _f64(origin if origin is not None else np.zeros(dim))
    d = None if damage is None else _f64(damage)
    buf = C.create_string_buffer(4096)
    _check(lib.pdgpu_write_snapshot(dim, (C.c_int * dim)(*dims), float(h), _dp(org), _dp(u),
                                    None if d is None else _dp(d), int(step), float(t), directory.encode(), buf, 4096))
    return buf.value.decode()


class MonitorWriter:
    """pdfast::MonitorWriter<Dim> (output.hpp:45-72) on the library's host writer:
    MonitorWriter(path, dims, h, origin, points); .nodes; .append(step, t, u)
    with a host field u (dim, N); .append_sim(engine) writes the rows an engine
    recorded on the device since the last call (FastForce.sim_monitor)."""

    def __init__(self, path: str, dims, h: float, origin, points):
        self.dims = tuple(int(d) for d in dims)
        self.dim = len(self.dims)
        pts = _f64(points).reshape(-1, self.dim)
        d = (C.c_int * self.dim)(*self.dims)
        self.nodes = np.zeros(len(pts), dtype=np.int64)
        lib = _lib.load()
        _check(lib.pdgpu_monitor_nodes(self.dim, d, float(h), _dp(_f64(origin)), _dp(pts), len(pts),
                                       self.nodes.ctypes.data_as(_lib.c_int64_p)))
        self._h = C.c_void_p()
        _check(lib.pdgpu_monitor_open(path.encode() if path else None, self.dim, d, float(h), _dp(_f64(origin)),
                                      _dp(pts), len(pts), C.byref(self._h)))
        self._lib = lib

    def append(self, step: int, t: float, u: np.ndarray):
        u = np.asarray(u).reshape(self.dim, -1)
        vals = _f64(u[:, self.nodes].T)
        _check(self._lib.pdgpu_monitor_append(self._h, int(step), float(t), _dp(vals)))

    def append_sim(self, engine: "FastForce") -> int:
        steps, ts, vals = engine.sim_monitor_read()
        for s_, t_, v_ in zip(steps, ts, vals):
            _check(self._lib.pdgpu_monitor_append(self._h, int(s_), float(t_), _dp(_f64(v_))))
        return len(steps)

    def close(self):
        if self._h:
            self._lib.pdgpu_monitor_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_snapshot(path: str, dim: int):
    """read_snapshot_dat (output.hpp:116-154) -> dict(dims, h, origin, step, t, u[dim, N], damage[N])."""
    lib = _lib.load()
    dims = (C.c_int * 3)()
    h = C.c_double()
    org = np.zeros(3)
    step = C.c_int64()
    t = C.c_double()
    p = path.encode()
    _check(lib.pdgpu_read_snapshot(p, dim, dims, C.byref(h), _dp(org), C.byref(step), C.byref(t), None, None))
    n = int(np.prod([dims[d] for d in range(dim)]))
    u = np.zeros((dim, n))
    dmg = np.zeros(n)
    _check(lib.pdgpu_read_snapshot(p, dim, dims, C.byref(h), _dp(org), C.byref(step), C.byref(t), _dp(u), _dp(dmg)))
    return {"dims": tuple(dims[d] for d in range(dim)), "h": h.value, "origin": org[:dim].copy(),
            "step": step.value, "t": t.value, "u": u, "damage": dmg}


def _ptr(x) -> int:
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    raise TypeError("expected a device pointer or a CUDA tensor")


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy default stream's explicit handle


def _stream(s, *tensors):
    """Stream for a device entry point.

    s = None: when any argument is a torch CUDA tensor, the caller's current
    torch stream on that tensor's device, so the engine is ordered after the
    torch kernels that produced its inputs and before those that consume its
    outputs; with raw pointers only, the engine's own stream.  A torch stream
    (or raw handle) -> that stream.  Torch's default stream has handle 0, which
    the C ABI reads as "engine stream", so it is passed as cudaStreamLegacy.

    One engine must not be driven from two streams at once: its spectral
    workspace and reduction scratch are shared by every entry point."""
    if s is None:
        dev = next((t.device for t in tensors if getattr(t, "is_cuda", False)), None)
        if dev is None:
            return None
        import torch
        s = torch.cuda.current_stream(dev)
    h = s.cuda_stream if hasattr(s, "cuda_stream") else int(s)
    return h if h else _CUDA_STREAM_LEGACY


class Convolver:
    """Single-pair spectral convolution, the reference's Convolver<Dim>
    (convolution.hpp:210-230): f = sum_o K_ab(o) u[p + o] over the lattice
    (zero outside), one scalar field in and out.  Built on the same engine as
    FastForce: a stencil stack holding only pair (a, b), the input placed in
    component b, the result read from component a."""

    def __init__(self, dims, M: int, stencils: np.ndarray, a: int = 0, b: int = 0, device: int = 0):
        dims = tuple(int(d) for d in dims)
        dim = len(dims)
        npairs = dim * (dim + 1) // 2
        side = 2 * M + 1
        K = np.asarray(stencils, dtype=np.float64).reshape(npairs, side ** dim)
        pr = pair_index(dim, a, b)
        only = np.zeros_like(K)
        only[pr] = K[pr]
        self.dim, self.a, self.b = dim, int(a), int(b)
        self.n = int(np.prod(dims))
        self._ff = FastForce(dims, M, only, device=device)

    def apply(self, u: np.ndarray) -> np.ndarray:
        """Convolver::apply(u, f) (convolution.hpp:217-221); u, f: N-vectors."""
        x = np.zeros((self.dim, self.n))
        x[self.b] = np.asarray(u, dtype=np.float64).reshape(self.n)
        return self._ff.apply(x)[self.a].copy()

    def last_imag_residue(self) -> float:
        return self._ff.last_imag_residue()

    def close(self):
        self._ff.close()
