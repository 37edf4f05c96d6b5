"""ctypes wrappers of the CPU checkers.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference legs, never by the product package.

  Oracle     -> oracle/liboracle.so   (plain-C restatement, oracle.c)
  RefProblem -> oracle/_ref/libpdref.so (the reference's own headers compiled
                against oracle/fftw_cpu; present only where it was built)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpdref.so")

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)


def _d(a):
    return a.ctypes.data_as(dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def build():
    """Compile the checkers (liboracle always; _ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_olib = None
_rlib = None


def olib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(HERE, "oracle.c")):
            subprocess.run(["make", "-s", "-C", HERE, ORACLE_SO], check=True)
        L = C.CDLL(ORACLE_SO)
        sig = {
            "orc_rng_new": (C.c_void_p, [C.c_uint32]),
            "orc_rng_free": (None, [C.c_void_p]),
            "orc_rng_next": (C.c_uint32, [C.c_void_p]),
            "orc_rng_uniform": (C.c_double, [C.c_void_p, C.c_double, C.c_double]),
            "orc_rng_fill": (None, [C.c_void_p, C.c_int64, C.c_double, C.c_double, dp]),
            "orc_alpha": (C.c_double, [C.c_double, C.c_double, C.c_int, C.c_double]),
            "orc_critical_stretch": (C.c_double, [C.c_double, C.c_double, C.c_double, C.c_int]),
            "orc_volume_correction": (C.c_double, [C.c_double, C.c_double, C.c_double]),
            "orc_build_kernel": (None, [C.c_int, C.c_double, C.c_double, C.c_int, C.c_double, C.c_double, dp]),
            "orc_offsets": (C.c_int, [C.c_int, C.c_int, ip]),
            "orc_new": (C.c_void_p, [C.c_int, ip, C.c_double, dp, C.c_double, C.c_double, C.c_int, C.c_double,
                                     C.c_double]),
            "orc_free": (None, [C.c_void_p]),
            "orc_get_kernel": (None, [C.c_void_p, dp]),
            "orc_set_kernel": (None, [C.c_void_p, dp]),
            "orc_get_regions": (None, [C.c_void_p, u8p, u8p]),
            "orc_get_de": (None, [C.c_void_p, dp]),
            "orc_add_constraint": (C.c_int, [C.c_void_p, dp, dp, C.c_int, C.c_int, C.c_double]),
            "orc_add_load": (None, [C.c_void_p, dp, dp, dp]),
            "orc_set_body": (None, [C.c_void_p, dp]),
            "orc_break_bond": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64]),
            "orc_total_broken": (C.c_int64, [C.c_void_p]),
            "orc_ledger_pairs": (C.c_int64, [C.c_void_p, i64p, C.c_int64]),
            "orc_random_ledger": (None, [C.c_void_p, C.c_void_p, C.c_int]),
            "orc_random_kernel": (None, [C.c_void_p, C.c_void_p]),
            "orc_apply_fast": (None, [C.c_void_p, dp, dp]),
            "orc_apply_corrections": (None, [C.c_void_p, dp, dp]),
            "orc_matvec": (None, [C.c_void_p, dp, dp]),
            "orc_dense_force": (None, [C.c_void_p, dp, dp]),
            "orc_evaluate_force": (None, [C.c_void_p, dp, dp]),
            "orc_cg": (C.c_int, [C.c_void_p, dp, dp, C.c_double, C.c_int, ip, dp, dp, C.c_int]),
            "orc_cg_rhs": (None, [C.c_void_p, dp, dp]),
            "orc_static_residual": (C.c_double, [C.c_void_p, dp, dp]),
            "orc_bond_stretch": (C.c_double, [C.c_int, dp, dp, dp, dp]),
            "orc_update_bonds": (C.c_int64, [C.c_void_p, dp, C.c_double, dp, i64p, C.c_int64]),
            "orc_seed_segment": (C.c_int64, [C.c_void_p, dp]),
            "orc_seed_notch": (C.c_int64, [C.c_void_p, dp]),
            "orc_sim_init": (None, [C.c_void_p, C.c_double]),
            "orc_sim_set_velocity": (None, [C.c_void_p, dp]),
            "orc_sim_init_adr": (None, [C.c_void_p, C.c_double, C.c_double]),
            "orc_sim_adr_damping": (C.c_double, [C.c_void_p]),
            "orc_sim_adr_mass": (None, [C.c_void_p, dp]),
            "orc_sim_step": (C.c_int64, [C.c_void_p, C.c_double, dp]),
            "orc_sim_get": (None, [C.c_void_p, dp, dp, dp, dp]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _olib = L
    return _olib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def rlib():
    global _rlib
    if _rlib is None:
        if not ref_available():
            raise FileNotFoundError("oracle/_ref/libpdref.so not built (needs /root/reference at build time)")
        L = C.CDLL(REF_SO)
        sig = {
            "ref_rng_new": (C.c_void_p, [C.c_uint32]),
            "ref_rng_free": (None, [C.c_void_p]),
            "ref_rng_next": (C.c_uint32, [C.c_void_p]),
            "ref_rng_uniform": (None, [C.c_void_p, C.c_int64, C.c_double, C.c_double, dp]),
            "ref_new": (C.c_void_p, [C.c_int, ip, C.c_double, dp, C.c_double, C.c_double, C.c_int, C.c_double,
                                     C.c_double]),
            "ref_free": (None, [C.c_void_p]),
            "ref_set_stencils": (None, [C.c_void_p, dp, C.c_int64]),
            "ref_add_constraint": (None, [C.c_void_p, dp, dp, C.c_int, C.c_int, C.c_double]),
            "ref_add_load": (None, [C.c_void_p, dp, dp, dp]),
            "ref_add_crack": (None, [C.c_void_p, dp, C.c_int]),
            "ref_add_bond": (None, [C.c_void_p, C.c_int64, C.c_int64]),
            "ref_finalize": (C.c_int, [C.c_void_p]),
            "ref_get_kernel": (None, [C.c_void_p, dp]),
            "ref_get_regions": (None, [C.c_void_p, u8p, u8p, dp]),
            "ref_matvec": (C.c_int, [C.c_void_p, dp, dp, C.c_int]),
            "ref_imag_residue": (C.c_double, [C.c_void_p]),
            "ref_dense": (None, [C.c_void_p, dp, dp]),
            "ref_ledger_pairs": (C.c_int64, [C.c_void_p, i64p, C.c_int64]),
            "ref_update_bonds": (C.c_int64, [C.c_void_p, dp, C.c_double, dp, i64p, C.c_int64]),
            "ref_bond_stretch": (C.c_double, [C.c_int, dp, dp, dp, dp]),
            "ref_cg": (C.c_int, [C.c_void_p, dp, dp, C.c_double, C.c_int, ip, dp, dp, C.c_int]),
            "ref_sim_init": (C.c_int, [C.c_void_p, C.c_double, C.c_double, dp]),
            "ref_sim_step": (C.c_int64, [C.c_void_p, C.c_int]),
            "ref_sim_init_adr": (C.c_int, [C.c_void_p, C.c_double, C.c_double, dp, C.c_double]),
            "ref_sim_adr_damping": (C.c_double, [C.c_void_p]),
            "ref_sim_get": (None, [C.c_void_p, dp, dp, dp, dp]),
            "ref_bench": (C.c_double, [C.c_void_p, dp, C.c_int64, C.c_int]),
            "ref_random_kernel": (None, [C.c_void_p, C.c_int, C.c_int, C.c_double, dp]),
            "ref_random_field": (None, [C.c_void_p, C.c_int, C.c_int64, C.c_double, dp]),
            "ref_random_ledger": (C.c_int64, [C.c_void_p, C.c_int, ip, C.c_int, C.c_int, i64p, C.c_int64]),
            "ref_tbt_apply_all": (None, [C.c_void_p, dp, dp]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _rlib = L
    return _rlib


class Rng:
    """std::mt19937 + uniform_real_distribution restated (oracle.c); ref=True uses the real libstdc++ one."""

    def __init__(self, seed: int, ref: bool = False):
        self.ref = ref
        self.L = rlib() if ref else olib()
        self.h = (self.L.ref_rng_new if ref else self.L.orc_rng_new)(seed)

    def __del__(self):
        try:
            (self.L.ref_rng_free if self.ref else self.L.orc_rng_free)(self.h)
        except Exception:
            pass

    def next(self) -> int:
        return (self.L.ref_rng_next if self.ref else self.L.orc_rng_next)(self.h)

    def uniform(self, n: int, a: float = -1.0, b: float = 1.0) -> np.ndarray:
        out = np.empty(n)
        if self.ref:
            self.L.ref_rng_uniform(self.h, n, a, b, _d(out))
        else:
            self.L.orc_rng_fill(self.h, n, a, b, _d(out))
        return out


def random_field(rng: Rng, dim: int, n: int, amp: float = 1.0) -> np.ndarray:
    """oracles.hpp:113-119 random_field: (dim, n), component-major."""
    return rng.uniform(dim * n, -amp, amp).reshape(dim, n)


class Oracle:
    """One problem in the C restatement (oracle.c)."""

    def __init__(self, dims, h=1.0, delta=None, M=3, E=1.0, thickness=1.0, rho=1.0, origin=None):
        self.L = olib()
        self.dims = tuple(int(d) for d in dims)
        self.dim = len(self.dims)
        self.n = int(np.prod(self.dims))
        self.M = M
        d = (C.c_int * self.dim)(*self.dims)
        org = _f64(origin if origin is not None else np.zeros(self.dim))
        self.h = self.L.orc_new(self.dim, d, h, _d(org), thickness, M * h if delta is None else delta, M, E, rho)
        self.np = self.dim * (self.dim + 1) // 2
        self.ss = (2 * M + 1) ** self.dim

    def __del__(self):
        try:
            self.L.orc_free(self.h)
        except Exception:
            pass

    def kernel(self):
        K = np.zeros((self.np, self.ss))
        self.L.orc_get_kernel(self.h, _d(K))
        return K

    def set_kernel(self, K):
        self.L.orc_set_kernel(self.h, _d(_f64(K)))

    def random_kernel(self, rng: Rng):
        self.L.orc_random_kernel(self.h, rng.h)

    def random_ledger(self, rng: Rng, tries: int):
        self.L.orc_random_ledger(self.h, rng.h, tries)

    def regions(self):
        ns = np.zeros(self.n, dtype=np.uint8)
        cm = np.zeros(self.n, dtype=np.uint8)
        self.L.orc_get_regions(self.h, ns.ctypes.data_as(u8p), cm.ctypes.data_as(u8p))
        return ns, cm

    def de(self):
        out = np.zeros((self.np, self.n))
        self.L.orc_get_de(self.h, _d(out))
        return out

    def add_constraint(self, lo, hi, mask, kind=0, value=0.0):
        self.L.orc_add_constraint(self.h, _d(_f64(lo)), _d(_f64(hi)), mask, kind, value)

    def add_load(self, lo, hi, value):
        self.L.orc_add_load(self.h, _d(_f64(lo)), _d(_f64(hi)), _d(_f64(value)))

    def set_body(self, body):
        self.L.orc_set_body(self.h, _d(_f64(body)))

    def break_bond(self, p, q):
        return self.L.orc_break_bond(self.h, p, q)

    def seed_segment(self, a, b, width=0.0):
        return self.L.orc_seed_segment(self.h, _d(_f64([a[0], a[1], b[0], b[1], width])))

    def seed_notch(self, axis, plane, width, lo, hi):
        return self.L.orc_seed_notch(self.h, _d(_f64([axis, plane, width, *lo, *hi])))

    def ledger_pairs(self):
        n = self.L.orc_ledger_pairs(self.h, None, 0)
        out = np.zeros((max(n, 1), 2), dtype=np.int64)
        self.L.orc_ledger_pairs(self.h, out.ctypes.data_as(i64p), n)
        return out[:n]

    def _op(self, fn, u):
        u = _f64(u).reshape(self.dim, self.n)
        f = np.zeros_like(u)
        fn(self.h, _d(u), _d(f))
        return f

    def apply(self, u):
        return self._op(self.L.orc_apply_fast, u)

    def matvec(self, u):
        return self._op(self.L.orc_matvec, u)

    def dense(self, u):
        return self._op(self.L.orc_dense_force, u)

    def evaluate_force(self, u):
        return self._op(self.L.orc_evaluate_force, u)

    def cg(self, b, tol=1e-10, maxit=10000, nhist=0):
        b = _f64(b).reshape(self.dim, self.n)
        x = np.zeros_like(b)
        it = C.c_int()
        rel = C.c_double()
        hist = np.zeros((max(nhist, 1), self.dim, self.n)) if nhist else None
        self.L.orc_cg(self.h, _d(b), _d(x), tol, maxit, C.byref(it), C.byref(rel),
                      None if hist is None else _d(hist), nhist)
        return x, it.value, rel.value, hist

    def static_residual(self, b, x):
        return self.L.orc_static_residual(self.h, _d(_f64(b)), _d(_f64(x)))

    def update_bonds(self, u, s0, watch=None, cap=1 << 20):
        w = None if watch is None else _box6(watch, self.dim)
        out = np.zeros((cap, 2), dtype=np.int64)
        n = self.L.orc_update_bonds(self.h, _d(_f64(u)), s0, None if w is None else _d(w),
                                    out.ctypes.data_as(i64p), cap)
        return out[: min(n, cap)]

    def sim_init(self, dt, v0=None):
        self.L.orc_sim_init(self.h, dt)
        if v0 is not None:
            self.L.orc_sim_set_velocity(self.h, _d(_f64(v0)))

    def sim_init_adr(self, dt, fixed_damping=None):
        """Simulation with Integrator::Adr (timestepping.hpp:79-162)."""
        self.L.orc_sim_init_adr(self.h, dt, float("nan") if fixed_damping is None else float(fixed_damping))

    def adr_damping(self):
        return self.L.orc_sim_adr_damping(self.h)

    def adr_mass(self):
        m = np.zeros(3)
        self.L.orc_sim_adr_mass(self.h, _d(m))
        return m[: self.dim]

    def sim_step(self, n=1, s0=-1.0, watch=None):
        w = None if watch is None else _box6(watch, self.dim)
        tot = 0
        for _ in range(n):
            tot += self.L.orc_sim_step(self.h, s0, None if w is None else _d(w))
        return tot

    def sim_get(self):
        u = np.zeros((self.dim, self.n))
        v = np.zeros_like(u)
        f = np.zeros_like(u)
        t = C.c_double()
        self.L.orc_sim_get(self.h, _d(u), _d(v), _d(f), C.byref(t))
        return u, v, f, t.value


class RefProblem:
    """One problem built by the reference's own code (oracle/_ref/libpdref.so)."""

    def __init__(self, dims, h=1.0, delta=None, M=3, E=1.0, thickness=1.0, rho=1.0, origin=None):
        self.L = rlib()
        self.dims = tuple(int(d) for d in dims)
        self.dim = len(self.dims)
        self.n = int(np.prod(self.dims))
        self.M = M
        d = (C.c_int * self.dim)(*self.dims)
        org = _f64(origin if origin is not None else np.zeros(self.dim))
        self.h = self.L.ref_new(self.dim, d, h, _d(org), thickness, M * h if delta is None else delta, M, E, rho)
        self.np = self.dim * (self.dim + 1) // 2
        self.ss = (2 * M + 1) ** self.dim
        self.final = False

    def __del__(self):
        try:
            self.L.ref_free(self.h)
        except Exception:
            pass

    def set_stencils(self, K):
        K = _f64(K)
        self.L.ref_set_stencils(self.h, _d(K), K.size)

    def add_constraint(self, lo, hi, mask, kind=0, value=0.0):
        self.L.ref_add_constraint(self.h, _d(_f64(lo)), _d(_f64(hi)), mask, kind, value)

    def add_load(self, lo, hi, value):
        self.L.ref_add_load(self.h, _d(_f64(lo)), _d(_f64(hi)), _d(_f64(value)))

    def add_segment(self, a, b, width=0.0):
        g = _f64([a[0], a[1], b[0], b[1], width])
        self.L.ref_add_crack(self.h, _d(g), 5)

    def add_notch(self, axis, plane, width, lo, hi):
        g = _f64([axis, plane, width, *lo, *hi])
        self.L.ref_add_crack(self.h, _d(g), 9)

    def add_bond(self, p, q):
        self.L.ref_add_bond(self.h, p, q)

    def finalize(self):
        rc = self.L.ref_finalize(self.h)
        if rc:
            raise RuntimeError(f"reference finalize failed ({rc})")
        self.final = True

    def kernel(self):
        K = np.zeros((self.np, self.ss))
        self.L.ref_get_kernel(self.h, _d(K))
        return K

    def regions(self):
        ns = np.zeros(self.n, dtype=np.uint8)
        cm = np.zeros(self.n, dtype=np.uint8)
        de = np.zeros((self.np, self.n))
        self.L.ref_get_regions(self.h, ns.ctypes.data_as(u8p), cm.ctypes.data_as(u8p), _d(de))
        return ns, cm, de

    def apply(self, u):
        u = _f64(u).reshape(self.dim, self.n)
        f = np.zeros_like(u)
        self.L.ref_matvec(self.h, _d(u), _d(f), 0)
        return f

    def matvec(self, u):
        u = _f64(u).reshape(self.dim, self.n)
        f = np.zeros_like(u)
        rc = self.L.ref_matvec(self.h, _d(u), _d(f), 1)
        if rc == 3:
            raise ValueError("LedgerOutOfBand")
        return f

    def imag_residue(self):
        return self.L.ref_imag_residue(self.h)

    def dense(self, u):
        u = _f64(u).reshape(self.dim, self.n)
        f = np.zeros_like(u)
        self.L.ref_dense(self.h, _d(u), _d(f))
        return f

    def ledger_pairs(self):
        n = self.L.ref_ledger_pairs(self.h, None, 0)
        out = np.zeros((max(n, 1), 2), dtype=np.int64)
        self.L.ref_ledger_pairs(self.h, out.ctypes.data_as(i64p), n)
        return out[:n]

    def update_bonds(self, u, s0, watch=None, cap=1 << 20):
        w = None if watch is None else _f64(np.concatenate([watch[0], watch[1]]))
        out = np.zeros((cap, 2), dtype=np.int64)
        n = self.L.ref_update_bonds(self.h, _d(_f64(u)), s0, None if w is None else _d(w),
                                    out.ctypes.data_as(i64p), cap)
        return out[: min(n, cap)]

    def cg(self, b, tol=1e-10, maxit=10000, nhist=0):
        b = _f64(b).reshape(self.dim, self.n)
        x = np.zeros_like(b)
        it = C.c_int()
        rel = C.c_double()
        hist = np.zeros((max(nhist, 1), self.dim, self.n)) if nhist else None
        self.L.ref_cg(self.h, _d(b), _d(x), tol, maxit, C.byref(it), C.byref(rel),
                      None if hist is None else _d(hist), nhist)
        return x, it.value, rel.value, hist

    def sim_init(self, dt, s0=-1.0, watch=None):
        w = None if watch is None else _f64(np.concatenate([watch[0], watch[1]]))
        self.L.ref_sim_init(self.h, dt, s0, None if w is None else _d(w))

    def sim_init_adr(self, dt, s0=-1.0, watch=None, fixed_damping=None):
        w = None if watch is None else _box6(watch, self.dim)
        self.L.ref_sim_init_adr(self.h, dt, s0, None if w is None else _d(w),
                                float("nan") if fixed_damping is None else float(fixed_damping))

    def adr_damping(self):
        return self.L.ref_sim_adr_damping(self.h)

    def sim_step(self, n=1):
        return self.L.ref_sim_step(self.h, n)

    def sim_get(self):
        u = np.zeros((self.dim, self.n))
        v = np.zeros_like(u)
        f = np.zeros_like(u)
        t = C.c_double()
        self.L.ref_sim_get(self.h, _d(u), _d(v), _d(f), C.byref(t))
        return u, v, f, t.value

    def bench(self, u_batch, threads):
        u = _f64(u_batch)
        nvec = u.shape[0]
        return self.L.ref_bench(self.h, _d(u), nvec, threads)


def _box6(watch, dim):
    """oracle.c boxes are {lo[0..3), hi[0..3)} regardless of dim."""
    b = np.zeros(6)
    b[:dim] = np.asarray(watch[0], dtype=np.float64)[:dim]
    b[3:3 + dim] = np.asarray(watch[1], dtype=np.float64)[:dim]
    return b
