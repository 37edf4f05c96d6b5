"""C-ABI boundary checks that need no GPU: libpdgpu.so loads, exports every
entry point include/pdgpu.h declares, and its host-side assembly
(build_kernel, near-surface flags) equals the oracle's restatement of the
reference; error codes map onto the reference's exception names."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle.oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "pdgpu.h")).read()
    return sorted(set(re.findall(r"\b(pdgpu_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2301_11828_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert not [s for s in syms if s not in _lib.SIGNATURES]


def test_version_and_error_string():
    from paper_2301_11828_b200 import _lib
    lib = _lib.load()
    assert b"sm_100a" in lib.pdgpu_version()
    out = C.c_void_p()
    dims = (C.c_int * 2)(4, 4)
    K = np.zeros(3 * 81)
    rc = lib.pdgpu_create(2, dims, 4, K.ctypes.data_as(_lib.c_double_p), 0, C.byref(out))
    assert rc == 1  # PDGPU_ERR_HORIZON_TOO_LARGE, checked before touching the device
    assert b"M+1" in lib.pdgpu_last_error()


@pytest.mark.parametrize("dim,M,delta_over_h", [(2, 3, 3.015), (2, 2, 2.0), (3, 3, 3.015), (3, 4, 4.0)])
def test_build_kernel_matches_oracle(dim, M, delta_over_h):
    from paper_2301_11828_b200 import build_kernel
    h = 0.0025
    K = build_kernel(dim, h, delta_over_h * h, M, 2e11, 0.0025)
    o = Oracle((8,) * dim, h=h, delta=delta_over_h * h, M=M, E=2e11, thickness=0.0025)
    assert np.array_equal(K, o.kernel())  # bit-identical assembly


def test_near_surface_matches_oracle():
    from paper_2301_11828_b200 import near_surface
    for dims, M in (((20, 14), 3), ((9, 7, 8), 2)):
        o = Oracle(dims, h=1.0, M=M)
        ns, _ = o.regions()
        assert np.array_equal(near_surface(dims, M), ns)


def test_band_offsets_order():
    from paper_2301_11828_b200 import band_offsets
    o = Oracle((8, 8), h=1.0, M=3)
    offs = np.zeros((28, 3), dtype=np.int32)
    assert o.L.orc_offsets(2, 3, offs.ctypes.data_as(C.POINTER(C.c_int))) == 28
    assert np.array_equal(band_offsets(2, 3), offs)
    assert len(band_offsets(3, 3)) == 122


@pytest.mark.parametrize("dims", [(64, 8192), (32768, 16), (1024, 1024, 1024), (64, 64, 2048)])
def test_lattice_too_large_is_refused_before_the_device(dims):
    """Transform lengths beyond the instantiated kernels: a clean
    PDGPU_ERR_NOT_SUPPORTED from pdgpu_create, without touching the device."""
    from paper_2301_11828_b200 import _lib
    lib = _lib.load()
    out = C.c_void_p()
    d = (C.c_int * len(dims))(*dims)
    K = np.zeros(6 * 7 ** len(dims))
    rc = lib.pdgpu_create(len(dims), d, 3, K.ctypes.data_as(_lib.c_double_p), 0, C.byref(out))
    assert rc == 7  # PDGPU_ERR_NOT_SUPPORTED
    assert b"too large" in lib.pdgpu_last_error()
