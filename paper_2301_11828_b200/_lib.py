"""ctypes binding of libpdgpu.so (C ABI declared in include/pdgpu.h).

The product path has no fallback: if the CUDA library cannot be built or
loaded, import of the engine fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

_lock = threading.Lock()
_lib = None

c_int_p = C.POINTER(C.c_int)
c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)
c_uint8_p = C.POINTER(C.c_uint8)

# name -> (restype, argtypes); mirrors include/pdgpu.h
SIGNATURES = {
    "pdgpu_last_error": (C.c_char_p, []),
    "pdgpu_version": (C.c_char_p, []),
    "pdgpu_create": (C.c_int, [C.c_int, c_int_p, C.c_int, c_double_p, C.c_int, C.POINTER(C.c_void_p)]),
    "pdgpu_destroy": (None, [C.c_void_p]),
    "pdgpu_set_geometry": (C.c_int, [C.c_void_p, C.c_double, c_double_p, C.c_double, C.c_double]),
    "pdgpu_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "pdgpu_apply_direct": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "pdgpu_apply_host": (C.c_int, [C.c_void_p, c_double_p, c_double_p, C.c_int64, C.c_int]),
    "pdgpu_last_imag_residue": (C.c_double, [C.c_void_p]),
    "pdgpu_footprint_bytes": (C.c_size_t, [C.c_void_p]),
    "pdgpu_n_nodes": (C.c_int64, [C.c_void_p]),
    "pdgpu_symbol_is_real": (C.c_int, [C.c_void_p]),
    "pdgpu_symbol_mode": (C.c_int, [C.c_void_p]),
    "pdgpu_symbol_stream_bytes": (C.c_size_t, [C.c_void_p]),
    "pdgpu_embedding": (C.c_int, [C.c_void_p]),
    "pdgpu_set_ghosts": (C.c_int, [C.c_void_p, C.c_void_p]),
    "pdgpu_set_ghosts_strided": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64]),
    "pdgpu_halo_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "pdgpu_comm_unique_id": (C.c_int, [C.c_void_p]),
    "pdgpu_comm_init": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "pdgpu_slab_rows": (C.c_int, [C.c_int, C.c_int, C.c_int, c_int_p, c_int_p]),
    "pdgpu_set_regions": (C.c_int, [C.c_void_p, c_uint8_p, c_uint8_p]),
    "pdgpu_set_surface_diag": (C.c_int, [C.c_void_p, c_double_p]),
    "pdgpu_set_slab": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "pdgpu_write_snapshot": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_double, c_double_p, c_double_p, c_double_p,
                                       C.c_int64, C.c_double, C.c_char_p, C.c_char_p, C.c_int]),
    "pdgpu_monitor_open": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_int), C.c_double, c_double_p, c_double_p,
                                     C.c_int, C.POINTER(C.c_void_p)]),
    "pdgpu_monitor_nodes": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_double, c_double_p, c_double_p, C.c_int,
                                      c_int64_p]),
    "pdgpu_monitor_append": (C.c_int, [C.c_void_p, C.c_int64, C.c_double, c_double_p]),
    "pdgpu_monitor_close": (None, [C.c_void_p]),
    "pdgpu_sim_monitor": (C.c_int, [C.c_void_p, c_int64_p, C.c_int]),
    "pdgpu_set_cg_operator": (C.c_int, [C.c_void_p, C.c_int]),
    "pdgpu_set_transpose": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, c_int_p, c_int_p]),
    "pdgpu_group_matvec_transpose": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_void_p),
                                              C.POINTER(C.c_void_p), C.c_int]),
    "pdgpu_sim_monitor_read": (C.c_int, [C.c_void_p, c_int64_p, c_double_p, c_double_p, C.c_int64, c_int64_p]),
    "pdgpu_read_snapshot": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_int), c_double_p, c_double_p,
                                      C.POINTER(C.c_int64), c_double_p, c_double_p, c_double_p]),
    "pdgpu_constraint_values": (C.c_int, [C.c_void_p, c_uint8_p, c_double_p]),
    "pdgpu_set_ledger": (C.c_int, [C.c_void_p, c_int64_p, c_int64_p]),
    "pdgpu_break_bonds": (C.c_int, [C.c_void_p, c_int64_p, C.c_int64]),
    "pdgpu_ledger_pairs": (C.c_int, [C.c_void_p, c_int64_p, C.c_int64, c_int64_p]),
    "pdgpu_apply_corrections": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "pdgpu_apply_corrections_host": (C.c_int, [C.c_void_p, c_double_p, c_double_p, C.c_int64, C.c_int]),
    "pdgpu_matvec": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "pdgpu_matvec_host": (C.c_int, [C.c_void_p, c_double_p, c_double_p, C.c_int64, C.c_int]),
    "pdgpu_evaluate_force": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "pdgpu_add_constraint": (C.c_int, [C.c_void_p, c_double_p, c_double_p, C.c_int, C.c_int, C.c_double]),
    "pdgpu_add_load": (C.c_int, [C.c_void_p, c_double_p, c_double_p, c_double_p]),
    "pdgpu_set_body": (C.c_int, [C.c_void_p, c_double_p]),
    "pdgpu_seed_segment": (C.c_int, [C.c_void_p, c_double_p, c_int64_p]),
    "pdgpu_seed_notch": (C.c_int, [C.c_void_p, c_double_p, c_int64_p]),
    "pdgpu_update_bonds": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, c_double_p, c_int64_p, C.c_int64, c_int64_p]),
    "pdgpu_cg_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, c_int_p, c_double_p,
                                 C.c_void_p]),
    "pdgpu_cg_solve_host": (C.c_int, [C.c_void_p, c_double_p, c_double_p, C.c_double, C.c_int, c_int_p, c_double_p,
                                      c_double_p, C.c_int]),
    "pdgpu_sim_init": (C.c_int, [C.c_void_p, C.c_double, c_double_p]),
    "pdgpu_sim_step": (C.c_int, [C.c_void_p, C.c_int, C.c_double, c_double_p, c_int64_p]),
    "pdgpu_sim_init_adr": (C.c_int, [C.c_void_p, C.c_double, C.c_double]),
    "pdgpu_sim_adr_damping": (C.c_int, [C.c_void_p, c_double_p]),
    "pdgpu_sim_get": (C.c_int, [C.c_void_p, c_double_p, c_double_p, c_double_p, c_double_p]),
    "pdgpu_sim_get_aux": (C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    "pdgpu_sim_set_velocity": (C.c_int, [C.c_void_p, c_double_p]),
    "pdgpu_sim_newly_broken": (C.c_int, [C.c_void_p, c_int64_p, C.c_int64, c_int64_p]),
    "pdgpu_sim_finite": (C.c_int, [C.c_void_p, c_int_p]),
    "pdgpu_group_sim_step": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_double, c_double_p, c_int64_p]),
    "pdgpu_evaluate_force_host": (C.c_int, [C.c_void_p, c_double_p, c_double_p, C.c_int64]),
    "pdgpu_update_bonds_host": (C.c_int, [C.c_void_p, c_double_p, C.c_int64, C.c_double, c_double_p, c_int64_p,
                                          C.c_int64, c_int64_p]),
    "pdgpu_last_new_pairs": (C.c_int, [C.c_void_p, c_int64_p, C.c_int64, c_int64_p]),
    "pdgpu_timing_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "pdgpu_timing_read": (C.c_int, [C.c_void_p, c_double_p, c_int64_p, C.c_int]),
    "pdgpu_launch_count": (C.c_int64, [C.c_void_p]),
    "pdgpu_build_kernel": (C.c_int, [C.c_int, C.c_double, C.c_double, C.c_int, C.c_double, C.c_double, c_double_p]),
    "pdgpu_near_surface": (C.c_int, [C.c_int, c_int_p, C.c_int, c_uint8_p]),
}


def lib_path() -> str:
    return _build.LIB


def load(build_if_needed: bool = True):
    """Load libpdgpu.so, building it first when missing or stale."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_needed and not _build.up_to_date():
            _build.build()
        if not os.path.exists(_build.LIB):
            raise RuntimeError("libpdgpu.so is missing and could not be built: the CUDA engine is required")
        lib = C.CDLL(_build.LIB)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib
