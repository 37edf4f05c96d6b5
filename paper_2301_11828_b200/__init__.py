"""B200-native MSBFM (matrix-structure-based fast method) K.u engine for
linear bond-based peridynamics -- drop-in GPU path for the reference
`pdfast` FastForce / apply_corrections / update_bonds and new CG / VV
drivers.  See DESIGN.md and include/pdgpu.h."""
from .engine import (Convolver, Error, FastForce, HorizonTooLargeForGrid, IoError, LedgerOutOfBand, MonitorWriter,
                     ShapeMismatch, band_offsets, build_kernel, n_pairs, near_surface, pair_index)

__all__ = ["Convolver", "Error", "FastForce", "HorizonTooLargeForGrid", "IoError", "LedgerOutOfBand", "MonitorWriter",
           "ShapeMismatch", "band_offsets", "build_kernel", "n_pairs", "near_surface", "pair_index"]
