// assembly.h -- host-side operator assembly ("Phase I"), restated from the
// reference so the GPU library can build a problem without the reference
// headers.  Each function cites the reference routine it mirrors.
#pragma once
#include <stdint.h>

#include <vector>

namespace pdgpu {
namespace assembly {

int n_pairs(int dim);
int pair_index(int dim, int a, int b);                       // kernel.hpp:19-28
std::vector<int> band_offsets(int dim, int M);               // kernel.hpp:71-89 order
int64_t stencil_index(int dim, int M, const int* o);         // kernel.hpp:50-54
double volume_correction(double dist, double delta, double h);  // grid.hpp:135-139
double micromodulus_alpha(double E, double delta, int dim, double thickness);  // material.hpp:15-24
// build_kernel, kernel.hpp:99-127 -> np * (2M+1)^dim
std::vector<double> build_kernel(int dim, double h, double delta, int M, double E, double thickness);
// Slab frame: the lattice is rows [off, off + dims[dim-1]) of a lattice whose
// slowest axis has `global` rows (off = 0, global = dims[dim-1]: the whole
// lattice).  Faces of the slab that are not faces of the global lattice are
// not surfaces.
struct SlabFrame {
    int off = 0;
    int global = -1;  // < 0: dims[dim-1]
};
// Regions near-surface flag (grid.hpp:181-189)
std::vector<uint8_t> near_surface(int dim, const int* dims, int M, SlabFrame slab = {});
// SurfaceDiag raw diagonal on near-surface rows (corrections.hpp:24-42):
// rows (ascending) and np values per row
void surface_diag(int dim, const int* dims, int M, const double* stencils, const std::vector<uint8_t>& near,
                  std::vector<long long>& rows, std::vector<double>& de, SlabFrame slab = {});
// node position, grid.hpp:53-57
void node_pos(int dim, const int* dims, double h, const double* origin, int64_t p, double* x);
bool box_contains(int dim, const double* lo, const double* hi, const double* x);  // geometry.hpp:58-62
// crack seeding predicates (fracture.hpp:38-55, 75-92, 122-146)
bool segment_crosses(const double* seg5, const double* p, const double* q);
bool notch_crosses(const double* notch9, const double* p, const double* q);

}  // namespace assembly
}  // namespace pdgpu
