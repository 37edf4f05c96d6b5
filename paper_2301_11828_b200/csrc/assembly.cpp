// assembly.cpp -- host-side operator assembly for the GPU engine.  Restates
// the reference's setup routines (cited per function) in plain C++ so that
// the stencils, region masks and surface diagonal the GPU consumes are the
// same numbers the reference builds.  Compiled without FMA contraction.
#include "assembly.h"

#include <math.h>

#include <algorithm>

namespace pdgpu {
namespace assembly {

int n_pairs(int dim) { return dim * (dim + 1) / 2; }

int pair_index(int dim, int a, int b) {
    if (a > b) std::swap(a, b);
    if (dim == 2) return a + b;
    static const int row_start[3] = {0, 3, 5};
    return row_start[a] + b - a;
}

std::vector<int> band_offsets(int dim, int M) {
    std::vector<int> out;
    const long M2 = (long)M * M;
    const int zr = dim == 3 ? M : 0;
    for (int a = -M; a <= M; ++a)
        for (int b = -M; b <= M; ++b)
            for (int c = -zr; c <= zr; ++c) {
                const long n2 = (long)a * a + (long)b * b + (long)c * c;
                if (n2 == 0 || n2 > M2) continue;
                out.push_back(a);
                out.push_back(b);
                out.push_back(c);
            }
    return out;
}

int64_t stencil_index(int dim, int M, const int* o) {
    const int side = 2 * M + 1;
    int64_t idx = 0;
    for (int d = dim - 1; d >= 0; --d) idx = idx * side + (o[d] + M);
    return idx;
}

double volume_correction(double dist, double delta, double h) {
    if (dist <= delta - 0.5 * h) return 1.0;
    if (dist <= delta) return 0.5 + (delta - dist) / h;
    return 0.0;
}

double micromodulus_alpha(double E, double delta, int dim, double thickness) {
    const double pi = 3.141592653589793238462643383279502884;
    if (dim == 2) return 9.0 * E / (pi * delta * delta * delta * thickness);
    return 12.0 * E / (pi * delta * delta * delta * delta);
}

std::vector<double> build_kernel(int dim, double h, double delta, int M, double E, double thickness) {
    const int np = n_pairs(dim);
    int64_t ss = 1;
    for (int d = 0; d < dim; ++d) ss *= (2 * M + 1);
    std::vector<double> K((size_t)(np * ss), 0.0);
    const double alpha = micromodulus_alpha(E, delta, dim, thickness);
    const double vol = dim == 2 ? h * h * thickness : h * h * h;
    const std::vector<int> offs = band_offsets(dim, M);
    const size_t nof = offs.size() / 3;
    for (size_t k = 0; k < nof; ++k) {
        const int* o = &offs[3 * k];
        long n2 = 0;
        for (int d = 0; d < dim; ++d) n2 += (long)o[d] * o[d];
        const double dist = h * sqrt((double)n2);
        const double lam = volume_correction(dist, delta, h);
        const double scale = alpha * lam * vol / (dist * dist * dist);
        for (int a = 0; a < dim; ++a)
            for (int b = a; b < dim; ++b)
                K[(size_t)(pair_index(dim, a, b) * ss + stencil_index(dim, M, o))] = scale * (o[a] * h) * (o[b] * h);
    }
    const int zero[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a)
        for (int b = a; b < dim; ++b) {
            double* Kp = &K[(size_t)(pair_index(dim, a, b) * ss)];
            double sum = 0.0;
            for (size_t k = 0; k < nof; ++k) sum += Kp[stencil_index(dim, M, &offs[3 * k])];
            Kp[stencil_index(dim, M, zero)] = -sum;
        }
    return K;
}

// global extent / coordinate of axis d under the slab frame
static inline int frame_lim(int dim, const int* dims, int d, const SlabFrame& s) {
    return (d == dim - 1 && s.global >= 0) ? s.global : dims[d];
}
static inline int frame_off(int dim, int d, const SlabFrame& s) { return d == dim - 1 ? s.off : 0; }

std::vector<uint8_t> near_surface(int dim, const int* dims, int M, SlabFrame slab) {
    const int nz = dim == 3 ? dims[2] : 1;
    const int64_t n = (int64_t)dims[0] * dims[1] * nz;
    std::vector<uint8_t> out((size_t)n, 0);
    for (int64_t p = 0; p < n; ++p) {
        int c[3];
        c[0] = (int)(p % dims[0]);
        c[1] = (int)((p / dims[0]) % dims[1]);
        c[2] = (int)(p / ((int64_t)dims[0] * dims[1]));
        for (int d = 0; d < dim; ++d)
            if (c[d] + frame_off(dim, d, slab) < M ||
                c[d] + frame_off(dim, d, slab) >= frame_lim(dim, dims, d, slab) - M) {
                out[(size_t)p] = 1;
                break;
            }
    }
    return out;
}

void surface_diag(int dim, const int* dims, int M, const double* K, const std::vector<uint8_t>& near,
                  std::vector<long long>& rows, std::vector<double>& de, SlabFrame slab) {
    const int np = n_pairs(dim);
    int64_t ss = 1;
    for (int d = 0; d < dim; ++d) ss *= (2 * M + 1);
    const std::vector<int> offs = band_offsets(dim, M);
    const size_t nof = offs.size() / 3;
    rows.clear();
    de.clear();
    const int64_t n = (int64_t)near.size();
    const int nz = dim == 3 ? dims[2] : 1;
    for (int64_t p = 0; p < n; ++p) {
        if (!near[(size_t)p]) continue;
        int c[3];
        c[0] = (int)(p % dims[0]);
        c[1] = (int)((p / dims[0]) % dims[1]);
        c[2] = (int)(p / ((int64_t)dims[0] * dims[1]));
        double acc[6] = {0, 0, 0, 0, 0, 0};
        for (size_t k = 0; k < nof; ++k) {
            const int* o = &offs[3 * k];
            bool inside = true;
            for (int d = 0; d < dim; ++d) {
                const int q = c[d] + frame_off(dim, d, slab) + o[d];
                inside = inside && q >= 0 && q < frame_lim(dim, dims, d, slab);
            }
            if (inside) continue;
            const int64_t si = stencil_index(dim, M, o);
            for (int a = 0; a < dim; ++a)
                for (int b = a; b < dim; ++b) {
                    const int pi = pair_index(dim, a, b);
                    acc[pi] += K[pi * ss + si];
                }
        }
        rows.push_back(p);
        for (int k = 0; k < np; ++k) de.push_back(acc[k]);
    }
}

void node_pos(int dim, const int* dims, double h, const double* origin, int64_t p, double* x) {
    int c[3];
    c[0] = (int)(p % dims[0]);
    c[1] = (int)((p / dims[0]) % dims[1]);
    c[2] = dim == 3 ? (int)(p / ((int64_t)dims[0] * dims[1])) : 0;
    for (int d = 0; d < dim; ++d) x[d] = origin[d] + (c[d] + 0.5) * h;
}

bool box_contains(int dim, const double* lo, const double* hi, const double* x) {
    for (int d = 0; d < dim; ++d)
        if (x[d] < lo[d] || x[d] > hi[d]) return false;
    return true;
}

static int orient2_sign(const double* a, const double* b, const double* c) {
    const double t1 = (b[0] - a[0]) * (c[1] - a[1]);
    const double t2 = (b[1] - a[1]) * (c[0] - a[0]);
    const double det = t1 - t2;
    const double tol = 1e-10 * (fabs(t1) + fabs(t2));
    if (fabs(det) <= tol) return 0;
    return det > 0.0 ? 1 : -1;
}

static bool segments_cross(const double* a, const double* b, const double* p, const double* q) {
    const int o1 = orient2_sign(a, b, p), o2 = orient2_sign(a, b, q);
    const int o3 = orient2_sign(p, q, a), o4 = orient2_sign(p, q, b);
    return o1 * o2 < 0 && o3 * o4 < 0;
}

bool segment_crosses(const double* seg, const double* p, const double* q) {
    const double a[2] = {seg[0], seg[1]}, b[2] = {seg[2], seg[3]};
    const double width = seg[4];
    if (width <= 0.0) return segments_cross(a, b, p, q);
    const double t[2] = {b[0] - a[0], b[1] - a[1]};
    const double len = sqrt(t[0] * t[0] + t[1] * t[1]);
    if (len == 0.0) return false;
    const double nrm[2] = {-t[1] / len, t[0] / len};
    for (double side : {0.5 * width, -0.5 * width}) {
        const double fa[2] = {a[0] + side * nrm[0], a[1] + side * nrm[1]};
        const double fb[2] = {b[0] + side * nrm[0], b[1] + side * nrm[1]};
        if (segments_cross(fa, fb, p, q)) return true;
    }
    return false;
}

bool notch_crosses(const double* nt, const double* p, const double* q) {
    const int axis = (int)nt[0];
    const double plane = nt[1], width = nt[2];
    const double faces[2] = {plane - 0.5 * width, plane + 0.5 * width};
    const int n_faces = width > 0.0 ? 2 : 1;
    for (int fi = 0; fi < n_faces; ++fi) {
        const double face = width > 0.0 ? faces[fi] : plane;
        const double dp = p[axis] - face, dq = q[axis] - face;
        const double tol = 1e-12 * (fabs(p[axis]) + fabs(q[axis]) + fabs(face));
        if (fabs(dp) <= tol || fabs(dq) <= tol) continue;
        if (!((dp > 0.0 && dq < 0.0) || (dp < 0.0 && dq > 0.0))) continue;
        const double t = dp / (dp - dq);
        bool inside = true;
        for (int d = 0; d < 3; ++d) {
            if (d == axis) continue;
            const double x = p[d] + t * (q[d] - p[d]);
            inside = inside && x >= nt[3 + d] && x <= nt[6 + d];
        }
        if (inside) return true;
    }
    return false;
}

}  // namespace assembly
}  // namespace pdgpu
