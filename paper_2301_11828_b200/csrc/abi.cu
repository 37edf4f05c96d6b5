// abi.cu -- the C ABI (include/pdgpu.h) over the engine.  Host-side
// orchestration only: setup, stream-ordered launches, error mapping.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pdgpu.h"
#include "assembly.h"
#include "engine.h"

namespace pdgpu {
namespace snapshot {
std::string write(const std::string& dir, int dim, const int* dims, double h, const double* origin,
                  const double* u, const double* damage, int64_t step, double t);
bool read(const std::string& path, int dim, int* dims, double* h, double* origin, int64_t* step, double* t,
          double* u, double* damage, std::string& err);
struct Monitor;
int64_t nearest_node(int dim, const int* dims, double h, const double* origin, const double* x);
Monitor* monitor_open(const char* path, int dim, const int* dims, double h, const double* origin, const double* pts,
                      int npts, std::string& err);
void monitor_append(Monitor* m, int64_t step, double t, const double* vals);
void monitor_close(Monitor* m);
}  // namespace snapshot
}  // namespace pdgpu

using namespace pdgpu;

struct pdgpu_engine : public Engine {};

namespace {

thread_local std::string g_err;

struct PdError : std::runtime_error {
    int code;
    PdError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) throw PdError(PDGPU_ERR_OUT_OF_MEMORY, std::string(what) + ": out of memory");
    if (e != cudaSuccess) throw PdError(PDGPU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return PDGPU_OK;
    } catch (const PdError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host out of memory";
        return PDGPU_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_err = e.what();
        const std::string w = e.what();
        if (w.find("out of memory") != std::string::npos) return PDGPU_ERR_OUT_OF_MEMORY;
        return PDGPU_ERR_CUDA;
    }
}

template <class T>
void dalloc(T*& p, size_t count, const char* what) {
    if (p) cudaFree(p);
    p = nullptr;
    cuda_check(cudaMalloc((void**)&p, sizeof(T) * std::max<size_t>(count, 1)), what);
}

cudaStream_t pick_stream(Engine& e, void* s) { return s ? (cudaStream_t)s : e.stream; }

void coords_of(const Engine& e, int64_t p, int* c) {
    c[0] = (int)(p % e.plan.N[0]);
    c[1] = (int)((p / e.plan.N[0]) % e.plan.N[1]);
    c[2] = (int)(p / ((int64_t)e.plan.N[0] * e.plan.N[1]));
}

// node position in GLOBAL coordinates (grid.hpp:53-57): a slab engine's rows
// are rows [slab.off, ...) of the global lattice; origin is the global origin
void pos_of(const Engine& e, int64_t p, double* x) {
    int c[3];
    coords_of(e, p, c);
    if (e.slab.global >= 0) c[e.dim - 1] += e.slab.off;
    for (int d = 0; d < e.dim; ++d) x[d] = e.origin[d] + (c[d] + 0.5) * e.h;
}

int64_t global_offset(const Engine& e) {
    const int64_t plane = e.dim == 3 ? (int64_t)e.plan.N[0] * e.plan.N[1] : e.plan.N[0];
    return e.slab.global >= 0 ? (int64_t)e.slab.off * plane : 0;
}

int find_offset(const Engine& e, const int* o) {
    for (int k = 0; k < e.nof; ++k)
        if (e.offs[3 * k] == o[0] && e.offs[3 * k + 1] == o[1] && e.offs[3 * k + 2] == o[2]) return k;
    return -1;
}

void ensure_ledger(Engine& e) {
    if (e.d_ledger) return;
    touch_state(e);
    const int64_t N = e.plan.nodes;
    dalloc(e.d_ledger, (size_t)(N * e.lw), "alloc ledger");
    dalloc(e.d_bond_rows, (size_t)N, "alloc bond rows");
    dalloc(e.d_listed, (size_t)N, "alloc listed");
    cuda_check(cudaMemset(e.d_ledger, 0, sizeof(uint32_t) * N * e.lw), "zero ledger");
    cuda_check(cudaMemset(e.d_listed, 0, sizeof(int) * N), "zero listed");
    cuda_check(cudaMemset(e.d_counters, 0, sizeof(unsigned long long) * 4), "zero counters");
    e.n_bond_rows = 0;
    e.bond_rows_on_device = false;
    e.total_broken = 0;
    e.new_pairs_cap = std::max<int64_t>(1 << 20, N / 4);
    dalloc(e.d_new_pairs, (size_t)(2 * e.new_pairs_cap), "alloc new pairs");
}

void upload_surface(Engine& e, const std::vector<long long>& rows, const std::vector<double>& de) {
    touch_state(e);
    e.surf_default = false;
    e.n_surf = (int64_t)rows.size();
    dalloc(e.d_surf_rows, rows.size(), "alloc surface rows");
    dalloc(e.d_surf_de, de.size(), "alloc surface de");
    if (!rows.empty()) {
        cuda_check(cudaMemcpy(e.d_surf_rows, rows.data(), sizeof(long long) * rows.size(), cudaMemcpyHostToDevice),
                   "copy surface rows");
        cuda_check(cudaMemcpy(e.d_surf_de, de.data(), sizeof(double) * de.size(), cudaMemcpyHostToDevice),
                   "copy surface de");
    }
}

// recompute the constraint mask and the constrained-dof list (last writer wins,
// identical to applying the constraints in order, corrections.hpp:142-160)
void rebuild_constraints(Engine& e) {
    touch_state(e);
    const int64_t N = e.plan.nodes;
    const int dim = e.dim;
    e.h_cmask.assign((size_t)N, 0);
    std::map<long long, std::pair<int, double>> dofs;
    std::map<long long, double> ucv;  // prescribed displacements (kind 0 only, later boxes win)
    for (const auto& cs : e.constraints) {
        for (int64_t p = 0; p < N; ++p) {
            double x[3];
            pos_of(e, p, x);
            if (!assembly::box_contains(dim, cs.lo, cs.hi, x)) continue;
            e.h_cmask[(size_t)p] |= cs.dir_mask;
            for (int d = 0; d < dim; ++d)
                if ((cs.dir_mask >> d) & 1u) {
                    dofs[(long long)d * N + p] = {cs.kind, cs.value};
                    if (cs.kind == 0) ucv[(long long)d * N + p] = cs.value;
                }
        }
    }
    // u_c for CG as a sparse list (the solve scatters it on the device)
    {
        std::vector<long long> uid;
        std::vector<double> uval;
        for (const auto& kv : ucv)
            if (kv.second != 0.0) {
                uid.push_back(kv.first);
                uval.push_back(kv.second);
            }
        e.n_uc = (int64_t)uid.size();
        dalloc(e.d_uc_ids, std::max<size_t>(uid.size(), 1), "alloc uc ids");
        dalloc(e.d_uc_val, std::max<size_t>(uval.size(), 1), "alloc uc val");
        if (!uid.empty()) {
            cuda_check(cudaMemcpy(e.d_uc_ids, uid.data(), sizeof(long long) * uid.size(), cudaMemcpyHostToDevice), "uc");
            cuda_check(cudaMemcpy(e.d_uc_val, uval.data(), sizeof(double) * uval.size(), cudaMemcpyHostToDevice), "uc");
        }
    }
    cuda_check(cudaMemcpy(e.d_cmask, e.h_cmask.data(), (size_t)N, cudaMemcpyHostToDevice), "copy cmask");
    std::vector<long long> ids;
    std::vector<double> vals;
    std::vector<int> kinds;
    for (const auto& kv : dofs) {
        ids.push_back(kv.first);
        kinds.push_back(kv.second.first);
        vals.push_back(kv.second.second);
    }
    e.n_cdofs = (int64_t)ids.size();
    dalloc(e.d_cdofs, ids.size(), "alloc cdofs");
    dalloc(e.d_cval, vals.size(), "alloc cval");
    dalloc(e.d_ckind, kinds.size(), "alloc ckind");
    if (!ids.empty()) {
        cuda_check(cudaMemcpy(e.d_cdofs, ids.data(), sizeof(long long) * ids.size(), cudaMemcpyHostToDevice), "cdofs");
        cuda_check(cudaMemcpy(e.d_cval, vals.data(), sizeof(double) * vals.size(), cudaMemcpyHostToDevice), "cval");
        cuda_check(cudaMemcpy(e.d_ckind, kinds.data(), sizeof(int) * kinds.size(), cudaMemcpyHostToDevice), "ckind");
    }
}

bool has_constraints(const Engine& e) { return !e.constraints.empty() || e.any_cmask; }

// set bits for (p, q) pairs on the device; returns the number newly broken
__global__ void k_break_pairs(uint32_t* ledger, int lw, const long long* quad, int64_t n, long long* bond_rows,
                              int* listed, unsigned long long* counters) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long p = quad[4 * i], k = quad[4 * i + 1], q = quad[4 * i + 2], kn = quad[4 * i + 3];
    const unsigned old = atomicOr(&ledger[p * lw + (k >> 5)], 1u << (k & 31));
    if ((old >> (k & 31)) & 1u) return;
    atomicOr(&ledger[q * lw + (kn >> 5)], 1u << (kn & 31));
    atomicAdd(&counters[1], 1ull);
    if (atomicExch(&listed[p], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = p;
    if (atomicExch(&listed[q], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = q;
}

// ---- on-device assembly (set-up) --------------------------------------
// Crack seeding (seed_cracks, fracture.hpp:164-198) with the predicates of
// fracture.hpp:38-55 / 75-92 / 122-146 in explicitly rounded fp64 (no FMA
// contraction: bit-identical to the host restatement and the reference),
// thread per node of the crack's bounding box; the lower node of each bond
// tests it (q > p) and sets both ledger bits as k_break_pairs does.
struct SeedGeom {
    double g[9];
};

__device__ int d_orient2_sign(const double* a, const double* b, const double* c) {
    const double t1 = __dmul_rn(__dsub_rn(b[0], a[0]), __dsub_rn(c[1], a[1]));
    const double t2 = __dmul_rn(__dsub_rn(b[1], a[1]), __dsub_rn(c[0], a[0]));
    const double det = __dsub_rn(t1, t2);
    const double tol = __dmul_rn(1e-10, __dadd_rn(fabs(t1), fabs(t2)));
    if (fabs(det) <= tol) return 0;
    return det > 0.0 ? 1 : -1;
}

__device__ bool d_segments_cross(const double* a, const double* b, const double* p, const double* q) {
    const int o1 = d_orient2_sign(a, b, p), o2 = d_orient2_sign(a, b, q);
    const int o3 = d_orient2_sign(p, q, a), o4 = d_orient2_sign(p, q, b);
    return o1 * o2 < 0 && o3 * o4 < 0;
}

__device__ bool d_segment_crosses(const double* seg, const double* p, const double* q) {
    const double a[2] = {seg[0], seg[1]}, b[2] = {seg[2], seg[3]};
    const double width = seg[4];
    if (width <= 0.0) return d_segments_cross(a, b, p, q);
    const double t[2] = {__dsub_rn(b[0], a[0]), __dsub_rn(b[1], a[1])};
    const double len = __dsqrt_rn(__dadd_rn(__dmul_rn(t[0], t[0]), __dmul_rn(t[1], t[1])));
    if (len == 0.0) return false;
    const double nrm[2] = {__ddiv_rn(-t[1], len), __ddiv_rn(t[0], len)};
    for (int si = 0; si < 2; ++si) {
        const double side = si == 0 ? __dmul_rn(0.5, width) : __dmul_rn(-0.5, width);
        const double fa[2] = {__dadd_rn(a[0], __dmul_rn(side, nrm[0])), __dadd_rn(a[1], __dmul_rn(side, nrm[1]))};
        const double fb[2] = {__dadd_rn(b[0], __dmul_rn(side, nrm[0])), __dadd_rn(b[1], __dmul_rn(side, nrm[1]))};
        if (d_segments_cross(fa, fb, p, q)) return true;
    }
    return false;
}

__device__ bool d_notch_crosses(const double* nt, const double* p, const double* q) {
    const int axis = (int)nt[0];
    const double plane = nt[1], width = nt[2];
    const int n_faces = width > 0.0 ? 2 : 1;
    for (int fi = 0; fi < n_faces; ++fi) {
        const double face = width > 0.0 ? (fi == 0 ? __dsub_rn(plane, __dmul_rn(0.5, width))
                                                   : __dadd_rn(plane, __dmul_rn(0.5, width)))
                                         : plane;
        const double dp = __dsub_rn(p[axis], face), dq = __dsub_rn(q[axis], face);
        const double tol = __dmul_rn(1e-12, __dadd_rn(__dadd_rn(fabs(p[axis]), fabs(q[axis])), fabs(face)));
        if (fabs(dp) <= tol || fabs(dq) <= tol) continue;
        if (!((dp > 0.0 && dq < 0.0) || (dp < 0.0 && dq > 0.0))) continue;
        const double t = __ddiv_rn(dp, __dsub_rn(dp, dq));
        bool inside = true;
        for (int d = 0; d < 3; ++d) {
            if (d == axis) continue;
            const double x = __dadd_rn(p[d], __dmul_rn(t, __dsub_rn(q[d], p[d])));
            inside = inside && x >= nt[3 + d] && x <= nt[6 + d];
        }
        if (inside) return true;
    }
    return false;
}

template <bool NOTCH>
__global__ void k_seed(SeedGeom geom, int dim, int N0, int N1, int N2, int lo0, int lo1, int lo2, int n0, int n1,
                       int64_t total, double h, double o0, double o1, double o2, const int* __restrict__ offs, int nof,
                       uint32_t* ledger, int lw, long long* bond_rows, int* listed, unsigned long long* counters) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int c[3] = {lo0 + (int)(i % n0), lo1 + (int)((i / n0) % n1), lo2 + (int)(i / ((int64_t)n0 * n1))};
    const double org[3] = {o0, o1, o2};
    double xp[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) xp[d] = __dadd_rn(org[d], __dmul_rn(__dadd_rn((double)c[d], 0.5), h));
    const int Nd[3] = {N0, N1, N2};
    const int64_t p = ((int64_t)c[2] * N1 + c[1]) * N0 + c[0];
    for (int k = 0; k < nof; ++k) {
        const int qc[3] = {c[0] + offs[3 * k], c[1] + offs[3 * k + 1], c[2] + offs[3 * k + 2]};
        bool in = true;
        for (int d = 0; d < dim; ++d) in = in && qc[d] >= 0 && qc[d] < Nd[d];
        if (!in) continue;
        const int64_t q = ((int64_t)qc[2] * N1 + qc[1]) * N0 + qc[0];
        if (q < p) continue;  // visited from q
        double xq[3] = {0, 0, 0};
        for (int d = 0; d < dim; ++d) xq[d] = __dadd_rn(org[d], __dmul_rn(__dadd_rn((double)qc[d], 0.5), h));
        const bool cross = NOTCH ? d_notch_crosses(geom.g, xp, xq) : d_segment_crosses(geom.g, xp, xq);
        if (!cross) continue;
        const int kn = offs[3 * nof + k];  // index of -offset
        const unsigned old = atomicOr(&ledger[p * lw + (k >> 5)], 1u << (k & 31));
        if ((old >> (k & 31)) & 1u) continue;
        atomicOr(&ledger[q * lw + (kn >> 5)], 1u << (kn & 31));
        atomicAdd(&counters[1], 1ull);
        if (atomicExch(&listed[p], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = p;
        if (atomicExch(&listed[q], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = q;
    }
}

// SurfaceDiag (corrections.hpp:24-42) on the device for the engine's own
// lattice: near-surface rows enumerated row by row (a whole x row when y / z
// is within M of a face, else its 2M end nodes), so rows come out ascending
// like the host scan; D^e sums the kernel entries of the offsets that leave
// the lattice in for_each_offset order (koff), i.e. the same sums.
__global__ void k_surface_rows(int dim, int M, int N0, int N1, int N2, const long long* __restrict__ rowoff,
                               int64_t nrows, const int* __restrict__ offs, int nof,
                               const double* __restrict__ koff, int np, long long* out_rows, double* out_de) {
    const int64_t r = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;  // (z, y) row
    if (r >= nrows) return;
    const long long b0 = rowoff[r], cnt = rowoff[r + 1] - b0;
    const int y = (int)(r % N1), z = (int)(r / N1);
    for (long long i = threadIdx.x; i < cnt; i += blockDim.x) {
        const int x = cnt == N0 ? (int)i : (i < M ? (int)i : N0 - 2 * M + (int)i);
        const int c[3] = {x, y, z};
        const int Nd[3] = {N0, N1, N2};
        double acc[6] = {0, 0, 0, 0, 0, 0};
        for (int k = 0; k < nof; ++k) {
            bool inside = true;
            for (int d = 0; d < dim; ++d) {
                const int q = c[d] + offs[3 * k + d];
                inside = inside && q >= 0 && q < Nd[d];
            }
            if (inside) continue;
            for (int pp = 0; pp < np; ++pp) acc[pp] = __dadd_rn(acc[pp], koff[(int64_t)k * np + pp]);
        }
        out_rows[b0 + i] = ((long long)z * N1 + y) * N0 + x;
        for (int pp = 0; pp < np; ++pp) out_de[(b0 + i) * np + pp] = acc[pp];
    }
}

// engine's own lattice (no slab frame): D^e and the near-surface row list on
// the device; the host near flags are filled lazily (ensure_h_near)
void build_surface_device(Engine& e) {
    const int dim = e.dim, M = e.M;
    const int* N = e.plan.N;
    const int nz = dim == 3 ? N[2] : 1;
    const int64_t nrows = (int64_t)N[1] * nz;
    std::vector<long long> rowoff((size_t)nrows + 1, 0);
    for (int64_t r = 0; r < nrows; ++r) {
        const int y = (int)(r % N[1]), z = (int)(r / N[1]);
        bool full = y < M || y >= N[1] - M;
        if (dim == 3) full = full || z < M || z >= N[2] - M;
        const long long cnt = full || N[0] <= 2 * M ? N[0] : 2 * M;
        rowoff[(size_t)r + 1] = rowoff[(size_t)r] + cnt;
    }
    const int64_t n = rowoff[(size_t)nrows];
    touch_state(e);
    e.n_surf = n;
    dalloc(e.d_surf_rows, (size_t)n, "alloc surface rows");
    dalloc(e.d_surf_de, (size_t)(n * e.np), "alloc surface de");
    long long* d_rowoff = nullptr;
    cuda_check(cudaMalloc(&d_rowoff, sizeof(long long) * rowoff.size()), "alloc row offsets");
    cuda_check(cudaMemcpy(d_rowoff, rowoff.data(), sizeof(long long) * rowoff.size(), cudaMemcpyHostToDevice), "rowoff");
    const unsigned gx = (unsigned)std::min<int64_t>(nrows, 65535);
    const unsigned gy = (unsigned)((nrows + gx - 1) / gx);
    k_surface_rows<<<dim3(gx, gy), 128, 0, e.stream>>>(dim, M, N[0], N[1], nz, d_rowoff, nrows, e.d_offs, e.nof,
                                                       e.d_K + e.np * e.ss, e.np, e.d_surf_rows, e.d_surf_de);
    cuda_check(cudaGetLastError(), "surface rows");
    cuda_check(cudaStreamSynchronize(e.stream), "surface rows");
    cudaFree(d_rowoff);
    e.h_near.clear();
    e.surf_default = true;
}

void ensure_h_near(Engine& e) {
    if ((int64_t)e.h_near.size() == e.plan.nodes) return;
    e.h_near = assembly::near_surface(e.dim, e.plan.N, e.M, e.slab);
}

// host (p,q) pairs -> device bits; dedups within the call by sequential
// semantics of break_bond (a pair listed twice breaks once).
int64_t break_pairs(Engine& e, const int64_t* pairs, int64_t n) {
    ensure_ledger(e);
    std::vector<long long> quad;
    quad.reserve((size_t)(4 * n));
    std::vector<std::pair<long long, long long>> seen;
    for (int64_t i = 0; i < n; ++i) {
        int64_t p = pairs[2 * i], q = pairs[2 * i + 1];
        if (p < 0 || q < 0 || p >= e.plan.nodes || q >= e.plan.nodes)
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bond endpoint out of range");
        int cp[3], cq[3], o[3], no[3];
        coords_of(e, p, cp);
        coords_of(e, q, cq);
        for (int d = 0; d < 3; ++d) {
            o[d] = cq[d] - cp[d];
            no[d] = -o[d];
        }
        const int k = find_offset(e, o), kn = find_offset(e, no);
        if (k < 0 || kn < 0) throw PdError(PDGPU_ERR_LEDGER_OUT_OF_BAND, "broken bond exceeds the horizon band");
        const long long a = std::min(p, q), b = std::max(p, q);
        if (std::find(seen.begin(), seen.end(), std::make_pair(a, b)) != seen.end()) continue;
        if (n < 4096) seen.push_back({a, b});
        quad.push_back(p);
        quad.push_back(k);
        quad.push_back(q);
        quad.push_back(kn);
    }
    const int64_t m = (int64_t)quad.size() / 4;
    if (m == 0) return 0;
    touch_state(e);
    long long* d_quad = nullptr;
    cuda_check(cudaMalloc(&d_quad, sizeof(long long) * quad.size()), "alloc quad");
    cuda_check(cudaMemcpy(d_quad, quad.data(), sizeof(long long) * quad.size(), cudaMemcpyHostToDevice), "copy quad");
    cuda_check(cudaMemsetAsync(e.d_counters + 1, 0, sizeof(unsigned long long), e.stream), "reset");
    k_break_pairs<<<(unsigned)((m + 127) / 128), 128, 0, e.stream>>>(e.d_ledger, e.lw, d_quad, m, e.d_bond_rows,
                                                                     e.d_listed, e.d_counters);
    cuda_check(cudaGetLastError(), "break pairs");
    unsigned long long cnt[2];
    cuda_check(cudaMemcpyAsync(cnt, e.d_counters, sizeof(cnt), cudaMemcpyDeviceToHost, e.stream), "counters");
    cuda_check(cudaStreamSynchronize(e.stream), "break pairs sync");
    cudaFree(d_quad);
    e.n_bond_rows = (int64_t)cnt[0];
    e.total_broken += (int64_t)cnt[1];
    return (int64_t)cnt[1];
}

// one-sided breaks of bonds whose partner lives in another slab: (p, k,
// counted) triples; counted = this slab owns the pair (its node is the lower)
__global__ void k_break_halves(uint32_t* ledger, int lw, const long long* tri, int64_t n, long long* bond_rows,
                               int* listed, unsigned long long* counters) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long p = tri[3 * i], k = tri[3 * i + 1];
    const unsigned old = atomicOr(&ledger[p * lw + (k >> 5)], 1u << (k & 31));
    if ((old >> (k & 31)) & 1u) return;
    if (tri[3 * i + 2]) atomicAdd(&counters[1], 1ull);
    if (atomicExch(&listed[p], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = p;
}

int64_t break_halves(Engine& e, const std::vector<long long>& tri) {
    const int64_t m = (int64_t)tri.size() / 3;
    if (m == 0) return 0;
    ensure_ledger(e);
    touch_state(e);
    long long* d_tri = nullptr;
    cuda_check(cudaMalloc(&d_tri, sizeof(long long) * tri.size()), "alloc halves");
    cuda_check(cudaMemcpy(d_tri, tri.data(), sizeof(long long) * tri.size(), cudaMemcpyHostToDevice), "copy halves");
    cuda_check(cudaMemsetAsync(e.d_counters + 1, 0, sizeof(unsigned long long), e.stream), "reset");
    k_break_halves<<<(unsigned)((m + 127) / 128), 128, 0, e.stream>>>(e.d_ledger, e.lw, d_tri, m, e.d_bond_rows,
                                                                      e.d_listed, e.d_counters);
    cuda_check(cudaGetLastError(), "break halves");
    unsigned long long cnt[2];
    cuda_check(cudaMemcpyAsync(cnt, e.d_counters, sizeof(cnt), cudaMemcpyDeviceToHost, e.stream), "counters");
    cuda_check(cudaStreamSynchronize(e.stream), "break halves sync");
    cudaFree(d_tri);
    e.n_bond_rows = (int64_t)cnt[0];
    e.total_broken += (int64_t)cnt[1];
    return (int64_t)cnt[1];
}

// Separable symbol (2D): if every stencil component has a definite parity
// in each axis (true for build_kernel output, kernel.hpp:109-116: K^xx, K^yy
// even/even, K^xy odd/odd), H_p(kx, ky) = sum_m D_p[kx][m] * (cos|sin)(2 pi ky m/Py)
// with D_p[kx][0] = C_p[0] for pairs even in y, D_p[kx][m] = 2 C_p[m], and
// C_p[m] = sign_p / (Px Py) sum_ox K_p(ox, m) (cos|sin)(2 pi kx ox / Px),
// sign_p = -1 for odd/odd pairs (i*i).  Exact rewrite of the direct DFT of
// the stencil; the kernel evaluates H per frequency instead of streaming an
// O(N) table.  Enabled by PDGPU_SYMBOL=separable.
// 3D: the column axis is z, columns are (kx, ky), and the per-column
// coefficients fold the x and y phases; pairs odd in z (xz, yz) use sin.
// Opt-in (PDGPU_SYMBOL=separable): it removes the O(N) symbol stream (half of
// the 3D spectral pass's HBM bytes at batch 1) but measured slower in 2D and
// 3D, both fp64-issue bound; it remains a memory-footprint option.
void build_coltab(Engine& e) {
    if (e.d_coltab) {
        cudaFree(e.d_coltab);
        e.d_coltab = nullptr;
    }
    e.coltab_oddmask = 0;
    if (!e.real_symbol) return;
    // off by default: measured slower in both 2D and 3D on B200 (the spectral
    // pass is fp64-issue bound); it saves the O(N) symbol memory (3.2 GB at 256^3)
    bool want = false;
    if (const char* env = getenv("PDGPU_SYMBOL")) {
        if (std::string(env) == "separable") want = true;
        if (std::string(env) == "table") want = false;
    }
    if (!want) return;
    const int dim = e.dim, M = e.M, side = 2 * M + 1, np = e.np, l = dim - 1;
    auto Kat = [&](int p, const int* o) {
        int64_t idx = 0;
        for (int d = dim - 1; d >= 0; --d) idx = idx * side + (o[d] + M);
        return e.stencils[(size_t)(p * e.ss + idx)];
    };
    // parity per pair and axis: +1 even, -1 odd, 0 neither.  The centre
    // (-row sum, kernel.hpp:119-125) is a constant term of the symbol and is
    // excluded: an odd pair's centre is round-off of the row sum.
    std::vector<int> par((size_t)np * dim, 0);
    for (int p = 0; p < np; ++p)
        for (int ax = 0; ax < dim; ++ax) {
            bool even = true, odd = true;
            for (int64_t si = 0; si < e.ss; ++si) {
                int o[3] = {0, 0, 0};
                int64_t rem = si;
                for (int d = 0; d < dim; ++d) {
                    o[d] = (int)(rem % side) - M;
                    rem /= side;
                }
                if (o[0] == 0 && o[1] == 0 && o[2] == 0) continue;
                int r[3] = {o[0], o[1], o[2]};
                r[ax] = -r[ax];
                const double a = Kat(p, o), b = Kat(p, r);
                even = even && a == b;
                odd = odd && a == -b;
            }
            par[(size_t)(p * dim + ax)] = even ? 1 : (odd ? -1 : 0);
        }
    int oddmask = 0;
    for (int p = 0; p < np; ++p) {
        int nodd = 0;
        for (int ax = 0; ax < dim; ++ax) {
            if (par[(size_t)(p * dim + ax)] == 0) return;
            nodd += par[(size_t)(p * dim + ax)] == -1;
        }
        if (nodd & 1) return;  // imaginary symbol
        if (par[(size_t)(p * dim + l)] == -1) oddmask |= 1 << p;
    }
    if (dim == 2 && oddmask != 0b010) return;  // the 2D kernel hard-wires xx, yy even and xy odd along y
    const Plan& pl = e.plan;
    const int ND = np * (M + 1);
    const long double pi2 = 2.0L * 3.141592653589793238462643383279502884L;
    const long double scale = 1.0L / ((long double)pl.P[0] * (long double)pl.P[1] * (long double)pl.P[2]);
    // per-axis trig tables cos/sin(2 pi k o / P_d), o = -M..M
    std::vector<std::vector<double>> cs(2), sn(2);
    for (int d = 0; d < dim - 1; ++d) {
        const int P = pl.P[d], n = d == 0 ? pl.Hx : pl.P[1];
        cs[d].resize((size_t)n * side);
        sn[d].resize((size_t)n * side);
        for (int k = 0; k < n; ++k)
            for (int o = -M; o <= M; ++o) {
                const long double ang = pi2 * (long double)(((int64_t)k * (o + P)) % P) / P;
                cs[d][(size_t)k * side + o + M] = (double)cosl(ang);
                sn[d][(size_t)k * side + o + M] = (double)sinl(ang);
            }
    }
    std::vector<double> tab((size_t)pl.ncols * ND, 0.0);
    for (int col = 0; col < pl.ncols; ++col) {
        const int kx = dim == 2 ? col : col / pl.P[1], ky = dim == 2 ? 0 : col % pl.P[1];
        for (int p = 0; p < np; ++p) {
            int nodd = 0;
            for (int ax = 0; ax < dim; ++ax) nodd += par[(size_t)(p * dim + ax)] == -1;
            const double sign = nodd == 2 ? -1.0 : 1.0;  // i * i
            const bool oddx = par[(size_t)(p * dim)] == -1, oddy = dim == 3 && par[(size_t)(p * dim + 1)] == -1;
            for (int m = 0; m <= M; ++m) {
                double c = 0.0;
                const int oy_lo = dim == 3 ? -M : 0, oy_hi = dim == 3 ? M : 0;
                for (int oy = oy_lo; oy <= oy_hi; ++oy)
                    for (int ox = -M; ox <= M; ++ox) {
                        int o[3] = {ox, dim == 3 ? oy : m, dim == 3 ? m : 0};
                        if (ox == 0 && oy == 0 && m == 0) continue;  // centre added below
                        const double kv = Kat(p, o);
                        if (kv == 0.0) continue;
                        double fx = oddx ? sn[0][(size_t)kx * side + ox + M] : cs[0][(size_t)kx * side + ox + M];
                        double fy = 1.0;
                        if (dim == 3) fy = oddy ? sn[1][(size_t)ky * side + oy + M] : cs[1][(size_t)ky * side + oy + M];
                        c += kv * fx * fy;
                    }
                c *= sign * (double)scale;
                const bool evl = par[(size_t)(p * dim + l)] == 1;
                int zero[3] = {0, 0, 0};
                const double centre = Kat(p, zero) * (double)scale;
                tab[(size_t)col * ND + p * (M + 1) + m] = m == 0 ? (evl ? c : 0.0) + centre : 2.0 * c;
            }
        }
    }
    cuda_check(cudaMalloc(&e.d_coltab, sizeof(double) * tab.size()), "alloc coltab");
    cuda_check(cudaMemcpy(e.d_coltab, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice), "coltab");
    e.coltab_oddmask = oddmask;
    // the O(N) table is no longer read
    if (e.d_sym) cudaFree(e.d_sym);
    e.d_sym = nullptr;
}

void matvec_impl(Engine& e, const double* u, double* f, int batch, cudaStream_t s) {
    e.fold_surface_next = true;  // the corrections follow: the 3D face passes may take D^e
    launch_fast_apply(e, u, f, batch, s, 1.0, nullptr, nullptr);
    launch_corrections(e, u, f, batch, s, 1.0);
}

void evaluate_force_impl(Engine& e, const double* u, double* f, cudaStream_t s) {
    const bool cons = has_constraints(e);
    e.fold_surface_next = true;
    launch_fast_apply(e, u, f, 1, s, 1.0, cons ? e.d_cmask : nullptr, e.d_body);
    launch_corrections(e, u, f, 1, s, 1.0);
}

void ensure_stage(Engine& e, int64_t elems) {
    if (elems <= e.stage_cap) return;
    dalloc(e.d_u_stage, (size_t)elems, "alloc stage u");
    dalloc(e.d_f_stage, (size_t)elems, "alloc stage f");
    e.stage_cap = elems;
}

}  // namespace

extern "C" {

const char* pdgpu_last_error(void) { return g_err.c_str(); }
const char* pdgpu_version(void) { return "pdgpu 0.1 (sm_100a)"; }

int pdgpu_create(int dim, const int* dims, int M, const double* stencils, int device, pdgpu_t* out) {
    return guarded([&] {
        if (!out || !dims || !stencils) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        *out = nullptr;
        if (dim != 2 && dim != 3) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "dim must be 2 or 3");
        if (M < 1 || M > 8) throw PdError(PDGPU_ERR_NOT_SUPPORTED, "band half-width M must be in [1, 8]");
        for (int d = 0; d < dim; ++d)
            if (dims[d] < M + 1)
                throw PdError(PDGPU_ERR_HORIZON_TOO_LARGE, "need at least M+1 nodes per axis for the embedding");
        {
            // transform lengths the kernels are instantiated for (checked before touching the device):
            // x rows up to 2 * 4096-point halves, columns up to 4096 points per transform (3D: 512)
            Plan pl;
            plan_init(pl, dim, dims, M);
            const int lq = pl.logPl - (pl.nh == 2 ? 1 : 0);
            const int lqy = dim == 3 ? pl.logP[1] - 1 : 0;
            if (pl.logQx > 12 || lq > (dim == 2 ? 12 : 9) || lqy > 9)
                throw PdError(PDGPU_ERR_NOT_SUPPORTED, "lattice too large for the single-CTA transform tiles");
        }
        cuda_check(cudaSetDevice(device), "set device");
        auto* e = new pdgpu_engine();
        try {
            e->device = device;
            cuda_check(cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, device), "sm count");
            e->dim = dim;
            e->M = M;
            e->np = assembly::n_pairs(dim);
            e->ss = 1;
            for (int d = 0; d < dim; ++d) e->ss *= (2 * M + 1);
            e->stencils.assign(stencils, stencils + e->np * e->ss);
            e->offs = assembly::band_offsets(dim, M);
            e->nof = (int)e->offs.size() / 3;
            e->lw = (e->nof + 31) / 32;
            e->delta = M;
            plan_init(e->plan, dim, dims, M);
            const Plan& pl = e->plan;
            const int64_t N = pl.nodes;
            if (pl.P[0] / 4 * 2 * 16 > 227 * 1024 || pl.Pl / 2 * dim * 16 > 227 * 1024)
                throw PdError(PDGPU_ERR_NOT_SUPPORTED, "lattice too large for the single-CTA transform tiles");
            // physical (even) stencils give a real symbol
            e->real_symbol = true;
            {
                const int side = 2 * M + 1;
                for (int p = 0; p < e->np && e->real_symbol; ++p)
                    for (int64_t si = 0; si < e->ss; ++si) {
                        int64_t rem = si;
                        int o[3] = {0, 0, 0};
                        for (int d = 0; d < dim; ++d) {
                            o[d] = (int)(rem % side) - M;
                            rem /= side;
                        }
                        int no[3] = {-o[0], -o[1], -o[2]};
                        const int64_t sj = assembly::stencil_index(dim, M, no);
                        if (e->stencils[p * e->ss + si] != e->stencils[p * e->ss + sj]) {
                            e->real_symbol = false;
                            break;
                        }
                    }
            }
            set_kernel_attributes();
            cuda_check(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking), "stream");
            // stencils + per-offset coefficient table koff[k*np + pair]
            std::vector<double> kbuf(e->stencils);
            for (int k = 0; k < e->nof; ++k)
                for (int p = 0; p < e->np; ++p)
                    kbuf.push_back(e->stencils[p * e->ss + assembly::stencil_index(dim, M, &e->offs[3 * k])]);
            dalloc(e->d_K, kbuf.size(), "alloc K");
            cuda_check(cudaMemcpy(e->d_K, kbuf.data(), sizeof(double) * kbuf.size(), cudaMemcpyHostToDevice), "K");
            std::vector<int> obuf(e->offs);
            std::vector<long long> disp;
            for (int k = 0; k < e->nof; ++k) {
                const int* o = &e->offs[3 * k];
                int no[3] = {-o[0], -o[1], -o[2]};
                obuf.push_back(find_offset(*e, no));
                disp.push_back((long long)o[2] * pl.N[0] * pl.N[1] + (long long)o[1] * pl.N[0] + o[0]);
            }
            dalloc(e->d_offs, obuf.size(), "alloc offs");
            cuda_check(cudaMemcpy(e->d_offs, obuf.data(), sizeof(int) * obuf.size(), cudaMemcpyHostToDevice), "offs");
            dalloc(e->d_disp, disp.size(), "alloc disp");
            cuda_check(cudaMemcpy(e->d_disp, disp.data(), sizeof(long long) * disp.size(), cudaMemcpyHostToDevice),
                       "disp");
            build_twiddles(*e);
            build_symbol(*e);
            build_coltab(*e);
            build_wrap_table(*e);  // wrap correction and slab ghost rows (built before any graph capture)
            // regions + surface diagonal from the geometry (build_de)
            if (getenv("PDGPU_HOST_ASSEMBLY")) {
                e->h_near = assembly::near_surface(dim, dims, M);
                std::vector<long long> rows;
                std::vector<double> de;
                assembly::surface_diag(dim, dims, M, e->stencils.data(), e->h_near, rows, de);
                upload_surface(*e, rows, de);
                e->surf_default = true;
            } else {
                build_surface_device(*e);  // D^e and the near-surface rows on the device
            }
            dalloc(e->d_cmask, (size_t)N, "alloc cmask");
            cuda_check(cudaMemset(e->d_cmask, 0, (size_t)N), "zero cmask");
            e->h_cmask.assign((size_t)N, 0);
            dalloc(e->d_counters, 4, "alloc counters");
            cuda_check(cudaMemset(e->d_counters, 0, 32), "zero counters");
            dalloc(e->d_red, 4096, "alloc red");
            dalloc(e->d_scal, 16, "alloc scal");
            dalloc(e->d_ticket, 4, "alloc ticket");
            cuda_check(cudaMemset(e->d_ticket, 0, 16), "zero ticket");
            cuda_check(cudaDeviceSynchronize(), "create");
        } catch (...) {
            pdgpu_destroy(e);
            throw;
        }
        *out = e;
    });
}

void pdgpu_destroy(pdgpu_t h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    void* ptrs[] = {h->d_xstrip, h->d_lidx, h->d_loff, h->d_lK, h->d_sidx, h->d_stab, h->d_fidx, h->d_ftab, h->d_vh, h->d_wrows, h->d_wo0, h->d_wK, h->d_tw, h->d_sym, h->d_K, h->d_offs, h->d_disp, h->d_S1, h->d_S2, h->d_u_stage, h->d_f_stage,
                    h->d_cmask, h->d_surf_rows, h->d_surf_de, h->d_ledger, h->d_bond_rows, h->d_listed,
                    h->d_counters, h->d_new_pairs, h->d_body, h->d_cdofs, h->d_cval, h->d_ckind, h->d_u, h->d_v,
                    h->d_f, h->d_fprev, h->d_red, h->d_scal, h->d_ticket, h->d_cg, h->d_coltab, h->d_symh,
                    h->d_scratch, h->d_kc, h->d_uc_ids, h->d_uc_val, h->d_face_recv, h->d_halo,
                    h->d_mon_nodes, h->d_mon_rows};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h->cg_graph) cudaGraphExecDestroy(h->cg_graph);
    a2a_free(*h);
    h->d_face_recv = nullptr;  // freed with the other buffers above
    h->d_halo = nullptr;
    try {
        comm_destroy(*h);
    } catch (...) {
    }
    if (h->stream) cudaStreamDestroy(h->stream);
    if (h->copy_in) cudaStreamDestroy(h->copy_in);
    if (h->copy_out) cudaStreamDestroy(h->copy_out);
    for (cudaEvent_t ev : h->ev_pool) cudaEventDestroy(ev);
    delete h;
}

int pdgpu_set_geometry(pdgpu_t h, double spacing, const double* origin, double delta, double rho) {
    return guarded([&] {
        if (!h || !(spacing > 0)) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad geometry");
        cuda_check(cudaSetDevice(h->device), "set device");
        h->h = spacing;
        for (int d = 0; d < 3; ++d) h->origin[d] = (origin && d < h->dim) ? origin[d] : 0.0;
        h->delta = delta;
        h->rho = rho > 0 ? rho : 1.0;
        if (!h->constraints.empty()) rebuild_constraints(*h);
    });
}

int pdgpu_apply(pdgpu_t h, const double* u, double* f, int batch, void* stream) {
    return guarded([&] {
        if (!h || !u || !f || batch < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad apply arguments");
        cuda_check(cudaSetDevice(h->device), "set device");
        launch_fast_apply(*h, u, f, batch, pick_stream(*h, stream), 1.0, nullptr, nullptr);
    });
}

int pdgpu_apply_direct(pdgpu_t h, const double* u, double* f, int batch, void* stream) {
    return guarded([&] {
        if (!h || !u || !f || batch < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad apply arguments");
        cuda_check(cudaSetDevice(h->device), "set device");
        launch_direct_apply(*h, u, f, batch, pick_stream(*h, stream), 1.0);
    });
}

int pdgpu_apply_host(pdgpu_t h, const double* u, double* f, int64_t n_nodes, int batch) {
    return guarded([&] {
        if (!h || !u || !f || batch < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad apply arguments");
        if (n_nodes != h->plan.nodes) throw PdError(PDGPU_ERR_SHAPE_MISMATCH, "field length does not match the lattice");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t m = (int64_t)batch * h->dim * n_nodes;
        ensure_stage(*h, m);
        cuda_check(cudaMemcpyAsync(h->d_u_stage, u, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream), "H2D");
        launch_fast_apply(*h, h->d_u_stage, h->d_f_stage, batch, h->stream, 1.0, nullptr, nullptr);
        cuda_check(cudaMemcpyAsync(f, h->d_f_stage, sizeof(double) * m, cudaMemcpyDeviceToHost, h->stream), "D2H");
        cuda_check(cudaStreamSynchronize(h->stream), "apply_host");
    });
}

// The reference records max|Im|/max|Re| after each inverse C2C transform
// (convolution.hpp:158-172).  The R2C/C2R pipeline here never forms an
// imaginary part of the output field, so the residue is identically 0.
double pdgpu_last_imag_residue(pdgpu_t) { return 0.0; }

size_t pdgpu_footprint_bytes(pdgpu_t h) {
    if (!h) return 0;
    const Plan& pl = h->plan;
    const int64_t N = pl.nodes;
    size_t b = 0;
    if (h->d_sym) b += (size_t)pl.ncols * pl.Pl * (h->dim == 2 && h->real_symbol ? 4 : h->np) * (h->real_symbol ? 8 : 16);
    if (h->d_coltab) b += (size_t)pl.ncols * h->np * (h->M + 1) * 8;
    b += (size_t)(16 * (1 << pl.logTWN));
    b += (size_t)h->cap_batch * 16 * (pl.S1_per_vec + ((pl.dim == 3 || pl.k3_halves == 1) ? pl.S2_per_vec : 0));
    b += (size_t)N + (size_t)h->n_surf * (8 + 8 * h->np);
    if (h->d_ledger) b += (size_t)N * (4 * h->lw + 12);
    return b;
}

int64_t pdgpu_n_nodes(pdgpu_t h) { return h ? h->plan.nodes : 0; }
int pdgpu_symbol_is_real(pdgpu_t h) { return h && h->real_symbol ? 1 : 0; }
size_t pdgpu_symbol_stream_bytes(pdgpu_t h) {
    if (!h) return 0;
    const Plan& pl = h->plan;
    // (512/1024-point columns fall back to the full table on batches too small to
    // fill the SMs, launch_k3_2d; this reports the large-batch figure)
    const char* k3 = getenv("PDGPU_K3");
    if (h->d_symh && h->symh_for == h->d_sym && (k3 ? std::string(k3) == "tx3" : true))
        return (size_t)pl.ncols * 3 * h->symh_stride * 8;
    if (h->d_coltab) return (size_t)pl.ncols * h->np * (h->M + 1) * 8;
    return (size_t)pl.ncols * pl.Pl * (h->dim == 2 && h->real_symbol ? 4 : h->np) * (h->real_symbol ? 8 : 16);
}
int pdgpu_symbol_mode(pdgpu_t h) { return !h ? -1 : (h->d_coltab ? 2 : (h->real_symbol ? 1 : 0)); }
int pdgpu_embedding(pdgpu_t h) { return !h ? -1 : h->plan.circ_mask; }

int pdgpu_set_regions(pdgpu_t h, const uint8_t* near_surface, const uint8_t* cmask) {
    return guarded([&] {
        if (!h) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null handle");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t N = h->plan.nodes;
        if (near_surface) {
            h->h_near.assign(near_surface, near_surface + N);
            std::vector<long long> rows;
            std::vector<double> de;
            assembly::surface_diag(h->dim, h->plan.N, h->M, h->stencils.data(), h->h_near, rows, de, h->slab);
            upload_surface(*h, rows, de);
        }
        if (cmask) {
            h->h_cmask.assign(cmask, cmask + N);
            h->any_cmask = false;
            for (int64_t p = 0; p < N; ++p) h->any_cmask = h->any_cmask || cmask[p] != 0;
            cuda_check(cudaMemcpy(h->d_cmask, cmask, (size_t)N, cudaMemcpyHostToDevice), "copy cmask");
        }
    });
}

int pdgpu_set_slab(pdgpu_t h, int global_rows, int row_offset) {
    return guarded([&] {
        if (!h) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null handle");
        const int n_last = h->plan.N[h->dim - 1];
        if (global_rows < n_last || row_offset < 0 || row_offset + n_last > global_rows)
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "slab outside the global lattice");
        cuda_check(cudaSetDevice(h->device), "set device");
        h->slab.off = row_offset;
        h->slab.global = global_rows;
        h->h_near = assembly::near_surface(h->dim, h->plan.N, h->M, h->slab);
        std::vector<long long> rows;
        std::vector<double> de;
        assembly::surface_diag(h->dim, h->plan.N, h->M, h->stencils.data(), h->h_near, rows, de, h->slab);
        upload_surface(*h, rows, de);
        if (h->dim == 3) {
            // the tiled wrap face passes serve a slab whose own axis is short (their z
            // pass takes the ghost planes): rebuild the tables for the slab frame
            touch_state(*h);
            for (void** p : {(void**)&h->d_wrows, (void**)&h->d_wo0, (void**)&h->d_wK, (void**)&h->d_lidx, (void**)&h->d_loff,
                             (void**)&h->d_lK, (void**)&h->d_sidx, (void**)&h->d_stab, (void**)&h->d_fidx, (void**)&h->d_ftab}) {
                if (*p) cudaFree(*p);
                *p = nullptr;
            }
            build_wrap_table(*h);
        }
    });
}

int pdgpu_set_ghosts(pdgpu_t h, const double* ghosts) {
    return guarded([&] {
        if (!h) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null handle");
        if (ghosts && h->slab.global < 0) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "ghost rows need pdgpu_set_slab");
        h->d_ghost = ghosts;
        h->user_ghost_bc = 0;  // default layout [batch][dim][2][M][plane]
        h->user_ghost_side = 0;
        touch_state(*h);  // a captured CG iteration holds the old pointer
    });
}

int pdgpu_set_ghosts_strided(pdgpu_t h, const double* ghosts, int64_t vec_comp_stride, int64_t side_stride) {
    return guarded([&] {
        if (!h) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null handle");
        if (ghosts && h->slab.global < 0) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "ghost rows need pdgpu_set_slab");
        if (ghosts && (vec_comp_stride <= 0 || side_stride <= 0))
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "ghost strides must be positive");
        h->d_ghost = ghosts;
        h->user_ghost_bc = vec_comp_stride;
        h->user_ghost_side = side_stride;
        touch_state(*h);
    });
}

int pdgpu_halo_pack(pdgpu_t h, const double* u, int batch, double* send, void* stream) {
    return guarded([&] {
        if (!h || !u || !send || batch < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        if (h->plan.N[h->dim - 1] < h->M) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "slab thinner than the horizon");
        cuda_check(cudaSetDevice(h->device), "set device");
        halo_pack(*h, u, batch, send, pick_stream(*h, stream));
    });
}

int pdgpu_comm_unique_id(void* id_out) {
    return guarded([&] {
        if (!id_out) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        comm_unique_id(id_out);
    });
}

int pdgpu_comm_init(pdgpu_t h, int nranks, int rank, const void* id) {
    return guarded([&] {
        if (!h || !id || nranks < 1 || rank < 0 || rank >= nranks)
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad communicator arguments");
        if (nranks > 1 && h->slab.global < 0) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "multi-rank engines need pdgpu_set_slab");
        if (h->plan.N[h->dim - 1] < h->M) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "slab thinner than the horizon");
        cuda_check(cudaSetDevice(h->device), "set device");
        comm_init(*h, nranks, rank, id);
    });
}

int pdgpu_slab_rows(int global_rows, int nranks, int rank, int* row_begin, int* row_end) {
    return guarded([&] {
        if (!row_begin || !row_end || nranks < 1 || rank < 0 || rank >= nranks || global_rows < nranks)
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad slab arguments");
        *row_begin = (int)((int64_t)global_rows * rank / nranks);
        *row_end = (int)((int64_t)global_rows * (rank + 1) / nranks);
    });
}

int pdgpu_set_surface_diag(pdgpu_t h, const double* de) {
    return guarded([&] {
        if (!h || !de) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t N = h->plan.nodes;
        ensure_h_near(*h);
        std::vector<long long> rows;
        std::vector<double> vals;
        for (int64_t p = 0; p < N; ++p) {
            if (!h->h_near[(size_t)p]) continue;
            rows.push_back(p);
            for (int k = 0; k < h->np; ++k) vals.push_back(de[(int64_t)k * N + p]);
        }
        upload_surface(*h, rows, vals);
    });
}

int pdgpu_set_ledger(pdgpu_t h, const int64_t* row_start, const int64_t* partners) {
    return guarded([&] {
        if (!h || !row_start) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        ensure_ledger(*h);
        touch_state(*h);
        const int64_t N = h->plan.nodes;
        std::vector<uint32_t> bits((size_t)(N * h->lw), 0u);
        std::vector<long long> rows;
        std::vector<int> listed((size_t)N, 0);
        int64_t halves = 0;
        for (int64_t p = 0; p < N; ++p) {
            for (int64_t j = row_start[p]; j < row_start[p + 1]; ++j) {
                const int64_t q = partners[j];
                if (q < 0 || q >= N) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "partner out of range");
                int cp[3], cq[3], o[3];
                coords_of(*h, p, cp);
                coords_of(*h, q, cq);
                for (int d = 0; d < 3; ++d) o[d] = cq[d] - cp[d];
                const int k = find_offset(*h, o);
                if (k < 0) throw PdError(PDGPU_ERR_LEDGER_OUT_OF_BAND, "broken bond exceeds the horizon band");
                bits[(size_t)(p * h->lw + (k >> 5))] |= 1u << (k & 31);
                ++halves;
            }
            if (row_start[p + 1] > row_start[p]) {
                rows.push_back(p);
                listed[(size_t)p] = 1;
            }
        }
        cuda_check(cudaMemcpy(h->d_ledger, bits.data(), sizeof(uint32_t) * bits.size(), cudaMemcpyHostToDevice),
                   "copy ledger");
        cuda_check(cudaMemcpy(h->d_listed, listed.data(), sizeof(int) * listed.size(), cudaMemcpyHostToDevice),
                   "copy listed");
        if (!rows.empty())
            cuda_check(cudaMemcpy(h->d_bond_rows, rows.data(), sizeof(long long) * rows.size(), cudaMemcpyHostToDevice),
                       "copy rows");
        unsigned long long cnt[2] = {(unsigned long long)rows.size(), 0ull};
        cuda_check(cudaMemcpy(h->d_counters, cnt, sizeof(cnt), cudaMemcpyHostToDevice), "copy counters");
        h->n_bond_rows = (int64_t)rows.size();
        h->total_broken = halves / 2;
    });
}

int pdgpu_break_bonds(pdgpu_t h, const int64_t* pairs, int64_t n) {
    return guarded([&] {
        if (!h || (n > 0 && !pairs)) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        break_pairs(*h, pairs, n);
    });
}

int pdgpu_ledger_pairs(pdgpu_t h, int64_t* out, int64_t cap, int64_t* count) {
    return guarded([&] {
        if (!h || !count) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        *count = 0;
        if (!h->d_ledger) return;
        const int64_t N = h->plan.nodes;
        std::vector<uint32_t> bits((size_t)(N * h->lw));
        cuda_check(cudaStreamSynchronize(h->stream), "sync");
        cuda_check(cudaMemcpy(bits.data(), h->d_ledger, sizeof(uint32_t) * bits.size(), cudaMemcpyDeviceToHost),
                   "read ledger");
        // partner order per row = ascending q = ascending displacement
        std::vector<int> order(h->nof);
        std::vector<long long> disp(h->nof);
        for (int k = 0; k < h->nof; ++k) {
            order[k] = k;
            const int* o = &h->offs[3 * k];
            disp[k] = (long long)o[2] * h->plan.N[0] * h->plan.N[1] + (long long)o[1] * h->plan.N[0] + o[0];
        }
        std::sort(order.begin(), order.end(), [&](int a, int b) { return disp[a] < disp[b]; });
        // global node ids: a slab engine reports the pairs whose lower node it
        // holds (partners may lie in the next slab), so the union over ranks is
        // the global ledger
        const int64_t goff = global_offset(*h);
        int64_t c = 0;
        for (int64_t p = 0; p < N; ++p)
            for (int k : order) {
                if (disp[k] <= 0) continue;
                if (!((bits[(size_t)(p * h->lw + (k >> 5))] >> (k & 31)) & 1u)) continue;
                if (out && c < cap) {
                    out[2 * c] = goff + p;
                    out[2 * c + 1] = goff + p + disp[k];
                }
                ++c;
            }
        *count = c;
    });
}

int pdgpu_apply_corrections(pdgpu_t h, const double* u, double* f, int batch, void* stream) {
    return guarded([&] {
        if (!h || !u || !f || batch < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        cuda_check(cudaSetDevice(h->device), "set device");
        launch_corrections(*h, u, f, batch, pick_stream(*h, stream), 1.0);
    });
}

int pdgpu_apply_corrections_host(pdgpu_t h, const double* u, double* f, int64_t n_nodes, int batch) {
    return guarded([&] {
        if (!h || !u || !f || batch < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        if (n_nodes != h->plan.nodes) throw PdError(PDGPU_ERR_SHAPE_MISMATCH, "field length does not match the lattice");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t m = (int64_t)batch * h->dim * n_nodes;
        ensure_stage(*h, m);
        cuda_check(cudaMemcpyAsync(h->d_u_stage, u, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream), "H2D");
        cuda_check(cudaMemcpyAsync(h->d_f_stage, f, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream), "H2D");
        launch_corrections(*h, h->d_u_stage, h->d_f_stage, batch, h->stream, 1.0);
        cuda_check(cudaMemcpyAsync(f, h->d_f_stage, sizeof(double) * m, cudaMemcpyDeviceToHost, h->stream), "D2H");
        cuda_check(cudaStreamSynchronize(h->stream), "apply_corrections_host");
    });
}

int pdgpu_matvec(pdgpu_t h, const double* u, double* f, int batch, void* stream) {
    return guarded([&] {
        if (!h || !u || !f || batch < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        cuda_check(cudaSetDevice(h->device), "set device");
        matvec_impl(*h, u, f, batch, pick_stream(*h, stream));
    });
}

int pdgpu_matvec_host(pdgpu_t h, const double* u, double* f, int64_t n_nodes, int batch) {
    return guarded([&] {
        if (!h || !u || !f || batch < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        if (n_nodes != h->plan.nodes) throw PdError(PDGPU_ERR_SHAPE_MISMATCH, "field length does not match the lattice");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t mv = (int64_t)h->dim * n_nodes;
        ensure_stage(*h, (int64_t)batch * mv);
        if (!h->copy_in) {
            cuda_check(cudaStreamCreateWithFlags(&h->copy_in, cudaStreamNonBlocking), "stream");
            cuda_check(cudaStreamCreateWithFlags(&h->copy_out, cudaStreamNonBlocking), "stream");
        }
        // pipeline: H2D of chunk c+1 and D2H of chunk c-1 overlap the mat-vec of
        // chunk c.  PCIe-bound (the copies take ~4x the mat-vec), so one-vector
        // chunks: the exposed first H2D and last D2H are as short as possible
        const int chunk = 1;
        const int nch = (batch + chunk - 1) / chunk;
        std::vector<cudaEvent_t> evh(nch), evc(nch);
        for (int c = 0; c < nch; ++c) {
            cuda_check(cudaEventCreateWithFlags(&evh[c], cudaEventDisableTiming), "event");
            cuda_check(cudaEventCreateWithFlags(&evc[c], cudaEventDisableTiming), "event");
        }
        for (int c = 0; c < nch; ++c) {
            const int b0 = c * chunk, nb = std::min(chunk, batch - b0);
            const size_t off = (size_t)b0 * mv, bytes = sizeof(double) * (size_t)nb * mv;
            cuda_check(cudaMemcpyAsync(h->d_u_stage + off, u + off, bytes, cudaMemcpyHostToDevice, h->copy_in), "H2D");
            cuda_check(cudaEventRecord(evh[c], h->copy_in), "record");
            cuda_check(cudaStreamWaitEvent(h->stream, evh[c], 0), "wait");
            matvec_impl(*h, h->d_u_stage + off, h->d_f_stage + off, nb, h->stream);
            cuda_check(cudaEventRecord(evc[c], h->stream), "record");
            cuda_check(cudaStreamWaitEvent(h->copy_out, evc[c], 0), "wait");
            cuda_check(cudaMemcpyAsync(f + off, h->d_f_stage + off, bytes, cudaMemcpyDeviceToHost, h->copy_out), "D2H");
        }
        cuda_check(cudaStreamSynchronize(h->copy_out), "matvec_host");
        for (int c = 0; c < nch; ++c) {
            cudaEventDestroy(evh[c]);
            cudaEventDestroy(evc[c]);
        }
    });
}

int pdgpu_evaluate_force(pdgpu_t h, const double* u, double* f, void* stream) {
    return guarded([&] {
        if (!h || !u || !f) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        cuda_check(cudaSetDevice(h->device), "set device");
        evaluate_force_impl(*h, u, f, pick_stream(*h, stream));
    });
}

int pdgpu_evaluate_force_host(pdgpu_t h, const double* u, double* f, int64_t n_nodes) {
    return guarded([&] {
        if (!h || !u || !f) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        if (n_nodes != h->plan.nodes) throw PdError(PDGPU_ERR_SHAPE_MISMATCH, "field length does not match the lattice");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t m = (int64_t)h->dim * n_nodes;
        ensure_stage(*h, m);
        cuda_check(cudaMemcpyAsync(h->d_u_stage, u, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream), "H2D");
        evaluate_force_impl(*h, h->d_u_stage, h->d_f_stage, h->stream);
        cuda_check(cudaMemcpyAsync(f, h->d_f_stage, sizeof(double) * m, cudaMemcpyDeviceToHost, h->stream), "D2H");
        cuda_check(cudaStreamSynchronize(h->stream), "evaluate_force_host");
    });
}

int pdgpu_add_constraint(pdgpu_t h, const double* lo, const double* hi, int dir_mask, int kind, double value) {
    return guarded([&] {
        if (!h || !lo || !hi) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        Constraint c;
        memset(&c, 0, sizeof(c));
        for (int d = 0; d < h->dim; ++d) {
            c.lo[d] = lo[d];
            c.hi[d] = hi[d];
        }
        c.dir_mask = (uint8_t)dir_mask;
        c.kind = kind;
        c.value = value;
        h->constraints.push_back(c);
        rebuild_constraints(*h);
    });
}

int pdgpu_add_load(pdgpu_t h, const double* lo, const double* hi, const double* value) {
    return guarded([&] {
        if (!h || !lo || !hi || !value) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t N = h->plan.nodes;
        if (h->h_body.empty()) h->h_body.assign((size_t)(h->dim * N), 0.0);
        for (int64_t p = 0; p < N; ++p) {
            double x[3];
            pos_of(*h, p, x);
            if (!assembly::box_contains(h->dim, lo, hi, x)) continue;
            for (int d = 0; d < h->dim; ++d) h->h_body[(size_t)(d * N + p)] += value[d];
        }
        dalloc(h->d_body, h->h_body.size(), "alloc body");
        cuda_check(cudaMemcpy(h->d_body, h->h_body.data(), sizeof(double) * h->h_body.size(), cudaMemcpyHostToDevice),
                   "copy body");
    });
}

int pdgpu_set_body(pdgpu_t h, const double* body) {
    return guarded([&] {
        if (!h || !body) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t N = h->plan.nodes;
        h->h_body.assign(body, body + h->dim * N);
        dalloc(h->d_body, h->h_body.size(), "alloc body");
        cuda_check(cudaMemcpy(h->d_body, body, sizeof(double) * h->h_body.size(), cudaMemcpyHostToDevice), "copy body");
    });
}

static void seed_impl(Engine& e, const double* geom, bool notch, int64_t* added) {
    const int dim = e.dim;
    double lo[3], hi[3];
    if (!notch) {
        for (int d = 0; d < 2; ++d) {
            const double a = geom[d], b = geom[2 + d], w = geom[4];
            lo[d] = std::min(a - w, b - w);
            hi[d] = std::max(a + w, b + w);
        }
    } else {
        const int axis = (int)geom[0];
        for (int d = 0; d < 3; ++d) {
            lo[d] = d == axis ? geom[1] - geom[2] : geom[3 + d];
            hi[d] = d == axis ? geom[1] + geom[2] : geom[6 + d];
        }
    }
    // visit the nodes within delta + h of the crack hull (fracture.hpp:164-198),
    // in global lattice coordinates; a slab engine visits its own rows and
    // also sees partners in the neighbouring slabs (the bond's lower node owns
    // it, q > p as in fracture.hpp:189, and each side keeps its own half)
    const int SA = dim - 1;
    const int zoff = e.slab.global >= 0 ? e.slab.off : 0;
    int G[3] = {e.plan.N[0], e.plan.N[1], e.plan.N[2]};
    if (e.slab.global >= 0) G[SA] = e.slab.global;
    int clo[3] = {0, 0, 0}, chi[3] = {0, 0, 0};
    const double pad = e.delta + e.h;
    for (int d = 0; d < dim; ++d) {
        clo[d] = std::max(0, (int)floor((lo[d] - pad - e.origin[d]) / e.h));
        chi[d] = std::min(G[d] - 1, (int)ceil((hi[d] + pad - e.origin[d]) / e.h));
    }
    clo[SA] = std::max(clo[SA], zoff);
    chi[SA] = std::min(chi[SA], zoff + e.plan.N[SA] - 1);
    if (e.slab.global < 0 && !getenv("PDGPU_HOST_ASSEMBLY")) {
        // the engine's own lattice: the box sweep runs on the device (k_seed)
        for (int d = 0; d < dim; ++d)
            if (chi[d] < clo[d]) {
                if (added) *added = 0;
                return;
            }
        ensure_ledger(e);
        touch_state(e);
        SeedGeom sg;
        for (int i = 0; i < 9; ++i) sg.g[i] = i < (notch ? 9 : 5) ? geom[i] : 0.0;
        const int n0 = chi[0] - clo[0] + 1, n1 = dim >= 2 ? chi[1] - clo[1] + 1 : 1, n2 = dim == 3 ? chi[2] - clo[2] + 1 : 1;
        const int64_t total = (int64_t)n0 * n1 * n2;
        cuda_check(cudaMemsetAsync(e.d_counters + 1, 0, sizeof(unsigned long long), e.stream), "reset");
        const unsigned blocks = (unsigned)((total + 127) / 128);
        if (notch)
            k_seed<true><<<blocks, 128, 0, e.stream>>>(sg, dim, e.plan.N[0], e.plan.N[1], e.plan.N[2], clo[0], clo[1],
                                                       clo[2], n0, n1, total, e.h, e.origin[0], e.origin[1], e.origin[2],
                                                       e.d_offs, e.nof, e.d_ledger, e.lw, e.d_bond_rows, e.d_listed,
                                                       e.d_counters);
        else
            k_seed<false><<<blocks, 128, 0, e.stream>>>(sg, dim, e.plan.N[0], e.plan.N[1], e.plan.N[2], clo[0], clo[1],
                                                        clo[2], n0, n1, total, e.h, e.origin[0], e.origin[1],
                                                        e.origin[2], e.d_offs, e.nof, e.d_ledger, e.lw, e.d_bond_rows,
                                                        e.d_listed, e.d_counters);
        cuda_check(cudaGetLastError(), "seed");
        unsigned long long cnt[2];
        cuda_check(cudaMemcpyAsync(cnt, e.d_counters, sizeof(cnt), cudaMemcpyDeviceToHost, e.stream), "counters");
        cuda_check(cudaStreamSynchronize(e.stream), "seed sync");
        e.n_bond_rows = (int64_t)cnt[0];
        e.total_broken += (int64_t)cnt[1];
        if (added) *added = (int64_t)cnt[1];
        return;
    }
    auto gpos = [&](const int* cg, double* x) {
        for (int d = 0; d < dim; ++d) x[d] = e.origin[d] + (cg[d] + 0.5) * e.h;
    };
    auto glin = [&](const int* cg) { return ((int64_t)cg[2] * G[1] + cg[1]) * G[0] + cg[0]; };
    std::vector<int64_t> pairs;
    std::vector<long long> halves;  // (p, k, counted): the partner lives in another slab
    const int* N = e.plan.N;
    int c[3];
    for (c[2] = clo[2]; c[2] <= chi[2]; ++c[2])
        for (c[1] = clo[1]; c[1] <= chi[1]; ++c[1])
            for (c[0] = clo[0]; c[0] <= chi[0]; ++c[0]) {
                int cl[3] = {c[0], c[1], c[2]};
                cl[SA] -= zoff;
                const int64_t p = ((int64_t)cl[2] * N[1] + cl[1]) * N[0] + cl[0];
                const int64_t gp = glin(c);
                double xp[3];
                gpos(c, xp);
                for (int k = 0; k < e.nof; ++k) {
                    const int* o = &e.offs[3 * k];
                    int qc[3] = {c[0] + o[0], c[1] + o[1], c[2] + o[2]};
                    bool in = true;
                    for (int d = 0; d < dim; ++d) in = in && qc[d] >= 0 && qc[d] < G[d];
                    if (!in) continue;
                    const bool local = qc[SA] >= zoff && qc[SA] < zoff + N[SA];
                    const int64_t gq = glin(qc);
                    if (gq < gp && local) continue;  // visited from q
                    double xq[3];
                    gpos(qc, xq);
                    const double* a = gq > gp ? xp : xq;  // lower node first, as the reference visits it
                    const double* b = gq > gp ? xq : xp;
                    const bool cross = notch ? assembly::notch_crosses(geom, a, b) : assembly::segment_crosses(geom, a, b);
                    if (!cross) continue;
                    if (local) {
                        int ql[3] = {qc[0], qc[1], qc[2]};
                        ql[SA] -= zoff;
                        pairs.push_back(p);
                        pairs.push_back(((int64_t)ql[2] * N[1] + ql[1]) * N[0] + ql[0]);
                    } else {
                        halves.insert(halves.end(), {(long long)p, (long long)k, gq > gp ? 1LL : 0LL});
                    }
                }
            }
    int64_t n = break_pairs(e, pairs.data(), (int64_t)pairs.size() / 2);
    n += break_halves(e, halves);
    if (added) *added = n;
}

int pdgpu_seed_segment(pdgpu_t h, const double* seg, int64_t* added) {
    return guarded([&] {
        if (!h || !seg) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        if (h->dim != 2) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "segments are 2D cracks");
        cuda_check(cudaSetDevice(h->device), "set device");
        seed_impl(*h, seg, false, added);
    });
}

int pdgpu_seed_notch(pdgpu_t h, const double* notch, int64_t* added) {
    return guarded([&] {
        if (!h || !notch) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        if (h->dim != 3) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "notches are 3D cracks");
        cuda_check(cudaSetDevice(h->device), "set device");
        seed_impl(*h, notch, true, added);
    });
}

// one stretch sweep on device-resident u; the newly broken pairs are kept on
// the host (e.last_pairs) in the reference's visiting order
static int64_t update_bonds_impl(Engine& e, const double* u, double s0, const double* watch) {
    ensure_ledger(e);
    halo_exchange_now(e, u, e.stream);  // slabs: the rows beyond the upper face, for the bonds this slab owns
    const int64_t N = e.plan.nodes;
    const size_t lbytes = sizeof(uint32_t) * (size_t)(N * e.lw);
    // ledger before the sweep: if one sweep breaks more bonds than the device
    // pair buffer holds, the new pairs are recovered as the ledger difference
    // instead of being truncated
    uint32_t* d_prev = nullptr;
    cuda_check(cudaMallocAsync((void**)&d_prev, lbytes, e.stream), "alloc ledger snapshot");
    cuda_check(cudaMemcpyAsync(d_prev, e.d_ledger, lbytes, cudaMemcpyDeviceToDevice, e.stream), "snapshot");
    const int64_t n = launch_update_bonds(e, u, s0, watch, e.stream);
    if (halo_active(e)) {
        ledger_exchange(e, e.stream);  // slabs: mirror the bits of bonds broken across the face below
        unsigned long long rows = 0;
        cuda_check(cudaMemcpyAsync(&rows, e.d_counters, sizeof(rows), cudaMemcpyDeviceToHost, e.stream), "rows");
        cuda_check(cudaStreamSynchronize(e.stream), "merge");
        e.n_bond_rows = (int64_t)rows;
    }
    std::vector<std::pair<long long, long long>> pk;  // (p, offset index)
    if (n > 0 && n <= e.new_pairs_cap) {
        std::vector<long long> raw((size_t)(2 * n));
        cuda_check(cudaMemcpy(raw.data(), e.d_new_pairs, sizeof(long long) * raw.size(), cudaMemcpyDeviceToHost),
                   "read pairs");
        for (int64_t i = 0; i < n; ++i) pk.push_back({raw[2 * i], raw[2 * i + 1]});
    } else if (n > 0) {
        std::vector<uint32_t> now((size_t)(N * e.lw)), before((size_t)(N * e.lw));
        cuda_check(cudaMemcpy(now.data(), e.d_ledger, lbytes, cudaMemcpyDeviceToHost), "read ledger");
        cuda_check(cudaMemcpy(before.data(), d_prev, lbytes, cudaMemcpyDeviceToHost), "read ledger snapshot");
        for (int64_t p = 0; p < N; ++p)
            for (int k = 0; k < e.nof; ++k) {
                const int* o = &e.offs[3 * k];
                const long long disp = (long long)o[2] * e.plan.N[0] * e.plan.N[1] + (long long)o[1] * e.plan.N[0] + o[0];
                if (disp <= 0) continue;  // q > p owns the pair (fracture.hpp:220)
                const size_t w = (size_t)(p * e.lw + (k >> 5));
                if (((now[w] & ~before[w]) >> (k & 31)) & 1u) pk.push_back({p, k});
            }
    }
    cuda_check(cudaFreeAsync(d_prev, e.stream), "free ledger snapshot");
    cuda_check(cudaStreamSynchronize(e.stream), "update_bonds");
    // the reference's visiting order: p ascending, then for_each_offset order
    std::sort(pk.begin(), pk.end());
    const int* Nd = e.plan.N;
    const int64_t goff = global_offset(e);
    e.last_pairs.resize(2 * pk.size());
    for (size_t i = 0; i < pk.size(); ++i) {
        const int* o = &e.offs[3 * pk[i].second];
        e.last_pairs[2 * i] = goff + pk[i].first;
        e.last_pairs[2 * i + 1] = goff + pk[i].first + (long long)o[2] * Nd[0] * Nd[1] + (long long)o[1] * Nd[0] + o[0];
    }
    return n;
}

static void copy_pairs(const std::vector<int64_t>& pairs, int64_t* out, int64_t cap) {
    const int64_t n = (int64_t)pairs.size() / 2;
    if (out && cap > 0) std::copy(pairs.begin(), pairs.begin() + 2 * std::min(n, cap), out);
}

int pdgpu_update_bonds(pdgpu_t h, const double* u, double s0, const double* watch, int64_t* out, int64_t cap,
                       int64_t* count) {
    return guarded([&] {
        if (!h || !u) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t n = update_bonds_impl(*h, u, s0, watch);
        if (count) *count = n;
        copy_pairs(h->last_pairs, out, cap);
    });
}

int pdgpu_update_bonds_host(pdgpu_t h, const double* u, int64_t n_nodes, double s0, const double* watch,
                            int64_t* out, int64_t cap, int64_t* count) {
    return guarded([&] {
        if (!h || !u) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        if (n_nodes != h->plan.nodes) throw PdError(PDGPU_ERR_SHAPE_MISMATCH, "field length does not match the lattice");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t m = (int64_t)h->dim * n_nodes;
        ensure_stage(*h, m);
        cuda_check(cudaMemcpyAsync(h->d_u_stage, u, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream), "H2D");
        const int64_t n = update_bonds_impl(*h, h->d_u_stage, s0, watch);
        if (count) *count = n;
        copy_pairs(h->last_pairs, out, cap);
    });
}

int pdgpu_last_new_pairs(pdgpu_t h, int64_t* out, int64_t cap, int64_t* count) {
    return guarded([&] {
        if (!h || !count) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        *count = (int64_t)h->last_pairs.size() / 2;
        copy_pairs(h->last_pairs, out, cap);
    });
}

// prescribed displacement values u_c over all DOFs (displacement constraints,
// later boxes win -- corrections.hpp:142-160 applied in order); true if any != 0
static bool prescribed_values(const Engine& e, std::vector<double>& huc) {
    const int64_t N = e.plan.nodes, m = (int64_t)e.dim * N;
    huc.assign((size_t)m, 0.0);
    for (const auto& cs : e.constraints) {
        if (cs.kind != 0) continue;
        for (int64_t pn = 0; pn < N; ++pn) {
            double xx[3];
            pos_of(e, pn, xx);
            if (!assembly::box_contains(e.dim, cs.lo, cs.hi, xx)) continue;
            for (int d = 0; d < e.dim; ++d)
                if ((cs.dir_mask >> d) & 1u) huc[(size_t)(d * N + pn)] = cs.value;
        }
    }
    bool any = false;
    for (double v : huc) any = any || v != 0.0;
    return any;
}

int pdgpu_constraint_values(pdgpu_t h, uint8_t* mask, double* uc) {
    return guarded([&] {
        if (!h) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null handle");
        const int64_t N = h->plan.nodes;
        if (mask) {
            if ((int64_t)h->h_cmask.size() == N) std::copy(h->h_cmask.begin(), h->h_cmask.end(), mask);
            else std::fill(mask, mask + N, (uint8_t)0);
        }
        if (uc) {
            std::vector<double> huc;
            prescribed_values(*h, huc);
            std::copy(huc.begin(), huc.end(), uc);
        }
    });
}

// ------------------------------------------------------------------ CG ---
// q = -A_ff p on the free rows (zero on constrained ones): MSBFM (default) or,
// with pdgpu_set_cg_operator(h, 1), the direct stencil sum of the same
// operator (csrc/direct.cu; no symbol, no FFT) plus the same corrections
static void cg_operator(Engine& e, const double* p, double* q, cudaStream_t s) {
    if (e.cg_direct && !e.ghost_view && e.slab.global < 0) {
        launch_direct_apply(e, p, q, 1, s, -1.0, e.d_cmask);
    } else {
        e.fold_surface_next = true;
        launch_fast_apply(e, p, q, 1, s, -1.0, e.d_cmask, nullptr);
    }
    launch_corrections(e, p, q, 1, s, -1.0);
}

// CG iterations per captured graph: small systems replay several per launch
// (the host's graph-launch cadence would otherwise bound the iteration rate);
// iterations past convergence find the done flag and update nothing.  The
// slab (NCCL) path keeps one.
static int cg_iters_per_graph(const Engine& e, int64_t m) {
    if (const char* env = getenv("PDGPU_CG_IPG")) return std::max(1, atoi(env));
    return (m <= (1 << 21) && !comm_attached(e)) ? 8 : 1;
}

static void cg_impl(Engine& e, const double* b, double* x, double tol, int maxit, int* iters, double* relres,
                    cudaStream_t s, double* hist_host, int nhist) {
    const int64_t N = e.plan.nodes, m = (int64_t)e.dim * N;
    if (!e.d_cg || e.cg_cap < m) {
        dalloc(e.d_cg, (size_t)(4 * m), "alloc cg");
        e.cg_cap = m;
    }
    double* r = e.d_cg;
    double* p = r + m;
    double* q = p + m;
    double* uc = q + m;
    // prescribed displacement values u_c (displacement constraints only), scattered
    // on the device from the list rebuild_constraints keeps (no host O(N) pass per solve)
    const bool any_uc = e.n_uc > 0;
    if (any_uc) {
        cuda_check(cudaMemsetAsync(uc, 0, sizeof(double) * m, s), "zero uc");
        launch_scatter(uc, e.d_uc_ids, e.d_uc_val, e.n_uc, s);
    }
    if (any_uc) {
        matvec_impl(e, uc, q, 1, s);
        launch_mask_rhs(r, b, q, e.d_cmask, N, e.dim, s);
    } else {
        launch_mask_rhs(r, b, nullptr, e.d_cmask, N, e.dim, s);
    }
    cuda_check(cudaMemsetAsync(x, 0, sizeof(double) * m, s), "zero x");
    cuda_check(cudaMemcpyAsync(p, r, sizeof(double) * m, cudaMemcpyDeviceToDevice, s), "p = r");
    launch_dot(e, r, r, m, e.d_scal + 0, s);
    // slabs over NCCL: every dot product is this rank's share, all-reduced in place
    const bool multi = comm_attached(e);
    comm_allreduce(e, e.d_scal + 0, 1, s);
    if (multi && halo_active(e)) ensure_halo(e, 1);  // the captured iteration's halo buffers exist before capture
    double rr0 = 0;
    cuda_check(cudaMemcpyAsync(&rr0, e.d_scal, sizeof(double), cudaMemcpyDeviceToHost, s), "read rr");
    cuda_check(cudaStreamSynchronize(s), "cg init");
    const double bnorm = sqrt(rr0);
    int k = 0;
    double rel = bnorm > 0 ? 1.0 : 0.0;
    if (!hist_host && bnorm > 0 && !getenv("PDGPU_CG_HOSTLOOP")) {
        // One iteration captured as a CUDA graph and replayed in chunks; the
        // convergence test runs on the device (k_cg_update_dev), so the host
        // synchronises once per chunk instead of once per iteration.
        engine_alloc_workspace(e, 1);
        const bool timing = e.timing;
        e.timing = false;
        if (!e.cg_graph || e.cg_graph_x != x || e.cg_graph_stream != s || e.cg_cap != m ||
            e.cg_graph_version != e.state_version) {
            if (e.cg_graph) cudaGraphExecDestroy(e.cg_graph);
            e.cg_graph = nullptr;
            cudaGraph_t g;
            const int64_t l0 = e.launches;
            cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
            // small systems: programmatic dependent launch between the latency-bound kernels
            const char* pdlenv = getenv("PDGPU_PDL");
            e.pdl = pdlenv && pdlenv[0] == '1';  // opt-in: measured neutral (32.1 vs 32.5 us at 128^2)
            for (int rep = 0; rep < cg_iters_per_graph(e, m); ++rep) {
                cg_operator(e, p, q, s);
                if (multi) {
                    launch_dot(e, p, q, m, e.d_scal + 1, s);
                    comm_allreduce(e, e.d_scal + 1, 1, s);
                    launch_cg_step_dev_comm(e, x, r, p, q, m, e.d_scal, s);
                } else if (!launch_cg_fused(e, x, r, p, q, m, e.d_scal, s)) {  // one cooperative kernel
                    launch_dot(e, p, q, m, e.d_scal + 1, s);
                    launch_cg_step_dev(e, x, r, p, q, m, e.d_scal, s);
                }
            }
            e.pdl = false;
            cuda_check(cudaStreamEndCapture(s, &g), "end capture");
            e.cg_graph_launches = e.launches - l0;  // kernels per replay (capture itself launches none)
            e.launches = l0;
            cuda_check(cudaGraphInstantiate(&e.cg_graph, g, 0), "instantiate");
            cudaGraphDestroy(g);
            e.cg_graph_x = x;
            e.cg_graph_stream = s;
            e.cg_graph_version = e.state_version;
        }
        e.timing = timing;
        const double init[7] = {rr0, 0.0, rr0, tol * tol * rr0, 0.0, 0.0, (double)maxit};  // [6]: iteration cap
        cuda_check(cudaMemcpyAsync(e.d_scal, init, sizeof(init), cudaMemcpyHostToDevice, s), "scal init");
        double st[6] = {0, 0, 0, 0, 0, 0};
        int launched = 0;
        const int ipg = cg_iters_per_graph(e, m);
        const int chunk = m > (1 << 22) ? 4 : 16;
        while (launched < maxit) {
            const int nl = std::min(chunk, (maxit - launched + ipg - 1) / ipg);
            for (int i = 0; i < nl; ++i) cuda_check(cudaGraphLaunch(e.cg_graph, s), "graph launch");
            launched += nl * ipg;
            e.launches += (int64_t)nl * e.cg_graph_launches;
            cuda_check(cudaMemcpyAsync(st, e.d_scal, sizeof(st), cudaMemcpyDeviceToHost, s), "read scal");
            cuda_check(cudaStreamSynchronize(s), "cg chunk");
            if (st[4] != 0.0) break;
        }
        k = (int)st[5];
        rel = sqrt(st[2]) / bnorm;
    }
    while (!(!hist_host && bnorm > 0 && !getenv("PDGPU_CG_HOSTLOOP")) && bnorm > 0 && k < maxit) {
        cg_operator(e, p, q, s);
        launch_dot(e, p, q, m, e.d_scal + 1, s);
        comm_allreduce(e, e.d_scal + 1, 1, s);
        launch_cg_update(e, x, r, p, q, m, e.d_scal, e.d_scal + 2, s);
        comm_allreduce(e, e.d_scal + 2, 1, s);
        double rr1 = 0;
        cuda_check(cudaMemcpyAsync(&rr1, e.d_scal + 2, sizeof(double), cudaMemcpyDeviceToHost, s), "read rr");
        ++k;
        if (hist_host && k <= nhist)
            cuda_check(cudaMemcpyAsync(hist_host + (size_t)(k - 1) * m, x, sizeof(double) * m, cudaMemcpyDeviceToHost, s),
                       "hist");
        cuda_check(cudaStreamSynchronize(s), "cg iter");
        rel = sqrt(rr1) / bnorm;
        if (rel <= tol) break;
        launch_cg_direction(p, r, m, e.d_scal, s);
    }
    if (any_uc) launch_axpy(x, uc, 1.0, m, s);
    cuda_check(cudaStreamSynchronize(s), "cg done");
    if (iters) *iters = k;
    if (relres) *relres = rel;
}

int pdgpu_cg_solve(pdgpu_t h, const double* b, double* x, double tol, int maxit, int* iters, double* relres,
                   void* stream) {
    return guarded([&] {
        if (!h || !b || !x) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        cudaStream_t s = pick_stream(*h, stream);
        if (s == cudaStreamLegacy || s == cudaStreamPerThread) {
            // default streams cannot be captured into the CG graph: run on the
            // engine stream, ordered after the caller's work (cg_impl syncs at exit)
            cuda_check(cudaStreamSynchronize(s), "sync caller stream");
            s = h->stream;
        }
        cg_impl(*h, b, x, tol, maxit, iters, relres, s, nullptr, 0);
    });
}

int pdgpu_cg_solve_host(pdgpu_t h, const double* b, double* x, double tol, int maxit, int* iters, double* relres,
                        double* hist, int nhist) {
    return guarded([&] {
        if (!h || !b || !x) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t m = (int64_t)h->dim * h->plan.nodes;
        ensure_stage(*h, m);
        cuda_check(cudaMemcpyAsync(h->d_u_stage, b, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream), "H2D");
        cg_impl(*h, h->d_u_stage, h->d_f_stage, tol, maxit, iters, relres, h->stream, hist, nhist);
        cuda_check(cudaMemcpy(x, h->d_f_stage, sizeof(double) * m, cudaMemcpyDeviceToHost), "D2H");
    });
}

// ------------------------------------------------------------------ VV ---
int pdgpu_sim_init(pdgpu_t h, double dt, const double* v0) {
    return guarded([&] {
        if (!h) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null handle");
        cuda_check(cudaSetDevice(h->device), "set device");
        const int64_t m = (int64_t)h->dim * h->plan.nodes;
        dalloc(h->d_u, (size_t)m, "alloc u");
        dalloc(h->d_v, (size_t)m, "alloc v");
        dalloc(h->d_f, (size_t)m, "alloc f");
        dalloc(h->d_fprev, (size_t)m, "alloc fprev");
        cuda_check(cudaMemset(h->d_u, 0, sizeof(double) * m), "zero");
        cuda_check(cudaMemset(h->d_v, 0, sizeof(double) * m), "zero");
        cuda_check(cudaMemset(h->d_f, 0, sizeof(double) * m), "zero");
        cuda_check(cudaMemset(h->d_fprev, 0, sizeof(double) * m), "zero");
        if (v0) cuda_check(cudaMemcpy(h->d_v, v0, sizeof(double) * m, cudaMemcpyHostToDevice), "copy v0");
        h->dt = dt;
        h->t = 0.0;
        h->step = 0;
        h->force_ready = false;
        h->integrator = 0;
        launch_enforce(h->d_u, h->d_v, h->d_cdofs, h->d_cval, h->d_ckind, h->n_cdofs, 0.0, h->stream);
        cuda_check(cudaStreamSynchronize(h->stream), "sim init");
    });
}

int pdgpu_sim_init_adr(pdgpu_t h, double dt, double fixed_damping) {
    const int rc = pdgpu_sim_init(h, dt, nullptr);
    if (rc != PDGPU_OK) return rc;
    return guarded([&] {
        Engine& e = *h;
        const int64_t m = (int64_t)e.dim * e.plan.nodes;
        dalloc(e.d_vh, (size_t)m, "alloc v_half");
        cuda_check(cudaMemset(e.d_vh, 0, sizeof(double) * m), "zero v_half");
        // adr_mass (timestepping.hpp:150-162): 1/4 dt^2 sum_b 2 sum_off |K_ab(off)|,
        // offsets in for_each_offset order (kernel.hpp:71-89)
        for (int a = 0; a < e.dim; ++a) {
            double row = 0.0;
            for (int b = 0; b < e.dim; ++b) {
                double off_abs = 0.0;
                const int pr = assembly::pair_index(e.dim, a, b);
                for (int k = 0; k < e.nof; ++k)
                    off_abs += fabs(e.stencils[(size_t)(pr * e.ss + assembly::stencil_index(e.dim, e.M, &e.offs[3 * k]))]);
                row += 2.0 * off_abs;
            }
            e.adr_mass[a] = 0.25 * dt * dt * row;
        }
        e.integrator = 1;
        e.adr_fixed = fixed_damping == fixed_damping;  // NaN: adaptive (std::nullopt)
        e.adr_fixed_c = e.adr_fixed ? fixed_damping : 0.0;
        cuda_check(cudaMemset(e.d_scal + 10, 0, sizeof(double)), "zero damping");
    });
}

int pdgpu_sim_adr_damping(pdgpu_t h, double* c) {
    return guarded([&] {
        if (!h || !c) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        cuda_check(cudaStreamSynchronize(h->stream), "sync");
        cuda_check(cudaMemcpy(c, h->d_scal + 10, sizeof(double), cudaMemcpyDeviceToHost), "damping");
    });
}

// ---- one Simulation::step (timestepping.hpp:209-241) in phases, so the
// single-process slab group (pdgpu_group_sim_step) can exchange halo rows and
// face ledgers between them; pdgpu_sim_step runs them back to back (the NCCL
// exchanges happen inside the force and after the sweep).
static void sim_initial_force(Engine& e) {
    if (e.force_ready) return;
    evaluate_force_impl(e, e.d_u, e.d_f, e.stream);
    e.force_ready = true;
}

static void sim_pre(Engine& e) {
    const int64_t N = e.plan.nodes;
    if (e.integrator == 1) {  // ADR branch (timestepping.hpp:215-220)
        launch_adr_step(e, e.step == 0, e.stream);
    } else if (e.drift_done) {
        e.drift_done = false;  // done with the previous step's kick (sim_post)
    } else {
        launch_vv_drift(e.d_u, e.d_v, e.d_f, e.d_cmask, N, e.dim, e.dt, 1.0 / e.rho, e.stream);
    }
    e.t += e.dt;
    launch_enforce(e.d_u, e.d_v, e.d_cdofs, e.d_cval, e.d_ckind, e.n_cdofs, e.t, e.stream);
    std::swap(e.d_f, e.d_fprev);
}

static void sim_force(Engine& e) { evaluate_force_impl(e, e.d_u, e.d_f, e.stream); }

// fuse_next: another VV step follows in this call and nothing reads the state
// in between -- the stretch test moves in front (it reads u only), then the
// kick and the next step's drift run as one kernel (both skip constrained
// DOFs, which launch_enforce owns)
static void sim_post(Engine& e, double s0, const double* watch, bool fuse_next = false) {
    const int64_t N = e.plan.nodes;
    if (e.integrator != 1 && fuse_next) {
        if (s0 >= 0) launch_update_bonds(e, e.d_u, s0, watch, e.stream, /*sync=*/false);
        launch_vv_kick_drift(e.d_u, e.d_v, e.d_fprev, e.d_f, e.d_cmask, N, e.dim, e.dt, 1.0 / e.rho, e.stream);
        launch_enforce(e.d_u, e.d_v, e.d_cdofs, e.d_cval, e.d_ckind, e.n_cdofs, e.t, e.stream);
        e.drift_done = true;
        ++e.step;
        return;
    }
    if (e.integrator != 1) {
        launch_vv_kick(e.d_v, e.d_fprev, e.d_f, e.d_cmask, N, e.dim, e.dt, 1.0 / e.rho, e.stream);
        launch_enforce(e.d_u, e.d_v, e.d_cdofs, e.d_cval, e.d_ckind, e.n_cdofs, e.t, e.stream);
    }
    // the stretch test reads u's halo rows from this step's force exchange
    if (s0 >= 0) launch_update_bonds(e, e.d_u, s0, watch, e.stream, /*sync=*/false);
    ++e.step;
}

// one MonitorWriter row per step: u at the monitored nodes, gathered on the
// device (no field download); a full device buffer moves to the host spill
static void monitor_spill(Engine& e) {
    if (!e.mon_dev_rows) return;
    const size_t cnt = (size_t)e.mon_dev_rows * e.n_mon * e.dim;
    const size_t off = e.mon_spill.size();
    e.mon_spill.resize(off + cnt);
    cuda_check(cudaMemcpyAsync(e.mon_spill.data() + off, e.d_mon_rows, sizeof(double) * cnt, cudaMemcpyDeviceToHost,
                               e.stream), "monitor rows");
    cuda_check(cudaStreamSynchronize(e.stream), "monitor rows");
    e.mon_dev_rows = 0;
}

static void monitor_record(Engine& e) {
    if (!e.n_mon) return;
    if (e.mon_dev_rows == e.mon_cap) monitor_spill(e);
    launch_monitor_gather(e.d_u, e.d_mon_nodes, e.n_mon, e.dim, e.plan.nodes,
                          e.d_mon_rows + (size_t)e.mon_dev_rows * e.n_mon * e.dim, e.stream);
    e.launches += 1;
    ++e.mon_dev_rows;
    e.mon_step.push_back(e.step);
    e.mon_t.push_back(e.t);
}

static void sim_begin(Engine& e, int n_steps, double s0) {
    if (!e.d_u) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "simulation not initialised");
    e.sim_swept = s0 >= 0 && n_steps > 0;
    if (s0 >= 0) {
        ensure_ledger(e);
        cuda_check(cudaMemsetAsync(e.d_counters + 2, 0, sizeof(unsigned long long), e.stream), "reset breaks");
    }
}

static int64_t sim_end(Engine& e, double s0) {
    int64_t nb = 0;
    if (s0 >= 0) {
        // one read-back per call: row count and breaks of all steps
        unsigned long long cnt[3];
        cuda_check(cudaMemcpyAsync(cnt, e.d_counters, sizeof(cnt), cudaMemcpyDeviceToHost, e.stream), "counters");
        cuda_check(cudaStreamSynchronize(e.stream), "sim step");
        e.n_bond_rows = (int64_t)cnt[0];
        e.bond_rows_on_device = false;
        nb = (int64_t)cnt[2];
        e.total_broken += nb;
    }
    cuda_check(cudaStreamSynchronize(e.stream), "sim step");
    return nb;
}

int pdgpu_sim_step(pdgpu_t h, int n_steps, double s0, const double* watch, int64_t* broken) {
    return guarded([&] {
        if (!h || !h->d_u) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "simulation not initialised");
        cuda_check(cudaSetDevice(h->device), "set device");
        Engine& e = *h;
        sim_begin(e, n_steps, s0);
        // single lattice, no monitor: kick + next drift fused (PDGPU_VV_NOFUSE=1: separate kernels)
        const bool can_fuse = e.integrator != 1 && !e.n_mon && e.slab.global < 0 && !e.nccl_comm && !getenv("PDGPU_VV_NOFUSE");
        for (int i = 0; i < n_steps; ++i) {
            sim_initial_force(e);
            sim_pre(e);
            sim_force(e);
            sim_post(e, s0, watch, can_fuse && i + 1 < n_steps);
            if (s0 >= 0) ledger_exchange(e, e.stream);  // NCCL slabs: mirror bonds broken across the face below
            monitor_record(e);
        }
        const int64_t nb = sim_end(e, s0);
        if (broken) *broken = nb;
    });
}

// ---- single-process slab group: n engines holding consecutive row slabs of
// one lattice (pdgpu_set_slab), on one or several devices, stepped together;
// halo rows and face ledgers move by device copies instead of NCCL.
static void group_halo(pdgpu_t* hs, int n) {
    for (int r = 0; r < n; ++r) {
        Engine& e = *hs[r];
        cuda_check(cudaSetDevice(e.device), "set device");
        ensure_halo(e, 1);
        halo_pack(e, e.d_u, 1, e.d_halo, e.stream);
        if (!e.ev_fork) cuda_check(cudaEventCreateWithFlags(&e.ev_fork, cudaEventDisableTiming), "event");
        cuda_check(cudaEventRecord(e.ev_fork, e.stream), "pack done");
    }
    for (int r = 0; r < n; ++r) {
        Engine& e = *hs[r];
        cuda_check(cudaSetDevice(e.device), "set device");
        const int64_t plane = e.dim == 3 ? (int64_t)e.plan.N[0] * e.plan.N[1] : e.plan.N[0];
        const size_t side = (size_t)e.dim * e.M * plane;  // batch 1
        double* recv = e.d_halo + (size_t)2 * e.halo_cap * e.dim * e.M * plane;
        for (int sd = 0; sd < 2; ++sd) {
            const int nb = sd == 0 ? r - 1 : r + 1;
            if (nb < 0 || nb >= n) continue;
            Engine& o = *hs[nb];
            cuda_check(cudaStreamWaitEvent(e.stream, o.ev_fork, 0), "wait pack");
            // the neighbour's high rows arrive as side 0, its low rows as side 1
            const double* src = o.d_halo + (sd == 0 ? side : 0);
            cuda_check(cudaMemcpyPeerAsync(recv + sd * side, e.device, src, o.device, sizeof(double) * side, e.stream),
                       "halo copy");
        }
        e.ghost_view = recv;
        e.ghost_bc_stride = e.M * plane;
        e.ghost_side_stride = (int64_t)side;
        e.halo_external = true;
    }
}

static void group_faces(pdgpu_t* hs, int n) {
    for (int r = 0; r < n; ++r) {
        Engine& e = *hs[r];
        cuda_check(cudaSetDevice(e.device), "set device");
        cuda_check(cudaEventRecord(e.ev_fork, e.stream), "sweep done");
    }
    for (int r = 1; r < n; ++r) {
        Engine& e = *hs[r];
        Engine& o = *hs[r - 1];
        cuda_check(cudaSetDevice(e.device), "set device");
        ledger_face_buffer(e);
        const int64_t plane = e.dim == 3 ? (int64_t)e.plan.N[0] * e.plan.N[1] : e.plan.N[0];
        const size_t bytes = sizeof(uint32_t) * (size_t)e.M * plane * e.lw;
        cuda_check(cudaStreamWaitEvent(e.stream, o.ev_fork, 0), "wait sweep");
        cuda_check(cudaMemcpyPeerAsync(e.d_face_recv, e.device, ledger_face_send(o), o.device, bytes, e.stream),
                   "face copy");
        launch_merge_face(e, e.d_face_recv, e.stream);
    }
}

// ---- distributed FFT (transpose.cu) ------------------------------------
int pdgpu_set_transpose(pdgpu_t h, int nranks, int rank, int global_rows, const int* row_bounds,
                        const int* col_bounds) {
    return guarded([&] {
        if (!h || !row_bounds || !col_bounds) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        try {
            a2a_setup(*h, nranks, rank, global_rows, row_bounds, col_bounds);
        } catch (const std::runtime_error& ex) {
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, ex.what());
        }
        // D^e, near-surface flags, positions and ids of the global lattice
        Engine& e = *h;
        e.h_near = assembly::near_surface(e.dim, e.plan.N, e.M, e.slab);
        std::vector<long long> rows;
        std::vector<double> de;
        assembly::surface_diag(e.dim, e.plan.N, e.M, e.stencils.data(), e.h_near, rows, de, e.slab);
        upload_surface(e, rows, de);
    });
}

// One K.u (apply + corrections) of a lattice split over the n engines of one
// process (pdgpu_set_transpose on each, rank r = engine r), the all-to-all
// transposes done by device copies: the single-process stand-in for the NCCL
// path, for tests on one GPU.
int pdgpu_group_matvec_transpose(pdgpu_t* hs, int n, const double* const* us, double* const* fs, int batch) {
    return guarded([&] {
        if (!hs || !us || !fs || n < 1 || batch < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad group");
        for (int r = 0; r < n; ++r)
            if (!hs[r] || hs[r]->a2a.G != n || hs[r]->a2a.rank != r)
                throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "group engine without the matching pdgpu_set_transpose");
        struct Reset {
            pdgpu_t* hs;
            int n;
            ~Reset() {
                for (int r = 0; r < n; ++r) hs[r]->a2a_external = false;
            }
        } reset{hs, n};
        std::vector<cudaEvent_t> ev(n);
        for (int r = 0; r < n; ++r) {
            cuda_check(cudaSetDevice(hs[r]->device), "set device");
            cuda_check(cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming), "event");
            hs[r]->a2a_external = true;
        }
        auto each = [&](auto&& fn) {
            for (int r = 0; r < n; ++r) {
                cuda_check(cudaSetDevice(hs[r]->device), "set device");
                fn(r, *hs[r]);
                cuda_check(cudaEventRecord(ev[r], hs[r]->stream), "record");
            }
        };
        // every engine's block g of d_send -> engine g's d_recv block r
        auto exchange = [&]() {
            const int64_t blk = a2a_block(*hs[0], batch);
            for (int r = 0; r < n; ++r) {
                Engine& e = *hs[r];
                cuda_check(cudaSetDevice(e.device), "set device");
                for (int g = 0; g < n; ++g) {
                    Engine& o = *hs[g];
                    cuda_check(cudaStreamWaitEvent(e.stream, ev[g], 0), "wait peer");
                    cuda_check(cudaMemcpyPeerAsync(e.a2a.d_recv + (size_t)g * blk, e.device, o.a2a.d_send + (size_t)r * blk,
                                                   o.device, sizeof(double2) * blk, e.stream),
                               "a2a copy");
                }
            }
            for (int r = 0; r < n; ++r) {
                cuda_check(cudaSetDevice(hs[r]->device), "set device");
                cuda_check(cudaEventRecord(ev[r], hs[r]->stream), "record");
            }
            for (int r = 0; r < n; ++r) {  // senders wait for their readers before reusing d_send
                cuda_check(cudaSetDevice(hs[r]->device), "set device");
                for (int g = 0; g < n; ++g) cuda_check(cudaStreamWaitEvent(hs[r]->stream, ev[g], 0), "wait readers");
            }
        };
        each([&](int r, Engine& e) { a2a_phase1(e, us[r], batch, e.stream); });
        exchange();
        each([&](int, Engine& e) { a2a_phase2(e, batch, e.stream); });
        exchange();
        each([&](int r, Engine& e) {
            a2a_phase3(e, fs[r], batch, e.stream, 1.0, nullptr, nullptr);
            halo_pack(e, us[r], batch, e.a2a.d_alias, e.stream);  // [side][batch][dim][M][Nx]
        });
        // the ring halo: engine r's side 0 <- engine r-1's last M rows, side 1 <-
        // engine r+1's first M rows (mod n)
        for (int r = 0; r < n; ++r) {
            Engine& e = *hs[r];
            Engine& lo = *hs[(r + n - 1) % n];
            Engine& hi = *hs[(r + 1) % n];
            const size_t side = (size_t)batch * e.dim * e.M * e.plan.N[0];
            cuda_check(cudaSetDevice(e.device), "set device");
            cuda_check(cudaStreamWaitEvent(e.stream, ev[(r + n - 1) % n], 0), "wait");
            cuda_check(cudaStreamWaitEvent(e.stream, ev[(r + 1) % n], 0), "wait");
            cuda_check(cudaMemcpyPeerAsync(a2a_alias_recv(e, batch), e.device, lo.a2a.d_alias + side, lo.device,
                                           sizeof(double) * side, e.stream),
                       "ring low");
            cuda_check(cudaMemcpyPeerAsync(a2a_alias_recv(e, batch) + side, e.device, hi.a2a.d_alias, hi.device,
                                           sizeof(double) * side, e.stream),
                       "ring high");
        }
        each([&](int r, Engine& e) {
            const size_t side = (size_t)batch * e.dim * e.M * e.plan.N[0];
            e.ghost_bc_stride = (int64_t)e.M * e.plan.N[0];
            e.ghost_side_stride = (int64_t)side;
            e.ghost_view = a2a_alias_recv(e, batch);
            launch_wrap_correction(e, us[r], fs[r], batch, e.stream, 1.0, nullptr);
            launch_corrections(e, us[r], fs[r], batch, e.stream, 1.0);
        });
        for (int r = 0; r < n; ++r) {
            cuda_check(cudaSetDevice(hs[r]->device), "set device");
            cuda_check(cudaStreamSynchronize(hs[r]->stream), "group matvec");
            cudaEventDestroy(ev[r]);
        }
    });
}

int pdgpu_group_sim_step(pdgpu_t* hs, int n, int n_steps, double s0, const double* watch, int64_t* broken) {
    return guarded([&] {
        if (!hs || n < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "empty group");
        for (int r = 0; r < n; ++r) {
            if (!hs[r] || !hs[r]->d_u) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "simulation not initialised");
            if (n > 1 && hs[r]->slab.global < 0) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "group engines need pdgpu_set_slab");
            if (comm_attached(*hs[r])) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "group engines carry no communicator");
        }
        struct Reset {
            pdgpu_t* hs;
            int n;
            ~Reset() {
                for (int r = 0; r < n; ++r) hs[r]->halo_external = false;
            }
        } reset{hs, n};
        for (int r = 0; r < n; ++r) {
            cuda_check(cudaSetDevice(hs[r]->device), "set device");
            sim_begin(*hs[r], n_steps, s0);
        }
        auto each = [&](auto&& fn) {
            for (int r = 0; r < n; ++r) {
                cuda_check(cudaSetDevice(hs[r]->device), "set device");
                fn(*hs[r]);
            }
        };
        for (int i = 0; i < n_steps; ++i) {
            if (!hs[0]->force_ready) {
                group_halo(hs, n);
                each([](Engine& e) { sim_initial_force(e); });
            }
            each([](Engine& e) { sim_pre(e); });
            group_halo(hs, n);
            each([](Engine& e) { sim_force(e); });
            each([&](Engine& e) { sim_post(e, s0, watch); });
            if (s0 >= 0) group_faces(hs, n);
        }
        int64_t nb = 0;
        each([&](Engine& e) { nb += sim_end(e, s0); });
        if (broken) *broken = nb;
    });
}

int pdgpu_sim_get(pdgpu_t h, double* u, double* v, double* f, double* t) {
    return guarded([&] {
        if (!h || !h->d_u) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "simulation not initialised");
        cuda_check(cudaSetDevice(h->device), "set device");
        const size_t m = sizeof(double) * h->dim * h->plan.nodes;
        cuda_check(cudaStreamSynchronize(h->stream), "sync");
        if (u) cuda_check(cudaMemcpy(u, h->d_u, m, cudaMemcpyDeviceToHost), "u");
        if (v) cuda_check(cudaMemcpy(v, h->d_v, m, cudaMemcpyDeviceToHost), "v");
        if (f) cuda_check(cudaMemcpy(f, h->d_f, m, cudaMemcpyDeviceToHost), "f");
        if (t) *t = h->t;
    });
}

int pdgpu_sim_get_aux(pdgpu_t h, double* f_prev, double* v_half) {
    return guarded([&] {
        if (!h || !h->d_u) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "simulation not initialised");
        cuda_check(cudaSetDevice(h->device), "set device");
        const size_t m = sizeof(double) * h->dim * h->plan.nodes;
        cuda_check(cudaStreamSynchronize(h->stream), "sync");
        if (f_prev) cuda_check(cudaMemcpy(f_prev, h->d_fprev, m, cudaMemcpyDeviceToHost), "f_prev");
        if (v_half) {
            if (h->d_vh) cuda_check(cudaMemcpy(v_half, h->d_vh, m, cudaMemcpyDeviceToHost), "v_half");
            else memset(v_half, 0, m);
        }
    });
}

int pdgpu_sim_set_velocity(pdgpu_t h, const double* v) {
    return guarded([&] {
        if (!h || !h->d_u || !v) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "simulation not initialised");
        cuda_check(cudaSetDevice(h->device), "set device");
        const size_t m = sizeof(double) * h->dim * h->plan.nodes;
        cuda_check(cudaMemcpyAsync(h->d_v, v, m, cudaMemcpyHostToDevice, h->stream), "copy v");
        launch_enforce(h->d_u, h->d_v, h->d_cdofs, h->d_cval, h->d_ckind, h->n_cdofs, h->t, h->stream);
        cuda_check(cudaStreamSynchronize(h->stream), "set velocity");
    });
}

int pdgpu_sim_newly_broken(pdgpu_t h, int64_t* out, int64_t cap, int64_t* count) {
    return guarded([&] {
        if (!h || !count) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        *count = 0;
        if (!h->sim_swept || !h->d_counters) return;
        unsigned long long n = 0;
        cuda_check(cudaStreamSynchronize(h->stream), "sync");
        cuda_check(cudaMemcpy(&n, h->d_counters + 1, sizeof(n), cudaMemcpyDeviceToHost), "count");
        *count = (int64_t)n;
        if (!out || cap <= 0 || n == 0) return;
        if ((int64_t)n > h->new_pairs_cap)
            throw PdError(PDGPU_ERR_NOT_SUPPORTED, "the last step broke more bonds than the device pair buffer holds");
        std::vector<long long> raw((size_t)(2 * n));
        cuda_check(cudaMemcpy(raw.data(), h->d_new_pairs, sizeof(long long) * raw.size(), cudaMemcpyDeviceToHost),
                   "read pairs");
        std::vector<std::pair<long long, long long>> pk;
        for (size_t i = 0; i < n; ++i) pk.push_back({raw[2 * i], raw[2 * i + 1]});
        std::sort(pk.begin(), pk.end());
        const int* Nd = h->plan.N;
        const int64_t goff = global_offset(*h);
        for (int64_t i = 0; i < std::min<int64_t>((int64_t)n, cap); ++i) {
            const int* o = &h->offs[3 * pk[(size_t)i].second];
            out[2 * i] = goff + pk[(size_t)i].first;
            out[2 * i + 1] = goff + pk[(size_t)i].first + (long long)o[2] * Nd[0] * Nd[1] + (long long)o[1] * Nd[0] + o[0];
        }
    });
}

int pdgpu_sim_finite(pdgpu_t h, int* ok) {
    return guarded([&] {
        if (!h || !h->d_u || !ok) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "simulation not initialised");
        cuda_check(cudaSetDevice(h->device), "set device");
        int* d_ok = (int*)(h->d_ticket + 2);  // spare slots of the ticket allocation
        const int one = 1;
        cuda_check(cudaMemcpyAsync(d_ok, &one, sizeof(int), cudaMemcpyHostToDevice, h->stream), "finite init");
        launch_finite(h->d_u, (int64_t)h->dim * h->plan.nodes, d_ok, h->stream);
        cuda_check(cudaMemcpyAsync(ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, h->stream), "finite read");
        cuda_check(cudaStreamSynchronize(h->stream), "finite");
    });
}

// --------------------------------------------------------- diagnostics ---
int pdgpu_timing_enable(pdgpu_t h, int on) {
    return guarded([&] {
        if (!h) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null handle");
        h->timing = on != 0;
    });
}

int pdgpu_timing_read(pdgpu_t h, double* ms, int64_t* cnt, int npass) {
    return guarded([&] {
        if (!h) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null handle");
        cuda_check(cudaSetDevice(h->device), "set device");
        cuda_check(cudaDeviceSynchronize(), "timing sync");
        for (int i = 0; i < npass; ++i) {
            if (ms) ms[i] = 0.0;
            if (cnt) cnt[i] = 0;
        }
        for (size_t k = 0; k < h->mark_pass.size(); ++k) {
            const int id = h->mark_pass[k];
            if (id >= npass) continue;
            float t = 0.f;
            cuda_check(cudaEventElapsedTime(&t, h->mark_a[k], h->mark_b[k]), "elapsed");
            if (ms) ms[id] += t;
            if (cnt) cnt[id] += 1;
        }
        h->mark_pass.clear();
        h->mark_a.clear();
        h->mark_b.clear();
        h->ev_used = 0;
    });
}

int64_t pdgpu_launch_count(pdgpu_t h) { return h ? h->launches : 0; }

// ------------------------------------------------------------ assembly ---
int pdgpu_build_kernel(int dim, double spacing, double delta, int M, double E, double thickness, double* out) {
    return guarded([&] {
        if (!out || (dim != 2 && dim != 3) || M < 1) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        if (dim == 2 && !(thickness > 0)) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "2D micromodulus requires the plate thickness");
        const std::vector<double> K = assembly::build_kernel(dim, spacing, delta, M, E, thickness);
        memcpy(out, K.data(), sizeof(double) * K.size());
    });
}

int pdgpu_near_surface(int dim, const int* dims, int M, uint8_t* out) {
    return guarded([&] {
        if (!out || !dims) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        const std::vector<uint8_t> v = assembly::near_surface(dim, dims, M);
        memcpy(out, v.data(), v.size());
    });
}

}  // extern "C"

/* ------------------------------------------------------------ snapshots -- */
int pdgpu_set_cg_operator(pdgpu_t h, int direct) {
    return guarded([&] {
        if (!h) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null handle");
        if (direct && (h->dim == 2 ? (h->M < 1 || h->M > 5) : false))
            throw PdError(PDGPU_ERR_NOT_SUPPORTED, "direct stencil: 2D horizon M must be 1..5");
        cuda_check(cudaSetDevice(h->device), "set device");
        if (direct) direct_prepare(*h);
        h->cg_direct = direct != 0;
        touch_state(*h);
    });
}

int pdgpu_sim_monitor(pdgpu_t h, const int64_t* nodes, int n) {
    return guarded([&] {
        if (!h || n < 0 || (n > 0 && !nodes)) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad monitor nodes");
        cuda_check(cudaSetDevice(h->device), "set device");
        Engine& e = *h;
        for (int k = 0; k < n; ++k)
            if (nodes[k] < 0 || nodes[k] >= e.plan.nodes) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "monitor node out of range");
        cuda_check(cudaStreamSynchronize(e.stream), "sync");
        e.n_mon = n;
        e.mon_dev_rows = 0;
        e.mon_step.clear();
        e.mon_t.clear();
        e.mon_spill.clear();
        if (!n) return;
        dalloc(e.d_mon_nodes, (size_t)n, "alloc monitor nodes");
        cuda_check(cudaMemcpy(e.d_mon_nodes, nodes, sizeof(long long) * n, cudaMemcpyHostToDevice), "copy monitor nodes");
        e.mon_cap = (int)std::max<int64_t>(64, std::min<int64_t>(4096, (1 << 22) / ((int64_t)n * e.dim)));
        dalloc(e.d_mon_rows, (size_t)e.mon_cap * n * e.dim, "alloc monitor rows");
    });
}

int pdgpu_sim_monitor_read(pdgpu_t h, int64_t* steps, double* t, double* values, int64_t cap, int64_t* count) {
    return guarded([&] {
        if (!h || !count) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        cuda_check(cudaSetDevice(h->device), "set device");
        Engine& e = *h;
        const int64_t rows = (int64_t)e.mon_step.size();
        *count = rows;
        if (!steps || !t || !values) return;
        if (cap < rows) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "monitor buffer too small");
        monitor_spill(e);
        const size_t per = (size_t)e.n_mon * e.dim;
        std::copy(e.mon_step.begin(), e.mon_step.end(), steps);
        std::copy(e.mon_t.begin(), e.mon_t.end(), t);
        std::copy(e.mon_spill.begin(), e.mon_spill.begin() + (size_t)rows * per, values);
        e.mon_step.clear();
        e.mon_t.clear();
        e.mon_spill.clear();
    });
}

int pdgpu_monitor_open(const char* path, int dim, const int* dims, double spacing, const double* origin,
                       const double* points, int npts, pdgpu_monitor_t* out) {
    return guarded([&] {
        if (!out || !dims || !origin || (npts > 0 && !points) || npts < 0 || dim < 2 || dim > 3 || !(spacing > 0))
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad monitor arguments");
        std::string err;
        snapshot::Monitor* m = snapshot::monitor_open(path, dim, dims, spacing, origin, points, npts, err);
        if (!m) throw PdError(PDGPU_ERR_IO, err);
        *out = reinterpret_cast<pdgpu_monitor_t>(m);
    });
}

int pdgpu_monitor_nodes(int dim, const int* dims, double spacing, const double* origin, const double* points, int npts,
                        int64_t* nodes) {
    return guarded([&] {
        if (!dims || !origin || !nodes || (npts > 0 && !points) || dim < 2 || dim > 3)
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        for (int k = 0; k < npts; ++k) nodes[k] = snapshot::nearest_node(dim, dims, spacing, origin, points + (size_t)k * dim);
    });
}

int pdgpu_monitor_append(pdgpu_monitor_t m, int64_t step, double t, const double* values) {
    return guarded([&] {
        if (!m || !values) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "null argument");
        snapshot::monitor_append(reinterpret_cast<snapshot::Monitor*>(m), step, t, values);
    });
}

void pdgpu_monitor_close(pdgpu_monitor_t m) {
    if (m) snapshot::monitor_close(reinterpret_cast<snapshot::Monitor*>(m));
}

int pdgpu_write_snapshot(int dim, const int* dims, double spacing, const double* origin, const double* u,
                         const double* damage, int64_t step, double t, const char* dir, char* path_out, int path_cap) {
    return guarded([&] {
        if (!dims || !origin || !dir || !u || dim < 1 || dim > 3) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        const std::string path = pdgpu::snapshot::write(dir, dim, dims, spacing, origin, u, damage, step, t);
        if (path.empty()) throw PdError(PDGPU_ERR_INVALID_ARGUMENT, std::string("cannot write snapshot in ") + dir);
        if (path_out && path_cap > 0) {
            strncpy(path_out, path.c_str(), (size_t)path_cap - 1);
            path_out[path_cap - 1] = 0;
        }
    });
}

int pdgpu_read_snapshot(const char* path, int dim, int* dims, double* spacing, double* origin, int64_t* step,
                        double* t, double* u, double* damage) {
    return guarded([&] {
        if (!path || !dims || !spacing || !origin || !step || !t || dim < 1 || dim > 3)
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, "bad arguments");
        std::string err;
        if (!pdgpu::snapshot::read(path, dim, dims, spacing, origin, step, t, u, damage, err))
            throw PdError(PDGPU_ERR_INVALID_ARGUMENT, err);
    });
}
