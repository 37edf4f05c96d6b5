// corrections.cu -- sparse correction SpMV and the bond-breaking kernel.
//
// K6a surface: f_a[p] += sum_b De_ab[p] u_b[p] on near-surface rows not
//     constrained in a (reference corrections.hpp:80-87).
// K6b bonds: warp per row with broken bonds, lane k <-> stencil offset k:
//     f_a[p] += sum_b K_ab(q-p) (u_b[p] - u_b[q]) over broken partners q
//     (corrections.hpp:89-109); deterministic xor-shuffle reduction.
// K7 update_bonds: thread per node over forward offsets (q > p), exact
//     non-linear stretch with IEEE round-to-nearest intrinsics (no FMA
//     contraction) so the break decision matches the reference's
//     bond_stretch bit for bit (fracture.hpp:17-29, 204-231).
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "engine.h"

namespace pdgpu {

template <int D>
__device__ __forceinline__ int pair_idx(int a, int b) {
    if (a > b) { const int t = a; a = b; b = t; }
    if (D == 2) return a + b;
    return (a == 0 ? 0 : (a == 1 ? 3 : 5)) + b - a;
}

template <int D>
__global__ void k_surface(const double* __restrict__ u, double* __restrict__ f, const long long* __restrict__ rows,
                          const double* __restrict__ de, const uint8_t* __restrict__ cmask, int64_t nrows,
                          int64_t nodes, int batch, double scale) {
    constexpr int NP = D * (D + 1) / 2;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows * batch) return;
    const int b = (int)(i / nrows);
    const int64_t r = i - (int64_t)b * nrows;
    const int64_t p = rows[r];
    const uint8_t cm = cmask[p];
    double up[D], dv[NP];
#pragma unroll
    for (int c = 0; c < D; ++c) up[c] = u[((int64_t)b * D + c) * nodes + p];
#pragma unroll
    for (int k = 0; k < NP; ++k) dv[k] = de[r * NP + k];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        if ((cm >> a) & 1u) continue;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) acc += dv[pair_idx<D>(a, c)] * up[c];
        f[((int64_t)b * D + a) * nodes + p] += scale * acc;
    }
}

template <int D>
__global__ void k_bonds(const double* __restrict__ u, double* __restrict__ f, const long long* __restrict__ rows,
                        int64_t nrows, const uint32_t* __restrict__ ledger, int lw, const long long* __restrict__ disp,
                        const double* __restrict__ koff, int nof, const uint8_t* __restrict__ cmask, int64_t nodes,
                        int batch, double scale) {
    constexpr int NP = D * (D + 1) / 2;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= nrows * batch) return;
    const int b = (int)(warp / nrows);
    const int64_t r = warp - (int64_t)b * nrows;
    const int64_t p = rows[r];
    const double* ub = u + (int64_t)b * D * nodes;
    double up[D];
#pragma unroll
    for (int c = 0; c < D; ++c) up[c] = ub[(int64_t)c * nodes + p];
    double acc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[a] = 0.0;
    for (int w = 0; w < lw; ++w) {
        const uint32_t word = ledger[p * lw + w];
        const int k = w * 32 + lane;
        if (k < nof && ((word >> lane) & 1u)) {
            const int64_t q = p + disp[k];
            double du[D];
#pragma unroll
            for (int c = 0; c < D; ++c) du[c] = up[c] - ub[(int64_t)c * nodes + q];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) s += koff[k * NP + pair_idx<D>(a, c)] * du[c];
                acc[a] += s;
            }
        }
    }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[a] += __shfl_xor_sync(0xffffffffu, acc[a], o);
    if (lane == 0) {
        const uint8_t cm = cmask[p];
#pragma unroll
        for (int a = 0; a < D; ++a)
            if (!((cm >> a) & 1u)) f[((int64_t)b * D + a) * nodes + p] += scale * acc[a];
    }
}

static void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void launch_corrections(Engine& e, const double* u, double* f, int batch, cudaStream_t s, double scale) {
    const int64_t N = e.plan.nodes;
    if (e.n_surf > 0) {
        PassTimer pt(e, kPassCorr, s);
        const int64_t tot = e.n_surf * batch;
        const int th = 256;
        if (e.dim == 2)
            k_surface<2><<<(unsigned)((tot + th - 1) / th), th, 0, s>>>(u, f, e.d_surf_rows, e.d_surf_de, e.d_cmask,
                                                                       e.n_surf, N, batch, scale);
        else
            k_surface<3><<<(unsigned)((tot + th - 1) / th), th, 0, s>>>(u, f, e.d_surf_rows, e.d_surf_de, e.d_cmask,
                                                                       e.n_surf, N, batch, scale);
    }
    if (e.n_bond_rows > 0) {
        PassTimer pt(e, kPassBonds, s);
        const int64_t warps = e.n_bond_rows * batch;
        const int th = 256;
        const int64_t blocks = (warps * 32 + th - 1) / th;
        // koff is stored right after the stencils in d_K (see abi.cu)
        const double* koff = e.d_K + e.np * e.ss;
        if (e.dim == 2)
            k_bonds<2><<<(unsigned)blocks, th, 0, s>>>(u, f, e.d_bond_rows, e.n_bond_rows, e.d_ledger, e.lw, e.d_disp,
                                                      koff, e.nof, e.d_cmask, N, batch, scale);
        else
            k_bonds<3><<<(unsigned)blocks, th, 0, s>>>(u, f, e.d_bond_rows, e.n_bond_rows, e.d_ledger, e.lw, e.d_disp,
                                                      koff, e.nof, e.d_cmask, N, batch, scale);
    }
    check(cudaGetLastError(), "corrections launch");
}

// ---------------------------------------------------------------- K7 -----
struct BondArgs {
    int dim, Nx, Ny, Nz, nof, lw;
    double h, o0, o1, o2;
    double s0;
    int has_watch;
    double wlo[3], whi[3];
};

__device__ __forceinline__ double pos_rn(double origin, int c, double h) {
    return __dadd_rn(origin, __dmul_rn((double)c + 0.5, h));
}

__global__ void k_update_bonds(const double* __restrict__ u, uint32_t* ledger, const int* __restrict__ offs,
                               const long long* __restrict__ disp, const int* __restrict__ negk, BondArgs A,
                               int64_t nodes, long long* new_pairs, int64_t cap, unsigned long long* counters,
                               long long* bond_rows, int* listed) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nodes) return;
    int c[3];
    c[0] = (int)(p % A.Nx);
    const int64_t t = p / A.Nx;
    c[1] = (int)(t % A.Ny);
    c[2] = (int)(t / A.Ny);
    const double org[3] = {A.o0, A.o1, A.o2};
    double xp[3], up[3];
    for (int d = 0; d < A.dim; ++d) xp[d] = pos_rn(org[d], c[d], A.h);
    if (A.has_watch)
        for (int d = 0; d < A.dim; ++d)
            if (xp[d] < A.wlo[d] || xp[d] > A.whi[d]) return;
    for (int d = 0; d < A.dim; ++d) up[d] = u[(int64_t)d * nodes + p];
    const int dims[3] = {A.Nx, A.Ny, A.Nz};
    for (int k = 0; k < A.nof; ++k) {
        if (disp[k] <= 0) continue;  // q < p: visited from the other end (fracture.hpp:220)
        int cq[3];
        bool inside = true;
        for (int d = 0; d < A.dim; ++d) {
            cq[d] = c[d] + offs[3 * k + d];
            inside = inside && cq[d] >= 0 && cq[d] < dims[d];
        }
        if (!inside) continue;
        double xq[3];
        for (int d = 0; d < A.dim; ++d) xq[d] = pos_rn(org[d], cq[d], A.h);
        if (A.has_watch) {
            bool in = true;
            for (int d = 0; d < A.dim; ++d) in = in && !(xq[d] < A.wlo[d] || xq[d] > A.whi[d]);
            if (!in) continue;
        }
        if ((ledger[p * A.lw + (k >> 5)] >> (k & 31)) & 1u) continue;
        const int64_t q = p + disp[k];
        double len0 = 0.0, len1 = 0.0;
        for (int d = 0; d < A.dim; ++d) {
            const double r = __dsub_rn(xq[d], xp[d]);
            const double ev = __dsub_rn(__dadd_rn(r, u[(int64_t)d * nodes + q]), up[d]);
            len0 = __dadd_rn(len0, __dmul_rn(r, r));
            len1 = __dadd_rn(len1, __dmul_rn(ev, ev));
        }
        len0 = __dsqrt_rn(len0);
        len1 = __dsqrt_rn(len1);
        const double s = __ddiv_rn(__dsub_rn(len1, len0), len0);
        if (s >= A.s0) {
            atomicOr(&ledger[p * A.lw + (k >> 5)], 1u << (k & 31));
            const int kn = negk[k];
            atomicOr(&ledger[q * A.lw + (kn >> 5)], 1u << (kn & 31));
            const unsigned long long slot = atomicAdd(&counters[1], 1ull);
            if ((int64_t)slot < cap) {
                new_pairs[2 * slot] = p;
                new_pairs[2 * slot + 1] = k;
            }
            if (atomicExch(&listed[p], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = p;
            if (atomicExch(&listed[q], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = q;
        }
    }
}

// Returns the number of newly broken bonds; new pairs are left in
// e.d_new_pairs as (p, offset index) and bond rows are appended.
int64_t launch_update_bonds(Engine& e, const double* u, double s0, const double* watch, cudaStream_t s) {
    const Plan& pl = e.plan;
    BondArgs A;
    A.dim = e.dim;
    A.Nx = pl.N[0];
    A.Ny = pl.N[1];
    A.Nz = pl.N[2];
    A.nof = e.nof;
    A.lw = e.lw;
    A.h = e.h;
    A.o0 = e.origin[0];
    A.o1 = e.origin[1];
    A.o2 = e.origin[2];
    A.s0 = s0;
    A.has_watch = watch != nullptr;
    for (int d = 0; d < 3; ++d) {
        A.wlo[d] = watch && d < e.dim ? watch[d] : 0.0;
        A.whi[d] = watch && d < e.dim ? watch[e.dim + d] : 0.0;
    }
    // reset the new-pair counter, keep the row counter
    check(cudaMemsetAsync(e.d_counters + 1, 0, sizeof(unsigned long long), s), "reset counter");
    const int th = 128;
    const int64_t N = pl.nodes;
    const int* negk = (const int*)(e.d_offs + 3 * e.nof);
    e.launches += 1;
    k_update_bonds<<<(unsigned)((N + th - 1) / th), th, 0, s>>>(u, e.d_ledger, e.d_offs, e.d_disp, negk, A, N,
                                                               e.d_new_pairs, e.new_pairs_cap, e.d_counters,
                                                               e.d_bond_rows, e.d_listed);
    check(cudaGetLastError(), "update_bonds launch");
    unsigned long long cnt[2];
    check(cudaMemcpyAsync(cnt, e.d_counters, sizeof(cnt), cudaMemcpyDeviceToHost, s), "read counters");
    check(cudaStreamSynchronize(s), "update_bonds");
    e.n_bond_rows = (int64_t)cnt[0];
    e.total_broken += (int64_t)cnt[1];
    return (int64_t)cnt[1];
}

}  // namespace pdgpu
