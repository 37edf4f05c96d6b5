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
#include <stdlib.h>

#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

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
                        int64_t nrows, const unsigned long long* __restrict__ nrows_dev,
                        const uint32_t* __restrict__ ledger, int lw, const long long* __restrict__ disp,
                        const double* __restrict__ koff, int nof, const uint8_t* __restrict__ cmask, int64_t nodes,
                        int batch, double scale, const double* __restrict__ ghost, int64_t gs_bc, int64_t gs_side,
                        int64_t plane, int R, int M) {
    constexpr int NP = D * (D + 1) / 2;
    // row count from the device when bonds broke since the host last looked
    // (sim_step does not synchronise per step); grid-stride over warps
    const int64_t nr = nrows_dev ? (int64_t)*nrows_dev : nrows;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; warp < nr * batch; warp += nwarps) {
        const int b = (int)(warp / nr);
        const int64_t r = warp - (int64_t)b * nr;
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
                if (ghost && (q < 0 || q >= nodes)) {
                    // partner beyond an interior slab face: the neighbour's halo rows
                    const int64_t qrow = q >= 0 ? q / plane : -((-q + plane - 1) / plane);
                    const int64_t qin = q - qrow * plane;
                    const int side = qrow < 0 ? 0 : 1;
                    const int64_t layer = side ? qrow - R : qrow + M;
#pragma unroll
                    for (int c = 0; c < D; ++c)
                        du[c] = up[c] - ghost[(int64_t)(b * D + c) * gs_bc + side * gs_side + layer * plane + qin];
                } else {
#pragma unroll
                    for (int c = 0; c < D; ++c) du[c] = up[c] - ub[(int64_t)c * nodes + q];
                }
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    double sacc = 0.0;
#pragma unroll
                    for (int c = 0; c < D; ++c) sacc += koff[k * NP + pair_idx<D>(a, c)] * du[c];
                    acc[a] += sacc;
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
}

static void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// K6w wrap correction of the periodic embedding (engine.h, Plan).  Along a
// periodic axis the FFT product evaluates sum_o K(o) u[(p+o) mod P]; the
// reference's padded transform (convolution.hpp:58-71,183-195) sees zeros
// outside the lattice.  The two differ exactly by the aliased terms: offsets
// o with p+o outside the lattice along some axis, every such axis periodic
// (P = N, so the wrapped coordinate lands back inside).  Only nodes within M
// layers of a periodic face have any; thread per such node, enumerated face
// by face (a node in the bands of several periodic axes is handled by the
// first), the full (2M+1)^d box of every stencil component (the same
// entries the symbol is built from, so arbitrary stencils stay exact).
// f_a[p] -= scale * sum_o sum_b K_ab(o) u_b[wrap(p+o)] on rows not
// constrained in a (K5 has zeroed those).
// 3D: the x-face strips u[b][c][z][y][x in [0,2M) u [N0-2M,N0)] copied to
// strip[b][c][slot][z][y] (slot = x for the low side, 2M + x - (N0-2M) for the
// high side), so the x-band's aliased reads -- a warp spans consecutive y --
// are unit-stride instead of one cache line per lane.
__global__ void k_xstrip(const double* __restrict__ u, double* __restrict__ strip, int N0, int N1, int N2, int M,
                         int64_t nrows) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // ((b*3 + c)*N2 + z)*N1 + y
    if (i >= nrows) return;
    const int64_t plane = (int64_t)N1 * N2;
    const int64_t bc = i / plane, zy = i - bc * plane;
    const double* row = u + i * N0;
    double* dst = strip + bc * 4 * M * plane + zy;
    for (int x = 0; x < 2 * M; ++x) {
        dst[(int64_t)x * plane] = row[x];
        dst[(int64_t)(2 * M + x) * plane] = row[N0 - 2 * M + x];
    }
}

template <int D>
__global__ void __launch_bounds__(128) k_wrap(const double* __restrict__ u, double* __restrict__ f,
                                              const int* __restrict__ wrows, const int* __restrict__ wo0,
                                              const double* __restrict__ wK, int M, int N0, int N1, int N2,
                                              int circ_mask, const uint8_t* __restrict__ cmask, int64_t nodes,
                                              int batch, double scale, int64_t band0, int64_t band1, int64_t band2,
                                              const double* __restrict__ ghost, int64_t gs_bc, int64_t gs_side,
                                              int lo_int, int hi_int, const int* __restrict__ lidx, const int* __restrict__ loff,
                                              const double* __restrict__ lK, const double* __restrict__ xstrip) {
    constexpr int NP = D * (D + 1) / 2;
    const int64_t per_vec = band0 + band1 + band2;
    const int64_t gidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gidx >= per_vec * batch) return;
    const int b = (int)(gidx / per_vec);
    int64_t r = gidx - (int64_t)b * per_vec;
    int ax = 0;
    if (r >= band0) {
        r -= band0;
        ax = 1;
        if (r >= band1) {
            r -= band1;
            ax = 2;
        }
    }
    // mixed radix over the two other axes (lower axis fastest), the band
    // layer (2M values) slowest: a warp shares one depth, so one trip count.
    // Scalars, not arrays: a runtime-indexed array would live in local memory.
    auto layer = [&](int64_t l, int n) { return (int)l < M ? (int)l : n - 2 * M + (int)l; };
    int c0, c1, c2;
    if (ax == 0) {
        c1 = (int)(r % N1);
        r /= N1;
        c2 = (int)(r % N2);
        r /= N2;
        c0 = layer(r, N0);
    } else if (ax == 1) {
        c0 = (int)(r % N0);
        r /= N0;
        c2 = (int)(r % N2);
        r /= N2;
        c1 = layer(r, N1);
    } else {
        c0 = (int)(r % N0);
        r /= N0;
        c1 = (int)(r % N1);
        r /= N1;
        c2 = layer(r, N2);
    }
    // already covered by an earlier periodic axis
    if (ax >= 1 && (circ_mask & 1) && (c0 < M || c0 >= N0 - M)) return;
    if (ax >= 2 && ((circ_mask >> 1) & 1) && (c1 < M || c1 >= N1 - M)) return;
    const int64_t p = ((int64_t)c2 * N1 + c1) * N0 + c0;
    const uint8_t cm = cmask ? cmask[p] : 0;
    const double* ub = u + (int64_t)b * D * nodes;
    constexpr int KS = (NP + 1) & ~1;  // entry stride: 16-byte aligned pairs
    double acc[D], gacc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[a] = gacc[a] = 0.0;
    const int64_t plane = D == 3 ? (int64_t)N0 * N1 : N0;
    // fast path: the node is M or more away from every face of the other axes,
    // so the aliased entries are exactly the precomputed list of its layer
    // (uniform across the warp: one depth per warp, no row bookkeeping)
    {
        const bool in0 = ax == 0 || (c0 >= M && c0 < N0 - M);
        const bool in1 = ax == 1 || (c1 >= M && c1 < N1 - M);
        const bool in2 = D == 2 || ax == 2 || (c2 >= M && c2 < N2 - M);
        if (in0 && in1 && in2) {
            const int cax = ax == 0 ? c0 : (ax == 1 ? c1 : c2);
            const int nax = ax == 0 ? N0 : (ax == 1 ? N1 : N2);
            const int sd = cax < M ? 0 : 1;
            const int l = sd ? nax - 1 - cax : cax;
            const bool per = (circ_mask >> ax) & 1;
            const bool gface = ghost && ax == D - 1 && (sd ? hi_int : lo_int);
            const int li = (ax * 2 + sd) * M + l;
            const int e0 = __ldg(lidx + li), e1 = __ldg(lidx + li + 1);
            const int wrapd = sd ? -nax : nax;
#pragma unroll 2
            for (int e = e0; e < e1; ++e) {
                const int4 o = __ldg(reinterpret_cast<const int4*>(loff) + e);
                const int q0 = c0 + o.x, q1 = c1 + o.y, q2 = c2 + o.z;
                double kv[KS];
                const double2* ke = reinterpret_cast<const double2*>(lK + (int64_t)e * KS);
#pragma unroll
                for (int k = 0; k < KS / 2; ++k) {
                    const double2 v2 = __ldg(ke + k);
                    kv[2 * k] = v2.x;
                    kv[2 * k + 1] = v2.y;
                }
                if (per) {
                    double uq[D];
                    if (D == 3 && ax == 0 && xstrip) {
                        // x-face strip: slot of the wrapped x, [b][c][slot][z][y]
                        const int slot = sd ? q0 - N0 : q0 + 4 * M;  // x = q0 - N0 (low strip) or q0 + N0 (high)
                        const int64_t pl = (int64_t)N1 * N2;
                        const double* sp = xstrip + (int64_t)b * D * 4 * M * pl + (int64_t)slot * pl +
                                           (int64_t)q2 * N1 + q1;
#pragma unroll
                        for (int bb = 0; bb < D; ++bb) uq[bb] = sp[(int64_t)bb * 4 * M * pl];
                    } else {
                        const int64_t q = ((int64_t)(q2 + (ax == 2 ? wrapd : 0)) * N1 + q1 + (ax == 1 ? wrapd : 0)) * N0 +
                                          q0 + (ax == 0 ? wrapd : 0);
#pragma unroll
                        for (int bb = 0; bb < D; ++bb) uq[bb] = ub[(int64_t)bb * nodes + q];
                    }
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int bb = 0; bb < D; ++bb) acc[a] += kv[pair_idx<D>(a, bb)] * uq[bb];
                }
                if (gface) {
                    const int qs = D == 3 ? q2 : q1;
                    const int layer = sd ? qs - nax : qs + M;
                    const int64_t pidx = D == 3 ? (int64_t)q1 * N0 + q0 : q0;
#pragma unroll
                    for (int bb = 0; bb < D; ++bb) {
                        const double g = ghost[(int64_t)(b * D + bb) * gs_bc + sd * gs_side + (int64_t)layer * plane + pidx];
#pragma unroll
                        for (int a = 0; a < D; ++a) gacc[a] += kv[pair_idx<D>(a, bb)] * g;
                    }
                }
            }
#pragma unroll
            for (int a = 0; a < D; ++a) {
                if ((cm >> a) & 1u) continue;
                f[((int64_t)b * D + a) * nodes + p] += scale * (gacc[a] - acc[a]);
            }
            return;
        }
    }
    // in-lattice o0 range of this node; entries outside it along x alias when x is periodic
    const int lo0 = -c0, hi0 = N0 - 1 - c0;
    const bool cx = circ_mask & 1;
    auto load_k = [&](int e, double (&kv)[KS]) {
        const double2* ke = reinterpret_cast<const double2*>(wK + (int64_t)e * KS);
#pragma unroll
        for (int k = 0; k < KS / 2; ++k) {
            const double2 v2 = __ldg(ke + k);
            kv[2 * k] = v2.x;
            kv[2 * k + 1] = v2.y;
        }
    };
    auto add = [&](int e, int64_t q) {
        double uq[D];
#pragma unroll
        for (int bb = 0; bb < D; ++bb) uq[bb] = ub[(int64_t)bb * nodes + q];
        double kv[KS];
        load_k(e, kv);
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int bb = 0; bb < D; ++bb) acc[a] += kv[pair_idx<D>(a, bb)] * uq[bb];
    };
    // halo slabs: rows beyond an interior face of the slowest axis come from
    // the neighbour's ghost rows, ghost[(b*D + c)*gs_bc + side*gs_side + layer*plane]
    auto add_ghost = [&](int e, int side, int layer, int64_t pidx) {
        double kv[KS];
        load_k(e, kv);
#pragma unroll
        for (int bb = 0; bb < D; ++bb) {
            const double g = ghost[(int64_t)(b * D + bb) * gs_bc + side * gs_side + (int64_t)layer * plane + pidx];
#pragma unroll
            for (int a = 0; a < D; ++a) gacc[a] += kv[pair_idx<D>(a, bb)] * g;
        }
    };
    const int m2 = D == 3 ? M : 0;
    const int side = 2 * M + 1;
    for (int o2 = -m2; o2 <= m2; ++o2) {
        int w2 = c2 + o2;
        bool out2 = false, al2 = true, gh2 = false;
        int gside = 0, glayer = 0;
        if (D == 3 && (w2 < 0 || w2 >= N2)) {
            out2 = true;
            if (ghost && (w2 < 0 ? lo_int : hi_int)) {  // z is the slowest axis in 3D
                gh2 = true;
                gside = w2 < 0 ? 0 : 1;
                glayer = w2 < 0 ? w2 + M : w2 - N2;
            }
            if ((circ_mask >> 2) & 1) w2 = w2 < 0 ? w2 + N2 : w2 - N2;
            else al2 = false;
            if (!al2 && !gh2) continue;
        }
        for (int o1 = -M; o1 <= M; ++o1) {
            int w1 = c1 + o1;
            bool out1 = out2, al1 = al2, gh1 = gh2;
            int gs = gside, gl = glayer;
            if (w1 < 0 || w1 >= N1) {
                out1 = true;
                if (D == 2) {  // y is the slowest axis in 2D
                    gh1 = ghost && (w1 < 0 ? lo_int : hi_int);
                    gs = w1 < 0 ? 0 : 1;
                    gl = w1 < 0 ? w1 + M : w1 - N1;
                } else {
                    gh1 = false;  // the neighbour slab has no nodes outside the y range either
                }
                if ((circ_mask >> 1) & 1) w1 = w1 < 0 ? w1 + N1 : w1 - N1;
                else al1 = false;
            }
            if (!al1 && !gh1) continue;
            const int row = (o2 + m2) * side + (o1 + M);
            const int e0 = __ldg(wrows + 2 * row), e1 = __ldg(wrows + 2 * row + 1);
            const int64_t qrow = ((int64_t)w2 * N1 + w1) * N0;
            if (al1) {
                if (out1) {  // every entry of the row aliases (x in range) or is dropped (x out, padded)
                    for (int e = e0; e < e1; ++e) {
                        int w0 = c0 + __ldg(wo0 + e);
                        if (w0 < 0 || w0 >= N0) {
                            if (!cx) continue;
                            w0 = w0 < 0 ? w0 + N0 : w0 - N0;
                        }
                        add(e, qrow + w0);
                    }
                } else if (cx) {  // only the entries leaving along x
                    for (int e = e0; e < e1; ++e) {
                        const int o0 = __ldg(wo0 + e);
                        if (o0 >= lo0) break;
                        add(e, qrow + c0 + o0 + N0);
                    }
                    for (int e = e1 - 1; e >= e0; --e) {
                        const int o0 = __ldg(wo0 + e);
                        if (o0 <= hi0) break;
                        add(e, qrow + c0 + o0 - N0);
                    }
                }
            }
            if (gh1) {  // true neighbour values, x inside the lattice only
                const int64_t prow = D == 3 ? (int64_t)(c1 + o1) * N0 : 0;
                for (int e = e0; e < e1; ++e) {
                    const int x = c0 + __ldg(wo0 + e);
                    if (x < 0 || x >= N0) continue;
                    add_ghost(e, gs, gl, prow + x);
                }
            }
        }
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
        if ((cm >> a) & 1u) continue;
        f[((int64_t)b * D + a) * nodes + p] += scale * (gacc[a] - acc[a]);
    }
}

// K6w with per-state entry lists (the general form of k_wrap's fast path):
// every band node, including edges and corners, loops over one precomputed
// list of the entries that leave the lattice from its position class, with
// the wrapped displacement stored -- no per-row bookkeeping, independent loads
// (unrolled), and the ghost-row terms of halo slabs in the same pass.
template <int D, int LPN, bool FOLD = false>
__global__ void __launch_bounds__(128) k_wrap_tab(const double* __restrict__ u, double* __restrict__ f,
                                                  const int* __restrict__ sidx, const int4* __restrict__ stab,
                                                  const double* __restrict__ wK, int M, int N0, int N1, int N2,
                                                  int circ_mask, const uint8_t* __restrict__ cmask, int64_t nodes,
                                                  int batch, double scale, int64_t band0, int64_t band1,
                                                  int64_t band2, const double* __restrict__ ghost, int64_t gs_bc,
                                                  int64_t gs_side, int lo_int, int hi_int,
                                                  const double* __restrict__ xstrip,
                                                  const uint8_t* __restrict__ smask, double gsign, int glob) {
    pdl_entry();
    constexpr int NP = D * (D + 1) / 2;
    constexpr int KS = (NP + 1) & ~1;
    // FOLD (every axis periodic, the lattice's own D^e, corrections follow):
    // the node's aliased entries are exactly the offsets that leave the
    // lattice, whose kernel sum is D^e (corrections.hpp:24-42), so this pass
    // also adds D^e u_p under the surface mask and k_surface is skipped
    // LPN lanes per node (a quad of consecutive lanes), entries strided over them
    const int64_t per_vec = band0 + band1 + band2;
    const int64_t gidx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPN;
    const int sub = threadIdx.x % LPN;
    if (gidx >= per_vec * batch) return;
    const int b = (int)(gidx / per_vec);
    int64_t r = gidx - (int64_t)b * per_vec;
    int ax = 0;
    if (r >= band0) {
        r -= band0;
        ax = 1;
        if (r >= band1) {
            r -= band1;
            ax = 2;
        }
    }
    auto layer = [&](int64_t l, int n) { return (int)l < M ? (int)l : n - 2 * M + (int)l; };
    int c0, c1, c2;
    if (ax == 0) {
        c1 = (int)(r % N1);
        r /= N1;
        c2 = (int)(r % N2);
        r /= N2;
        c0 = layer(r, N0);
    } else if (ax == 1) {
        c0 = (int)(r % N0);
        r /= N0;
        c2 = (int)(r % N2);
        r /= N2;
        c1 = layer(r, N1);
    } else {
        c0 = (int)(r % N0);
        r /= N0;
        c1 = (int)(r % N1);
        r /= N1;
        c2 = layer(r, N2);
    }
    if (ax >= 1 && (circ_mask & 1) && (c0 < M || c0 >= N0 - M)) return;
    if (ax >= 2 && ((circ_mask >> 1) & 1) && (c1 < M || c1 >= N1 - M)) return;
    auto st = [&](int c, int n) { return c < M ? 1 + c : (c >= n - M ? M + n - c : 0); };
    const int S = 2 * M + 1;
    const int state = st(c0, N0) + S * (st(c1, N1) + (D == 3 ? S * st(c2, N2) : 0));
    const int64_t p = ((int64_t)c2 * N1 + c1) * N0 + c0;
    const uint8_t cm = cmask ? cmask[p] : 0;
    const double* ub = u + (int64_t)b * D * nodes + p;
    // 3D x band: every read has x within 2M of the node's x face, i.e. in the
    // compact strip [b][c][slot][z][y] (a warp spans y: unit stride)
    const bool strip = D == 3 && ax == 0 && xstrip;
    const int64_t spl = (int64_t)N1 * N2;
    const double* sb = strip ? xstrip + (int64_t)b * D * 4 * M * spl : nullptr;
    const int64_t plane = D == 3 ? (int64_t)N0 * N1 : N0;
    const int64_t pin = D == 3 ? (int64_t)c1 * N0 + c0 : c0;  // in-plane index of p
    double acc[D], gacc[D], ds[NP];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[a] = gacc[a] = 0.0;
#pragma unroll
    for (int k = 0; k < NP; ++k) ds[k] = 0.0;
    const int e0 = __ldg(sidx + state), e1 = __ldg(sidx + state + 1);
#pragma unroll 4
    for (int e = e0 + sub; e < e1; e += LPN) {
        const int4 rec = __ldg(stab + e);
        const int w0 = (int)(short)(rec.x & 0xffff), w1 = rec.x >> 16, w2 = rec.y;  // wrapped displacement
        const int fl = rec.w;
        double kv[KS];
        const double2* ke = reinterpret_cast<const double2*>(wK + (int64_t)rec.z * KS);
#pragma unroll
        for (int k = 0; k < KS / 2; ++k) {
            const double2 v2 = __ldg(ke + k);
            kv[2 * k] = v2.x;
            kv[2 * k + 1] = v2.y;
        }
        if (fl & 1) {
            double uq[D];
            if (strip) {
                const int q0 = c0 + w0;
                const int slot = q0 < 2 * M ? q0 : q0 - N0 + 4 * M;
                const double* sp = sb + (int64_t)slot * spl + (int64_t)(c2 + w2) * N1 + (c1 + w1);
#pragma unroll
                for (int bb = 0; bb < D; ++bb) uq[bb] = sp[(int64_t)bb * 4 * M * spl];
            } else {
                const int64_t lin = (int64_t)w0 + (int64_t)N0 * (w1 + (int64_t)N1 * w2);
#pragma unroll
                for (int bb = 0; bb < D; ++bb) uq[bb] = ub[(int64_t)bb * nodes + lin];
            }
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
                for (int bb = 0; bb < D; ++bb) acc[a] += kv[pair_idx<D>(a, bb)] * uq[bb];
            if (FOLD) {
#pragma unroll
                for (int k = 0; k < NP; ++k) ds[k] += kv[k];
            }
        }
        if ((fl & 2) && ghost) {
            const int sd = (fl >> 2) & 1;
            // distributed FFT (gsign < 0): across a global face every such entry
            // is aliased; across an interior face only those that also leave
            // along x (the FFT wrapped them circularly there)
            const bool use = gsign > 0.0 || ((glob >> sd) & 1) || (fl & 128);
            if ((sd ? hi_int : lo_int) && use) {
                const int gl = (fl >> 3) & 15;
                const int64_t pidx = pin + (fl >> 8);
#pragma unroll
                for (int bb = 0; bb < D; ++bb) {
                    const double g = ghost[(int64_t)(b * D + bb) * gs_bc + sd * gs_side + (int64_t)gl * plane + pidx];
#pragma unroll
                    for (int a = 0; a < D; ++a) gacc[a] += kv[pair_idx<D>(a, bb)] * g;
                }
            }
        }
    }
    if (LPN > 1) {  // the node's lanes: consecutive, all alive (the early returns are per node)
        const unsigned qm = ((1u << LPN) - 1u) << ((threadIdx.x & 31) & ~(LPN - 1));
#pragma unroll
        for (int o = 1; o < LPN; o <<= 1) {
#pragma unroll
            for (int a = 0; a < D; ++a) {
                acc[a] += __shfl_xor_sync(qm, acc[a], o);
                gacc[a] += __shfl_xor_sync(qm, gacc[a], o);
            }
            if (FOLD) {
#pragma unroll
                for (int k = 0; k < NP; ++k) ds[k] += __shfl_xor_sync(qm, ds[k], o);
            }
        }
        if (sub) return;
    }
    const uint8_t smk = FOLD && smask ? smask[p] : 0;
    double up[D];
    if (FOLD) {
#pragma unroll
        for (int c = 0; c < D; ++c) up[c] = ub[(int64_t)c * nodes];
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
        // gsign: +1 halo slabs (true neighbour rows), -1 distributed FFT (aliases
        // of the opposite global end, subtracted like the local ones)
        double dv = ((cm >> a) & 1u) ? 0.0 : gsign * gacc[a] - acc[a];
        if (FOLD && !((smk >> a) & 1u)) {
            double sa = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) sa += ds[pair_idx<D>(a, c)] * up[c];
            dv += sa;
        }
        f[((int64_t)b * D + a) * nodes + p] += scale * dv;
    }
}

// ---- 3D wrap correction as three tiled face passes (every axis periodic,
// no ghost rows).  Each aliased (node, entry) term is taken by exactly one
// pass: the x pass takes entries leaving along x, the y pass those leaving
// along y but not x, the z pass those leaving along z only.  A CTA covers a
// 32 x 8 tile of the face's node columns (tile axes B fast, C slow) on one
// side, for the M depths; the M layers of u beyond the opposite face (with an
// M halo in B and C, wrapped where that axis may wrap in this pass) are staged
// in SMEM once, so the ~70 entries per column read SMEM instead of L2.  The x
// pass stages from the x-face strip copy (unit stride along y).  Passes run
// back to back, each node's row updated by one thread per pass.
constexpr int kFaceTB = 32, kFaceTC = 8;

template <int A, bool FOLD>
__global__ void __launch_bounds__(kFaceTB * kFaceTC) k_wrap_face(
    const double* __restrict__ u, double* __restrict__ f, const int* __restrict__ fidx,
    const int4* __restrict__ ftab, const double* __restrict__ wK, int M, int N0, int N1, int N2,
    const uint8_t* __restrict__ cmask, const uint8_t* __restrict__ smask, int64_t nodes, double scale,
    int nrec_max, const double* __restrict__ xstrip, double* __restrict__ fx,
    const double* __restrict__ ghost = nullptr, int64_t gs_bc = 0, int64_t gs_side = 0, int lo_int = 0,
    int hi_int = 0) {
    constexpr int D = 3, KS = 6;
    extern __shared__ double tile[];  // [layer][comp][c'][b'] (b' fastest), then the records and their K
    const int NA = A == 0 ? N0 : (A == 1 ? N1 : N2);
    const int NB = A == 0 ? N1 : N0;
    const int NC = A == 2 ? N1 : N2;
    const int side = blockIdx.z & 1, b = blockIdx.z >> 1;
    const int b0 = blockIdx.x * kFaceTB, c0 = blockIdx.y * kFaceTC;
    const int WB = kFaceTB + 2 * M, WC = kFaceTC + 2 * M;
    const int layer_sz = WB * WC;
    const int tot = M * D * layer_sz;
    // this pass's entry records (the M depths of one side) and their stencil
    // values, staged once: every thread of the CTA walks the same list
    const int r0 = __ldg(fidx + (A * 2 + side) * M), r1 = __ldg(fidx + (A * 2 + side) * M + M);
    int4* srec = reinterpret_cast<int4*>(tile + tot);
    double* sK = reinterpret_cast<double*>(srec + nrec_max);
    for (int e = threadIdx.x; e < r1 - r0; e += blockDim.x) {
        const int4 r = __ldg(ftab + r0 + e);
        srec[e] = r;
#pragma unroll
        for (int k = 0; k < KS; ++k) sK[e * KS + k] = __ldg(wK + (int64_t)r.w * KS + k);
    }
    // the M layers beyond the opposite face, eight loads of a thread in flight
    // before its SMEM stores; the x pass walks the layers fastest (24
    // contiguous bytes of a row end), the others the B axis (x)
    const double* ub = u + (int64_t)b * D * nodes;
    const int64_t spl = (int64_t)N1 * N2;
    auto coords = [&](int idx, int& i, int& comp, int& cc, int& bb) {
        if (A == 0 && !xstrip) {
            i = idx % M;
            const int rest = idx / M;
            bb = rest % WB;
            const int rest2 = rest / WB;
            cc = rest2 % WC;
            comp = rest2 / WC;
        } else {
            bb = idx % WB;
            const int rest = idx / WB;
            cc = rest % WC;
            const int rest2 = rest / WC;
            comp = rest2 % D;
            i = rest2 / D;
        }
    };
    auto fetch = [&](int i, int comp, int cc, int bb) -> double {
        int gb = b0 + bb - M, gc = c0 + cc - M;
        const int ga = side == 0 ? NA - M + i : i;
        // B wraps in the x pass only (y pass: x stays in range; z pass: x and y do)
        if (gb < 0 || gb >= NB) {
            if (A != 0) return 0.0;
            gb = gb < 0 ? gb + NB : gb - NB;
        }
        // C wraps in the x and y passes
        if (gc < 0 || gc >= NC) {
            if (A == 2) return 0.0;
            gc = gc < 0 ? gc + NC : gc - NC;
        }
        if (A == 0 && xstrip) {  // the strip K1 wrote: [b][c][slot][z][y], unit stride along y
            const int slot = ga < 2 * M ? ga : ga - N0 + 4 * M;
            return xstrip[((int64_t)(b * D + comp) * 4 * M + slot) * spl + (int64_t)gc * N1 + gb];
        }
        if (A == 0) return ub[(int64_t)comp * nodes + ((int64_t)gc * N1 + gb) * N0 + ga];
        if (A == 1) return ub[(int64_t)comp * nodes + ((int64_t)gc * N1 + ga) * N0 + gb];
        // z pass of a halo slab: across an interior face the entry's true
        // neighbour is ghost plane i of that side (k_wrap_tab's layer order), so
        // the staged value is alias - ghost and the pass subtracts both at once
        double v = ub[(int64_t)comp * nodes + ((int64_t)ga * N1 + gc) * N0 + gb];
        if (ghost && (side == 0 ? lo_int : hi_int))
            v -= ghost[(int64_t)(b * D + comp) * gs_bc + side * gs_side + (int64_t)i * N0 * N1 + (int64_t)gc * N0 + gb];
        return v;
    };
    for (int i0 = threadIdx.x; i0 < tot; i0 += 8 * (int)blockDim.x) {
        double v[8];
        int dst[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int idx = i0 + k * (int)blockDim.x;
            int i = 0, comp = 0, cc = 0, bb = 0;
            if (idx < tot) coords(idx, i, comp, cc, bb);
            dst[k] = idx < tot ? ((i * D + comp) * WC + cc) * WB + bb : -1;
            v[k] = idx < tot ? fetch(i, comp, cc, bb) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (dst[k] >= 0) tile[dst[k]] = v[k];
    }
    __syncthreads();
    const int tb = threadIdx.x % kFaceTB, tc = threadIdx.x / kFaceTB;
    const int gb = b0 + tb, gc = c0 + tc;
    if (gb >= NB || gc >= NC) return;
    for (int l = 0; l < M; ++l) {
        const int ga = side == 0 ? l : NA - 1 - l;
        const int x = A == 0 ? ga : gb, y = A == 0 ? gb : (A == 1 ? ga : gc), z = A == 2 ? ga : gc;
        const int64_t p = ((int64_t)z * N1 + y) * N0 + x;
        const int e0 = __ldg(fidx + (A * 2 + side) * M + l) - r0, e1 = __ldg(fidx + (A * 2 + side) * M + l + 1) - r0;
        // FOLD: the surface diagonal D^e (corrections.hpp:24-42) is the sum of
        // exactly these entries (each taken by one pass), so the passes add
        // (sum K) u_p in place of k_surface, under the engine's constraint mask
        double acc[D] = {0.0, 0.0, 0.0};
        double ds[KS] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 2
        for (int e = e0; e < e1; ++e) {
            const int4 r = srec[e];  // {oB, oC, oA, box}
            if (A != 0 && (gb + r.x < 0 || gb + r.x >= NB)) continue;  // leaves along x: the x pass's
            if (A == 2 && (gc + r.y < 0 || gc + r.y >= NC)) continue;  // leaves along y: the y pass's
            const int i = side == 0 ? l + r.z + M : r.z - l - 1;
            const double* tp = tile + ((i * D) * WC + (tc + r.y + M)) * WB + (tb + r.x + M);
            const double2* k2 = reinterpret_cast<const double2*>(sK + e * KS);
            const double2 ka = k2[0], kb = k2[1], kc = k2[2];
            const double kv[KS] = {ka.x, ka.y, kb.x, kb.y, kc.x, kc.y};
            const double uq[3] = {tp[0], tp[layer_sz], tp[2 * layer_sz]};
            if (FOLD) {
#pragma unroll
                for (int k = 0; k < KS; ++k) ds[k] += kv[k];
            }
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
                for (int bb = 0; bb < D; ++bb) acc[a] += kv[pair_idx<D>(a, bb)] * uq[bb];
        }
        const uint8_t cm = cmask ? cmask[p] : 0;
        const uint8_t sm_ = FOLD && smask ? smask[p] : 0;
        double up[D] = {0.0, 0.0, 0.0};
        if (FOLD) {
            if (A == 0 && xstrip) {  // the node's own values are in the strip too (slot l / 4M-1-l)
                const int slot = side == 0 ? l : 4 * M - 1 - l;
#pragma unroll
                for (int c = 0; c < D; ++c)
                    up[c] = xstrip[((int64_t)(b * D + c) * 4 * M + slot) * spl + (int64_t)gc * N1 + gb];
            } else {
#pragma unroll
                for (int c = 0; c < D; ++c) up[c] = ub[(int64_t)c * nodes + p];
            }
        }
#pragma unroll
        for (int a = 0; a < D; ++a) {
            double dv = 0.0;
            if ((cm >> a) & 1u) dv = 0.0;
            else dv = -acc[a];
            if (FOLD && !((sm_ >> a) & 1u)) {
                double sa = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) sa += ds[pair_idx<D>(a, c)] * up[c];
                dv += sa;
            }
            if (A == 0 && fx)  // K5 adds it when it writes the row end: [b][a][z][y][slot 2M]
                fx[(((int64_t)(b * D + a) * N2 + gc) * N1 + gb) * 2 * M + (side == 0 ? l : 2 * M - 1 - l)] = scale * dv;
            else
                f[((int64_t)b * D + a) * nodes + p] += scale * dv;
        }
    }
}

static void build_face_table(Engine& e, const std::vector<int>& rows, const std::vector<int>& o0s) {
    const Plan& pl = e.plan;
    const int M = e.M, S = 2 * M + 1;
    if (e.dim != 3) return;
    // measured: 256^3 wrap + D^e 0.237 -> 0.161 ms; at 128^3 the per-state
    // kernel is as fast (0.081 vs 0.083 ms), so the passes start at 192
    // (a halo slab's own axis may be short: its z pass covers the full ghost faces)
    for (int a = 0; a < 3; ++a)
        if (!pl.circ[a] || pl.N[a] < (a == 2 && e.slab.global >= 0 ? std::max(S, 2 * M) : std::max(S, 192))) return;
    std::vector<int> fidx;
    std::vector<int4> ftab;
    for (int A = 0; A < 3; ++A)
        for (int side = 0; side < 2; ++side)
            for (int l = 0; l < M; ++l) {
                fidx.push_back((int)ftab.size());
                for (int row = 0; row < S * S; ++row)
                    for (int ei = rows[2 * row]; ei < rows[2 * row + 1]; ++ei) {
                        const int o[3] = {o0s[(size_t)ei], row % S - M, row / S - M};
                        if (!(side == 0 ? o[A] < -l : o[A] > l)) continue;
                        const int oB = A == 0 ? o[1] : o[0];
                        const int oC = A == 2 ? o[1] : o[2];
                        ftab.push_back(make_int4(oB, oC, o[A], ei));
                    }
            }
    fidx.push_back((int)ftab.size());
    e.face_rec_max = 0;
    for (int k = 0; k < 6; ++k) e.face_rec_max = std::max(e.face_rec_max, fidx[(size_t)(k + 1) * M] - fidx[(size_t)k * M]);
    check(cudaMalloc((void**)&e.d_fidx, sizeof(int) * fidx.size()), "alloc face index");
    check(cudaMemcpy(e.d_fidx, fidx.data(), sizeof(int) * fidx.size(), cudaMemcpyHostToDevice), "copy face index");
    check(cudaMalloc((void**)&e.d_ftab, sizeof(int4) * ftab.size()), "alloc face table");
    check(cudaMemcpy(e.d_ftab, ftab.data(), sizeof(int4) * ftab.size(), cudaMemcpyHostToDevice), "copy face table");
    for (const void* fn : {(const void*)k_wrap_face<0, false>, (const void*)k_wrap_face<1, false>,
                           (const void*)k_wrap_face<2, false>, (const void*)k_wrap_face<0, true>,
                           (const void*)k_wrap_face<1, true>, (const void*)k_wrap_face<2, true>})
        check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "face smem");
}

// per-state lists for k_wrap_tab (engine.h d_sidx / d_stab); entry ids index
// the d_wK table built below (same storage order)
static void build_state_table(Engine& e, const std::vector<int>& rows, const std::vector<int>& o0s) {
    const Plan& pl = e.plan;
    // distributed FFT: along the slowest axis (global, periodic over Nyg) an
    // entry leaving the slab aliases only at the global faces, onto the
    // opposite end's rows -- every such entry becomes a ghost entry (with the
    // wrapped x offset when it also leaves along x), none a local alias
    const bool a2a = e.a2a.G > 0;
    const int dim = e.dim, M = e.M, S = 2 * M + 1;
    for (int a = 0; a < dim; ++a)
        if (pl.N[a] < S || (a < 2 && pl.N[a] > 32767)) return;  // k_wrap's general path
    const int SA = dim - 1;
    const int nrows = dim == 3 ? S * S : S;
    int nstates = 1;
    for (int a = 0; a < dim; ++a) nstates *= S;
    std::vector<int> sidx;
    std::vector<int4> tab;
    for (int state = 0; state < nstates; ++state) {
        sidx.push_back((int)tab.size());
        int sa[3] = {0, 0, 0};
        int rem = state;
        for (int a = 0; a < dim; ++a) {
            sa[a] = rem % S;
            rem /= S;
        }
        for (int row = 0; row < nrows; ++row)
            for (int ei = rows[2 * row]; ei < rows[2 * row + 1]; ++ei) {
                const int o[3] = {o0s[(size_t)ei], (dim == 3 ? row % S : row) - M, dim == 3 ? row / S - M : 0};
                bool out[3] = {false, false, false};
                int shift[3] = {0, 0, 0};
                bool any = false, alias = true;
                for (int a = 0; a < dim; ++a) {
                    const int s_ = sa[a];
                    if (s_ >= 1 && s_ <= M) out[a] = o[a] < -(s_ - 1);          // low face, depth s-1
                    else if (s_ > M) out[a] = o[a] > (s_ - M - 1);              // high face, depth s-M-1
                    if (!out[a]) continue;
                    any = true;
                    if (pl.circ[a] && !(a2a && a == SA)) shift[a] = s_ <= M ? pl.N[a] : -pl.N[a];
                    else alias = false;
                }
                if (!any) continue;
                // ghost rows: out along the slowest axis only (distributed FFT:
                // out along it at all, other axes wrapped where they alias)
                bool gh = out[SA];
                if (!a2a)
                    for (int a = 0; a < SA; ++a) gh = gh && !out[a];
                else
                    for (int a = 0; a < SA; ++a) gh = gh && (!out[a] || pl.circ[a]);
                if (!alias && !gh) continue;
                int fl = alias ? 1 : 0;
                if (gh) {
                    const int side = sa[SA] <= M ? 0 : 1;
                    const int depth = side == 0 ? sa[SA] - 1 : sa[SA] - M - 1;
                    const int c = side == 0 ? depth : pl.N[SA] - 1 - depth;  // coordinate of p along SA
                    const int w = c + o[SA];
                    const int gl = side == 0 ? w + M : w - pl.N[SA];
                    int ow[3] = {o[0], o[1], o[2]};
                    if (a2a)
                        for (int a = 0; a < SA; ++a)
                            if (out[a]) ow[a] += sa[a] <= M ? pl.N[a] : -pl.N[a];
                    const int goff = dim == 3 ? ow[0] + pl.N[0] * ow[1] : ow[0];
                    bool xo = false;  // also leaves along a faster axis (distributed FFT: aliased there too)
                    for (int a = 0; a < SA; ++a) xo = xo || out[a];
                    fl |= 2 | (side << 2) | (gl << 3) | (xo ? 128 : 0) | (goff << 8);
                }
                // wrapped displacement: x and y in 16 bits each, z in 32
                const int w0 = o[0] + shift[0], w1 = o[1] + shift[1], w2 = o[2] + shift[2];
                tab.push_back(make_int4((int)(((uint32_t)w0 & 0xffffu) | ((uint32_t)w1 << 16)), w2, ei, fl));
            }
    }
    sidx.push_back((int)tab.size());
    if (tab.empty()) tab.push_back(make_int4(0, 0, 0, 0));
    if (e.d_sidx) cudaFree(e.d_sidx);
    if (e.d_stab) cudaFree(e.d_stab);
    check(cudaMalloc((void**)&e.d_sidx, sizeof(int) * sidx.size()), "alloc state index");
    check(cudaMemcpy(e.d_sidx, sidx.data(), sizeof(int) * sidx.size(), cudaMemcpyHostToDevice), "copy state index");
    check(cudaMalloc((void**)&e.d_stab, sizeof(int4) * tab.size()), "alloc state table");
    check(cudaMemcpy(e.d_stab, tab.data(), sizeof(int4) * tab.size(), cudaMemcpyHostToDevice), "copy state table");
}

void build_wrap_table(Engine& e) {
    const int dim = e.dim, M = e.M, side = 2 * M + 1, np = e.np;
    const int nrows = dim == 3 ? side * side : side;
    std::vector<int> rows(2 * (size_t)nrows), o0s;
    std::vector<double> kv;
    for (int row = 0; row < nrows; ++row) {
        rows[2 * row] = (int)o0s.size();
        for (int i0 = 0; i0 < side; ++i0) {
            const int64_t si = (int64_t)row * side + i0;  // KernelStack storage: axis 0 fastest (kernel.hpp:50-54)
            bool any = false;
            for (int pp = 0; pp < np; ++pp) any = any || e.stencils[(size_t)(pp * e.ss + si)] != 0.0;
            if (!any) continue;
            o0s.push_back(i0 - M);
            for (int pp = 0; pp < np; ++pp) kv.push_back(e.stencils[(size_t)(pp * e.ss + si)]);
            if (np & 1) kv.push_back(0.0);  // entry stride (np + 1) & ~1 (k_wrap's double2 loads)
        }
        rows[2 * row + 1] = (int)o0s.size();
    }
    if (o0s.empty()) {
        o0s.push_back(0);
        for (int pp = 0; pp < ((np + 1) & ~1); ++pp) kv.push_back(0.0);
    }
    auto up = [](void** dst, const void* src, size_t bytes) {
        check(cudaMalloc(dst, bytes), "alloc wrap table");
        check(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), "copy wrap table");
    };
    up((void**)&e.d_wrows, rows.data(), sizeof(int) * rows.size());
    up((void**)&e.d_wo0, o0s.data(), sizeof(int) * o0s.size());
    up((void**)&e.d_wK, kv.data(), sizeof(double) * kv.size());
    // layer lists (k_wrap fast path): for axis a, side s, depth l the entries
    // with o_a < -l (s = 0) or o_a > l (s = 1), storage order
    const int KSh = (np + 1) & ~1;
    std::vector<int> lidx, loff;
    std::vector<double> lk;
    for (int a = 0; a < 3; ++a)
        for (int sd = 0; sd < 2; ++sd)
            for (int l = 0; l < M; ++l) {
                lidx.push_back((int)(loff.size() / 4));
                if (a >= dim) continue;
                int64_t ent = 0;
                for (int row = 0; row < nrows; ++row)
                    for (int ei = rows[2 * row]; ei < rows[2 * row + 1]; ++ei, ++ent) {
                        const int o[3] = {o0s[(size_t)ei], (dim == 3 ? row % side : row) - M,
                                          dim == 3 ? row / side - M : 0};
                        if (!(sd == 0 ? o[a] < -l : o[a] > l)) continue;
                        loff.insert(loff.end(), {o[0], o[1], o[2], 0});
                        for (int k = 0; k < KSh; ++k) lk.push_back(kv[(size_t)ei * KSh + k]);
                    }
                (void)ent;
            }
    lidx.push_back((int)(loff.size() / 4));
    if (loff.empty()) {
        loff.assign(4, 0);
        lk.assign((size_t)KSh, 0.0);
    }
    up((void**)&e.d_lidx, lidx.data(), sizeof(int) * lidx.size());
    up((void**)&e.d_loff, loff.data(), sizeof(int) * loff.size());
    up((void**)&e.d_lK, lk.data(), sizeof(double) * lk.size());
    if (!getenv("PDGPU_WRAP_GENERIC")) build_state_table(e, rows, o0s);
    if (!getenv("PDGPU_WRAP_GENERIC") && !getenv("PDGPU_WRAP_NOFACE")) build_face_table(e, rows, o0s);
}

void launch_wrap_correction(Engine& e, const double* u, double* f, int batch, cudaStream_t s, double scale,
                            const uint8_t* cmask) {
    const Plan& pl = e.plan;
    const int SA = pl.dim - 1;
    // ghost faces: halo slabs add the true neighbour rows at interior faces;
    // the distributed FFT subtracts the opposite end's rows at the global faces
    const bool a2a = e.a2a.G > 0;
    const int lo_int = a2a ? 1 : (e.slab.global >= 0 && e.slab.off > 0);
    const int hi_int = a2a ? 1 : (e.slab.global >= 0 && e.slab.off + pl.N[SA] < e.slab.global);
    const double gsign = a2a ? -1.0 : 1.0;
    const int glob = a2a ? ((e.a2a.rank == 0 ? 1 : 0) | (e.a2a.rank == e.a2a.G - 1 ? 2 : 0)) : 0;
    const double* ghost = e.ghost_view && (lo_int || hi_int) ? e.ghost_view : nullptr;
    int64_t band[3] = {0, 0, 0};
    for (int d = 0; d < pl.dim; ++d) {
        if (!pl.circ[d] && !(d == SA && ghost)) continue;
        band[d] = 2 * e.M;
        for (int k = 0; k < 3; ++k)
            if (k != d) band[d] *= pl.N[k];
    }
    const int64_t tot = (band[0] + band[1] + band[2]) * batch;
    if (tot == 0) return;
    if (!e.d_wrows) build_wrap_table(e);
    const int th = 128;
    const unsigned blocks = (unsigned)((tot + th - 1) / th);
    const double* xstrip = nullptr;
    if (pl.dim == 3 && pl.circ[0] && e.d_xstrip && batch <= e.cap_batch && 4 * e.M <= pl.N[0] &&
        !(e.d_ftab && !a2a)) {
        const int64_t nrows = (int64_t)batch * 3 * pl.N[1] * pl.N[2];
        k_xstrip<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(u, e.d_xstrip, pl.N[0], pl.N[1], pl.N[2], e.M, nrows);
        xstrip = e.d_xstrip;
        e.launches += 1;
    }
    if (e.d_ftab && !a2a) {  // 3D, every axis periodic (halo slabs: ghost planes in the z pass): three tiled face passes
        const int M = e.M;
        const size_t smem = sizeof(double) * (size_t)M * 3 * (kFaceTB + 2 * M) * (kFaceTC + 2 * M) +
                            (sizeof(int4) + 6 * sizeof(double)) * (size_t)e.face_rec_max;
        const int* N = pl.N;
        const dim3 g0((N[1] + kFaceTB - 1) / kFaceTB, (N[2] + kFaceTC - 1) / kFaceTC, 2 * batch);
        const dim3 g1((N[0] + kFaceTB - 1) / kFaceTB, (N[2] + kFaceTC - 1) / kFaceTC, 2 * batch);
        const dim3 g2((N[0] + kFaceTB - 1) / kFaceTB, (N[1] + kFaceTC - 1) / kFaceTC, 2 * batch);
        const int th = kFaceTB * kFaceTC;
        // the surface diagonal folds in when the caller adds the corrections
        // right after (matvec / evaluate_force / CG) and D^e is the lattice's own
        const bool fold = e.fold_surface_next && e.surf_default && !ghost && e.slab.global < 0;
        if (fold) e.surface_folded = true;
        const double* xs = e.xstrip_ready ? e.d_xstrip : nullptr;  // written by this K.u's K1
        e.xstrip_ready = false;
#define PDGPU_WF(AX, G, FD)                                                                                         \
    k_wrap_face<AX, FD><<<G, th, smem, s>>>(u, f, e.d_fidx, e.d_ftab, e.d_wK, M, N[0], N[1], N[2], cmask, e.d_cmask, \
                                            pl.nodes, scale, e.face_rec_max, AX == 0 ? xs : nullptr, nullptr,        \
                                            AX == 2 ? ghost : nullptr, e.ghost_bc_stride, e.ghost_side_stride, lo_int, hi_int)
        const bool xdone = e.xpass_done;  // the x pass ran before K5 (launch_wrap_xpass)
        e.xpass_done = false;
        if (fold) {
            if (!xdone) PDGPU_WF(0, g0, true);
            PDGPU_WF(1, g1, true);
            PDGPU_WF(2, g2, true);
        } else {
            if (!xdone) PDGPU_WF(0, g0, false);
            PDGPU_WF(1, g1, false);
            PDGPU_WF(2, g2, false);
        }
#undef PDGPU_WF
        e.launches += xdone ? 1 : 2;  // the caller counts one
        return;
    }
    if (e.d_stab) {  // per-state lists (every band node)
        // few band nodes (small lattices, latency-bound): four lanes per node
        const bool quad = tot < (int64_t)e.num_sms * 256;
        const unsigned tb = (unsigned)((tot * (quad ? 4 : 1) + th - 1) / th);
        // D^e folds in when every axis is periodic (the band is then exactly
        // the near-surface set) and the corrections follow this K.u
        const bool fold = e.fold_surface_next && e.surf_default && !ghost && e.slab.global < 0 &&
                          pl.circ_mask == (1 << pl.dim) - 1;
        if (fold) e.surface_folded = true;
#define PDGPU_WT(D, L, FD, XS)                                                                                        \
    launch_maybe_pdl(e.pdl, k_wrap_tab<D, L, FD>, dim3(tb), dim3(th), 0, s, u, f, e.d_sidx, e.d_stab, e.d_wK, e.M,    \
                     pl.N[0], pl.N[1], pl.N[2], pl.circ_mask, cmask, pl.nodes, batch, scale, band[0], band[1],       \
                     band[2], ghost, e.ghost_bc_stride, e.ghost_side_stride, lo_int, hi_int, XS, e.d_cmask,   \
                     gsign, glob)
        if (pl.dim == 2) {
            if (quad) {
                if (fold) PDGPU_WT(2, 4, true, nullptr);
                else PDGPU_WT(2, 4, false, nullptr);
            } else {
                if (fold) PDGPU_WT(2, 1, true, nullptr);
                else PDGPU_WT(2, 1, false, nullptr);
            }
        } else {
            if (quad) {
                if (fold) PDGPU_WT(3, 4, true, xstrip);
                else PDGPU_WT(3, 4, false, xstrip);
            } else {
                if (fold) PDGPU_WT(3, 1, true, xstrip);
                else PDGPU_WT(3, 1, false, xstrip);
            }
        }
#undef PDGPU_WT
        return;
    }
    if (pl.dim == 2)
        k_wrap<2><<<blocks, th, 0, s>>>(u, f, e.d_wrows, e.d_wo0, e.d_wK, e.M, pl.N[0], pl.N[1], pl.N[2],
                                        pl.circ_mask, cmask, pl.nodes, batch, scale, band[0], band[1], band[2],
                                        ghost, e.ghost_bc_stride, e.ghost_side_stride, lo_int, hi_int, e.d_lidx,
                                        e.d_loff, e.d_lK, nullptr);
    else
        k_wrap<3><<<blocks, th, 0, s>>>(u, f, e.d_wrows, e.d_wo0, e.d_wK, e.M, pl.N[0], pl.N[1], pl.N[2],
                                        pl.circ_mask, cmask, pl.nodes, batch, scale, band[0], band[1], band[2],
                                        ghost, e.ghost_bc_stride, e.ghost_side_stride, lo_int, hi_int, e.d_lidx,
                                        e.d_loff, e.d_lK, xstrip);
}

// 3D face path, before K5: the x pass into d_fx (needs the strip K1 wrote);
// returns true when it ran (K5 then adds d_fx at the row ends)
bool launch_wrap_xpass(Engine& e, const double* u, int batch, cudaStream_t s, double scale, const uint8_t* cmask) {
    const Plan& pl = e.plan;
    e.xpass_done = false;
    // opt-in (PDGPU_XFOLD=1): the x pass's f writes leave the wrap, but K5's
    // row-end reads of d_fx put a dependent load at the end of every K5 CTA:
    // measured 256^3 x pass 70 -> 46 us, K5 0.211 -> 0.250 ms, net slower
    const char* xf = getenv("PDGPU_XFOLD");
    if (!(xf && xf[0] == '1') ||
        !(e.d_ftab && e.d_fx && e.xstrip_ready && e.slab.global < 0 && !e.ghost_view && batch <= e.cap_batch))
        return false;
    const int M = e.M;
    const size_t smem = sizeof(double) * (size_t)M * 3 * (kFaceTB + 2 * M) * (kFaceTC + 2 * M) +
                        (sizeof(int4) + 6 * sizeof(double)) * (size_t)e.face_rec_max;
    const int* N = pl.N;
    const dim3 g0((N[1] + kFaceTB - 1) / kFaceTB, (N[2] + kFaceTC - 1) / kFaceTC, 2 * batch);
    const bool fold = e.fold_surface_next && e.surf_default;
    if (fold)
        k_wrap_face<0, true><<<g0, kFaceTB * kFaceTC, smem, s>>>(u, nullptr, e.d_fidx, e.d_ftab, e.d_wK, M, N[0], N[1],
                                                                 N[2], cmask, e.d_cmask, pl.nodes, scale,
                                                                 e.face_rec_max, e.d_xstrip, e.d_fx);
    else
        k_wrap_face<0, false><<<g0, kFaceTB * kFaceTC, smem, s>>>(u, nullptr, e.d_fidx, e.d_ftab, e.d_wK, M, N[0],
                                                                  N[1], N[2], cmask, e.d_cmask, pl.nodes, scale,
                                                                  e.face_rec_max, e.d_xstrip, e.d_fx);
    e.launches += 1;
    e.xpass_done = true;
    return true;
}

void launch_corrections(Engine& e, const double* u, double* f, int batch, cudaStream_t s, double scale) {
    const int64_t N = e.plan.nodes;
    const bool folded = e.surface_folded;  // D^e already added by the face passes of this K.u
    e.surface_folded = false;
    e.fold_surface_next = false;
    if (e.n_surf > 0 && !folded) {
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
    if (e.n_bond_rows > 0 || e.bond_rows_on_device) {
        PassTimer pt(e, kPassBonds, s);
        const int th = 256;
        // host count known: exact grid; otherwise a resident grid reading the count
        const int64_t blocks = e.bond_rows_on_device ? (int64_t)e.num_sms * 8
                                                     : (e.n_bond_rows * batch * 32 + th - 1) / th;
        const unsigned long long* nd = e.bond_rows_on_device ? e.d_counters : nullptr;
        // koff is stored right after the stencils in d_K (see abi.cu)
        const double* koff = e.d_K + e.np * e.ss;
        const int SA = e.dim - 1;
        const int64_t plane = e.dim == 3 ? (int64_t)e.plan.N[0] * e.plan.N[1] : e.plan.N[0];
        const double* gh = slab_has_faces(e) ? e.ghost_view : nullptr;
        if (e.dim == 2)
            k_bonds<2><<<(unsigned)blocks, th, 0, s>>>(u, f, e.d_bond_rows, e.n_bond_rows, nd, e.d_ledger, e.lw,
                                                      e.d_disp, koff, e.nof, e.d_cmask, N, batch, scale, gh,
                                                      e.ghost_bc_stride, e.ghost_side_stride, plane, e.plan.N[SA],
                                                      e.M);
        else
            k_bonds<3><<<(unsigned)blocks, th, 0, s>>>(u, f, e.d_bond_rows, e.n_bond_rows, nd, e.d_ledger, e.lw,
                                                      e.d_disp, koff, e.nof, e.d_cmask, N, batch, scale, gh,
                                                      e.ghost_bc_stride, e.ghost_side_stride, plane, e.plan.N[SA],
                                                      e.M);
    }
    check(cudaGetLastError(), "corrections launch");
}

// ---------------------------------------------------------------- K7 -----
struct BondArgs {
    int dim, Nx, Ny, Nz, nof, lw;
    double h, o0, o1, o2;
    double s0;
    double s1sq;  // (1 + s0)^2
    // tiled 2D test: (1 + s0)^2 h^2 (1 -+ 1e-9), times the offset's integer |o|^2 the
    // squared-length thresholds of the unambiguous decisions (below)
    double thr_lo, thr_hi;
    int fast;     // squared-length pre-test enabled (s0 > -1)
    int has_watch;
    double wlo[3], whi[3];
    // halo slabs: global row offset of the slowest axis (positions are global,
    // grid.hpp:53-57), and the rows beyond the upper interior face (ghost side
    // 1, read for bonds the lower slab owns: q > p, fracture.hpp:220)
    int zoff, ghi;
    const double* ghost;
    int64_t gs_bc, gs_side, plane;
};

// counters[2] += counters[1] (breaks of this sweep, for a later host read)
__global__ void k_accumulate(unsigned long long* counters) { counters[2] += counters[1]; }

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
    const int SA = A.dim - 1;
    double xp[3], up[3];
    for (int d = 0; d < A.dim; ++d) xp[d] = pos_rn(org[d], c[d] + (d == SA ? A.zoff : 0), A.h);
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
            inside = inside && cq[d] >= 0 && cq[d] < dims[d] + (d == SA ? A.ghi : 0);
        }
        if (!inside) continue;
        const bool remote = cq[SA] >= dims[SA];  // in the next slab (ghost side 1)
        double xq[3];
        for (int d = 0; d < A.dim; ++d) xq[d] = pos_rn(org[d], cq[d] + (d == SA ? A.zoff : 0), A.h);
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
            // ghost side 1, vector 0: layer * plane + in-plane index == q - nodes
            const double uq = remote ? A.ghost[(int64_t)d * A.gs_bc + A.gs_side + (q - nodes)] : u[(int64_t)d * nodes + q];
            const double ev = __dsub_rn(__dadd_rn(r, uq), up[d]);
            len0 = __dadd_rn(len0, __dmul_rn(r, r));
            len1 = __dadd_rn(len1, __dmul_rn(ev, ev));
        }
        // Decide on squared lengths when the answer is unambiguous (s >= s0
        // <=> |xi+eta|^2 >= (1+s0)^2 |xi|^2); the margin (1e-12 relative) is
        // far above the few-ulp error of either side, so only bonds within
        // it take the reference's exact sqrt/div sequence below and every
        // decision stays the reference's (fracture.hpp:17-29, 224).
        bool brk;
        const double thr = A.s1sq * len0;
        if (A.fast && len1 < thr * (1.0 - 1e-12)) {
            brk = false;
        } else if (A.fast && len1 > thr * (1.0 + 1e-12)) {
            brk = true;
        } else {
            len0 = __dsqrt_rn(len0);
            len1 = __dsqrt_rn(len1);
            const double s = __ddiv_rn(__dsub_rn(len1, len0), len0);
            brk = s >= A.s0;
        }
        if (brk) {
            atomicOr(&ledger[p * A.lw + (k >> 5)], 1u << (k & 31));
            const int kn = negk[k];
            if (!remote) atomicOr(&ledger[q * A.lw + (kn >> 5)], 1u << (kn & 31));  // remote: the face merge
            const unsigned long long slot = atomicAdd(&counters[1], 1ull);
            if ((int64_t)slot < cap) {
                new_pairs[2 * slot] = p;
                new_pairs[2 * slot + 1] = k;
            }
            if (atomicExch(&listed[p], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = p;
            if (!remote && atomicExch(&listed[q], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = q;
        }
    }
}

// 2D tiled variant of k_update_bonds (no watch box): 32 x 8 nodes per CTA,
// u of the tile plus its forward halo (x +-M, y +M) in SMEM, compile-time
// forward offsets (q > p: oy > 0, or oy == 0 and ox > 0), one ledger word per
// node.  Same arithmetic and decision rule as k_update_bonds.
constexpr int band_index2d(int M, int ox, int oy) {
    int idx = 0;
    for (int a = -M; a <= M; ++a)
        for (int b = -M; b <= M; ++b) {
            if (a == ox && b == oy) return idx;
            if (a * a + b * b > 0 && a * a + b * b <= M * M) ++idx;
        }
    return -1;
}

template <int M>
__global__ void __launch_bounds__(256) k_update_bonds_tile2d(const double* __restrict__ u, uint32_t* ledger, BondArgs A,
                                                             int64_t nodes, long long* new_pairs, int64_t cap,
                                                             unsigned long long* counters, long long* bond_rows,
                                                             int* listed) {
    constexpr int TX = 32, TY = 8, W = TX + 2 * M, H = TY + M;
    __shared__ double su[2][H][W + 1];
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    for (int i = threadIdx.x; i < H * W; i += 256) {
        const int yy = i / W, xx = i - yy * W;
        const int gx = x0 + xx - M, gy = y0 + yy;
        const bool in = gx >= 0 && gx < A.Nx && gy < A.Ny;
        const int64_t q = (int64_t)gy * A.Nx + gx;
        if (!in && gx >= 0 && gx < A.Nx && gy < A.Ny + A.ghi) {  // rows of the next slab (ghost side 1)
            su[0][yy][xx] = A.ghost[A.gs_side + (q - nodes)];
            su[1][yy][xx] = A.ghost[A.gs_bc + A.gs_side + (q - nodes)];
            continue;
        }
        su[0][yy][xx] = in ? u[q] : 0.0;
        su[1][yy][xx] = in ? u[nodes + q] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & (TX - 1), ty = threadIdx.x / TX;
    const int cx = x0 + tx, cy = y0 + ty;
    if (cx >= A.Nx || cy >= A.Ny) return;
    const int64_t p = (int64_t)cy * A.Nx + cx;
    const double xp0 = pos_rn(A.o0, cx, A.h), xp1 = pos_rn(A.o1, cy + A.zoff, A.h);
    const double up0 = su[0][ty][tx + M], up1 = su[1][ty][tx + M];
    const uint32_t word = ledger[p];  // lw == 1 (<= 32 in-band offsets)
    uint32_t newbits = 0;
    // tiles whose forward halo lies inside the lattice skip the per-bond range
    // tests (uniform per CTA); a bond is looked at again only if it is live and
    // not clearly below the threshold, so the common case is branch-free
    const bool interior = x0 >= M && x0 + TX + M <= A.Nx && y0 + TY + M <= A.Ny;
    auto sweep = [&](auto interior_c) {
        constexpr bool INTERIOR = decltype(interior_c)::value;
#pragma unroll
        for (int oy = 0; oy <= M; ++oy) {
#pragma unroll
            for (int ox = -M; ox <= M; ++ox) {
                if (ox * ox + oy * oy > M * M || (oy == 0 && ox <= 0)) continue;
                const int k = band_index2d(M, ox, oy);
                const int qx = cx + ox, qy = cy + oy;
                const bool inb = INTERIOR || (qx >= 0 && qx < A.Nx && qy < A.Ny + A.ghi);
                const bool live = inb && !((word >> k) & 1u);
                const double r0 = __dsub_rn(pos_rn(A.o0, qx, A.h), xp0);
                const double r1 = __dsub_rn(pos_rn(A.o1, qy + A.zoff, A.h), xp1);
                const double e0 = __dsub_rn(__dadd_rn(r0, su[0][ty + oy][tx + M + ox]), up0);
                const double e1 = __dsub_rn(__dadd_rn(r1, su[1][ty + oy][tx + M + ox]), up1);
                double len1 = __dadd_rn(__dadd_rn(0.0, __dmul_rn(e0, e0)), __dmul_rn(e1, e1));
                // Unambiguous decisions against the nominal reference length |o|^2 h^2:
                // the rounded node positions move |xi|^2 by a few ulp of the largest
                // coordinate over h (~1e-11 relative on a unit plate at 4096^2), the
                // reference's own s by a few ulp, so outside the band (1e-9 plus that
                // bound, launch_update_bonds) the reference decides the same way;
                // inside it the reference's exact sequence runs (fracture.hpp:17-29, 224).
                const double n2 = (double)(ox * ox + oy * oy);  // a constant once unrolled
                if (!live || (A.fast && len1 < A.thr_lo * n2)) continue;
                bool brk;
                if (A.fast && len1 > A.thr_hi * n2) {
                    brk = true;
                } else {
                    const double len0 = __dsqrt_rn(__dadd_rn(__dadd_rn(0.0, __dmul_rn(r0, r0)), __dmul_rn(r1, r1)));
                    len1 = __dsqrt_rn(len1);
                    brk = __ddiv_rn(__dsub_rn(len1, len0), len0) >= A.s0;
                }
                if (!brk) continue;
                newbits |= 1u << k;
                const int64_t q = p + (int64_t)oy * A.Nx + ox;
                const bool local = qy < A.Ny;  // else the next slab's node: its bit arrives by the face merge
                if (local) atomicOr(&ledger[q], 1u << band_index2d(M, -ox, -oy));
                const unsigned long long slot = atomicAdd(&counters[1], 1ull);
                if ((int64_t)slot < cap) {
                    new_pairs[2 * slot] = p;
                    new_pairs[2 * slot + 1] = k;
                }
                if (local && atomicExch(&listed[q], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = q;
            }
        }
    };
    if (interior) sweep(std::true_type{});
    else sweep(std::false_type{});
    if (newbits) {
        atomicOr(&ledger[p], newbits);
        if (atomicExch(&listed[p], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = p;
    }
}

// Halo slabs: the lower slab decides the bonds crossing its upper face (q > p,
// fracture.hpp:220) and sets only its own half; the ledger words of its last M
// rows reach this slab (recv, [M][plane][lw]) and every bit whose partner lies
// in this slab's rows becomes the mirrored bit here (ledger.hpp:21-26), the
// row listed for the correction SpMV.  Idempotent (the ledger is monotone).
__global__ void k_merge_face(uint32_t* ledger, int lw, const uint32_t* __restrict__ recv, const int* __restrict__ offs,
                             const int* __restrict__ negk, int nof, int dim, int N0, int N1, int M, int64_t plane,
                             long long* bond_rows, int* listed, unsigned long long* counters) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (layer, in-plane node)
    if (i >= (int64_t)M * plane) return;
    const int layer = (int)(i / plane);
    const int64_t pin = i - (int64_t)layer * plane;
    const int c0 = (int)(pin % N0), c1 = dim == 3 ? (int)(pin / N0) : 0;
    const int SA = dim - 1;
    for (int k = 0; k < nof; ++k) {
        if (!((recv[i * lw + (k >> 5)] >> (k & 31)) & 1u)) continue;
        const int* o = offs + 3 * k;
        const int row = layer - M + o[SA];  // local row of the partner
        if (row < 0) continue;              // a bond inside the lower slab
        const int q0 = c0 + o[0], q1 = dim == 3 ? c1 + o[1] : 0;
        const int64_t q = (int64_t)row * plane + (dim == 3 ? (int64_t)q1 * N0 : 0) + q0;
        (void)N1;
        const int kn = negk[k];
        const unsigned old = atomicOr(&ledger[q * lw + (kn >> 5)], 1u << (kn & 31));
        if (!((old >> (kn & 31)) & 1u) && atomicExch(&listed[q], 1) == 0) bond_rows[atomicAdd(&counters[0], 1ull)] = q;
    }
}

void launch_merge_face(Engine& e, const uint32_t* recv, cudaStream_t s) {
    const int64_t plane = e.dim == 3 ? (int64_t)e.plan.N[0] * e.plan.N[1] : e.plan.N[0];
    const int64_t n = (int64_t)e.M * plane;
    const int* negk = (const int*)(e.d_offs + 3 * e.nof);
    k_merge_face<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(e.d_ledger, e.lw, recv, e.d_offs, negk, e.nof, e.dim,
                                                           e.plan.N[0], e.plan.N[1], e.M, plane, e.d_bond_rows,
                                                           e.d_listed, e.d_counters);
    e.launches += 1;
    check(cudaGetLastError(), "merge face");
}

// Returns the number of newly broken bonds (sync = true); new pairs are left
// in e.d_new_pairs as (p, offset index) and bond rows are appended.  With
// sync = false nothing is read back: the row count stays on the device
// (k_bonds reads it) and counters[2] accumulates the breaks for the caller.
int64_t launch_update_bonds(Engine& e, const double* u, double s0, const double* watch, cudaStream_t s, bool sync) {
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
    A.s1sq = (1.0 + s0) * (1.0 + s0);
    {
        // band of the nominal-length decisions: the rounded positions move a bond
        // component (>= h) by a few ulp of the largest coordinate
        double xmax = 0.0;
        for (int d = 0; d < e.dim; ++d)
            xmax = std::max(xmax, std::fabs(e.origin[d]) + (pl.N[d] + (e.slab.global >= 0 && d == e.dim - 1 ? e.slab.global : 0)) * e.h);
        const double band = 1e-9 + 32.0 * 2.2204460492503131e-16 * xmax / e.h;
        A.thr_lo = A.s1sq * A.h * A.h * (1.0 - band);
        A.thr_hi = A.s1sq * A.h * A.h * (1.0 + band);
    }
    A.fast = s0 > -1.0 + 1e-6 && !getenv("PDGPU_EXACT_STRETCH");
    A.has_watch = watch != nullptr;
    for (int d = 0; d < 3; ++d) {
        A.wlo[d] = watch && d < e.dim ? watch[d] : 0.0;
        A.whi[d] = watch && d < e.dim ? watch[e.dim + d] : 0.0;
    }
    A.zoff = e.slab.global >= 0 ? e.slab.off : 0;
    const bool hi_ghost = slab_hi_face(e) && e.ghost_view;
    A.ghi = hi_ghost ? e.M : 0;
    A.ghost = hi_ghost ? e.ghost_view : nullptr;
    A.gs_bc = e.ghost_bc_stride;
    A.gs_side = e.ghost_side_stride;
    A.plane = e.dim == 3 ? (int64_t)pl.N[0] * pl.N[1] : pl.N[0];
    touch_state(e);  // the bond-row count changes under any captured launch sequence
    // reset the new-pair counter, keep the row counter
    check(cudaMemsetAsync(e.d_counters + 1, 0, sizeof(unsigned long long), s), "reset counter");
    const int th = 128;
    const int64_t N = pl.nodes;
    const int* negk = (const int*)(e.d_offs + 3 * e.nof);
    e.launches += 1;
    if (e.dim == 2 && e.lw == 1 && !watch && e.M >= 1 && e.M <= 3 && !getenv("PDGPU_BONDS_GENERIC")) {
        dim3 grid((pl.N[0] + 31) / 32, (pl.N[1] + 7) / 8);
#define PDGPU_UB(MM)                                                                                      \
    k_update_bonds_tile2d<MM><<<grid, 256, 0, s>>>(u, e.d_ledger, A, N, e.d_new_pairs, e.new_pairs_cap, \
                                                  e.d_counters, e.d_bond_rows, e.d_listed)
        if (e.M == 1) PDGPU_UB(1);
        else if (e.M == 2) PDGPU_UB(2);
        else PDGPU_UB(3);
#undef PDGPU_UB
    } else {
        k_update_bonds<<<(unsigned)((N + th - 1) / th), th, 0, s>>>(u, e.d_ledger, e.d_offs, e.d_disp, negk, A, N,
                                                                   e.d_new_pairs, e.new_pairs_cap, e.d_counters,
                                                                   e.d_bond_rows, e.d_listed);
    }
    check(cudaGetLastError(), "update_bonds launch");
    if (!sync) {
        e.bond_rows_on_device = true;
        k_accumulate<<<1, 1, 0, s>>>(e.d_counters);
        return 0;
    }
    unsigned long long cnt[2];
    check(cudaMemcpyAsync(cnt, e.d_counters, sizeof(cnt), cudaMemcpyDeviceToHost, s), "read counters");
    check(cudaStreamSynchronize(s), "update_bonds");
    e.n_bond_rows = (int64_t)cnt[0];
    e.bond_rows_on_device = false;
    e.total_broken += (int64_t)cnt[1];
    return (int64_t)cnt[1];
}

}  // namespace pdgpu
