// spectral.cu -- the MSBFM spectral product f = A_hat u on sm_100a.
//
// Replaces FastForce<Dim>::apply (reference convolution.hpp:249-259): d
// forward padded FFTs (forward_field :119-128), the d x d per-frequency
// product with conj(G_hat) (hadamard :135-154) and d inverse FFTs with window
// extraction (inverse_extract :158-172).
//
// Pass structure (one vector; B vectors batch into the grid):
//   K1 rfft_rows   : real rows along x -> half spectrum (Hx = Px/2+1 columns),
//                    written transposed [kx][row] so K3 reads contiguously.
//   K2 cfft_y_fwd  : (3D) padded y FFT, written transposed [kx][ky][z].
//   K3 spectral    : padded FFT along the last axis, d x d symbol multiply,
//                    inverse FFT, truncation to the window -- one fused pass,
//                    spectra never leave registers between the transforms;
//                    in place.
//   K4 cfft_y_inv  : (3D) inverse y FFT + truncation, transposed back.
//   K5 irfft_rows  : C2R along x + truncation + epilogue (scale, constraint
//                    mask, body force), written in the reference's node order.
// All transforms are register-resident Stockham FFTs (fft.cuh).  The symbol
// (K9) is conj(G_hat)/prod(P) by a direct DFT of the (2M+1)^d stencil: real
// for the physical (even) stencils, complex for arbitrary ones (the
// reference's random-stencil tests).  Layout [col][half][k][pair] so each
// thread reads its n_pairs coefficients contiguously.
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point, no libcuda link)
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "engine.h"
#include "fft.cuh"

#ifndef PDGPU_PART
#define PDGPU_ALL_PARTS 1  // see "The host side is compiled in parts" below
#endif

namespace pdgpu {

// ------------------------------------------------ async copies / L2 hints ---
// mbarrier + 1D bulk copy (cp.async.bulk, TMA engine) helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// bulk prefetch of [src, src+bytes) into L2 (TMA engine, no SMEM, no registers)
__device__ __forceinline__ void l2_prefetch(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = pred ? 16 : 0;  // zero-fill outside the window
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
// L2 eviction-priority hints (createpolicy, sm_80+): data re-read within the
// same CTA a few microseconds later is loaded/stored evict_last, its last use
// evict_first, so the streaming traffic of the other CTAs does not push it out.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ld_hint(const double2* a, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ld_hint_rw(const double2* a, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(double2* a, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

static inline int ilog2(int64_t v) {
    int l = 0;
    while ((int64_t(1) << l) < v) ++l;
    return l;
}

constexpr int kSmemBudget = 210 * 1024;

static int xbuf_slots(int logq) { return (1 << logq) + ((1 << logq) >> 4) + 1; }
static int threads_per_transform(int logq, int logrmax) { return 1 << std::max(0, logq - logrmax); }
// TMA-gather / TMA-store row kernels (two rows per CTA): per-transform buffer
// stride with 2*stride = 4 (mod 8) 16-byte slots, so the two rows' buffers sit
// 64 bytes apart (mod 128): a quarter-warp spanning both rows hits all 32 banks
__host__ __device__ constexpr int xbuf_stride_rows(int xb) { return xb + ((2 - (xb & 3)) & 3); }
static int xbuf_stride_rows_h(int logq) { return xbuf_stride_rows(xbuf_slots(logq)); }
// row kernels with T < 8 threads per transform: 8/T transforms share a
// quarter-warp; per-transform buffers T (mod 8) 16-byte slots apart put them
// on distinct bank groups (T = 4: the two halves of a quarter-warp 64 B apart)
__host__ __device__ constexpr int xbuf_stride_t(int xb, int T) { return T >= 8 ? xb : xb + ((T - (xb & 7)) & 7); }
static int xbuf_stride_t_h(int logq) { return xbuf_stride_t(xbuf_slots(logq), threads_per_transform(logq, 4)); }

// box tensor map over S[slab][kx][row] (complex): dims {2*Nrow doubles, Hx, nslab},
// box {2*TR doubles, 256 kx, 1}; cuTensorMapEncodeTiled through the runtime's
// driver entry point
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// blocked: the row-blocked spectrum [slab][row / 8][kx][row % 8] (2D S2 between
// K3 and K5, launch_k3_2d) -- x = 2 * (row % 8), z = slab * (Nrow / 8) + row / 8
static bool encode_box_map(CUtensorMap& m, const double2* S, int Nrow, int Hx, int nslab, int TR,
                           bool blocked = false, int boxk = 256) {
    static EncodeTiledFn enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            enc = nullptr;
            return false;
        }
    }
    cuuint64_t dims[3] = {(cuuint64_t)2 * Nrow, (cuuint64_t)Hx, (cuuint64_t)nslab};
    cuuint64_t strides[2] = {(cuuint64_t)Nrow * 16, (cuuint64_t)Hx * Nrow * 16};
    if (blocked) {
        dims[0] = 16;
        dims[2] = (cuuint64_t)nslab * (Nrow / 8);
        strides[0] = 128;
        strides[1] = (cuuint64_t)Hx * 128;
    }
    cuuint32_t box[3] = {(cuuint32_t)(2 * TR), (cuuint32_t)boxk, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)S, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#if defined(PDGPU_ALL_PARTS) || PDGPU_PART == 0
void plan_init(Plan& pl, int dim, const int* dims, int M) {
    pl.dim = dim;
    bool periodic_ok = true;
    if (const char* env = getenv("PDGPU_EMBED")) periodic_ok = std::string(env) != "padded";
    pl.circ_mask = 0;
    for (int d = 0; d < 3; ++d) {
        pl.N[d] = d < dim ? dims[d] : 1;
        pl.circ[d] = 0;
        if (d < dim) {
            const int lp = ilog2(pl.N[d]);
            const bool pow2 = (1 << lp) == pl.N[d];
            // periodic needs a power of two with room for the whole stencil
            // (no self-overlap of the wrapped band) and the transform minimum
            // sizes (duo/3D spectral kernels: >= 16 points)
            pl.circ[d] = periodic_ok && pow2 && pl.N[d] >= 2 * M + 1 && pl.N[d] >= 16;
            pl.logP[d] = pl.circ[d] ? lp : lp + 1;
            pl.P[d] = 1 << pl.logP[d];
            pl.circ_mask |= pl.circ[d] << d;
        } else {
            pl.logP[d] = 0;
            pl.P[d] = 1;
        }
    }
    pl.nodes = (int64_t)pl.N[0] * pl.N[1] * pl.N[2];
    pl.Hx = pl.P[0] / 2 + 1;
    pl.logQx = pl.logP[0] - 2;
    if (dim == 2) {
        pl.ncols = pl.Hx;
        pl.Nl = pl.N[1];
        pl.Pl = pl.P[1];
        pl.logPl = pl.logP[1];
        pl.nh = pl.circ[1] ? 1 : 2;
        pl.S1_per_vec = (int64_t)dim * pl.Hx * pl.N[1];
        pl.S2_per_vec = pl.S1_per_vec;  // K3 output (out of place, z^0 parked in it)
    } else {
        pl.ncols = pl.Hx * pl.P[1];
        pl.Nl = pl.N[2];
        pl.Pl = pl.P[2];
        pl.logPl = pl.logP[2];
        pl.nh = pl.circ[2] ? 1 : 2;
        pl.S1_per_vec = (int64_t)dim * pl.N[2] * pl.Hx * pl.N[1];
        pl.S2_per_vec = (int64_t)dim * pl.Hx * pl.P[1] * pl.N[2];
    }
    pl.logTWN = std::max(pl.logP[0], std::max(pl.logP[1], pl.logP[2]));
    // K1/K5: two transforms (even/odd outputs) of Qx points per row
    {
        const int T = threads_per_transform(pl.logQx, 4);
        const int per_row = 2 * xbuf_slots(pl.logQx) * 16;
        int tr = 1;
        while (tr < 8 && 2 * (tr * 2) * T <= 512 && (tr * 2) * per_row <= kSmemBudget) tr *= 2;
        if (const char* env = getenv("PDGPU_K1_ROWS")) tr = std::max(1, std::min(tr, atoi(env)));
        while (tr > 1 && tr > pl.N[1]) tr /= 2;  // power of two (K1 pipe template)
        pl.k1_rows = tr;
    }
    // K3: columns per CTA
    {
        const int logq = pl.logPl - (pl.nh == 2 ? 1 : 0);
        const int logr = dim == 3 ? 3 : 4;
        const int T = threads_per_transform(logq, logr);
        // 2D columns are too long to park z^0 on chip; periodic: no z^0 at all
        const bool zsmem = dim == 3 && pl.nh == 2;
        const int per_col = (xbuf_slots(logq) + (zsmem ? 2 * dim - 1 : dim - 1) * (1 << logq)) * 16;
        int nc = 1;
        while ((nc * 2) * T <= 256 && (nc * 2) * per_col <= kSmemBudget) nc *= 2;
        pl.k3_cols = nc;
        pl.k3_halves = dim == 3 ? 2 : 1;  // 3D: in place on S2; 2D: out of place S1 -> S2
    }
    if (dim == 3) {
        const int logq = pl.logP[1] - 1;
        const int T = threads_per_transform(logq, 4);
        const int per_z = 2 * xbuf_slots(logq) * 16;
        int zt = 1;
        while (zt < 8 && 2 * (zt * 2) * T <= 512 && (zt * 2) * per_z <= kSmemBudget) zt *= 2;
        pl.k2_zt = std::min(zt, pl.N[2]);
    }
}
#endif

// ------------------------------------------------------------------ K1 ---
// Row transform of Nx reals zero-padded to Px = 4*Qx: z[n] = x[2n] + i x[2n+1]
// (n < Qx carries all data); Z = FFT_{2Qx}(z) via even (E) and odd (O)
// outputs, each a Qx-point FFT; X[k] = Fe + e^{-2 pi i k/Px} Fo.
// CIRC (periodic embedding, Px = Nx): z fills all 2Qx points and the even /
// odd split is a decimation-in-frequency stage, E <- z[n] + z[n+Qx],
// O <- (z[n] - z[n+Qx]) e^{-2 pi i n/(2Qx)}.
template <int LOGQ, bool CIRC>
__global__ void __launch_bounds__(512) k_rfft_rows(const double* __restrict__ u, double2* __restrict__ S, int Nx,
                                                   int Nrow, int Hx, int TR, const double2* __restrict__ tw,
                                                   int logTWN) {
    using Sh = FftShape<LOGQ, 4>;
    constexpr int Q = Sh::Q, T = Sh::T, R = Sh::R, XB = xbuf_stride_t(Sh::XBUF, Sh::T);
    extern __shared__ double2 sm[];
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    const int r = gi >> 1, eo = gi & 1;
    const int slab = blockIdx.y;
    const int row0 = blockIdx.x * TR;
    const int nr = min(TR, Nrow - row0);
    const bool valid = r < nr;
    const double* src = u + ((int64_t)slab * Nrow + row0 + r) * Nx;
    double2* xb = sm + gi * XB;
    double2 v[R];
    const int shE = logTWN - (LOGQ + 1);
    const bool vec = (Nx & 1) == 0;
    const double2 wbase = __ldg(tw + (t << shE));  // e^{-2 pi i t/(2Qx)}
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int n = t + j * T;
        const int i0 = 2 * n;
        double2 z = make_double2(0.0, 0.0);
        if (valid && i0 < Nx) {
            if (vec) z = __ldg(reinterpret_cast<const double2*>(src + i0));
            else z = make_double2(src[i0], i0 + 1 < Nx ? src[i0 + 1] : 0.0);
        }
        if (CIRC) {  // Nx = 4Q, even
            const double2 z2 = valid ? __ldg(reinterpret_cast<const double2*>(src + i0 + 2 * Q)) : make_double2(0.0, 0.0);
            z = eo ? csub(z, z2) : cadd(z, z2);
        }
        v[j] = eo ? cmul(z, tw32r<-1>(j * (16 / R), wbase)) : z;
    }
    reg_fft<LOGQ, 4, -1>(v, t, xb, make_fft_tw<LOGQ, 4>(t, tw, logTWN), BlockBar{});
#pragma unroll
    for (int j = 0; j < R; ++j) xb[spad(t + j * T)] = v[j];
    __syncthreads();
    constexpr int halfP = 2 * Q;
    const int shX = logTWN - (LOGQ + 2);
    // e^{-2 pi i kx/Px} by recurrence along the thread's kx sequence
    const bool rec = (blockDim.x % nr) == 0;
    const int kstep = rec ? (int)blockDim.x / nr : 0;
    double2 Wk = __ldg(tw + ((threadIdx.x / nr) << shX));
    const double2 Wstep = __ldg(tw + ((kstep & (2 * halfP - 1)) << shX));
    for (int idx = threadIdx.x; idx < nr * Hx; idx += blockDim.x) {
        const int kx = idx / nr, rr = idx - kx * nr;
        const int k = kx & (halfP - 1);
        const int k2 = (halfP - kx) & (halfP - 1);
        const double2* Z = sm + 2 * rr * XB;
        const double2 A = Z[(k & 1) * XB + spad(k >> 1)];
        const double2 B = cconj(Z[(k2 & 1) * XB + spad(k2 >> 1)]);
        const double2 Fe = cscale(cadd(A, B), 0.5);
        const double2 D = csub(A, B);
        const double2 Fo = make_double2(0.5 * D.y, -0.5 * D.x);
        const double2 W = rec ? Wk : __ldg(tw + (kx << shX));
        Wk = cmul(Wk, Wstep);
        S[((int64_t)slab * Hx + kx) * Nrow + row0 + rr] = cadd(Fe, cmul(W, Fo));
    }
}

// ------------------------------------------------------------------ K5 ---
// C2R: Z[k] = (X[k] + conj X[h-k]) + i e^{+2 pi i k/Px} (X[k] - conj X[h-k]),
// h = Px/2; z = IFFT_{2Qx}(Z) on its first Qx outputs = E'[n] + e^{+2 pi i n/(2Qx)} O'[n];
// x[2n] = Re z, x[2n+1] = Im z.  CIRC (Px = Nx): all 2Qx outputs are kept,
// z[n + Qx] = E'[n] - e^{+2 pi i n/(2Qx)} O'[n].
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* m, void* dst, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(m), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* m, int x, int y, int z) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(m), "r"(x), "r"(y), "r"(z)
                 : "memory");
}

// TMAG: the tile's [kx][row] spectrum block lands in SMEM through TMA boxes
// ({2*TR doubles, 256 kx} per box, the box tensor map tm over S) instead of
// per-thread global gathers; the pre-processing then reads it from SMEM.
template <int LOGQ, int LOGTR, bool CIRC, bool TMAG = false>
__global__ void __launch_bounds__(512) k_irfft_rows(const double2* __restrict__ S, double* __restrict__ f, int Nx,
                                                    int Nrow, int Nz, int dim, int Hx,
                                                    const double2* __restrict__ tw, int logTWN, double scale,
                                                    const uint8_t* __restrict__ cmask,
                                                    const double* __restrict__ body, int64_t nodes,
                                                    const __grid_constant__ CUtensorMap tm, int pf,
                                                    const double* __restrict__ fx, int Mfx, int blk = 0) {
    pdl_entry();
    using Sh = FftShape<LOGQ, 4>;
    constexpr int Q = Sh::Q, T = Sh::T, R = Sh::R;
    constexpr int XB = TMAG ? xbuf_stride_rows(Sh::XBUF) : xbuf_stride_t(Sh::XBUF, Sh::T);  // per-transform stride
    constexpr int TR = 1 << LOGTR;
    extern __shared__ double2 sm[];
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    const int eo = gi & 1;
    const int slab = blockIdx.y;
    const int row0 = blockIdx.x * TR;
    const int nr = min(TR, Nrow - row0);
    constexpr int halfP = 2 * Q;
    const int shX = logTWN - (LOGQ + 2);
    const double2* src = S + (int64_t)slab * Hx * Nrow + row0;
    // Z[k] and Z[halfP-k] from X[k], X[halfP-k] for k < Q; thread item u has
    // j = j0 + 2T*u, k = 2j (j < Q/2) or 2(j - Q/2) + 1, so Z lands in E[j],
    // E[Q-j] or O[j'], O[Q-1-j'] -- consecutive slots of one buffer per
    // quarter-warp.  Thread i -> j0 = 8*(i >> (3+LOGTR)) + (i & 7), row
    // rr = (i >> 3) & (TR-1) (rows adjacent in S fill whole sectors).  The U
    // item loads are issued together (the gather is latency bound).
    // e^{+2 pi i k/Px} = e^{2 pi i 2 j0/Px} e^{2 pi i u/R} (x e^{2 pi i/Px} e^{-i pi/2} for odd k).
    {
        // TMAG: quarter-warp = 4 consecutive j x the 2 rows (LA = 2), and the
        // even / odd k of the same j swapped on (j >> 1) & 1 -- the landed
        // [k][row] block is then read conflict-free (8 distinct 16-byte bank
        // groups per quarter-warp instead of 2 or 4)
        constexpr int LA = TMAG ? 2 : ((2 * T >= 8) ? 3 : 0);
        constexpr int U = R / 2;
        const int rr = (threadIdx.x >> LA) & (TR - 1);
        const int j0 = ((threadIdx.x >> (LA + LOGTR)) << LA) + (threadIdx.x & ((1 << LA) - 1));
        const bool live = rr < nr;
        const double2 W0 = twiddle<1>(tw, (2 * j0) << shX);
        const double2 W1 = cmul(W0, twiddle<1>(tw, 1 << shX));
        double2 Xa[U], Xb[U];
        double2 xq = make_double2(0.0, 0.0);
        if constexpr (TMAG) {
            __shared__ __align__(8) uint64_t bar;
            // (an element offset from sm, not a pointer rounded through an integer:
            // the accesses stay in the shared window instead of becoming generic)
            double2* land = sm + ((128u - (smem_u32(sm) & 127u)) & 127u) / 16u;
            const int nbox = (Hx + 255) / 256;
            if (threadIdx.x == 0) mbar_init(&bar, 1);
            __syncthreads();
            if (threadIdx.x == 0) {
                mbar_expect_tx(&bar, (unsigned)(nbox * 256 * TR * 16));
                // blk: S is row-blocked, [slab][row / 8][kx][row % 8] (see encode_box_map)
                const int cx0 = blk ? 2 * (row0 & 7) : 2 * row0;
                const int cz0 = blk ? slab * (Nrow >> 3) + (row0 >> 3) : slab;
                for (int bx = 0; bx < nbox; ++bx) tma_load_3d(&tm, land + bx * 256 * TR, &bar, cx0, bx * 256, cz0);
                // the block of the CTA that starts pf CTAs later (launch order:
                // x fastest) into L2, so its landing is an L2 hit
                if (pf) {
                    const int64_t nxt = (int64_t)blockIdx.y * gridDim.x + blockIdx.x + pf;
                    const int by = (int)(nxt / gridDim.x), bxx = (int)(nxt % gridDim.x);
                    if (by < (int)gridDim.y) {
                        const int r1 = bxx * TR;
                        const int cx1 = blk ? 2 * (r1 & 7) : 2 * r1;
                        const int cz1 = blk ? by * (Nrow >> 3) + (r1 >> 3) : by;
                        for (int bx = 0; bx < nbox; ++bx) tma_prefetch_3d(&tm, cx1, bx * 256, cz1);
                    }
                }
            }
            mbar_wait(&bar, 0);
            static_assert(U % 2 == 0, "even / odd k halves");
#pragma unroll
            for (int u = 0; u < U / 2; ++u) {
                // items u (k = 2j) and u + U/2 (k = 2j + 1) of the same j
                const int j = j0 + 2 * T * u;
                const int ke = 2 * j, ko = 2 * j + 1;
                const bool sw = (j >> 1) & 1;
                const double2 a1 = land[(sw ? ko : ke) * TR + rr], a2 = land[(sw ? ke : ko) * TR + rr];
                const double2 b1 = land[(halfP - (sw ? ko : ke)) * TR + rr], b2 = land[(halfP - (sw ? ke : ko)) * TR + rr];
                Xa[u] = sw ? a2 : a1;
                Xa[u + U / 2] = sw ? a1 : a2;
                Xb[u] = sw ? b2 : b1;
                Xb[u + U / 2] = sw ? b1 : b2;
            }
            if (threadIdx.x < nr) xq = land[Q * TR + threadIdx.x];
            __syncthreads();  // the landing area is about to be overwritten by E / O
        } else {
            if (pf) {
                // the gather region of the CTA launched pf later into L2: its
                // Hx + 1 row chunks (TR rows x 16 B each, Nrow apart), one per thread
                const int64_t nxt = (int64_t)blockIdx.y * gridDim.x + blockIdx.x + pf;
                const int by = (int)(nxt / gridDim.x), bxx = (int)(nxt % gridDim.x);
                if (by < (int)gridDim.y) {
                    const double2* nsrc = S + (int64_t)by * Hx * Nrow + bxx * TR;
                    for (int c = threadIdx.x; c < Hx; c += blockDim.x)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(nsrc + (int64_t)c * Nrow));
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + 2 * T * u;
                const int k = j < Q / 2 ? 2 * j : 2 * (j - Q / 2) + 1;
                Xa[u] = live ? src[(int64_t)k * Nrow + rr] : make_double2(0.0, 0.0);
                Xb[u] = live ? src[(int64_t)(halfP - k) * Nrow + rr] : make_double2(0.0, 0.0);
            }
            if (threadIdx.x < nr) xq = src[(int64_t)Q * Nrow + threadIdx.x];
        }
        double2* E = sm + 2 * rr * XB;
        double2* O = E + XB;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j0 + 2 * T * u;
            const bool even = j < Q / 2;
            const double2 W = R >= 4 ? (2 * T * u < Q / 2 ? tw32r<1>(u * (32 / R), W0)
                                                            : tw32r<1>(u * (32 / R) - 8, W1))
                                     : twiddle<1>(tw, (even ? 2 * j : 2 * (j - Q / 2) + 1) << shX);
            const double2 a = Xa[u], bb = Xb[u];
            const double2 s1 = cadd(a, cconj(bb));
            const double2 t1 = cmul(W, csub(a, cconj(bb)));
            const double2 W2 = make_double2(-W.x, W.y);  // e^{+2 pi i (halfP-k)/Px}
            const double2 s2 = cadd(bb, cconj(a));
            const double2 t2 = cmul(W2, csub(bb, cconj(a)));
            const double2 Zk = make_double2(s1.x - t1.y, s1.y + t1.x);
            const double2 Zm = make_double2(s2.x - t2.y, s2.y + t2.x);
            if (live) {
                if (even) {
                    E[spad(j)] = Zk;
                    if (j != 0) E[spad(Q - j)] = Zm;
                } else {
                    const int jo = j - Q / 2;
                    O[spad(jo)] = Zk;
                    O[spad(Q - 1 - jo)] = Zm;
                }
            }
        }
        // Nyquist k = Q (self-paired, W = e^{i pi/2} = i) -> E[Q/2]
        if (threadIdx.x < nr) {
            const double2 s1 = cadd(xq, cconj(xq));
            const double2 t1 = cmul(make_double2(0.0, 1.0), csub(xq, cconj(xq)));
            sm[2 * threadIdx.x * XB + (Q & 1) * XB + spad(Q >> 1)] = make_double2(s1.x - t1.y, s1.y + t1.x);
        }
    }
    __syncthreads();
    double2* xb = sm + gi * XB;
    double2 v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = xb[spad(t + j * T)];
    __syncthreads();
    reg_fft<LOGQ, 4, 1>(v, t, xb, make_fft_tw<LOGQ, 4>(t, tw, logTWN), BlockBar{});
    const int shE = logTWN - (LOGQ + 1);
    const double2 wbase = twiddle<1>(tw, t << shE);  // e^{+2 pi i t/(2Qx)}
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int n = t + j * T;
        xb[spad(n)] = eo ? cmul(tw32r<1>(j * (16 / R), wbase), v[j]) : v[j];
    }
    __syncthreads();
    const int a = (slab / Nz) % dim;
    const int z = slab % Nz;
    double* dst = f + ((int64_t)slab * Nrow + row0) * Nx;
    const bool vec = (Nx & 1) == 0;
    // item (rr, m), m < Q: z[m] = E'[m] + O'[m] (and, periodic, z[m + Q] =
    // E'[m] - O'[m] from the same two SMEM reads); x[2n] = Re z, x[2n+1] = Im z
    auto emit = [&](int rr, int n, double2 zz) {
        const int i0 = 2 * n;
        if (i0 >= Nx) return;
        double v0 = zz.x * scale, v1 = zz.y * scale;
        const int64_t node = ((int64_t)z * Nrow + row0 + rr) * Nx + i0;
        const bool two = i0 + 1 < Nx;
        if (body) {
            v0 += body[(int64_t)a * nodes + node];
            if (two) v1 += body[(int64_t)a * nodes + node + 1];
        }
        if (cmask) {
            if ((cmask[node] >> a) & 1u) v0 = 0.0;
            if (two && ((cmask[node + 1] >> a) & 1u)) v1 = 0.0;
        }
        if (fx && (i0 < Mfx || i0 + 1 >= Nx - Mfx)) {  // 3D: the wrap x pass's result at the row ends
            // fx[b][a][z][y][slot 2M]: the row's 2M values are contiguous
            const double* fr = fx + ((int64_t)(slab / Nz) * Nz * Nrow + (int64_t)z * Nrow + row0 + rr) * 2 * Mfx;
            if (i0 < Mfx) v0 += fr[i0];
            else if (i0 >= Nx - Mfx) v0 += fr[Mfx + i0 - (Nx - Mfx)];
            if (two) {
                if (i0 + 1 < Mfx) v1 += fr[i0 + 1];
                else if (i0 + 1 >= Nx - Mfx) v1 += fr[Mfx + i0 + 1 - (Nx - Mfx)];
            }
        }
        double* o = dst + (int64_t)rr * Nx + i0;
        if (vec) {
            *reinterpret_cast<double2*>(o) = make_double2(v0, v1);
        } else {
            o[0] = v0;
            if (two) o[1] = v1;
        }
    };
#pragma unroll 4
    for (int u = 0; u < R / 2; ++u) {  // nr*Q <= 2*TR*T * R/2 items
        const int idx = threadIdx.x + u * 2 * TR * T;
        const int rr = idx >> LOGQ, m = idx & (Q - 1);
        if (rr >= nr) continue;
        const double2 ze = sm[2 * rr * XB + spad(m)];
        const double2 zo = sm[(2 * rr + 1) * XB + spad(m)];
        emit(rr, m, cadd(ze, zo));
        if (CIRC) emit(rr, m + Q, csub(ze, zo));
    }
}

// ------------------------------------- K5, persistent, two row groups ---
// k_irfft_rows<10, 1, true, true> (periodic 4096-wide rows, two rows per tile,
// TMA-landed [kx][2 rows] blocks) as one persistent 512-thread CTA per SM made
// of two 256-thread groups.  Each group has its own work area (E / O spectra
// and FFT exchange) and its own named barrier; the landing buffer is shared:
// the moment a group has its block in registers it requests the next tile's
// block -- the other group's -- so a landing is always in flight behind the
// two groups' transforms, where the one-tile CTA waits for its block with
// nothing to do (20 % of its stall samples).  Same arithmetic and thread map
// per tile as the one-tile kernel.
struct GroupBar {
    int id, n;
    __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
};

// NG groups of 4T threads (512 threads in all) and NL landing buffers, NG % NL
// == 0: tile i of the CTA belongs to group i % NG and lands in buffer i % NL;
// the group that has just read buffer i % NL requests tile i + NL into it (for
// group (i + NL) % NG), so NL landings are in flight.  4096-wide rows: two
// 256-thread groups and one buffer; 2048-wide rows: four 128-thread groups and
// two buffers.
template <int LOGQ, int NG, int NL>
__global__ void __launch_bounds__(512, 1) k_irfft_rows_p2(double* __restrict__ f, int Nx, int Nrow, int Nz, int dim,
                                                         int Hx, const double2* __restrict__ tw, int logTWN,
                                                         double scale, const uint8_t* __restrict__ cmask,
                                                         const double* __restrict__ body, int64_t nodes,
                                                         const __grid_constant__ CUtensorMap tm, int pf, int blk,
                                                         int64_t ntiles) {
    using Sh = FftShape<LOGQ, 4>;
    constexpr int Q = Sh::Q, T = Sh::T, R = Sh::R;
    constexpr int XB = xbuf_stride_rows(Sh::XBUF);
    constexpr int TR = 2, LOGTR = 1;
    constexpr int GS = 2 * TR * T, LOGGS = Sh::LOGT + 2;  // threads per group (one two-row tile)
    static_assert(GS * NG == 512 && NG % NL == 0, "512 threads in NG groups, NL | NG landing buffers");
    constexpr int halfP = 2 * Q;
    // plain offsets from the array keep the accesses in the shared window (a
    // pointer rounded up through an integer compiles to generic loads / stores)
    extern __shared__ __align__(128) double2 smraw[];
    __shared__ __align__(8) uint64_t full[NG];
    const int g = threadIdx.x >> LOGGS;
    const int tid = threadIdx.x & (GS - 1);
    const GroupBar gbar{1 + g, GS};
    const int nbox = (Hx + 255) / 256;
    if (smem_u32(smraw) & 127u) __trap();  // TMA tensor boxes land on 128-byte boundaries
    const int lsz = nbox * 256 * TR;                          // double2 per landing buffer
    double2* sm = smraw + NL * lsz + g * 2 * TR * XB;         // this group's work area
    const int gi = tid >> Sh::LOGT;
    const int t = tid & (T - 1);
    const int eo = gi & 1;
    const int shX = logTWN - (LOGQ + 2);
    const int shE = logTWN - (LOGQ + 1);
    const int groups = Nrow / TR;
    if (threadIdx.x == 0)
        for (int i = 0; i < NG; ++i) mbar_init(&full[i], 1);
    __syncthreads();
    // tile i of this CTA: blockIdx.x + i * gridDim.x; group g takes i = g, g + NG, ...
    auto request = [&](int64_t tile, int gdst, double2* land) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const int cx0 = blk ? 2 * (row0 & 7) : 2 * row0;
        const int cz0 = blk ? slab * (Nrow >> 3) + (row0 >> 3) : slab;
        mbar_expect_tx(&full[gdst], (unsigned)(nbox * 256 * TR * 16));
        for (int bx = 0; bx < nbox; ++bx) tma_load_3d(&tm, land + bx * 256 * TR, &full[gdst], cx0, bx * 256, cz0);
    };
    auto prefetch = [&](int64_t tile) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const int cx0 = blk ? 2 * (row0 & 7) : 2 * row0;
        const int cz0 = blk ? slab * (Nrow >> 3) + (row0 >> 3) : slab;
        for (int bx = 0; bx < nbox; ++bx) tma_prefetch_3d(&tm, cx0, bx * 256, cz0);
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < NL; ++i)
            if ((int64_t)blockIdx.x + (int64_t)i * gridDim.x < ntiles)
                request((int64_t)blockIdx.x + (int64_t)i * gridDim.x, i % NG, smraw + i * lsz);
    constexpr int LA = 2;
    constexpr int U = R / 2;
    const int rr = (tid >> LA) & (TR - 1);
    const int j0 = ((tid >> (LA + LOGTR)) << LA) + (tid & ((1 << LA) - 1));
    const double2 W0 = twiddle<1>(tw, (2 * j0) << shX);
    const double2 W1 = cmul(W0, twiddle<1>(tw, 1 << shX));
    const double2 wbase = twiddle<1>(tw, t << shE);  // e^{+2 pi i t/(2Qx)}
    unsigned ph = 0;
    const int li = g % NL;  // this group's landing buffer: (g + k * NG) % NL
    for (int64_t tile = (int64_t)blockIdx.x + (int64_t)g * gridDim.x; tile < ntiles; tile += NG * (int64_t)gridDim.x) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        {
            double2* land = smraw + li * lsz;
            double2 Xa[U], Xb[U];
            double2 xq = make_double2(0.0, 0.0);
            mbar_wait(&full[g], ph);
            ph ^= 1;
#pragma unroll
            for (int u = 0; u < U / 2; ++u) {
                const int j = j0 + 2 * T * u;
                const int ke = 2 * j, ko = 2 * j + 1;
                const bool sw = (j >> 1) & 1;
                const double2 a1 = land[(sw ? ko : ke) * TR + rr], a2 = land[(sw ? ke : ko) * TR + rr];
                const double2 b1 = land[(halfP - (sw ? ko : ke)) * TR + rr], b2 = land[(halfP - (sw ? ke : ko)) * TR + rr];
                Xa[u] = sw ? a2 : a1;
                Xa[u + U / 2] = sw ? a1 : a2;
                Xb[u] = sw ? b2 : b1;
                Xb[u + U / 2] = sw ? b1 : b2;
            }
            if (tid < TR) xq = land[Q * TR + tid];
            gbar();  // the block is in this group's registers: the buffer takes the tile NL further on
            if (tid == 0) {
                const int64_t nxt = tile + NL * (int64_t)gridDim.x;
                if (nxt < ntiles) request(nxt, (g + NL) % NG, land);
                if (pf && nxt + (int64_t)pf * gridDim.x < ntiles) prefetch(nxt + (int64_t)pf * gridDim.x);
            }
            double2* E = sm + 2 * rr * XB;
            double2* O = E + XB;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + 2 * T * u;
                const bool even = j < Q / 2;
                const double2 W = 2 * T * u < Q / 2 ? tw32r<1>(u * (32 / R), W0) : tw32r<1>(u * (32 / R) - 8, W1);
                const double2 a = Xa[u], bb = Xb[u];
                const double2 s1 = cadd(a, cconj(bb));
                const double2 t1 = cmul(W, csub(a, cconj(bb)));
                const double2 W2 = make_double2(-W.x, W.y);  // e^{+2 pi i (halfP-k)/Px}
                const double2 s2 = cadd(bb, cconj(a));
                const double2 t2 = cmul(W2, csub(bb, cconj(a)));
                const double2 Zk = make_double2(s1.x - t1.y, s1.y + t1.x);
                const double2 Zm = make_double2(s2.x - t2.y, s2.y + t2.x);
                if (even) {
                    E[spad(j)] = Zk;
                    if (j != 0) E[spad(Q - j)] = Zm;
                } else {
                    const int jo = j - Q / 2;
                    O[spad(jo)] = Zk;
                    O[spad(Q - 1 - jo)] = Zm;
                }
            }
            if (tid < TR) {  // Nyquist k = Q (self-paired, W = i) -> E[Q/2]
                const double2 s1 = cadd(xq, cconj(xq));
                const double2 t1 = cmul(make_double2(0.0, 1.0), csub(xq, cconj(xq)));
                sm[2 * tid * XB + (Q & 1) * XB + spad(Q >> 1)] = make_double2(s1.x - t1.y, s1.y + t1.x);
            }
        }
        gbar();
        double2* xb = sm + gi * XB;
        double2 v[R];
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = xb[spad(t + j * T)];
        gbar();
        reg_fft<LOGQ, 4, 1>(v, t, xb, make_fft_tw<LOGQ, 4>(t, tw, logTWN), gbar);
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int n = t + j * T;
            xb[spad(n)] = eo ? cmul(tw32r<1>(j * (16 / R), wbase), v[j]) : v[j];
        }
        gbar();
        const int a = (slab / Nz) % dim;
        const int z = slab % Nz;
        double* dst = f + ((int64_t)slab * Nrow + row0) * Nx;
        auto emit = [&](int r2, int n, double2 zz) {
            const int i0 = 2 * n;
            double v0 = zz.x * scale, v1 = zz.y * scale;
            const int64_t node = ((int64_t)z * Nrow + row0 + r2) * Nx + i0;
            if (body) {
                v0 += body[(int64_t)a * nodes + node];
                v1 += body[(int64_t)a * nodes + node + 1];
            }
            if (cmask) {
                if ((cmask[node] >> a) & 1u) v0 = 0.0;
                if ((cmask[node + 1] >> a) & 1u) v1 = 0.0;
            }
            *reinterpret_cast<double2*>(dst + (int64_t)r2 * Nx + i0) = make_double2(v0, v1);
        };
#pragma unroll 4
        for (int u = 0; u < R / 2; ++u) {
            const int idx = tid + u * 2 * TR * T;
            const int r2 = idx >> LOGQ, m = idx & (Q - 1);
            const double2 ze = sm[2 * r2 * XB + spad(m)];
            const double2 zo = sm[(2 * r2 + 1) * XB + spad(m)];
            emit(r2, m, cadd(ze, zo));
            emit(r2, m + Q, csub(ze, zo));
        }
        gbar();  // the work area is read: the next tile's spectra may overwrite it
    }
}

// ------------------------------------------------------------------ K3 ---
// Columns in[((b*D + c)*ncols + col)*Nl + n], n < Nl, zero-padded to Pl = 2Ql.
// Half h (ky = 2k + h): U_c = FFT_Ql(x_c[n] e^{-2 pi i h n/Pl}); F_a = sum_c
// H[col][h][k][pair(a,c)] U_c; z_a^h = IFFT_Ql(F_a);  y_a[n] = z_a^0[n] +
// e^{+2 pi i n/Pl} z_a^1[n].  z^0 is parked in SMEM (thread-private slots).
// NH = 1 (periodic column, Pl = Ql = Nl): one pass, no pre-twiddle, no park.
template <int D>
__device__ __forceinline__ int pair_of(int a, int b) {
    if (a > b) {
        const int t = a;
        a = b;
        b = t;
    }
    if (D == 2) return a + b;
    return (a == 0 ? 0 : (a == 1 ? 3 : 5)) + b - a;
}

// Only one component's spectrum is live in registers at a time; the other
// d-1 wait in thread-private SMEM slots (`cpark`).  The half-0 result z^0 is
// parked either in SMEM (ZSMEM, small columns; in place allowed) or in `out`
// itself (large 2D columns; `out` must not alias `in`, the second half
// re-reads `in` and read-modify-writes `out`).
template <int D, bool REAL>
__device__ __forceinline__ void symbol_product(double2* F, const double2* U, const void* __restrict__ sym,
                                               int64_t fidx) {
    constexpr int NP = D * (D + 1) / 2;
    if (REAL) {
        double g[NP > 3 ? NP : 4];
        if constexpr (D == 2) {
            // 2D real symbol: 4 doubles per frequency (xx, xy, yy, 0), one 32-byte load
            const double* H = (const double*)sym + fidx * 4;
            asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                : "=d"(g[0]), "=d"(g[1]), "=d"(g[2]), "=d"(g[3])
                : "l"(H));
        } else if constexpr (NP % 2 == 0) {
            // 3D: six doubles per frequency, 48 bytes: three 16-byte loads
            const double2* H2 = reinterpret_cast<const double2*>((const double*)sym + fidx * NP);
#pragma unroll
            for (int p = 0; p < NP / 2; ++p) {
                const double2 h2 = __ldg(H2 + p);
                g[2 * p] = h2.x;
                g[2 * p + 1] = h2.y;
            }
        } else {
            const double* H = (const double*)sym + fidx * NP;
#pragma unroll
            for (int p = 0; p < NP; ++p) g[p] = __ldg(H + p);
        }
#pragma unroll
        for (int a = 0; a < D; ++a) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const double gg = g[pair_of<D>(a, c)];
                acc.x += gg * U[c].x;
                acc.y += gg * U[c].y;
            }
            F[a] = acc;
        }
    } else {
        const double2* H = (const double2*)sym + fidx * NP;
        double2 g[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) g[p] = __ldg(H + p);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int c = 0; c < D; ++c) acc = cadd(acc, cmul(g[pair_of<D>(a, c)], U[c]));
            F[a] = acc;
        }
    }
}

template <int LOGQ, int D, bool REAL, int LOGR, bool ZSMEM, bool SEP = false, int NH = 2>
__global__ void __launch_bounds__(256, NH == 1 ? 2 : 1) k_spectral(const double2* in, double2* out, const void* __restrict__ sym,
                                                     int ncols, int Nl, int NC, const double2* __restrict__ tw,
                                                     int logTWN, const double* __restrict__ coltab = nullptr,
                                                     int M = 0, int oddmask = 0) {
    using Sh = FftShape<LOGQ, LOGR>;
    constexpr int Q = Sh::Q, T = Sh::T, XB = Sh::XBUF;
    constexpr int RR = Sh::R;
    constexpr int NP = D * (D + 1) / 2;
    extern __shared__ double2 sm[];
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    // batch index fastest in launch order: the CTAs resident together share
    // a column's symbol in L2 instead of re-reading it per vector
    const int col = blockIdx.y * NC + gi;
    const int b = blockIdx.x;
    const bool valid = col < ncols;
    double2* xb = sm + gi * XB;
    // per column: (D-1)*Q component park, then (ZSMEM) D*Q half-0 park
    double2* cpark = sm + NC * XB + (int64_t)gi * (ZSMEM ? 2 * D - 1 : D - 1) * Q;
    double2* zpark = cpark + (D - 1) * Q;
    const int shP = logTWN - (LOGQ + NH - 1);  // Pl = NH * Q
    double2 v[RR];
    const FftTw tws = make_fft_tw<LOGQ, LOGR>(t, tw, logTWN);
    // separable symbol: this column's n_pairs x (M+1) coefficients in SMEM
    const int ND = NP * (M + 1);
    double* dsm = reinterpret_cast<double*>(sm + NC * XB + (int64_t)NC * (ZSMEM ? 2 * D - 1 : D - 1) * Q) + gi * ND;
    if (SEP)
        for (int i = t; i < ND; i += T) dsm[i] = valid ? __ldg(coltab + (int64_t)col * ND + i) : 0.0;
#pragma unroll 1
    for (int h = 0; h < NH; ++h) {
#pragma unroll 1
        for (int c = 0; c < D; ++c) {
            const double2* src = in + ((int64_t)(b * D + c) * ncols + col) * Nl;
#pragma unroll
            for (int j = 0; j < RR; ++j) {
                const int n = t + j * T;
                double2 x = make_double2(0.0, 0.0);
                if (valid && n < Nl) x = src[n];
                v[j] = h ? cmul(x, __ldg(tw + (n << shP))) : x;
            }
            reg_fft<LOGQ, LOGR, -1>(v, t, xb, tws, BlockBar{});
            if (c < D - 1) {
#pragma unroll
                for (int j = 0; j < RR; ++j) cpark[c * Q + j * T + t] = v[j];
            }
        }
        // per-frequency d x d product (ky = 2k + h); last component in v
        const int64_t sbase = ((int64_t)(valid ? col : 0) * NH + h) * Q;
        // e^{+2 pi i kz/Pl} for kz = 2(t + jT) + h: base(t, h) * e^{2 pi i j/RR}
        const double2 eh = SEP ? cconj(__ldg(tw + ((NH * t + h) << shP))) : make_double2(1.0, 0.0);
#pragma unroll
        for (int j = 0; j < RR; ++j) {
            const int k = t + j * T;
            double2 U[D], F[D];
#pragma unroll
            for (int c = 0; c < D - 1; ++c) U[c] = cpark[c * Q + j * T + t];
            U[D - 1] = v[j];
            if (SEP) {
                const double2 e = tw32r<1>(j * (32 / RR), eh);
                double g[NP];
#pragma unroll
                for (int p = 0; p < NP; ++p) g[p] = dsm[p * (M + 1)];
                double2 em = e;
                for (int m = 1; m <= M; ++m) {
#pragma unroll
                    for (int p = 0; p < NP; ++p) g[p] += dsm[p * (M + 1) + m] * (((oddmask >> p) & 1) ? em.y : em.x);
                    em = cmul(em, e);
                }
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        const double gg = g[pair_of<D>(a, c)];
                        acc.x += gg * U[c].x;
                        acc.y += gg * U[c].y;
                    }
                    F[a] = acc;
                }
            } else {
                symbol_product<D, REAL>(F, U, sym, sbase + k);
            }
#pragma unroll
            for (int a = 0; a < D - 1; ++a) cpark[a * Q + j * T + t] = F[a];
            v[j] = F[D - 1];
        }
#pragma unroll 1
        for (int ai = 0; ai < D; ++ai) {
            const int a = D - 1 - ai;  // the component already in registers first
            if (ai > 0) {
#pragma unroll
                for (int j = 0; j < RR; ++j) v[j] = cpark[a * Q + j * T + t];
            }
            reg_fft<LOGQ, LOGR, 1>(v, t, xb, tws, BlockBar{});
            double2* dst = out + ((int64_t)(b * D + a) * ncols + col) * Nl;
#pragma unroll
            for (int j = 0; j < RR; ++j) {
                const int n = t + j * T;
                if (ZSMEM) {
                    double2* zp = zpark + a * Q + j * T + t;
                    if (h == 0) *zp = v[j];
                    else if (valid && n < Nl) dst[n] = cadd(*zp, cmul(twiddle<1>(tw, n << shP), v[j]));
                } else if (valid && n < Nl) {
                    if (h == 0) dst[n] = v[j];
                    else dst[n] = cadd(dst[n], cmul(twiddle<1>(tw, n << shP), v[j]));
                }
            }
        }
    }
}

// ------------------------------------------------------ K3, pipelined ---
// 2D spectral pass as a persistent kernel: each CTA walks (vector, column)
// items in vector-fastest order, one column group of NC columns per item
// (NC*T = 256 threads).  Every global operand of the six FFTs of an item
// (x_0, x_1 for both halves, then z^0_1, z^0_0 for the read-modify-write of
// the second half) is fetched with cp.async into a staging buffer one FFT
// ahead of its use, so HBM/L2 latency hides behind the previous transform.

// ------------------------------------------------------ K1, pipelined ---
// Persistent x-forward pass: each CTA walks (slab, row-group) tiles; the next
// tile's TR rows of reals land in a staging buffer via cp.async while the
// current tile is transformed and written, so HBM latency overlaps compute.
// Requires even Nx (16-byte row alignment); the plain kernel covers the rest.
template <int LOGQ, int LOGTR, bool CIRC>
__global__ void __launch_bounds__(512, 1) k_rfft_rows_pipe(const double* __restrict__ u, double2* __restrict__ S,
                                                           int Nx, int Nrow, int nslab, int Hx,
                                                           const double2* __restrict__ tw, int logTWN,
                                                           double* __restrict__ xstrip, int M, int Nz) {
    pdl_entry();
    using Sh = FftShape<LOGQ, 4>;
    constexpr int Q = Sh::Q, T = Sh::T, R = Sh::R, XB = xbuf_stride_t(Sh::XBUF, Sh::T);
    constexpr int TR = 1 << LOGTR;
    extern __shared__ double2 sm[];
    double* stage = reinterpret_cast<double*>(sm + 2 * TR * XB);  // TR rows x rowlen reals
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    const int r = gi >> 1, eo = gi & 1;
    const int shE = logTWN - (LOGQ + 1);
    const int shX = logTWN - (LOGQ + 2);
    constexpr int halfP = 2 * Q;
    const double2 wbase = __ldg(tw + (t << shE));
    const FftTw tws = make_fft_tw<LOGQ, 4>(t, tw, logTWN);
    const int groups = (Nrow + TR - 1) / TR;
    const int64_t ntiles = (int64_t)groups * nslab;
    const int rowlen = CIRC ? 4 * Q : 2 * Q;  // staged doubles per row (>= Nx)
    auto fetch = [&](int64_t tile) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const int nr = min(TR, Nrow - row0);
        const double* src = u + ((int64_t)slab * Nrow + row0) * Nx;
        const int chunks_per_row = rowlen / 2;
        for (int c = threadIdx.x; c < TR * chunks_per_row; c += blockDim.x) {
            const int rr = c / chunks_per_row, i0 = 2 * (c - rr * chunks_per_row);
            const bool p = rr < nr && i0 < Nx;
            cp_async16(stage + rr * rowlen + i0, p ? src + (int64_t)rr * Nx + i0 : src, p);
        }
        cp_async_commit();
    };
    // Post-processing items (a, rr): one thread makes X[2a] (from E[a], E[Q-a])
    // and X[2a+1] (from O[a], O[Q-1-a]), a = a0 + 2T*u, plus X[halfP] for
    // a0 == 0.  Thread i -> a0 = 8*(i >> (3+LOGTR)) + (i & 7), rr = (i >> 3) &
    // (TR-1): each quarter-warp reads 8 consecutive slots of one buffer
    // (distinct banks for the 16-byte loads) and each warp store still fills
    // whole 32-byte sectors along rr.  W(2a) = e^{-2 pi i 2a/Px} =
    // W(2a0) e^{-2 pi i u/R}: two table reads per thread, hoisted.
    constexpr int LA = (2 * T >= 8) ? 3 : 0;  // tiny transforms: rr fastest
    const int rr = (threadIdx.x >> LA) & (TR - 1);
    const int a0 = ((threadIdx.x >> (LA + LOGTR)) << LA) + (threadIdx.x & ((1 << LA) - 1));
    const double2 W0 = __ldg(tw + ((2 * a0) << shX));
    const double2 W1 = cmul(W0, __ldg(tw + (1 << shX)));  // W(2a0 + 1)
    int64_t tile = blockIdx.x;
    if (tile < ntiles) fetch(tile);
    for (; tile < ntiles; tile += gridDim.x) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const int nr = min(TR, Nrow - row0);
        double2* xb = sm + gi * XB;
        double2 v[R];
        cp_async_wait_all();
        __syncthreads();
        if (xstrip) {
            // 3D: the 2M-wide row ends into the x-face strip [b][c][slot][z][y]
            // (slot x, or 2M + x - (Nx - 2M)) for the wrap correction's x pass
            const int S4 = 4 * M, bc = slab / Nz, z = slab - bc * Nz;
            for (int idx = threadIdx.x; idx < nr * S4; idx += blockDim.x) {
                const int rr2 = idx / S4, sl = idx - rr2 * S4;
                const int x = sl < 2 * M ? sl : Nx - 4 * M + sl;
                xstrip[(((int64_t)bc * S4 + sl) * Nz + z) * Nrow + row0 + rr2] = stage[rr2 * rowlen + x];
            }
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int n = t + j * T;
            double2 z = *reinterpret_cast<const double2*>(stage + r * rowlen + 2 * n);
            if (CIRC) {  // decimation in frequency (see k_rfft_rows)
                const double2 z2 = *reinterpret_cast<const double2*>(stage + r * rowlen + 2 * (n + Q));
                z = eo ? csub(z, z2) : cadd(z, z2);
            }
            v[j] = eo ? cmul(z, tw32r<-1>(j * (16 / R), wbase)) : z;
        }
        __syncthreads();
        if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);
        reg_fft<LOGQ, 4, -1>(v, t, xb, tws, BlockBar{});
#pragma unroll
        for (int j = 0; j < R; ++j) xb[nat_slot<T>(t, j)] = v[j];
        __syncthreads();
        // X[kx] = Fe + e^{-2 pi i kx/Px} Fo, Fe/Fo from Z[k], conj Z[halfP-k] (items: see top)
        const double2* E = sm + 2 * rr * XB;
        const double2* O = E + XB;
        double2* dst = S + (int64_t)slab * Hx * Nrow + row0 + rr;
        const bool live = rr < nr;
#pragma unroll 4
        for (int u = 0; u < R / 2; ++u) {
            const int a = a0 + 2 * T * u;
            // kx = 2a: A = E[a], B = conj Z[halfP - 2a] = conj E[(Q - a) mod Q]
            // kx = 2a+1: A = O[a], B = conj Z[halfP - 2a - 1] = conj O[Q - 1 - a]
            const double2 Ae = E[spad(a)];
            const double2 Be = cconj(E[spad((Q - a) & (Q - 1))]);
            const double2 Ao = O[spad(a)];
            const double2 Bo = cconj(O[spad(Q - 1 - a)]);
            {
                const double2 Fe = cscale(cadd(Ae, Be), 0.5);
                const double2 D = csub(Ae, Be);
                const double2 Fo = make_double2(0.5 * D.y, -0.5 * D.x);
                if (live) dst[(int64_t)(2 * a) * Nrow] = cadd(Fe, cmul(tw32r<-1>(u * (32 / R), W0), Fo));
            }
            {
                const double2 Fe = cscale(cadd(Ao, Bo), 0.5);
                const double2 D = csub(Ao, Bo);
                const double2 Fo = make_double2(0.5 * D.y, -0.5 * D.x);
                if (live) dst[(int64_t)(2 * a + 1) * Nrow] = cadd(Fe, cmul(tw32r<-1>(u * (32 / R), W1), Fo));
            }
        }
        if (a0 == 0 && live) {  // Nyquist: X[halfP] = Re Z0 - Im Z0 (k = k2 = 0)
            const double2 A = E[0];
            dst[(int64_t)halfP * Nrow] = make_double2(A.x - A.y, 0.0);
        }
        __syncthreads();  // xb reused by the next tile's exchanges
    }
    cp_async_wait_all();
}

// ------------------------------------------------- K1, two CTAs per SM ---
// Same transform and store pattern as k_rfft_rows_pipe with two rows per
// tile, sized for two co-resident CTAs per SM (256 threads, <= 128
// registers, ~104 KB SMEM each): the FFT exchanges use 8-byte slots (split
// real/imaginary), and one buffer per row serves first as the cp.async
// staging area of the input row and then as the natural-order spectrum the
// R2C post-processing reads.  The next tile's rows are fetched after the
// post-processing; its latency is covered by the other CTA on the SM.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, const void* src, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
                 "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
                 : "memory");
}

// K1 duo row buffers: max(two exchange buffers, staged row) doubles, rounded
// up to 8 mod 16 doubles so consecutive rows sit 64 bytes apart in the banks
// CFM (TSTORE tiles): 0 the plain stride; 1 rounded to 8 mod 16 doubles
// (rows 64 B apart in the banks) for the conflict-free thread map below.
__host__ __device__ constexpr int k1_duo_row_stride(int XB, int rowlen, int cfm = 0) {
    return (2 * 2 * XB > rowlen ? 2 * 2 * XB : rowlen) +
           (cfm ? ((24 - (2 * 2 * XB > rowlen ? 2 * 2 * XB : rowlen) % 16) % 16) : 0);
}

// TSTORE: the tile's [kx][row] spectrum block is assembled in SMEM (over the
// row buffers, after every spectrum value has been read into registers) and
// written by TMA boxes ({2*TR doubles, 256 kx}, tensor map tm over S) instead of
// per-thread scattered stores.
template <int LOGQ, bool CIRC, bool TSTORE = false, int CFM = 0>
__global__ void __launch_bounds__(256, 2) k_rfft_rows_duo(const double* __restrict__ u, double2* __restrict__ S,
                                                          int Nx, int Nrow, int nslab, int Hx,
                                                          const double2* __restrict__ tw, int logTWN,
                                                          const __grid_constant__ CUtensorMap tm, int pf,
                                                          int early) {
    using Sh = FftShape<LOGQ, 4>;
    constexpr int Q = Sh::Q, T = Sh::T, R = Sh::R, XB = Sh::XBUF;
    constexpr int LOGTR = 11 - LOGQ;  // rows per tile: 2 * TR * T = 256 threads
    constexpr int TR = 1 << LOGTR;
    static_assert(LOGQ >= 4 && LOGQ <= 10, "2048/Q rows of two Q-point transforms per 256-thread CTA");
    extern __shared__ double2 sm[];
    constexpr int rowlen = CIRC ? 4 * Q : 2 * Q;          // staged doubles per row (>= Nx)
    constexpr int RS = k1_duo_row_stride(XB, rowlen, CFM);  // doubles per row buffer
    constexpr bool CF = TSTORE && CFM == 1;  // conflict-free [kx][row] block writes
    double* rowbuf = reinterpret_cast<double*>(sm);        // TR x RS doubles
    double* xd = rowbuf + TR * RS;                          // 2*TR transforms x XB doubles
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    const int r = gi >> 1, eo = gi & 1;
    const int shE = logTWN - (LOGQ + 1);
    const int shX = logTWN - (LOGQ + 2);
    constexpr int halfP = 2 * Q;
    const int groups = (Nrow + TR - 1) / TR;
    const int64_t ntiles = (int64_t)groups * nslab;
    // rows exactly fill the staging length (periodic, or padded power-of-two
    // rows): one TMA bulk copy per row, else per-thread cp.async with zero fill
    const bool bulk = Nx == rowlen;
    __shared__ __align__(8) uint64_t bar, bar0;
    __shared__ double2 stw[FftTwTable<LOGQ, 4>::SIZE];
    fill_fft_tw_table<LOGQ, 4>(stw, tw, logTWN);
    if (bulk && threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar0, 1);
    }
    __syncthreads();
    unsigned ph = 0, ph0 = 0;
    // TSTORE tiles with `early`: row 0 of the next tile lands in the exchange
    // buffer (free from the end of the transforms to the next tile's first
    // exchange, and large enough for one row) while this tile is post-processed
    // and stored; only the remaining rows wait for the store to release the row
    // buffers.
    const bool split = TSTORE && early && bulk && rowlen <= 2 * TR * XB;
    auto fetch_row0 = [&](int64_t tile) {
        if (threadIdx.x == 0) {
            const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
            fence_proxy_async();
            mbar_expect_tx(&bar0, (unsigned)(rowlen * 8));
            bulk_load(xd, u + ((int64_t)slab * Nrow + row0) * Nx, rowlen * 8, &bar0);
        }
    };
    auto fetch_rest = [&](int64_t tile) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const int nr = min(TR, Nrow - row0);
        if (threadIdx.x == 0 && nr > 1) {
            const double* src = u + ((int64_t)slab * Nrow + row0) * Nx;
            fence_proxy_async();
            mbar_expect_tx(&bar, (unsigned)((nr - 1) * rowlen * 8));
            for (int rr = 1; rr < nr; ++rr) bulk_load(rowbuf + rr * RS, src + (int64_t)rr * Nx, rowlen * 8, &bar);
        }
    };
    auto fetch = [&](int64_t tile) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const int nr = min(TR, Nrow - row0);
        const double* src = u + ((int64_t)slab * Nrow + row0) * Nx;
        if (bulk) {
            if (threadIdx.x == 0) {
                fence_proxy_async();
                mbar_expect_tx(&bar, (unsigned)(nr * rowlen * 8));
                for (int rr = 0; rr < nr; ++rr) bulk_load(rowbuf + rr * RS, src + (int64_t)rr * Nx, rowlen * 8, &bar);
            }
            return;
        }
        constexpr int chunks_per_row = rowlen / 2;
        for (int c = threadIdx.x; c < TR * chunks_per_row; c += blockDim.x) {
            const int rr = c / chunks_per_row, i0 = 2 * (c - rr * chunks_per_row);
            const bool p = rr < nr && i0 < Nx;
            cp_async16(rowbuf + rr * RS + i0, p ? src + (int64_t)rr * Nx + i0 : u, p);
        }
        cp_async_commit();
    };
    // post-processing thread map: a quarter-warp covers 8 consecutive kx of one
    // row; with TSTORE (two rows) 4 consecutive kx of both rows, so that its
    // [kx][row] block writes land on 8 distinct 16-byte bank groups (below)
    constexpr int LA = CF ? 2 : (2 * T >= 8) ? 3 : 0;
    const int rr = (threadIdx.x >> LA) & (TR - 1);
    const int a0 = ((threadIdx.x >> (LA + LOGTR)) << LA) + (threadIdx.x & ((1 << LA) - 1));
    int64_t tile = blockIdx.x;
    if (tile < ntiles) {
        if (split) {
            fetch_row0(tile);
            fetch_rest(tile);
        } else {
            fetch(tile);
        }
    }
    for (; tile < ntiles; tile += gridDim.x) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const int nr = min(TR, Nrow - row0);
        if (pf && bulk && threadIdx.x == 0 && tile + (int64_t)pf * gridDim.x < ntiles) {
            // the rows this CTA fetches pf tiles later, into L2 now
            const int64_t nt = tile + (int64_t)pf * gridDim.x;
            const int ns = (int)(nt / groups), nr0 = (int)(nt % groups) * TR;
            const int nn = min(TR, Nrow - nr0);
            for (int rr2 = 0; rr2 < nn; ++rr2)
                l2_prefetch(u + ((int64_t)ns * Nrow + nr0 + rr2) * Nx, rowlen * 8);
        }
        double2 v[R];
        if (split) {
            mbar_wait(&bar0, ph0);
            ph0 ^= 1;
            if (nr > 1) {
                mbar_wait(&bar, ph);
                ph ^= 1;
            }
        } else if (bulk) {
            mbar_wait(&bar, ph);  // rows past the lattice (nr < TR) hold stale data: never stored
            ph ^= 1;
        } else {
            cp_async_wait_all();
        }
        __syncthreads();
        {
            const double* st = (split && r == 0) ? xd : rowbuf + r * RS;
            const double2 wbase = __ldg(tw + (opaque(t) << shE));
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int n = t + j * T;
                double2 z = *reinterpret_cast<const double2*>(st + 2 * n);
                if (CIRC) {
                    const double2 z2 = *reinterpret_cast<const double2*>(st + 2 * (n + Q));
                    z = eo ? csub(z, z2) : cadd(z, z2);
                }
                v[j] = eo ? cmul(z, tw32r<-1>(j * (16 / R), wbase)) : z;
            }
        }
        __syncthreads();  // row buffers free: they receive the spectra below
        reg_fft<LOGQ, 4, -1, BlockBar, true>(v, t, reinterpret_cast<double2*>(xd + gi * XB),
                                             make_fft_tw_s<LOGQ, 4>(opaque(t), stw), BlockBar{});
        double2* spec = reinterpret_cast<double2*>(rowbuf + r * RS) + eo * XB;
#pragma unroll
        for (int j = 0; j < R; ++j) spec[nat_slot<T>(t, j)] = v[j];
        __syncthreads();
        if (split && tile + gridDim.x < ntiles) fetch_row0(tile + gridDim.x);
        const double2* E = reinterpret_cast<const double2*>(rowbuf + rr * RS);
        const double2* O = E + XB;
        double2* dst = S + (int64_t)slab * Hx * Nrow + row0 + rr;
        const bool live = rr < nr;
        const double2 W0 = __ldg(tw + ((2 * opaque(a0)) << shX));
        const double2 W1 = cmul(W0, __ldg(tw + (1 << shX)));
        // Mirrored pairs share their two SMEM reads: X[2a] and X[2Q-2a] both come
        // from E[a], E[Q-a]; X[2a+1] and X[2Q-2a-1] from O[a], O[Q-1-a]; the
        // mirrored twiddle is e^{-2 pi i (2Q-k)/Px} = -conj(e^{-2 pi i k/Px}).
        auto post = [](double2 A, double2 B, double2 W) {
            const double2 Fe = cscale(cadd(A, B), 0.5);
            const double2 D = csub(A, B);
            return cadd(Fe, cmul(W, make_double2(0.5 * D.y, -0.5 * D.x)));
        };
        if constexpr (TSTORE) {
            constexpr int NU = R / 4;
            double2 e1[NU], e2[NU], o1[NU], o2[NU];
#pragma unroll
            for (int uu = 0; uu < NU; ++uu) {
                const int a = a0 + 2 * T * uu;
                e1[uu] = E[spad(a)];
                e2[uu] = E[spad((Q - a) & (Q - 1))];
                o1[uu] = O[spad(a)];
                o2[uu] = O[spad(Q - 1 - a)];
            }
            const double2 Aq = E[spad(Q / 2)];
            __syncthreads();  // every spectrum value is in registers: the block overwrites them
            double2* ob = sm + ((128u - (smem_u32(sm) & 127u)) & 127u) / 16u;  // shared-window offset, 128-byte aligned
#pragma unroll
            for (int uu = 0; uu < NU; ++uu) {
                const int a = a0 + 2 * T * uu;
                const double2 We = tw32r<-1>(uu * (32 / R), W0), Wo = tw32r<-1>(uu * (32 / R), W1);
                const double2 Wem = make_double2(-We.x, We.y), Wom = make_double2(-Wo.x, Wo.y);
                const double2 xe = post(e1[uu], cconj(e2[uu]), We), xem = post(e2[uu], cconj(e1[uu]), Wem);
                const double2 xo = post(o1[uu], cconj(o2[uu]), Wo), xom = post(o2[uu], cconj(o1[uu]), Wom);
                // kx pairs (2a, 2a+1) and (2Q-2a, 2Q-2a-1) are 64 contiguous bytes
                // of the block; threads with a bit 1 set store them in the other
                // order, so each store instruction of a quarter-warp (a..a+3, two
                // rows) covers all eight 16-byte slots of a 128-byte bank line
                const bool sw = CF && ((a >> 1) & 1);
                ob[(2 * a + sw) * TR + rr] = sw ? xo : xe;
                ob[(2 * a + 1 - sw) * TR + rr] = sw ? xe : xo;
                ob[(2 * Q - 2 * a - sw) * TR + rr] = sw ? xom : xem;
                ob[(2 * Q - 2 * a - 1 + sw) * TR + rr] = sw ? xem : xom;
            }
            if (a0 == 0) ob[Q * TR + rr] = post(Aq, cconj(Aq), make_double2(0.0, -1.0));
            fence_proxy_async();
            __syncthreads();
            if (threadIdx.x == 0) {
                const int nbox = (Hx + 255) / 256;
                for (int bx = 0; bx < nbox; ++bx) tma_store_3d(&tm, ob + bx * 256 * TR, 2 * row0, bx * 256, slab);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                // the block region takes the next tile's rows: wait until the stores have read it
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncthreads();
            if (tile + gridDim.x < ntiles) {
                if (split) fetch_rest(tile + gridDim.x);
                else fetch(tile + gridDim.x);
            }
            continue;
        }
#pragma unroll 2
        for (int uu = 0; uu < R / 4; ++uu) {
            const int a = a0 + 2 * T * uu;  // a < Q/2
            const double2 e1 = E[spad(a)], e2 = E[spad((Q - a) & (Q - 1))];
            const double2 o1 = O[spad(a)], o2 = O[spad(Q - 1 - a)];
            const double2 We = tw32r<-1>(uu * (32 / R), W0), Wo = tw32r<-1>(uu * (32 / R), W1);
            const double2 Wem = make_double2(-We.x, We.y), Wom = make_double2(-Wo.x, Wo.y);
            if (live) {
                dst[(int64_t)(2 * a) * Nrow] = post(e1, cconj(e2), We);
                dst[(int64_t)(2 * Q - 2 * a) * Nrow] = post(e2, cconj(e1), Wem);  // a = 0: Nyquist
                dst[(int64_t)(2 * a + 1) * Nrow] = post(o1, cconj(o2), Wo);
                dst[(int64_t)(2 * Q - 2 * a - 1) * Nrow] = post(o2, cconj(o1), Wom);
            }
        }
        if (a0 == 0 && live) {  // kx = Q (a = Q/2, self-paired), W = e^{-i pi/2}
            const double2 A = E[spad(Q / 2)];
            dst[(int64_t)Q * Nrow] = post(A, cconj(A), make_double2(0.0, -1.0));
        }
        __syncthreads();  // spectra read: the buffers take the next tile's rows
        if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);
    }
    cp_async_wait_all();
    if (TSTORE && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------- K1, persistent, two row groups ---
// k_rfft_rows_duo<10, true, true> (periodic 4096-wide rows, two rows per tile,
// TMA-stored [kx][2 rows] blocks) as one persistent 512-thread CTA per SM made
// of two 256-thread groups (k_irfft_rows_p2 is the inverse pass built the same
// way).  The two rows of a tile land in a buffer the groups share; a group
// has them in registers within a few hundred cycles and then requests the
// other group's next tile, so a landing is always in flight behind the
// transforms.  Each group's work area serves in turn as FFT exchange buffer,
// natural-order spectra and the [kx][row] block the TMA store reads; the wait
// for that store's read sits at the top of the group's next tile, behind the
// other group's work.  Same arithmetic and thread map per tile as the duo kernel.
// CF: the conflict-free [kx][row] block-write map of k_rfft_rows_duo<.., CFM = 1>.
// NG groups of 4T threads and NL landing buffers as in k_irfft_rows_p2 (4096-
// wide rows: 2 x 256 threads, one buffer; 2048-wide: 4 x 128 threads, two
// buffers); the block leaves in NBOX TMA boxes of BOXK kx (2049 = 9 boxes of
// 256, the last one clipped by the tensor map; 1025 = 4 boxes of 256 and the
// Nyquist kx by plain stores).
template <int LOGQ, bool CF, int NG, int NL, int BOXK, int NBOX>
__global__ void __launch_bounds__(512, 1) k_rfft_rows_p2(const double* __restrict__ u, double2* __restrict__ S, int Nx,
                                                        int Nrow, int Hx,
                                                        const double2* __restrict__ tw, int logTWN,
                                                        const __grid_constant__ CUtensorMap tm, int64_t ntiles) {
    using Sh = FftShape<LOGQ, 4>;
    constexpr int Q = Sh::Q, T = Sh::T, R = Sh::R, XB = Sh::XBUF;
    constexpr int TR = 2, LOGTR = 1;
    constexpr int GS = 2 * TR * T, LOGGS = Sh::LOGT + 2;  // threads per group (one two-row tile)
    static_assert(GS * NG == 512 && NG % NL == 0, "512 threads in NG groups, NL | NG landing buffers");
    constexpr int rowlen = 4 * Q;                       // doubles per row (= Nx)
    constexpr int RS = k1_duo_row_stride(XB, rowlen, CF ? 1 : 0);   // doubles per row of spectra (E | O)
    constexpr int WK = ((TR * RS * 8 > NBOX * BOXK * TR * 16 ? TR * RS * 8 : NBOX * BOXK * TR * 16) + 127) / 128 * 128;
    static_assert(2 * TR * XB * 16 <= WK, "four 16-byte-slot exchange buffers per work area");
    static_assert((TR * rowlen * 8) % 128 == 0, "landing buffers keep the work areas 128-byte aligned");
    // plain offsets from the array keep the accesses in the shared window (a
    // pointer rounded up through an integer compiles to generic loads / stores)
    extern __shared__ __align__(128) double2 smraw[];
    __shared__ __align__(8) uint64_t full[NG];
    __shared__ double2 stw[FftTwTable<LOGQ, 4>::SIZE];
    const int g = threadIdx.x >> LOGGS;
    const int tid = threadIdx.x & (GS - 1);
    const GroupBar gbar{1 + g, GS};
    if (smem_u32(smraw) & 127u) __trap();  // the TMA store reads its boxes from 128-byte boundaries
    double* lands = reinterpret_cast<double*>(smraw);                                   // NL x TR x rowlen doubles
    double* wk = reinterpret_cast<double*>(smraw) + NL * TR * rowlen + g * (WK / 8);    // this group's work area
    const int gi = tid >> Sh::LOGT;
    const int t = tid & (T - 1);
    const int r = gi >> 1, eo = gi & 1;
    const int shE = logTWN - (LOGQ + 1);
    const int shX = logTWN - (LOGQ + 2);
    const int groups = Nrow / TR;
    fill_fft_tw_table<LOGQ, 4>(stw, tw, logTWN);
    if (threadIdx.x == 0)
        for (int i = 0; i < NG; ++i) mbar_init(&full[i], 1);
    __syncthreads();
    auto request = [&](int64_t tile, int gdst, double* land) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const double* src = u + ((int64_t)slab * Nrow + row0) * Nx;
        mbar_expect_tx(&full[gdst], (unsigned)(TR * rowlen * 8));
        for (int rr = 0; rr < TR; ++rr)
            bulk_load(land + rr * rowlen, src + (int64_t)rr * Nx, rowlen * 8, &full[gdst]);
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < NL; ++i)
            if ((int64_t)blockIdx.x + (int64_t)i * gridDim.x < ntiles)
                request((int64_t)blockIdx.x + (int64_t)i * gridDim.x, i % NG, lands + i * TR * rowlen);
    constexpr int LA = CF ? 2 : 3;
    const int rr = (tid >> LA) & (TR - 1);
    const int a0 = ((tid >> (LA + LOGTR)) << LA) + (tid & ((1 << LA) - 1));
    const double2 wbase = __ldg(tw + (opaque(t) << shE));
    auto post = [](double2 A, double2 B, double2 W) {
        const double2 Fe = cscale(cadd(A, B), 0.5);
        const double2 D = csub(A, B);
        return cadd(Fe, cmul(W, make_double2(0.5 * D.y, -0.5 * D.x)));
    };
    unsigned ph = 0;
    double* land = lands + (g % NL) * TR * rowlen;  // this group's landing buffer: (g + k * NG) % NL
    for (int64_t tile = (int64_t)blockIdx.x + (int64_t)g * gridDim.x; tile < ntiles; tile += NG * (int64_t)gridDim.x) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        double2 v[R];
        mbar_wait(&full[g], ph);
        ph ^= 1;
        {
            const double* st = land + r * rowlen;
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int n = t + j * T;
                const double2 z = *reinterpret_cast<const double2*>(st + 2 * n);
                const double2 z2 = *reinterpret_cast<const double2*>(st + 2 * (n + Q));
                const double2 zz = eo ? csub(z, z2) : cadd(z, z2);
                v[j] = eo ? cmul(zz, tw32r<-1>(j * (16 / R), wbase)) : zz;
            }
        }
        // this group's previous block has been read by its TMA store: the work area is free
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        gbar();  // the rows are in this group's registers: the landing buffer takes the tile NL further on
        if (tid == 0 && tile + NL * (int64_t)gridDim.x < ntiles) request(tile + NL * (int64_t)gridDim.x, (g + NL) % NG, land);
        // 16-byte exchange slots: the work area holds all four transforms' buffers
        // (the duo kernel needs the split 8-byte exchange to fit two CTAs per SM)
        reg_fft<LOGQ, 4, -1, GroupBar, false>(v, t, reinterpret_cast<double2*>(wk) + gi * XB,
                                              make_fft_tw_s<LOGQ, 4>(opaque(t), stw), gbar);
        double2* spec = reinterpret_cast<double2*>(wk + r * RS) + eo * XB;
#pragma unroll
        for (int j = 0; j < R; ++j) spec[nat_slot<T>(t, j)] = v[j];
        gbar();
        const double2* E = reinterpret_cast<const double2*>(wk + rr * RS);
        const double2* O = E + XB;
        const double2 W0 = __ldg(tw + ((2 * opaque(a0)) << shX));
        const double2 W1 = cmul(W0, __ldg(tw + (1 << shX)));
        constexpr int NU = R / 4;
        double2 e1[NU], e2[NU], o1[NU], o2[NU];
#pragma unroll
        for (int uu = 0; uu < NU; ++uu) {
            const int a = a0 + 2 * T * uu;
            e1[uu] = E[spad(a)];
            e2[uu] = E[spad((Q - a) & (Q - 1))];
            o1[uu] = O[spad(a)];
            o2[uu] = O[spad(Q - 1 - a)];
        }
        const double2 Aq = E[spad(Q / 2)];
        gbar();  // every spectrum value is in registers: the block overwrites them
        double2* ob = reinterpret_cast<double2*>(wk);
#pragma unroll
        for (int uu = 0; uu < NU; ++uu) {
            const int a = a0 + 2 * T * uu;
            const double2 We = tw32r<-1>(uu * (32 / R), W0), Wo = tw32r<-1>(uu * (32 / R), W1);
            const double2 Wem = make_double2(-We.x, We.y), Wom = make_double2(-Wo.x, Wo.y);
            const double2 xe = post(e1[uu], cconj(e2[uu]), We), xem = post(e2[uu], cconj(e1[uu]), Wem);
            const double2 xo = post(o1[uu], cconj(o2[uu]), Wo), xom = post(o2[uu], cconj(o1[uu]), Wom);
            const bool sw = CF && ((a >> 1) & 1);  // see k_rfft_rows_duo
            ob[(2 * a + sw) * TR + rr] = sw ? xo : xe;
            ob[(2 * a + 1 - sw) * TR + rr] = sw ? xe : xo;
            ob[(2 * Q - 2 * a - sw) * TR + rr] = sw ? xom : xem;
            ob[(2 * Q - 2 * a - 1 + sw) * TR + rr] = sw ? xem : xom;
        }
        if (a0 == 0) ob[Q * TR + rr] = post(Aq, cconj(Aq), make_double2(0.0, -1.0));
        fence_proxy_async();
        gbar();
        if (tid == 0) {
            const int nbox = min(NBOX, (Hx + BOXK - 1) / BOXK);
            for (int bx = 0; bx < nbox; ++bx) tma_store_3d(&tm, ob + bx * BOXK * TR, 2 * row0, bx * BOXK, slab);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        // kx beyond the boxes (a box must start on a 128-byte boundary of the
        // block, so 1025 kx leave as 4 boxes of 256 and this one)
        for (int i = NBOX * BOXK * TR + tid; i < Hx * TR; i += GS)
            S[((int64_t)slab * Hx + i / TR) * Nrow + row0 + (i & (TR - 1))] = ob[i];
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static int k1_p2_smem(int logq, int cfm, int nl, int ng, int boxk, int nbox) {
    const int Q = 1 << logq;
    const int XB = xbuf_slots(logq);
    const int RS = k1_duo_row_stride(XB, 4 * Q, cfm);
    const int wk = (std::max(2 * RS * 8, nbox * boxk * 2 * 16) + 127) / 128 * 128;
    return nl * 2 * 4 * Q * 8 + ng * wk + 128;
}

static int k1_duo_smem(int logq, bool circ, int cfm = 0) {
    const int Q = 1 << logq;
    const int TR = 2048 >> logq;
    const int XB = xbuf_slots(logq);
    const int rowlen = circ ? 4 * Q : 2 * Q;
    const int RS = k1_duo_row_stride(XB, rowlen, cfm);
    // + alignment slack for the TMA-store block (it may run past the row
    // buffers into the exchange buffer, free at that point)
    return (int)sizeof(double) * TR * (RS + 2 * XB) + 128;
}

constexpr int kPipeLogR = 4;  // 16 points per thread: 256 threads per 4096-point column
constexpr int kPipeThreads = 256;

// Symbol modes: 0 complex table, 1 real table (both [col][h][k][pair]),
// 2 separable: for stencils of definite parity per axis (the physical
// kernels, kernel.hpp:109-116) the symbol along the column axis is
// H(ky) = D[0] + sum_{m=1..M} D[m] * (cos|sin)(2 pi ky m / Pl) with per-column
// coefficients D (coltab, O(Hx*M) doubles) -- no O(N) symbol stream.
template <int LOGQ, int SYM>
__global__ void __launch_bounds__(kPipeThreads, 1) k_spectral2d_pipe(const double2* __restrict__ in, double2* out,
                                                            const void* __restrict__ sym,
                                                            const double* __restrict__ coltab, int M, int ncols,
                                                            int Nl, int NC, int batch, const double2* __restrict__ tw,
                                                            int logTWN) {
    using Sh = FftShape<LOGQ, kPipeLogR>;
    constexpr int Q = Sh::Q, T = Sh::T, XB = Sh::XBUF, RR = Sh::R;
    extern __shared__ double2 sm[];
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    double2* xb = sm + gi * XB;
    double2* cpark = sm + NC * XB + gi * Q;        // component 0 park
    double2* stage = sm + NC * XB + NC * Q + gi * Q;  // staging, natural order [j*T + t]
    const int shP = logTWN - (LOGQ + 1);
    const FftTw tws = make_fft_tw<LOGQ, kPipeLogR>(t, tw, logTWN);
    // exp(-2 pi i t/Pl): the half-1 pre-twiddle of n = t + j*T is this times
    // exp(-2 pi i j/(2R)) (compile time); exp(+2 pi i (2t+h)/Pl) seeds the
    // symbol phases of ky = 2(t + j*T) + h.
    const double2 wt = __ldg(tw + (t << shP));
    const double2 eh0 = cconj(__ldg(tw + ((2 * t) << shP)));
    const double2 eh1 = cconj(__ldg(tw + ((2 * t + 1) << shP)));
    const int ND = 3 * (M + 1);
    double* dsm = reinterpret_cast<double*>(sm + NC * XB + 2 * NC * Q) + gi * ND;
    const int ngroups = (ncols + NC - 1) / NC;
    const int64_t nitems = (int64_t)ngroups * batch;
    const int64_t cstride = (int64_t)ncols * Nl;  // component stride

    // stage operand: src column (already offset), n < Nl valid
    auto fetch = [&](const double2* src, bool ok) {
#pragma unroll
        for (int j = 0; j < RR; ++j) {
            const int n = t + j * T;
            const bool p = ok && n < Nl;
            cp_async16(stage + j * T + t, p ? src + n : src, p);
        }
        cp_async_commit();
    };
    auto item_ptrs = [&](int64_t it, int& b, int& col, bool& valid) {
        b = (int)(it % batch);
        col = (int)(it / batch) * NC + gi;
        valid = col < ncols;
    };

    int64_t it = blockIdx.x;
    if (it < nitems) {
        int b, col;
        bool valid;
        item_ptrs(it, b, col, valid);
        fetch(in + ((int64_t)(b * 2 + 0) * ncols + (valid ? col : 0)) * Nl, valid);
    }
    for (; it < nitems; it += gridDim.x) {
        int b, col;
        bool valid;
        item_ptrs(it, b, col, valid);
        const int cc = valid ? col : 0;
        const double2* x0 = in + ((int64_t)(b * 2 + 0) * ncols + cc) * Nl;
        const double2* x1 = x0 + cstride;
        double2* z0 = out + ((int64_t)(b * 2 + 0) * ncols + cc) * Nl;
        double2* z1 = z0 + cstride;
        double2 v[RR];
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                cp_async_wait_all();
                __syncthreads();
                if (h == 0) {
#pragma unroll
                    for (int j = 0; j < RR; ++j) v[j] = stage[j * T + t];
                } else {
#pragma unroll
                    for (int j = 0; j < RR; ++j) v[j] = cmul(stage[j * T + t], tw32r<-1>(j * (16 / RR), wt));
                }
                __syncthreads();
                if (SYM == 2 && h == 0 && c == 0)
                    for (int i = t; i < ND; i += T) dsm[i] = valid ? __ldg(coltab + (int64_t)cc * ND + i) : 0.0;
                // next operand: x1 after x0; after x1 of half 0 -> x0 of half 1;
                // after x1 of half 1 -> z^0_1 for the read-modify-write
                if (c == 0) fetch(x1, valid);
                else if (h == 0) fetch(x0, valid);
                else fetch(z1, valid);
                reg_fft<LOGQ, kPipeLogR, -1>(v, t, xb, tws, BlockBar{});
                if (c == 0) {
#pragma unroll
                    for (int j = 0; j < RR; ++j) cpark[j * T + t] = v[j];
                }
            }
            // 2 x 2 product; component 1 stays in registers
            const int64_t sbase = ((int64_t)cc * 2 + h) * Q;
            const double2 eh = h ? eh1 : eh0;
#pragma unroll
            for (int j = 0; j < RR; ++j) {
                const int k = t + j * T;
                double2 U[2], F[2];
                U[0] = cpark[j * T + t];
                U[1] = v[j];
                if (SYM == 2) {
                    // e = exp(+2 pi i ky / Pl), ky = 2k + h
                    const double2 e = tw32r<1>(j * (32 / RR), eh);
                    double gxx = dsm[0], gyy = dsm[2 * (M + 1)], gxy = dsm[M + 1];
                    double2 em = e;
                    for (int m = 1; m <= M; ++m) {
                        gxx += dsm[m] * em.x;
                        gxy += dsm[(M + 1) + m] * em.y;
                        gyy += dsm[2 * (M + 1) + m] * em.x;
                        em = cmul(em, e);
                    }
                    F[0] = make_double2(gxx * U[0].x + gxy * U[1].x, gxx * U[0].y + gxy * U[1].y);
                    F[1] = make_double2(gxy * U[0].x + gyy * U[1].x, gxy * U[0].y + gyy * U[1].y);
                } else {
                    symbol_product<2, SYM == 1>(F, U, sym, sbase + k);
                }
                cpark[j * T + t] = F[0];
                v[j] = F[1];
            }
#pragma unroll 1
            for (int ai = 0; ai < 2; ++ai) {
                const int a = 1 - ai;
                if (ai == 1) {
#pragma unroll
                    for (int j = 0; j < RR; ++j) v[j] = cpark[j * T + t];
                }
                reg_fft<LOGQ, kPipeLogR, 1>(v, t, xb, tws, BlockBar{});
                double2* dst = a ? z1 : z0;
                if (h == 0) {
#pragma unroll
                    for (int j = 0; j < RR; ++j) {
                        const int n = t + j * T;
                        if (valid && n < Nl) dst[n] = v[j];
                    }
                } else {
                    cp_async_wait_all();
                    __syncthreads();
#pragma unroll
                    for (int j = 0; j < RR; ++j) {
                        const int n = t + j * T;
                        const double2 y = cadd(stage[j * T + t], cmul(tw32r<1>(j * (16 / RR), cconj(wt)), v[j]));
                        if (valid && n < Nl) dst[n] = y;
                    }
                    __syncthreads();
                    if (a == 1) {
                        fetch(z0, valid);
                    } else if (it + gridDim.x < nitems) {
                        int b2, col2;
                        bool valid2;
                        item_ptrs(it + gridDim.x, b2, col2, valid2);
                        fetch(in + ((int64_t)(b2 * 2 + 0) * ncols + (valid2 ? col2 : 0)) * Nl, valid2);
                    }
                }
            }
            if (h == 0) __syncthreads();  // z^0 stores visible before the half-1 re-read
        }
    }
    cp_async_wait_all();
}

// NH = 2: padded column (Pl = 2Q, data on [0, Q)), two half-spectra as above.
// NH = 1: periodic column (Pl = Q = Nl): one forward FFT per component, the
// product, one inverse FFT, stored directly (no z^0 read-modify-write).
// Two-CTA-per-SM variant of the 2D spectral pass: the exchange buffer holds
// 8-byte slots (split real/imaginary exchange) and operands come straight from
// global memory, so a CTA needs NC*(Q*16 + XBUF*8) bytes (~99 KB at Q = 4096)
// and 128 registers per thread.  Two co-resident CTAs overlap each other's
// load / symbol / store phases with FFT work (one CTA per SM leaves them
// exposed).  Same data flow and numerics as k_spectral2d_pipe.
template <int LOGQ, int SYM, int NH>
__global__ void __launch_bounds__(kPipeThreads, 2) k_spectral2d_duo(const double2* __restrict__ in, double2* out,
                                                                   const void* __restrict__ sym,
                                                                   const double* __restrict__ coltab, int M,
                                                                   int ncols, int Nl, int NC, int batch,
                                                                   const double2* __restrict__ tw, int logTWN) {
    pdl_entry();
    using Sh = FftShape<LOGQ, kPipeLogR>;
    constexpr int Q = Sh::Q, T = Sh::T, XB = Sh::XBUF, RR = Sh::R;
    extern __shared__ double2 sm[];
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    double2* park = sm + gi * Q;  // thread-private slots [j*T + t]
    double* xd = reinterpret_cast<double*>(sm + NC * Q);
    double2* xb = reinterpret_cast<double2*>(xd + gi * XB);
    const int ND = 3 * (M + 1);
    double* dsm = xd + NC * XB + gi * ND;
    // x_0 of the next half arrives in the park by a bulk copy (TMA engine)
    // issued while the previous half's last inverse transform runs
    uint64_t* bars = reinterpret_cast<uint64_t*>(xd + NC * XB + (SYM == 2 ? NC * ND : 0));
    const unsigned xbytes = (unsigned)Nl * 16u;
    const int shP = logTWN - (LOGQ + NH - 1);  // Pl = NH * Q
    // register budget (128): twiddle bases are re-read from the (L1-resident)
    // table where they are used, behind opaque indices so they stay there
    const int ngroups = (ncols + NC - 1) / NC;
    const int64_t nitems = (int64_t)ngroups * batch;
    const int64_t cstride = (int64_t)ncols * Nl;
    auto item_x0 = [&](int64_t item, bool& ok) {
        const int bb = (int)(item % batch);
        const int cl = (int)(item / batch) * NC + gi;
        ok = cl < ncols;
        return in + ((int64_t)(bb * 2 + 0) * ncols + (ok ? cl : 0)) * Nl;
    };
    // all threads call this after a CTA barrier (park no longer read)
    auto prefetch = [&](const double2* src, bool ok) {
        if (t == 0 && ok) {
            fence_proxy_async();
            mbar_expect_tx(&bars[gi], xbytes);
            bulk_load(park, src, xbytes, &bars[gi]);
        }
    };
    __shared__ double2 stw[FftTwTable<LOGQ, kPipeLogR>::SIZE];
    fill_fft_tw_table<LOGQ, kPipeLogR>(stw, tw, logTWN);
    if (t == 0) mbar_init(&bars[gi], 1);
    __syncthreads();
    unsigned ph = 0;
    if (blockIdx.x < nitems) {
        bool ok;
        const double2* x = item_x0(blockIdx.x, ok);
        prefetch(x, ok);
    }
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int b = (int)(it % batch);
        const int col = (int)(it / batch) * NC + gi;
        const bool valid = col < ncols;
        const int cc = valid ? col : 0;
        const double2* x0 = in + ((int64_t)(b * 2 + 0) * ncols + cc) * Nl;
        double2* z0 = out + ((int64_t)(b * 2 + 0) * ncols + cc) * Nl;
        if (SYM == 2)
            for (int i = t; i < ND; i += T) dsm[i] = valid ? __ldg(coltab + (int64_t)cc * ND + i) : 0.0;
        double2 v[RR];
#pragma unroll 1
        for (int h = 0; h < NH; ++h) {
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                if (c == 0) {
                    if (valid && t == 0) {
                        // operands of the rest of this half, pulled into L2 behind FFT(x_0):
                        // x_1, this half's symbol rows, and z^0 for the half-1 update
                        l2_prefetch(x0 + cstride, xbytes);
                        if (SYM != 2)
                            l2_prefetch((const char*)sym + (((int64_t)cc * NH + h) * Q) * (SYM == 1 ? 4 * 8 : 3 * 16),
                                        (unsigned)Q * (SYM == 1 ? 4 * 8 : 3 * 16));
                        if (NH == 2 && h) {
                            l2_prefetch(z0, xbytes);
                            l2_prefetch(z0 + cstride, xbytes);
                        }
                    }
                    if (valid) {
                        mbar_wait(&bars[gi], ph);
                        ph ^= 1;
                    }
#pragma unroll
                    for (int j = 0; j < RR; ++j) {
                        const int n = t + j * T;
                        v[j] = (valid && n < Nl) ? park[j * T + t] : make_double2(0.0, 0.0);
                    }
                } else {
                    const double2* src = x0 + cstride;
                    // x_1 is read again for half 1: keep it in L2 until then
                    const uint64_t pol = h == NH - 1 ? l2_policy_evict_first() : l2_policy_evict_last();
#pragma unroll
                    for (int j = 0; j < RR; ++j) {
                        const int n = t + j * T;
                        v[j] = (valid && n < Nl) ? ld_hint(src + n, pol) : make_double2(0.0, 0.0);
                    }
                }
                if (h) {
                    const double2 w = __ldg(tw + (opaque(t) << shP));  // exp(-2 pi i t/Pl)
#pragma unroll
                    for (int j = 0; j < RR; ++j) v[j] = cmul(v[j], tw32r<-1>(j * (16 / RR), w));
                }
                reg_fft<LOGQ, kPipeLogR, -1, BlockBar, true>(v, t, xb, make_fft_tw_s<LOGQ, kPipeLogR>(opaque(t), stw),
                                                             BlockBar{});
                if (c == 0) {
#pragma unroll
                    for (int j = 0; j < RR; ++j) park[j * T + t] = v[j];
                }
            }
            // 2 x 2 product; component 1 stays in registers
            const int64_t sbase = ((int64_t)cc * NH + h) * Q;
            const double2 eh = cconj(__ldg(tw + ((NH * opaque(t) + h) << shP)));  // exp(+2 pi i (NH t+h)/Pl)
#pragma unroll
            for (int j = 0; j < RR; ++j) {
                const int k = t + j * T;
                double2 U[2], F[2];
                U[0] = park[j * T + t];
                U[1] = v[j];
                if (SYM == 2) {
                    const double2 e = tw32r<1>(j * (32 / RR), eh);  // exp(+2 pi i (NH k+h)/Pl)
                    double gxx = dsm[0], gyy = dsm[2 * (M + 1)], gxy = dsm[M + 1];
                    double2 em = e;
                    for (int m = 1; m <= M; ++m) {
                        gxx += dsm[m] * em.x;
                        gxy += dsm[(M + 1) + m] * em.y;
                        gyy += dsm[2 * (M + 1) + m] * em.x;
                        em = cmul(em, e);
                    }
                    F[0] = make_double2(gxx * U[0].x + gxy * U[1].x, gxx * U[0].y + gxy * U[1].y);
                    F[1] = make_double2(gxy * U[0].x + gyy * U[1].x, gxy * U[0].y + gyy * U[1].y);
                } else {
                    symbol_product<2, SYM == 1>(F, U, sym, sbase + k);
                }
                park[j * T + t] = F[0];
                v[j] = F[1];
            }
#pragma unroll 1
            for (int ai = 0; ai < 2; ++ai) {
                const int a = 1 - ai;
                if (ai == 1) {
#pragma unroll
                    for (int j = 0; j < RR; ++j) v[j] = park[j * T + t];
                    __syncthreads();  // park free: fetch the next half's x_0 behind this transform
                    if (h + 1 < NH) {
                        prefetch(x0, valid);
                    } else if (it + gridDim.x < nitems) {
                        bool ok;
                        const double2* x = item_x0(it + gridDim.x, ok);
                        prefetch(x, ok);
                    }
                }
                reg_fft<LOGQ, kPipeLogR, 1, BlockBar, true>(v, t, xb, make_fft_tw_s<LOGQ, kPipeLogR>(opaque(t), stw),
                                                            BlockBar{});
                double2* dst = z0 + a * cstride;
                if (NH == 1) {
                    const uint64_t pol = l2_policy_evict_first();
#pragma unroll
                    for (int j = 0; j < RR; ++j) {
                        const int n = t + j * T;
                        if (valid && n < Nl) st_hint(dst + n, v[j], pol);
                    }
                } else if (h == 0) {
                    const uint64_t pol = l2_policy_evict_last();  // z^0: re-read by this thread in half 1
#pragma unroll
                    for (int j = 0; j < RR; ++j) {
                        const int n = t + j * T;
                        if (valid && n < Nl) st_hint(dst + n, v[j], pol);
                    }
                } else {
                    const uint64_t pol = l2_policy_evict_first();
                    // y = z^0 + exp(+2 pi i n/Pl) z^1; z^0 was stored by this thread
                    const double2 w = cconj(__ldg(tw + (opaque(t) << shP)));
#pragma unroll
                    for (int j = 0; j < RR; ++j) {
                        const int n = t + j * T;
                        if (valid && n < Nl)
                            st_hint(dst + n, cadd(ld_hint_rw(dst + n, pol), cmul(tw32r<1>(j * (16 / RR), w), v[j])), pol);
                    }
                }
            }
        }
    }
}

// ---------------------------------------------- K3, TMEM-parked variant ---
// Tensor memory as thread-private parking space.  A thread owns the 16
// frequencies t + j*T of its column; the other component's spectrum (X0 while
// FFT(x1) runs, then F0 while IFFT(F1) runs) waits in the thread's own TMEM
// lane (32x32b shape: warp w reaches lanes 32*(w%4).., 64 columns of 32 bits
// hold 16 complex values; warps w and w+4 take columns 0 / 64 of the CTA's
// 128-column allocation).  That takes the 64 KB park out of shared memory,
// so the FFT exchanges can use 16-byte slots (half the LDS/STS instructions
// and barriers of the split 8-byte exchange) and two CTAs still fit per SM
// (~74 KB each).  Operands come straight from global memory into registers,
// L2-prefetched one item ahead.  Periodic columns (NH = 1) of 2048 / 4096
// points; same data flow and numerics as k_spectral2d_duo<LOGQ, SYM, 1>.
__device__ __forceinline__ uint32_t dlo(double d) { return (uint32_t)__double2loint(d); }
__device__ __forceinline__ uint32_t dhi(double d) { return (uint32_t)__double2hiint(d); }

// 4 complex values <-> 16 TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_st4(uint32_t ta, const double2* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(ta),
        "r"(dlo(v[0].x)), "r"(dhi(v[0].x)), "r"(dlo(v[0].y)), "r"(dhi(v[0].y)), "r"(dlo(v[1].x)), "r"(dhi(v[1].x)),
        "r"(dlo(v[1].y)), "r"(dhi(v[1].y)), "r"(dlo(v[2].x)), "r"(dhi(v[2].x)), "r"(dlo(v[2].y)), "r"(dhi(v[2].y)),
        "r"(dlo(v[3].x)), "r"(dhi(v[3].x)), "r"(dlo(v[3].y)), "r"(dhi(v[3].y))
        : "memory");
}

struct TmemQuad {
    uint32_t r[16];
};

__device__ __forceinline__ void tmem_ld4(uint32_t ta, TmemQuad& q) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(q.r[0]), "=r"(q.r[1]), "=r"(q.r[2]), "=r"(q.r[3]), "=r"(q.r[4]), "=r"(q.r[5]), "=r"(q.r[6]),
          "=r"(q.r[7]), "=r"(q.r[8]), "=r"(q.r[9]), "=r"(q.r[10]), "=r"(q.r[11]), "=r"(q.r[12]), "=r"(q.r[13]),
          "=r"(q.r[14]), "=r"(q.r[15])
        : "r"(ta)
        : "memory");
}

// wait for every tcgen05.ld of this thread; the registers of q pass through
// the wait so no use of them is scheduled before it
__device__ __forceinline__ void tmem_wait_ld(TmemQuad& q) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(q.r[0]), "+r"(q.r[1]), "+r"(q.r[2]), "+r"(q.r[3]), "+r"(q.r[4]), "+r"(q.r[5]), "+r"(q.r[6]),
                   "+r"(q.r[7]), "+r"(q.r[8]), "+r"(q.r[9]), "+r"(q.r[10]), "+r"(q.r[11]), "+r"(q.r[12]),
                   "+r"(q.r[13]), "+r"(q.r[14]), "+r"(q.r[15])
                 :
                 : "memory");
}

__device__ __forceinline__ void tmem_unpack4(const TmemQuad& q, double2* v) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
        v[i] = make_double2(__hiloint2double((int)q.r[4 * i + 1], (int)q.r[4 * i]),
                            __hiloint2double((int)q.r[4 * i + 3], (int)q.r[4 * i + 2]));
}

// 2 complex values <-> 8 TMEM columns
__device__ __forceinline__ void tmem_st2(uint32_t ta, double2 a, double2 b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(ta),
                 "r"(dlo(a.x)), "r"(dhi(a.x)), "r"(dlo(a.y)), "r"(dhi(a.y)), "r"(dlo(b.x)), "r"(dhi(b.x)),
                 "r"(dlo(b.y)), "r"(dhi(b.y))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld2_wait(uint32_t ta, double2& a, double2& b) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
                 :
                 : "memory");
    a = make_double2(__hiloint2double((int)r[1], (int)r[0]), __hiloint2double((int)r[3], (int)r[2]));
    b = make_double2(__hiloint2double((int)r[5], (int)r[4]), __hiloint2double((int)r[7], (int)r[6]));
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// LAND = false: 16-byte exchange slots (XB * 16 bytes per column), operands
// loaded straight into registers.  LAND = true: x_0 lands by one TMA bulk copy
// in a Q * 16-byte buffer that is free again as soon as the thread has read
// it (the park is in TMEM), so the next item's x_0 is requested a whole item
// ahead; the exchange then uses 8-byte slots (split real/imaginary) to keep
// two CTAs per SM.
template <int LOGQ, int SYM, bool LAND, int CPS = 2>
__global__ void __launch_bounds__(kPipeThreads, CPS) k_spectral2d_tm(const double2* __restrict__ in, double2* out,
                                                                  const void* __restrict__ sym, int ncols, int NC,
                                                                  int batch, const double2* __restrict__ tw,
                                                                  int logTWN) {
    using Sh = FftShape<LOGQ, kPipeLogR>;
    constexpr int Q = Sh::Q, T = Sh::T, XB = Sh::XBUF, RR = Sh::R;
    static_assert(RR == 16 && T % 128 == 0, "16 points per thread, whole TMEM lane quadrants per column");
    extern __shared__ double2 sm[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bars[kPipeThreads / 128];
    __shared__ double2 stw[FftTwTable<LOGQ, kPipeLogR>::SIZE];
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    const int NCc = kPipeThreads / T;
    double2* land = sm + gi * Q;                                                       // LAND only
    double2* xb = LAND ? reinterpret_cast<double2*>(reinterpret_cast<double*>(sm + NCc * Q) + gi * XB)
                       : sm + gi * XB;
    const int warp = threadIdx.x >> 5;
    fill_fft_tw_table<LOGQ, kPipeLogR>(stw, tw, logTWN);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (LAND && t == 0) mbar_init(&bars[gi], 1);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t ta = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    const int ngroups = (ncols + NC - 1) / NC;
    const int64_t nitems = (int64_t)ngroups * batch;
    const int64_t cstride = (int64_t)ncols * Q;
    const uint64_t pol = l2_policy_evict_first();
    constexpr unsigned xbytes = (unsigned)Q * 16u;
    constexpr unsigned sbytes = (unsigned)Q * (SYM == 1 ? 4 * 8 : 3 * 16);
    auto item_col = [&](int64_t item, int& b, int& col) {
        b = (int)(item % batch);
        col = (int)(item / batch) * NC + gi;
        return col < ncols;
    };
    auto x0_of = [&](int b, int col) { return in + ((int64_t)(b * 2) * ncols + col) * Q; };
    // LAND: x_0 of an item into this column's landing buffer (one thread)
    auto land_x0 = [&](int64_t item) {
        int b, col;
        if (t == 0 && item < nitems && item_col(item, b, col)) {
            fence_proxy_async();
            mbar_expect_tx(&bars[gi], xbytes);
            bulk_load(land, x0_of(b, col), xbytes, &bars[gi]);
        }
    };
    if (LAND) land_x0(blockIdx.x);
    unsigned ph = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        int b, col;
        const bool valid = item_col(it, b, col);
        const int cc = valid ? col : 0;
        const double2* x0 = x0_of(b, cc);
        double2* z0 = out + ((int64_t)(b * 2) * ncols + cc) * Q;
        if (valid && t == 0) {
            // x_1 and the symbol rows into L2 behind FFT(x_0)
            l2_prefetch(x0 + cstride, xbytes);
            l2_prefetch((const char*)sym + (int64_t)cc * sbytes, sbytes);
        }
        double2 v[RR];
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
            if (LAND && c == 0) {
                if (valid) {
                    mbar_wait(&bars[gi], ph);
                    ph ^= 1;
                }
#pragma unroll
                for (int j = 0; j < RR; ++j) v[j] = valid ? land[t + j * T] : make_double2(0.0, 0.0);
                __syncthreads();  // landing buffer read by every thread: take the next item's x_0
                land_x0(it + gridDim.x);
            } else {
                const double2* src = x0 + c * cstride;
#pragma unroll
                for (int j = 0; j < RR; ++j) v[j] = valid ? ld_hint(src + t + j * T, pol) : make_double2(0.0, 0.0);
            }
            reg_fft<LOGQ, kPipeLogR, -1, BlockBar, LAND>(v, t, xb, make_fft_tw_s<LOGQ, kPipeLogR>(opaque(t), stw),
                                                         BlockBar{});
            if (c == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q) tmem_st4(ta + 16 * q, v + 4 * q);
                tmem_wait_st();
            }
        }
        // 2 x 2 product, two frequencies per TMEM round trip; F0 replaces X0
        const int64_t sbase = (int64_t)cc * Q;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            double2 x0v[2], f0[2];
            tmem_ld2_wait(ta + 8 * q, x0v[0], x0v[1]);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int j = 2 * q + i;
                double2 U[2], F[2];
                U[0] = x0v[i];
                U[1] = v[j];
                symbol_product<2, SYM == 1>(F, U, sym, sbase + t + j * T);
                f0[i] = F[0];
                v[j] = F[1];
            }
            tmem_st2(ta + 8 * q, f0[0], f0[1]);
        }
        if (!LAND && t == 0) {
            // the next item's x_0 into L2 behind the two inverse transforms (a
            // whole item ahead, 19 MB in flight over the GPU, it was partly
            // evicted again before use: DRAM reads +9 %)
            int b2, col2;
            if (it + gridDim.x < nitems && item_col(it + gridDim.x, b2, col2)) l2_prefetch(x0_of(b2, col2), xbytes);
        }
#pragma unroll 1
        for (int ai = 0; ai < 2; ++ai) {
            const int a = 1 - ai;
            if (ai == 1) {
                tmem_wait_st();
                TmemQuad tq[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) tmem_ld4(ta + 16 * q, tq[q]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    tmem_wait_ld(tq[q]);
                    tmem_unpack4(tq[q], v + 4 * q);
                }
            }
            reg_fft<LOGQ, kPipeLogR, 1, BlockBar, LAND>(v, t, xb, make_fft_tw_s<LOGQ, kPipeLogR>(opaque(t), stw),
                                                        BlockBar{});
            double2* dst = z0 + a * cstride;
            if (valid) {
#pragma unroll
                for (int j = 0; j < RR; ++j) st_hint(dst + t + j * T, v[j], pol);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

// ---------------------------------- K3, TMEM park + landed operands ---
// k_spectral2d_tm<LOGQ, SYM, false> with the operands landed by TMA bulk
// copies in the exchange buffer itself.  Behind the closing barrier of a
// transform's last exchange the buffer is idle while the last pass runs in
// registers: that is when the next operand column is requested (x_1 during
// FFT(x_0), the next item's x_0 during the last inverse transform; XL = 2 also
// the first half of the column's symbol rows during FFT(x_1); XL = 3 the
// column's mirror planes, build_symbol_half, which carry every frequency), so
// its latency sits behind the last pass, the TMEM park and the stores instead
// of in front of a transform.  Costs one SMEM read of the column and one extra
// barrier.
template <int LOGQ, int SYM, int XL>
__global__ void __launch_bounds__(kPipeThreads, 2) k_spectral2d_tx(const double2* __restrict__ in, double2* out,
                                                                 const void* __restrict__ sym, int ncols, int NC,
                                                                 int batch, const double2* __restrict__ tw,
                                                                 int logTWN, const double* __restrict__ symh,
                                                                 int HP, int blk) {
    using Sh = FftShape<LOGQ, kPipeLogR>;
    constexpr int Q = Sh::Q, T = Sh::T, XB = Sh::XBUF, RR = Sh::R;
    static_assert(RR == 16 && T % 32 == 0, "16 points per thread, whole warps (TMEM lane quadrants) per column");
    static_assert(XL == 1 || SYM == 1, "symbol landing: real table only");
    extern __shared__ double2 sm[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bars[kPipeThreads / 32];
    __shared__ double2 stw[FftTwTable<LOGQ, kPipeLogR>::SIZE];
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    double2* xb = sm + gi * XB;
    const int warp = threadIdx.x >> 5;
    fill_fft_tw_table<LOGQ, kPipeLogR>(stw, tw, logTWN);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) mbar_init(&bars[gi], 1);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t ta = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    const int ngroups = (ncols + NC - 1) / NC;
    const int64_t nitems = (int64_t)ngroups * batch;
    const int64_t cstride = (int64_t)ncols * Q;
    const uint64_t pol = l2_policy_evict_first();
    constexpr unsigned xbytes = (unsigned)Q * 16u;
    constexpr unsigned sbytes = (unsigned)Q * (SYM == 1 ? 4 * 8 : 3 * 16);
    auto item_col = [&](int64_t item, int& b, int& col) {
        b = (int)(item % batch);
        col = (int)(item / batch) * NC + gi;
        return col < ncols && gi < NC;  // NC below the CTA's column slots: small lattices, more CTAs
    };
    auto x0_of = [&](int b, int col) { return in + ((int64_t)(b * 2) * ncols + col) * Q; };
    // one column-sized block into this column's exchange buffer (one thread)
    auto land = [&](const void* src, unsigned bytes) {
        if (t == 0) {
            fence_proxy_async();
            mbar_expect_tx(&bars[gi], bytes);
            bulk_load(xb, src, bytes, &bars[gi]);
        }
    };
    unsigned ph = 0;
    auto landed = [&]() {
        mbar_wait(&bars[gi], ph);
        ph ^= 1;
    };
    {
        int b, col;
        if ((int64_t)blockIdx.x < nitems && item_col(blockIdx.x, b, col)) land(x0_of(b, col), xbytes);
    }
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        int b, col;
        const bool valid = item_col(it, b, col);
        const int cc = valid ? col : 0;
        const double2* x0 = x0_of(b, cc);
        double2* z0 = out + ((int64_t)(b * 2) * ncols + cc) * Q;
        int b2, col2;
        const bool nvalid = it + gridDim.x < nitems && item_col(it + gridDim.x, b2, col2);
        if (valid && t == 0) {
            // x_1 and the symbol rows into L2 behind FFT(x_0)
            l2_prefetch(x0 + cstride, xbytes);
            if (XL == 3) l2_prefetch(symh + (int64_t)cc * 3 * HP, (unsigned)(3 * HP * 8));
            else l2_prefetch((const char*)sym + (int64_t)cc * sbytes, sbytes);
        }
        double2 v[RR];
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
            if (valid) landed();
#pragma unroll
            for (int j = 0; j < RR; ++j) v[j] = valid ? xb[t + j * T] : make_double2(0.0, 0.0);
            __syncthreads();  // the column is in registers: the buffer takes the exchanges
            reg_fft<LOGQ, kPipeLogR, -1, BlockBar, false>(
                v, t, xb, make_fft_tw_s<LOGQ, kPipeLogR>(opaque(t), stw), BlockBar{}, [&]() {
                    if (!valid) return;
                    if (c == 0) land(x0 + cstride, xbytes);
                    else if (XL == 2) land((const char*)sym + (int64_t)cc * sbytes, sbytes / 2);
                    else if (XL == 3) land(symh + (int64_t)cc * 3 * HP, (unsigned)(3 * HP * 8));
                });
            if (c == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q) tmem_st4(ta + 16 * q, v + 4 * q);
                tmem_wait_st();
            }
        }
        // 2 x 2 product, two frequencies per TMEM round trip; F0 replaces X0
        const int64_t sbase = (int64_t)cc * Q;
        if (XL >= 2 && valid) landed();
        const double* hp = reinterpret_cast<const double*>(xb);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            double2 x0v[2], f0[2];
            tmem_ld2_wait(ta + 8 * q, x0v[0], x0v[1]);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int j = 2 * q + i;
                double2 U[2], F[2];
                U[0] = x0v[i];
                U[1] = v[j];
                if (XL == 3) {
                    // frequency k = t + j*T from the planes over [0, Q/2]: the upper
                    // half mirrored, xy odd
                    const int k = t + j * T;
                    const int kk = j < RR / 2 ? k : Q - k;
                    const double gxx = valid ? hp[kk] : 0.0;
                    const double gxy = valid ? (j < RR / 2 ? hp[HP + kk] : -hp[HP + kk]) : 0.0;
                    const double gyy = valid ? hp[2 * HP + kk] : 0.0;
                    F[0] = make_double2(gxx * U[0].x + gxy * U[1].x, gxx * U[0].y + gxy * U[1].y);
                    F[1] = make_double2(gxy * U[0].x + gyy * U[1].x, gxy * U[0].y + gyy * U[1].y);
                } else if (XL == 2 && j < RR / 2) {
                    // symbol rows t + j*T, j < 8: the landed first half of the column's table
                    const double2 g01 = valid ? xb[2 * (t + j * T)] : make_double2(0.0, 0.0);
                    const double2 g23 = valid ? xb[2 * (t + j * T) + 1] : make_double2(0.0, 0.0);
                    F[0] = make_double2(g01.x * U[0].x + g01.y * U[1].x, g01.x * U[0].y + g01.y * U[1].y);
                    F[1] = make_double2(g01.y * U[0].x + g23.x * U[1].x, g01.y * U[0].y + g23.x * U[1].y);
                } else {
                    symbol_product<2, SYM == 1>(F, U, sym, sbase + t + j * T);
                }
                f0[i] = F[0];
                v[j] = F[1];
            }
            tmem_st2(ta + 8 * q, f0[0], f0[1]);
        }
        if (XL >= 2) __syncthreads();  // symbol rows read: the buffer takes the exchanges
        if (nvalid && t == 0) l2_prefetch(x0_of(b2, col2), xbytes);
#pragma unroll 1
        for (int ai = 0; ai < 2; ++ai) {
            const int a = 1 - ai;
            if (ai == 1) {
                tmem_wait_st();
                TmemQuad tq[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) tmem_ld4(ta + 16 * q, tq[q]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    tmem_wait_ld(tq[q]);
                    tmem_unpack4(tq[q], v + 4 * q);
                }
            }
            reg_fft<LOGQ, kPipeLogR, 1, BlockBar, false>(v, t, xb, make_fft_tw_s<LOGQ, kPipeLogR>(opaque(t), stw),
                                                         BlockBar{}, [&]() {
                                                             if (ai == 1 && nvalid) land(x0_of(b2, col2), xbytes);
                                                         });
            // blk: the row-blocked layout [slab][n / 8][col][n % 8] -- eight
            // consecutive threads fill one 128-byte line, and K5's two-row gather
            // then reads 32-byte pieces 128 bytes apart instead of a column apart
            double2* dst = blk ? out + (int64_t)(b * 2 + a) * cstride + ((int64_t)(t >> 3) * ncols + cc) * 8 + (t & 7)
                               : z0 + a * cstride + t;
            const int64_t dj = blk ? (int64_t)T * ncols : T;
            if (valid) {
#pragma unroll
                for (int j = 0; j < RR; ++j) st_hint(dst + j * dj, v[j], pol);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

// ------------------------------------------------------- K2 / K4 (3D) ---
// CIRC (periodic y, Py = Ny = 2Q): even/odd outputs by a decimation-in-
// frequency stage (as in k_rfft_rows); K4 keeps all 2Q outputs.
template <int LOGQ, bool CIRC>
__global__ void __launch_bounds__(512) k_cfft_y_fwd(const double2* __restrict__ S1, double2* __restrict__ S2, int Ny,
                                                    int Nz, int Hx, int ZT, const double2* __restrict__ tw,
                                                    int logTWN) {
    using Sh = FftShape<LOGQ, 4>;
    constexpr int T = Sh::T, R = Sh::R, XB = Sh::XBUF;
    constexpr int Py = 2 * Sh::Q;
    extern __shared__ double2 sm[];
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    const int zz = gi >> 1, eo = gi & 1;
    const int z0 = blockIdx.x * ZT;
    const int nz = min(ZT, Nz - z0);
    const int kx = blockIdx.y;
    const int bd = blockIdx.z;
    const bool valid = zz < nz;
    const int shP = logTWN - (LOGQ + 1);
    const double2* src = S1 + (((int64_t)bd * Nz + z0 + zz) * Hx + kx) * Ny;
    double2* xb = sm + gi * XB;
    double2 v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int n = t + j * T;
        double2 x = make_double2(0.0, 0.0);
        if (valid && n < Ny) x = src[n];
        if (CIRC) {
            const double2 x2 = valid ? src[n + Sh::Q] : make_double2(0.0, 0.0);
            x = eo ? csub(x, x2) : cadd(x, x2);
        }
        v[j] = eo ? cmul(x, __ldg(tw + (n << shP))) : x;
    }
    reg_fft<LOGQ, 4, -1>(v, t, xb, make_fft_tw<LOGQ, 4>(t, tw, logTWN), BlockBar{});
#pragma unroll
    for (int j = 0; j < R; ++j) xb[spad(t + j * T)] = v[j];
    __syncthreads();
    // transposed store (runs of nz values per ky): a thread's SMEM reads first,
    // then its global stores (a full tile is exactly R per thread)
    {
        const int tot = Py * nz;
        double2* base = S2 + ((int64_t)bd * Hx + kx) * Py * Nz + z0;
        for (int i0 = 0; i0 < tot; i0 += R * (int)blockDim.x) {
            double2 g[R];
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int idx = i0 + threadIdx.x + u * (int)blockDim.x;
                const int ky = idx / nz, z = idx - ky * nz;
                g[u] = idx < tot ? sm[(2 * z + (ky & 1)) * XB + spad(ky >> 1)] : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int idx = i0 + threadIdx.x + u * (int)blockDim.x;
                const int ky = idx / nz, z = idx - ky * nz;
                if (idx < tot) base[(int64_t)ky * Nz + z] = g[u];
            }
        }
    }
}

template <int LOGQ, bool CIRC>
__global__ void __launch_bounds__(512) k_cfft_y_inv(const double2* __restrict__ S2, double2* __restrict__ S1, int Ny,
                                                    int Nz, int Hx, int ZT, const double2* __restrict__ tw,
                                                    int logTWN) {
    using Sh = FftShape<LOGQ, 4>;
    constexpr int T = Sh::T, R = Sh::R, XB = Sh::XBUF;
    constexpr int Py = 2 * Sh::Q;
    extern __shared__ double2 sm[];
    const int gi = threadIdx.x >> Sh::LOGT;
    const int t = threadIdx.x & (T - 1);
    const int eo = gi & 1;
    const int z0 = blockIdx.x * ZT;
    const int nz = min(ZT, Nz - z0);
    const int kx = blockIdx.y;
    const int bd = blockIdx.z;
    const int shP = logTWN - (LOGQ + 1);
    // the strided gather (runs of nz values per ky): every load of the thread
    // in flight before the SMEM stores (a full tile is exactly R per thread)
    {
        const int tot = Py * nz;
        const double2* base = S2 + ((int64_t)bd * Hx + kx) * Py * Nz + z0;
        for (int i0 = 0; i0 < tot; i0 += R * (int)blockDim.x) {
            double2 g[R];
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int idx = i0 + threadIdx.x + u * (int)blockDim.x;
                const int ky = idx / nz, z = idx - ky * nz;
                g[u] = idx < tot ? base[(int64_t)ky * Nz + z] : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int idx = i0 + threadIdx.x + u * (int)blockDim.x;
                const int ky = idx / nz, z = idx - ky * nz;
                if (idx < tot) sm[(2 * z + (ky & 1)) * XB + spad(ky >> 1)] = g[u];
            }
        }
    }
    __syncthreads();
    double2* xb = sm + gi * XB;
    double2 v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = xb[spad(t + j * T)];
    __syncthreads();
    reg_fft<LOGQ, 4, 1>(v, t, xb, make_fft_tw<LOGQ, 4>(t, tw, logTWN), BlockBar{});
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int n = t + j * T;
        xb[spad(n)] = eo ? cmul(twiddle<1>(tw, n << shP), v[j]) : v[j];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < nz * Ny; idx += blockDim.x) {
        const int z = idx / Ny, n = idx - z * Ny;
        const int m = n & (Sh::Q - 1);
        const double2 e0 = sm[2 * z * XB + spad(m)], o1 = sm[(2 * z + 1) * XB + spad(m)];
        S1[(((int64_t)bd * Nz + z0 + z) * Hx + kx) * Ny + n] = (CIRC && n >= Sh::Q) ? csub(e0, o1) : cadd(e0, o1);
    }
}

// ------------------------------------------------------------ symbol K9 --
// H(k) = scale * sum_o K(o) exp(+2 pi i k.o / P) = conj(G_hat(k)) / prod(P)
// (convolution.hpp:107-116 embeds K at wrapped offsets and FFTs; the product
// at :140-153 uses conj(G_hat)).  Exact rational phases via sincospi.
// Output layout [col][h][k][pair], ky = 2k + h.
#if defined(PDGPU_ALL_PARTS) || PDGPU_PART == 0
__global__ void k_build_symbol(void* sym, const double* __restrict__ K, int dim, int M, int np, int64_t ss,
                               int ncols, int Pl, int P0, int P1, int P2, int real, double scale, int NH, int ns,
                               int col0) {
    const int64_t nfreq = (int64_t)ncols * Pl;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nfreq) return;
    const int col = (int)(idx / Pl), kl = (int)(idx % Pl);
    int k0, k1, k2;
    if (dim == 2) {
        k0 = col + col0;  // col0: first column of a distributed-FFT rank's share
        k1 = kl;
        k2 = 0;
    } else {
        k0 = col / P1;
        k1 = col % P1;
        k2 = kl;
    }
    const int side = 2 * M + 1;
    double2 ex[17], ey[17], ez[17];
    for (int o = -M; o <= M; ++o) {
        double s, c;
        const int m0 = (int)(((int64_t)k0 * (o + P0)) % P0);
        sincospi(2.0 * (double)m0 / (double)P0, &s, &c);
        ex[o + M] = make_double2(c, s);
        const int m1 = (int)(((int64_t)k1 * (o + P1)) % P1);
        sincospi(2.0 * (double)m1 / (double)P1, &s, &c);
        ey[o + M] = make_double2(c, s);
        if (dim == 3) {
            const int m2 = (int)(((int64_t)k2 * (o + P2)) % P2);
            sincospi(2.0 * (double)m2 / (double)P2, &s, &c);
            ez[o + M] = make_double2(c, s);
        } else {
            ez[o + M] = make_double2(1.0, 0.0);
        }
    }
    double2 acc[6];
    for (int p = 0; p < np; ++p) acc[p] = make_double2(0.0, 0.0);
    const int s2n = dim == 3 ? side : 1;
    for (int i2 = 0; i2 < s2n; ++i2)
        for (int i1 = 0; i1 < side; ++i1) {
            const double2 e12 = cmul(ey[i1], dim == 3 ? ez[i2] : make_double2(1.0, 0.0));
            for (int i0 = 0; i0 < side; ++i0) {
                const int64_t si = ((int64_t)i2 * side + i1) * side + i0;
                const double2 e = cmul(ex[i0], e12);
                for (int p = 0; p < np; ++p) {
                    const double kv = K[p * ss + si];
                    if (kv != 0.0) {
                        acc[p].x += kv * e.x;
                        acc[p].y += kv * e.y;
                    }
                }
            }
        }
    const int Ql = Pl / NH;
    const int64_t o = (((int64_t)col * NH + (kl % NH)) * Ql + kl / NH) * ns;
    for (int p = 0; p < np; ++p) {
        if (real) ((double*)sym)[o + p] = acc[p].x * scale;
        else ((double2*)sym)[o + p] = make_double2(acc[p].x * scale, acc[p].y * scale);
    }
    for (int p = np; p < ns; ++p) {  // padding of the 2D real layout
        if (real) ((double*)sym)[o + p] = 0.0;
    }
}
#endif

// ------------------------------------------------------------------ host --
static void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

static void smem_attr(const void* fn) {
    cudaFuncAttributes fa;
    check(cudaFuncGetAttributes(&fa, fn), "func attributes");
    // the 227 KB per-block limit covers static + dynamic shared memory
    check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - (int)fa.sharedSizeBytes),
          "smem attr");
}


// The host side is compiled in parts (PDGPU_PART = 0..4, one object file
// each, built in parallel) so every translation unit instantiates only its
// own kernel templates; without PDGPU_PART everything is compiled at once.

void set_attrs_k1();
void set_attrs_k5();
void set_attrs_k3_2d();
void set_attrs_3d();
void launch_k1(Engine& e, const double* u, int batch, cudaStream_t s);
void launch_k5(Engine& e, const double2* xin, double* f, int batch, cudaStream_t s, double scale,
               const uint8_t* cmask, const double* body);
void launch_k3_2d(Engine& e, const double2* spec, int batch, cudaStream_t s, bool blocked_ok = false);
void launch_k2_3d(Engine& e, int batch, cudaStream_t s);
void launch_k3_3d(Engine& e, double2* spec, int batch, cudaStream_t s);
void launch_k4_3d(Engine& e, int batch, cudaStream_t s);

// runtime log2 -> compile-time template dispatch over [1, 12]
#define PDGPU_CASE(L, CALL) \
    case L: {               \
        constexpr int LQ = L; \
        CALL;               \
    } break;
#define PDGPU_DISPATCH_LOGQ(lq, CALL)                                                                       \
    switch (lq) {                                                                                           \
        PDGPU_CASE(1, CALL) PDGPU_CASE(2, CALL) PDGPU_CASE(3, CALL) PDGPU_CASE(4, CALL) PDGPU_CASE(5, CALL) \
        PDGPU_CASE(6, CALL) PDGPU_CASE(7, CALL) PDGPU_CASE(8, CALL) PDGPU_CASE(9, CALL)                     \
        PDGPU_CASE(10, CALL) PDGPU_CASE(11, CALL) PDGPU_CASE(12, CALL)                                      \
        default: throw std::runtime_error("transform length out of range");                                 \
    }
#define PDGPU_DISPATCH_LOGQ9(lq, CALL)                                                                      \
    switch (lq) {                                                                                           \
        PDGPU_CASE(1, CALL) PDGPU_CASE(2, CALL) PDGPU_CASE(3, CALL) PDGPU_CASE(4, CALL) PDGPU_CASE(5, CALL) \
        PDGPU_CASE(6, CALL) PDGPU_CASE(7, CALL) PDGPU_CASE(8, CALL) PDGPU_CASE(9, CALL)                     \
        default: throw std::runtime_error("3D transform length out of range");                              \
    }


#if defined(PDGPU_ALL_PARTS) || PDGPU_PART == 1
template <int L, bool C>
static void set_attrs_k1_l() {
    smem_attr((const void*)k_rfft_rows<L, C>);
    smem_attr((const void*)k_rfft_rows_pipe<L, 0, C>);
    smem_attr((const void*)k_rfft_rows_pipe<L, 1, C>);
    smem_attr((const void*)k_rfft_rows_pipe<L, 2, C>);
    smem_attr((const void*)k_rfft_rows_pipe<L, 3, C>);
    if constexpr (L >= 6 && L <= 10) smem_attr((const void*)k_rfft_rows_duo<L, C>);
    if constexpr (C && L == 10) {
        smem_attr((const void*)k_rfft_rows_duo<L, C, true, 0>);
        smem_attr((const void*)k_rfft_rows_duo<L, C, true, 1>);
        if constexpr (L == 10 && C) {
            smem_attr((const void*)k_rfft_rows_p2<10, false, 2, 1, 256, 9>);
            smem_attr((const void*)k_rfft_rows_p2<10, true, 2, 1, 256, 9>);
            smem_attr((const void*)k_rfft_rows_p2<9, true, 4, 2, 256, 4>);
            smem_attr((const void*)k_rfft_rows_p2<8, true, 8, 2, 256, 2>);
        }
    }
}
template <int... Ls>
static void set_attrs_k1_all(std::integer_sequence<int, Ls...>) {
    (set_attrs_k1_l<Ls + 1, false>(), ...);
    (set_attrs_k1_l<Ls + 1, true>(), ...);
}
void set_attrs_k1() { set_attrs_k1_all(std::make_integer_sequence<int, 12>{}); }

void launch_k1(Engine& e, const double* u, int batch, cudaStream_t s) {
    const Plan& pl = e.plan;
    e.xstrip_ready = false;  // set below when this pass writes the x-face strip
    const int Nx = pl.N[0], Ny = pl.N[1], Nz = pl.N[2];
    const int nslab = batch * pl.dim * Nz;
    const int lqx = pl.logQx;
    const bool cx = pl.circ[0] != 0;
    int TR = pl.k1_rows;
    const int T = threads_per_transform(lqx, 4);
    // two-CTA/SM variant: two rows of two transforms fill a 256-thread CTA
    if ((Nx & 1) == 0 && lqx >= 7 && lqx <= 10 && !getenv("PDGPU_NO_K1_DUO")) {  // lqx 6 (256-wide rows): the pipelined kernel measured faster
        // PDGPU_K1_CF=1: conflict-free [kx][row] block writes (4 kx x 2 rows per
        // quarter-warp).  SMEM bank conflicts 129M -> 18M per launch, and 6 %
        // faster at batch 2, but 22 % slower at batch 16 (long-scoreboard
        // stalls 23 -> 38 %, same DRAM bytes): off by default
        // L2 prefetch of the rows this CTA loads PDGPU_K1_PF tiles later: off
        // (measured 2.21 -> 2.7 / 3.1 ms at 4096^2 x 16 with 1 / 2 tiles ahead)
        const char* pfenv = getenv("PDGPU_K1_PF");
        const int k1pf = pfenv ? atoi(pfenv) : 0;
        // PDGPU_K1_EARLY=1: row 0 of the next tile is requested into the
        // exchange buffer before the post-processing, the rest after the TMA
        // store has read its block (measured slower: K1 2.25 -> 2.30 ms; off)
        const char* eenv = getenv("PDGPU_K1_EARLY");
        const int k1early = (eenv && eenv[0] == '1') ? 1 : 0;
        const char* cfenv = getenv("PDGPU_K1_CF");
        // (with the persistent two-group kernel below the landing latency is off
        // the critical path and the conflict-free map wins, 2.24 -> 2.15 ms: it is
        // the default there, PDGPU_K1_CF=0 disables)
        const char* p2e = getenv("PDGPU_K1_P2");
        const bool p2on = !(p2e && p2e[0] == '0');
        const int cfm = (cx && lqx == 10 && (cfenv ? cfenv[0] == '1' : p2on)) ? 1 : 0;
        const size_t dsm = (size_t)k1_duo_smem(lqx, cx, cfm);
        const int DTR = 2048 >> lqx;
        if (2 * (dsm + 1024) <= 228 * 1024) {
            const int64_t ntiles = (int64_t)((Ny + DTR - 1) / DTR) * nslab;
            const unsigned dgrid = (unsigned)std::min<int64_t>(ntiles, (int64_t)e.num_sms * 2);
            CUtensorMap tm;
            memset(&tm, 0, sizeof(tm));
            // TMA-stored spectrum blocks (periodic 4096-wide rows, two per tile:
            // K1 2.71 -> 2.32 ms at 4096^2 x 16; neutral at 2048, slower at 1024):
            // PDGPU_K1_TMA=0 disables
            const char* tenv = getenv("PDGPU_K1_TMA");
            const bool tst = cx && DTR <= 2 && !(tenv && tenv[0] == '0') && encode_box_map(tm, e.d_S1, Ny, pl.Hx, nslab, DTR) &&
                             (size_t)(((pl.Hx + 255) / 256) * 256 * DTR * 16 + 128) <= dsm;
            // 4096-wide periodic rows: the persistent two-group kernel (PDGPU_K1_P2=0:
            // the two-CTA duo kernel)
            const char* p2env = getenv("PDGPU_K1_P2");
            // 2048- / 1024-wide periodic rows: four 128-thread (eight 64-thread) groups, two
            // landing buffers, two rows per tile stored as 4 (2) TMA boxes of 256 kx + the
            // Nyquist kx: K1 0.626 -> 0.409 ms at 2048^2 x 16, 0.146 -> 0.137 ms at 1024^2 x 16
            // (PDGPU_K1_P2=0 disables)
            if (cx && (lqx == 9 || lqx == 8) && Nx == (4 << lqx) && Ny % 2 == 0 && pl.Hx == (2 << lqx) + 1 &&
                !(p2env && p2env[0] == '0') && !(tenv && tenv[0] == '0') && encode_box_map(tm, e.d_S1, Ny, pl.Hx, nslab, 2)) {
                const int64_t nt2 = (int64_t)(Ny / 2) * nslab;
                const int ng = lqx == 9 ? 4 : 8;
                const unsigned pgrid = (unsigned)std::min<int64_t>((nt2 + ng - 1) / ng, (int64_t)e.num_sms);
                if (lqx == 9)
                    k_rfft_rows_p2<9, true, 4, 2, 256, 4><<<pgrid, 512, k1_p2_smem(9, 1, 2, 4, 256, 4), s>>>(
                        u, e.d_S1, Nx, Ny, pl.Hx, e.d_tw, pl.logTWN, tm, nt2);
                else
                    k_rfft_rows_p2<8, true, 8, 2, 256, 2><<<pgrid, 512, k1_p2_smem(8, 1, 2, 8, 256, 2), s>>>(
                        u, e.d_S1, Nx, Ny, pl.Hx, e.d_tw, pl.logTWN, tm, nt2);
                return;
            }
            if (tst && lqx == 10 && Nx == (4 << lqx) && Ny % 2 == 0 && pl.Hx <= 9 * 256 &&
                !(p2env && p2env[0] == '0')) {
                const unsigned pgrid = (unsigned)std::min<int64_t>((ntiles + 1) / 2, (int64_t)e.num_sms);
                const int psm = k1_p2_smem(10, cfm, 1, 2, 256, 9);
                if (cfm)
                    k_rfft_rows_p2<10, true, 2, 1, 256, 9><<<pgrid, 512, psm, s>>>(u, e.d_S1, Nx, Ny, pl.Hx, e.d_tw, pl.logTWN,
                                                                                 tm, ntiles);
                else
                    k_rfft_rows_p2<10, false, 2, 1, 256, 9><<<pgrid, 512, psm, s>>>(u, e.d_S1, Nx, Ny, pl.Hx, e.d_tw, pl.logTWN,
                                                                                  tm, ntiles);
                return;
            }
#define PDGPU_K1T(CF) k_rfft_rows_duo<LQ, true, true, CF><<<dgrid, 256, dsm, s>>>(u, e.d_S1, Nx, Ny, nslab, pl.Hx, \
                                                                                e.d_tw, pl.logTWN, tm, k1pf, k1early)
#define PDGPU_K1D(C) (tst ? (cfm == 1 ? PDGPU_K1T(1) : PDGPU_K1T(0))                                     \
                      : k_rfft_rows_duo<LQ, C><<<dgrid, 256, dsm, s>>>(u, e.d_S1, Nx, Ny, nslab, pl.Hx, e.d_tw, \
                                                                      pl.logTWN, tm, k1pf, k1early))
            switch (lqx) {
                PDGPU_CASE(6, (cx ? PDGPU_K1D(true) : PDGPU_K1D(false)))
                PDGPU_CASE(7, (cx ? PDGPU_K1D(true) : PDGPU_K1D(false)))
                PDGPU_CASE(8, (cx ? PDGPU_K1D(true) : PDGPU_K1D(false)))
                PDGPU_CASE(9, (cx ? PDGPU_K1D(true) : PDGPU_K1D(false)))
                PDGPU_CASE(10, (cx ? PDGPU_K1D(true) : PDGPU_K1D(false)))
                default: goto no_duo;
            }
#undef PDGPU_K1D
#undef PDGPU_K1T
            return;
        }
    }
no_duo:
    const size_t rowlen = (size_t)(cx ? 4 : 2) << lqx;  // staged reals per row
    auto smem_of = [&](int tr) { return sizeof(double2) * (size_t)2 * tr * xbuf_stride_t_h(lqx); };
    auto psmem_of = [&](int tr) { return smem_of(tr) + sizeof(double) * (size_t)tr * rowlen; };
    int PTR = TR;  // pipelined kernel: shrink the tile until the staging buffer fits
    while (PTR > 1 && psmem_of(PTR) > 227 * 1024) PTR /= 2;
    // small lattices: down until the grid covers the SMs twice
    while (PTR > 1 && (int64_t)((Ny + PTR - 1) / PTR) * nslab < 2 * e.num_sms) PTR /= 2;
    if ((Nx & 1) == 0 && psmem_of(PTR) <= 227 * 1024 && !getenv("PDGPU_NO_K1_PIPE")) {
        const size_t psmem = psmem_of(PTR);
        const int64_t ntiles = (int64_t)((Ny + PTR - 1) / PTR) * nslab;
        // CTAs resident per SM (128 registers/thread under the 512-thread bound)
        const int per_sm = std::max(1, std::min((int)(228 * 1024 / (psmem + 1024)), 65536 / (2 * PTR * T * 128)));
        const unsigned pgrid = (unsigned)std::min<int64_t>(ntiles, (int64_t)e.num_sms * per_sm);
        const int ltr = PTR == 8 ? 3 : PTR == 4 ? 2 : PTR == 2 ? 1 : 0;
        // 3D with the tiled wrap passes: the x-face strip comes out of this pass
        double* xs = (pl.dim == 3 && e.d_ftab && pl.circ[0] && e.d_xstrip && batch <= e.cap_batch &&
                      e.slab.global < 0 && 4 * e.M <= Nx)
                         ? e.d_xstrip
                         : nullptr;
        e.xstrip_ready = xs != nullptr;
#define PDGPU_K1P(LT, C) launch_maybe_pdl(e.pdl, k_rfft_rows_pipe<LQ, LT, C>, dim3(pgrid), dim3(2 * PTR * T), psmem, s, \
                                          u, e.d_S1, Nx, Ny, nslab, pl.Hx, e.d_tw, pl.logTWN, xs, e.M, Nz)
#define PDGPU_K1PC(C) (ltr == 3 ? PDGPU_K1P(3, C) : ltr == 2 ? PDGPU_K1P(2, C) : ltr == 1 ? PDGPU_K1P(1, C) \
                                                                                 : PDGPU_K1P(0, C))
        if (cx) PDGPU_DISPATCH_LOGQ(lqx, PDGPU_K1PC(true))
        else PDGPU_DISPATCH_LOGQ(lqx, PDGPU_K1PC(false))
#undef PDGPU_K1PC
#undef PDGPU_K1P
    } else {
        dim3 grid((Ny + TR - 1) / TR, nslab);
        const size_t smem = smem_of(TR);
        if (cx)
            PDGPU_DISPATCH_LOGQ(lqx, (k_rfft_rows<LQ, true><<<grid, 2 * TR * T, smem, s>>>(u, e.d_S1, Nx, Ny, pl.Hx, TR,
                                                                                      e.d_tw, pl.logTWN)))
        else
            PDGPU_DISPATCH_LOGQ(lqx, (k_rfft_rows<LQ, false><<<grid, 2 * TR * T, smem, s>>>(u, e.d_S1, Nx, Ny, pl.Hx,
                                                                                       TR, e.d_tw, pl.logTWN)))
    }
}
#endif

#if defined(PDGPU_ALL_PARTS) || PDGPU_PART == 2
template <int L, bool C>
static void set_attrs_k5_l() {
    smem_attr((const void*)k_irfft_rows<L, 0, C>);
    smem_attr((const void*)k_irfft_rows<L, 1, C>);
    smem_attr((const void*)k_irfft_rows<L, 2, C>);
    smem_attr((const void*)k_irfft_rows<L, 3, C>);
    if constexpr (C && L >= 8) smem_attr((const void*)k_irfft_rows<L, 1, C, true>);
}
template <int... Ls>
static void set_attrs_k5_all(std::integer_sequence<int, Ls...>) {
    (set_attrs_k5_l<Ls + 1, false>(), ...);
    (set_attrs_k5_l<Ls + 1, true>(), ...);
}
void set_attrs_k5() {
    set_attrs_k5_all(std::make_integer_sequence<int, 12>{});
    smem_attr((const void*)k_irfft_rows_p2<10, 2, 1>);
    smem_attr((const void*)k_irfft_rows_p2<9, 4, 2>);
    smem_attr((const void*)k_irfft_rows_p2<8, 8, 2>);
}

void launch_k5(Engine& e, const double2* xin, double* f, int batch, cudaStream_t s, double scale,
               const uint8_t* cmask, const double* body) {
    const double* fxs = e.xpass_done ? e.d_fx : nullptr;  // the wrap x pass ran before this pass
    const Plan& pl = e.plan;
    const int Nx = pl.N[0], Ny = pl.N[1], Nz = pl.N[2], d = pl.dim;
    const int nslab = batch * d * Nz;
    const int lqx = pl.logQx;
    const bool cx = pl.circ[0] != 0;
    // padded rows: one row per CTA, two 256-thread CTAs co-reside per SM
    // (measured faster than two rows per CTA or a persistent double-buffered
    // variant); periodic rows (half the length): several rows per CTA (wider
    // gather chunks), 2.87 vs 3.22 ms at 4096^2 x 16
    // periodic rows: up to 256 threads / 4 rows per CTA (measured at 1024..4096 x 16:
    // 4096 -> 2 rows (2.73 ms), 2048 -> 4 rows (0.65 vs 0.68 ms with 2))
    int TR = pl.circ[0] ? std::min(std::min(4, pl.k1_rows), std::max(1, 128 / threads_per_transform(pl.logQx, 4))) : 1;
    const char* tenv = getenv("PDGPU_K5_TMA");
    const bool use_tma = !(tenv && tenv[0] == '0');
    // TMA-landed gathers run two rows per CTA (1024..4096-wide rows: 0.146 -> 0.131,
    // 0.673 -> 0.560, 2.74 -> 2.49 ms at batch 16)
    const bool tma_rows = pl.circ[0] && pl.logQx >= 8 && use_tma && pl.k1_rows >= 2;
    if (tma_rows) TR = 2;
    // short rows: at least 128 threads per CTA (up to the 8-row template limit)
    while (!tma_rows && TR < pl.k1_rows && 2 * TR * threads_per_transform(pl.logQx, 4) < 128) TR *= 2;
    // small lattices (latency-bound: CG on 128^2): rows per CTA down until the
    // grid covers the SMs twice
    while (!tma_rows && TR > 1 && (int64_t)((Ny + TR - 1) / TR) * nslab < 2 * e.num_sms) TR /= 2;
    if (const char* env = getenv("PDGPU_K5_ROWS")) TR = std::max(1, std::min(pl.k1_rows, atoi(env)));
    while (TR & (TR - 1)) TR &= TR - 1;  // power of two (template)
    const int ltr = TR == 8 ? 3 : TR == 4 ? 2 : TR == 2 ? 1 : 0;
    const int T = threads_per_transform(lqx, 4);
    dim3 grid((Ny + TR - 1) / TR, nslab);
    const size_t smem = sizeof(double2) * (size_t)2 * TR * xbuf_stride_t_h(lqx);
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    // L2 prefetch of the TMA-landed block of the CTA launched num_sms later
    // (its landing then hits L2: the block is 2049 32-byte pieces 64 KB apart):
    // K5 2.22 -> 1.97 ms at 4096^2 x 16, 0.479 -> 0.465 at 2048^2, but
    // 0.113 -> 0.136 at 1024^2, so from 2048-wide rows up (PDGPU_K5_PF = distance)
    const char* pfenv = getenv("PDGPU_K5_PF");
    const int k5pf = pfenv ? atoi(pfenv) : (lqx >= 9 ? e.num_sms : 0);
    // TMA-landed gathers (periodic rows, two per CTA; PDGPU_K5_TMA=0 disables)
    const bool blk = e.s2_blocked;  // set by launch_k3_2d for the spectrum it just wrote
    e.s2_blocked = false;
    if (blk && !(cx && TR == 2 && lqx >= 8 && use_tma && d == 2))
        throw std::runtime_error("K5: row-blocked spectrum without the TMA row gather");
    if (cx && TR == 2 && lqx >= 8 && use_tma && encode_box_map(tm, xin, Ny, pl.Hx, nslab, TR, blk)) {
        const int nbox = (pl.Hx + 255) / 256;
        const size_t tsm = std::max(sizeof(double2) * (size_t)2 * TR * xbuf_stride_rows_h(lqx),
                                    sizeof(double2) * (size_t)nbox * 256 * TR) + 128;
        // 4096-wide rows of a 2D lattice: the persistent two-group kernel
        // (PDGPU_K5_P2=0 keeps the one-tile CTAs; PDGPU_K5_P2PF = L2 prefetch distance in tiles)
        const char* p2env = getenv("PDGPU_K5_P2");
        // (2048-wide rows: four 128-thread groups and two landing buffers, 0.523 -> 0.456 ms
        // at 2048^2 x 16; 1024-wide rows: eight 64-thread groups, measured slower, 0.128 ->
        // 0.146 ms at 1024^2 x 16, opt-in PDGPU_K5_P2=1)
        const bool p2ok = d == 2 && Nz == 1 && !fxs && (Nx & 1) == 0 && Ny % TR == 0;
        if (p2ok && (((lqx == 10 || lqx == 9) && !(p2env && p2env[0] == '0')) || (lqx == 8 && p2env && p2env[0] == '1'))) {
            const int ng = lqx == 10 ? 2 : lqx == 9 ? 4 : 8, nl = lqx == 10 ? 1 : 2;
            const size_t psm = sizeof(double2) * ((size_t)nl * nbox * 256 * TR + (size_t)ng * 2 * TR * xbuf_stride_rows_h(lqx)) + 128;
            const int64_t ntiles = (int64_t)(Ny / TR) * nslab;
            const char* ppf = getenv("PDGPU_K5_P2PF");
            const int p2pf = ppf ? atoi(ppf) : 0;
            const unsigned pgrid = (unsigned)std::min<int64_t>((ntiles + ng - 1) / ng, (int64_t)e.num_sms);
#define PDGPU_K5P2(LQV, NGV, NLV)                                                                                       \
    k_irfft_rows_p2<LQV, NGV, NLV><<<pgrid, 512, psm, s>>>(f, Nx, Ny, Nz, d, pl.Hx, e.d_tw, pl.logTWN, scale, cmask, body, \
                                                          pl.nodes, tm, p2pf, blk ? 1 : 0, ntiles)
            if (lqx == 10) PDGPU_K5P2(10, 2, 1);
            else if (lqx == 9) PDGPU_K5P2(9, 4, 2);
            else PDGPU_K5P2(8, 8, 2);
#undef PDGPU_K5P2
            return;
        }
        switch (lqx) {
            PDGPU_CASE(8, (k_irfft_rows<LQ, 1, true, true><<<grid, 2 * TR * T, tsm, s>>>(xin, f, Nx, Ny, Nz, d, pl.Hx,
                                                      e.d_tw, pl.logTWN, scale, cmask, body, pl.nodes, tm, k5pf, fxs, e.M, blk ? 1 : 0)))
            PDGPU_CASE(9, (k_irfft_rows<LQ, 1, true, true><<<grid, 2 * TR * T, tsm, s>>>(xin, f, Nx, Ny, Nz, d, pl.Hx,
                                                      e.d_tw, pl.logTWN, scale, cmask, body, pl.nodes, tm, k5pf, fxs, e.M, blk ? 1 : 0)))
            PDGPU_CASE(10, (k_irfft_rows<LQ, 1, true, true><<<grid, 2 * TR * T, tsm, s>>>(xin, f, Nx, Ny, Nz, d, pl.Hx,
                                                      e.d_tw, pl.logTWN, scale, cmask, body, pl.nodes, tm, k5pf, fxs, e.M, blk ? 1 : 0)))
            PDGPU_CASE(11, (k_irfft_rows<LQ, 1, true, true><<<grid, 2 * TR * T, tsm, s>>>(xin, f, Nx, Ny, Nz, d, pl.Hx,
                                                      e.d_tw, pl.logTWN, scale, cmask, body, pl.nodes, tm, k5pf, fxs, e.M, blk ? 1 : 0)))
            PDGPU_CASE(12, (k_irfft_rows<LQ, 1, true, true><<<grid, 2 * TR * T, tsm, s>>>(xin, f, Nx, Ny, Nz, d, pl.Hx,
                                                      e.d_tw, pl.logTWN, scale, cmask, body, pl.nodes, tm, k5pf, fxs, e.M, blk ? 1 : 0)))
            default: break;
        }
        return;
    }
    if (blk) throw std::runtime_error("K5: row-blocked spectrum but no tensor map");
    // gathers (short rows, 3D): prefetch distance PDGPU_K5_GPF (CTAs)
    const char* gpfenv = getenv("PDGPU_K5_GPF");
    const int gpf = gpfenv ? atoi(gpfenv) : 0;
#define PDGPU_K5(LT, C) launch_maybe_pdl(e.pdl, k_irfft_rows<LQ, LT, C>, grid, dim3(2 * TR * T), smem, s, xin, f, Nx, Ny, \
                                         Nz, d, pl.Hx, e.d_tw, pl.logTWN, scale, cmask, body, pl.nodes, tm, gpf, fxs, e.M, 0)
#define PDGPU_K5C(C) (ltr == 3 ? PDGPU_K5(3, C) : ltr == 2 ? PDGPU_K5(2, C) : ltr == 1 ? PDGPU_K5(1, C) : PDGPU_K5(0, C))
    if (cx) PDGPU_DISPATCH_LOGQ(lqx, PDGPU_K5C(true))
    else PDGPU_DISPATCH_LOGQ(lqx, PDGPU_K5C(false))
#undef PDGPU_K5C
#undef PDGPU_K5
}
#endif

#if defined(PDGPU_ALL_PARTS) || PDGPU_PART == 3
template <int L>
static void set_attrs_k3_l() {
    if constexpr (L >= 4) {
        smem_attr((const void*)k_spectral2d_duo<L, 0, 1>);
        smem_attr((const void*)k_spectral2d_duo<L, 1, 1>);
        smem_attr((const void*)k_spectral2d_duo<L, 2, 1>);
        smem_attr((const void*)k_spectral2d_duo<L, 0, 2>);
        smem_attr((const void*)k_spectral2d_duo<L, 1, 2>);
        smem_attr((const void*)k_spectral2d_duo<L, 2, 2>);
    }
    if constexpr (L == 11 || L == 12) {
        smem_attr((const void*)k_spectral2d_tm<L, 0, false>);
        smem_attr((const void*)k_spectral2d_tm<L, 1, false>);
        smem_attr((const void*)k_spectral2d_tm<L, 1, false, 3>);
        smem_attr((const void*)k_spectral2d_tm<L, 0, true>);
        smem_attr((const void*)k_spectral2d_tm<L, 1, true>);
        smem_attr((const void*)k_spectral2d_tx<L, 0, 1>);
        smem_attr((const void*)k_spectral2d_tx<L, 1, 1>);
        smem_attr((const void*)k_spectral2d_tx<L, 1, 2>);
        smem_attr((const void*)k_spectral2d_tx<L, 1, 3>);
    }
    if constexpr (L == 9 || L == 10) smem_attr((const void*)k_spectral2d_tx<L, 1, 3>);
    smem_attr((const void*)k_spectral2d_pipe<L, 0>);
    smem_attr((const void*)k_spectral2d_pipe<L, 1>);
    smem_attr((const void*)k_spectral2d_pipe<L, 2>);
}
template <int... Ls>
static void set_attrs_k3_all(std::integer_sequence<int, Ls...>) {
    (set_attrs_k3_l<Ls + 1>(), ...);
}
void set_attrs_k3_2d() { set_attrs_k3_all(std::make_integer_sequence<int, 12>{}); }

#define PDGPU_DISPATCH_LOGQ_4_12(lq, CALL)                                                                  \
    switch (lq) {                                                                                           \
        PDGPU_CASE(4, CALL) PDGPU_CASE(5, CALL) PDGPU_CASE(6, CALL) PDGPU_CASE(7, CALL) PDGPU_CASE(8, CALL) \
        PDGPU_CASE(9, CALL) PDGPU_CASE(10, CALL) PDGPU_CASE(11, CALL) PDGPU_CASE(12, CALL)                  \
        default: throw std::runtime_error("transform length out of range");                                 \
    }

// 2D K3: out of place S1 -> S2 (padded: z^0 parked in S2)
// blocked_ok: the caller hands e.d_S2 straight to launch_k5, so the spectrum
// may be written row-blocked (e.s2_blocked tells K5)
void launch_k3_2d(Engine& e, const double2* spec, int batch, cudaStream_t s, bool blocked_ok) {
    const Plan& pl = e.plan;
    e.s2_blocked = false;
    const int nh = pl.nh;
    const int lq = pl.logPl - (nh == 2 ? 1 : 0);
    // persistent, cp.async-pipelined variant: NC*(XB + 2Q) slots
    const int Tp = threads_per_transform(lq, kPipeLogR);
    const int mode = e.d_coltab ? 2 : (e.real_symbol ? 1 : 0);
    const int ND = 3 * (e.M + 1);
    const size_t per_col = sizeof(double2) * (size_t)(xbuf_slots(lq) + 2 * (1 << lq)) +
                           (mode == 2 ? sizeof(double) * (size_t)ND : 0);
    // two-CTA/SM split-exchange kernel (default) unless PDGPU_K3=pipe
    // (the pipe variant handles padded columns only)
    const char* k3env = getenv("PDGPU_K3");
    // periodic 2048/4096-point columns: TMEM-parked kernel, operands by
    // register loads, 16-byte exchange (PDGPU_K3=tmland: x_0 TMA-landed with
    // the split exchange; PDGPU_K3=split: the SMEM-parked k_spectral2d_duo)
    const bool k3split = k3env && std::string(k3env) == "split";
    // 512/1024-point periodic columns with symbol mirror planes: the landed-operand
    // TMEM kernel with eight / four columns per CTA (K3 0.188 -> 0.156 ms at 1024^2 x 16,
    // 0.056 -> 0.050 ms at 512^2 x 16; any other PDGPU_K3 value: k_spectral2d_duo)
    // batches too small to cover the SMs twice with full CTAs (CG on 1024^2: 191 ->
    // 225 ms per solve) stay on k_spectral2d_duo unless PDGPU_K3=tx3 forces it
    const bool tx3_forced = k3env && std::string(k3env) == "tx3";
    const bool tx3_fits = (int64_t)((pl.ncols + kPipeThreads / Tp - 1) / (kPipeThreads / Tp)) * batch >= 2 * e.num_sms;
    if (nh == 1 && (lq == 9 || lq == 10) && mode == 1 && e.d_symh && e.symh_for == e.d_sym &&
        (tx3_forced || (!k3env && tx3_fits))) {
        int NCt = kPipeThreads / Tp;
        const size_t tsmem = (size_t)NCt * sizeof(double2) * xbuf_slots(lq);
        // forced on a small batch: fewer columns per CTA until the grid covers the SMs twice
        while (NCt > 1 && (int64_t)((pl.ncols + NCt - 1) / NCt) * batch < 2 * e.num_sms) NCt /= 2;
        const int64_t nitems = (int64_t)((pl.ncols + NCt - 1) / NCt) * batch;
        const unsigned tgrid = (unsigned)std::min<int64_t>(nitems, (int64_t)e.num_sms * 2);
        if (lq == 10)
            k_spectral2d_tx<10, 1, 3><<<tgrid, kPipeThreads, tsmem, s>>>(spec, e.d_S2, e.d_sym, pl.ncols, NCt, batch, e.d_tw,
                                                                        pl.logTWN, e.d_symh, e.symh_stride, 0);
        else
            k_spectral2d_tx<9, 1, 3><<<tgrid, kPipeThreads, tsmem, s>>>(spec, e.d_S2, e.d_sym, pl.ncols, NCt, batch, e.d_tw,
                                                                       pl.logTWN, e.d_symh, e.symh_stride, 0);
        return;
    }
    if (nh == 1 && (lq == 11 || lq == 12) && mode != 2 && !k3split) {
        const bool land = k3env && std::string(k3env) == "tmland";
        const int NCt = kPipeThreads / Tp;
        const size_t tsmem = land ? (size_t)NCt * (sizeof(double2) * ((size_t)1 << lq) + sizeof(double) * xbuf_slots(lq))
                                  : (size_t)NCt * sizeof(double2) * xbuf_slots(lq);
        const int64_t nitems = (int64_t)((pl.ncols + NCt - 1) / NCt) * batch;
        const unsigned tgrid = (unsigned)std::min<int64_t>(nitems, (int64_t)e.num_sms * 2);
#define TM_ARGS spec, e.d_S2, e.d_sym, pl.ncols, NCt, batch, e.d_tw, pl.logTWN
#define TM_L(LQV, LANDV)                                                                          \
    (mode == 1 ? k_spectral2d_tm<LQV, 1, LANDV><<<tgrid, kPipeThreads, tsmem, s>>>(TM_ARGS)       \
               : k_spectral2d_tm<LQV, 0, LANDV><<<tgrid, kPipeThreads, tsmem, s>>>(TM_ARGS))
        // PDGPU_K3=tx / tx2: operands (tx2: and half the symbol rows) landed in
        // the exchange buffer behind each transform's last exchange
        // (4096-point columns, measured on one B200 at 4096^2 x 16: 2.68 -> 2.51 ms;
        // tx2 2.55 ms -- the 32-byte symbol rows read at a two-way bank conflict;
        // tx3 2.39 ms; 2048-point columns: tm 0.640, tx 0.636, tx3 0.607 ms).
        // PDGPU_K3=tm: the register-load kernel at every length.
        const std::string k3s = k3env ? k3env : "";
        // tx3: the symbol from the column's mirror planes, landed the same way
        // (no symbol load left in the product; needs build_symbol_half's table)
        const bool symh_ok = e.d_symh && e.symh_for == e.d_sym && mode == 1;
        int xl = k3s == "tx2" ? 2 : k3s == "tx" ? 1 : (k3s == "tx3" || k3s.empty()) ? 3 : 0;
        // without the planes: landed operands at 4096 points, register loads at 2048
        if (xl == 3 && !symh_ok) xl = (lq == 12 || k3s == "tx3") ? 1 : 0;
        if (xl == 2 && mode != 1) xl = 1;
        const char* t3 = getenv("PDGPU_K3_TM3");  // three CTAs per SM (80 registers, spills)
        // row-blocked S2 (landed-operand kernel only; opt-in, PDGPU_S2_BLOCKED=1):
        // K5's TMA row gather must be the one that reads it (same conditions as
        // launch_k5).  Measured neutral to slightly slower at 4096^2 x 16 (K3 2.39
        // -> 2.42 ms, K5 2.13 -> 2.14 ms): K5 is not bound by its gather pattern.
        const char* k5t = getenv("PDGPU_K5_TMA");
        const char* sbe = getenv("PDGPU_S2_BLOCKED");
        const bool blk = blocked_ok && xl && lq == 12 && pl.dim == 2 && pl.circ[0] && pl.logQx >= 8 && pl.k1_rows >= 2 &&
                         !(k5t && k5t[0] == '0') && !getenv("PDGPU_K5_ROWS") && pl.Nl % 8 == 0 &&
                         (sbe && sbe[0] == '1');
        e.s2_blocked = blk;
        if (xl) {
#define TX_ARGS TM_ARGS, e.d_symh, e.symh_stride, blk ? 1 : 0
#define TX_L(LQV)                                                                                          \
    (mode == 1 ? (xl == 3   ? k_spectral2d_tx<LQV, 1, 3><<<tgrid, kPipeThreads, tsmem, s>>>(TX_ARGS)        \
                  : xl == 2 ? k_spectral2d_tx<LQV, 1, 2><<<tgrid, kPipeThreads, tsmem, s>>>(TX_ARGS)        \
                            : k_spectral2d_tx<LQV, 1, 1><<<tgrid, kPipeThreads, tsmem, s>>>(TX_ARGS))       \
               : k_spectral2d_tx<LQV, 0, 1><<<tgrid, kPipeThreads, tsmem, s>>>(TX_ARGS))
            if (lq == 12) TX_L(12);
            else TX_L(11);
#undef TX_L
#undef TX_ARGS
        } else if (lq == 12 && mode == 1 && !land && t3 && t3[0] == '1') {
            const unsigned g3 = (unsigned)std::min<int64_t>(nitems, (int64_t)e.num_sms * 3);
            k_spectral2d_tm<12, 1, false, 3><<<g3, kPipeThreads, tsmem, s>>>(TM_ARGS);
        } else if (lq == 12) {
            if (land) TM_L(12, true);
            else TM_L(12, false);
        } else {
            if (land) TM_L(11, true);
            else TM_L(11, false);
        }
#undef TM_L
#undef TM_ARGS
        return;
    }
    if ((nh == 1 || !(k3env && std::string(k3env) == "pipe")) && lq >= 4) {
        int NCd = kPipeThreads / Tp;
        // small lattices: fewer columns per CTA until the grid covers the SMs twice
        while (NCd > 1 && (int64_t)((pl.ncols + NCd - 1) / NCd) * batch < 2 * e.num_sms) NCd /= 2;
        const size_t dsmem = (size_t)NCd * (sizeof(double2) * (1 << lq) + sizeof(double) * xbuf_slots(lq) +
                                            (mode == 2 ? sizeof(double) * ND : 0) + sizeof(uint64_t));
        const int per_sm = std::max(1, std::min(2, (int)(228 * 1024 / (dsmem + 1024))));
        const int64_t nitems = (int64_t)((pl.ncols + NCd - 1) / NCd) * batch;
        const unsigned dgrid = (unsigned)std::min<int64_t>(nitems, (int64_t)e.num_sms * per_sm);
#define DUO_ARGS spec, e.d_S2, e.d_sym, e.d_coltab, e.M, pl.ncols, pl.Nl, NCd, batch, e.d_tw, pl.logTWN
#define DUO_NH(NHV)                                                                                           \
    if (mode == 2)                                                                                            \
        PDGPU_DISPATCH_LOGQ_4_12(lq, (launch_maybe_pdl(e.pdl, k_spectral2d_duo<LQ, 2, NHV>, dim3(dgrid), dim3(NCd * Tp), dsmem, s, DUO_ARGS))) \
    else if (mode == 1)                                                                                       \
        PDGPU_DISPATCH_LOGQ_4_12(lq, (launch_maybe_pdl(e.pdl, k_spectral2d_duo<LQ, 1, NHV>, dim3(dgrid), dim3(NCd * Tp), dsmem, s, DUO_ARGS))) \
    else                                                                                                      \
        PDGPU_DISPATCH_LOGQ_4_12(lq, (launch_maybe_pdl(e.pdl, k_spectral2d_duo<LQ, 0, NHV>, dim3(dgrid), dim3(NCd * Tp), dsmem, s, DUO_ARGS)))
        if (nh == 1) {
            DUO_NH(1)
        } else {
            DUO_NH(2)
        }
#undef DUO_NH
#undef DUO_ARGS
    } else {
        if (nh != 2) throw std::runtime_error("periodic column too short for the spectral kernel");
        const int NCp = (int)std::max<size_t>(1, std::min<size_t>(kPipeThreads / Tp, 225 * 1024 / per_col));
        const size_t psmem = per_col * NCp;
        const int64_t nitems = (int64_t)((pl.ncols + NCp - 1) / NCp) * batch;
        const unsigned pgrid = (unsigned)std::min<int64_t>(nitems, e.num_sms);
#define PIPE_ARGS spec, e.d_S2, e.d_sym, e.d_coltab, e.M, pl.ncols, pl.Nl, NCp, batch, e.d_tw, pl.logTWN
        if (mode == 2)
            PDGPU_DISPATCH_LOGQ(lq, (k_spectral2d_pipe<LQ, 2><<<pgrid, NCp * Tp, psmem, s>>>(PIPE_ARGS)))
        else if (mode == 1)
            PDGPU_DISPATCH_LOGQ(lq, (k_spectral2d_pipe<LQ, 1><<<pgrid, NCp * Tp, psmem, s>>>(PIPE_ARGS)))
        else
            PDGPU_DISPATCH_LOGQ(lq, (k_spectral2d_pipe<LQ, 0><<<pgrid, NCp * Tp, psmem, s>>>(PIPE_ARGS)))
#undef PIPE_ARGS
    }
}
#endif

#if defined(PDGPU_ALL_PARTS) || PDGPU_PART == 4
template <int L, bool C>
static void set_attrs_3d_l() {
    smem_attr((const void*)k_cfft_y_fwd<L, C>);
    smem_attr((const void*)k_cfft_y_inv<L, C>);
    if constexpr (!C) {
        smem_attr((const void*)k_spectral<L, 3, true, 3, true>);
        smem_attr((const void*)k_spectral<L, 3, false, 3, true>);
        smem_attr((const void*)k_spectral<L, 3, true, 3, true, true>);
    } else {
        smem_attr((const void*)k_spectral<L, 3, true, 3, false, false, 1>);
        smem_attr((const void*)k_spectral<L, 3, false, 3, false, false, 1>);
        smem_attr((const void*)k_spectral<L, 3, true, 3, false, true, 1>);
        if constexpr (L == 7 || L == 8) smem_attr((const void*)k_spectral<L, 3, true, 4, false, false, 1>);
    }
}
template <int... Ls>
static void set_attrs_3d_all(std::integer_sequence<int, Ls...>) {
    (set_attrs_3d_l<Ls + 1, false>(), ...);
    (set_attrs_3d_l<Ls + 1, true>(), ...);
}
void set_attrs_3d() { set_attrs_3d_all(std::make_integer_sequence<int, 9>{}); }

void launch_k2_3d(Engine& e, int batch, cudaStream_t s) {
    const Plan& pl = e.plan;
    const int Ny = pl.N[1], Nz = pl.N[2];
    const int ZT = pl.k2_zt;
    const int lq = pl.logP[1] - 1;
    const int T = threads_per_transform(lq, 4);
    dim3 grid((Nz + ZT - 1) / ZT, pl.Hx, batch * pl.dim);
    const size_t smem = sizeof(double2) * (size_t)2 * ZT * xbuf_slots(lq);
    if (pl.circ[1])
        PDGPU_DISPATCH_LOGQ9(lq, (k_cfft_y_fwd<LQ, true><<<grid, 2 * ZT * T, smem, s>>>(e.d_S1, e.d_S2, Ny, Nz, pl.Hx,
                                                                                    ZT, e.d_tw, pl.logTWN)))
    else
        PDGPU_DISPATCH_LOGQ9(lq, (k_cfft_y_fwd<LQ, false><<<grid, 2 * ZT * T, smem, s>>>(e.d_S1, e.d_S2, Ny, Nz, pl.Hx,
                                                                                     ZT, e.d_tw, pl.logTWN)))
}

void launch_k4_3d(Engine& e, int batch, cudaStream_t s) {
    const Plan& pl = e.plan;
    const int Ny = pl.N[1], Nz = pl.N[2];
    const int ZT = pl.k2_zt;
    const int lq = pl.logP[1] - 1;
    const int T = threads_per_transform(lq, 4);
    dim3 grid((Nz + ZT - 1) / ZT, pl.Hx, batch * pl.dim);
    const size_t smem = sizeof(double2) * (size_t)2 * ZT * xbuf_slots(lq);
    if (pl.circ[1])
        PDGPU_DISPATCH_LOGQ9(lq, (k_cfft_y_inv<LQ, true><<<grid, 2 * ZT * T, smem, s>>>(e.d_S2, e.d_S1, Ny, Nz, pl.Hx,
                                                                                    ZT, e.d_tw, pl.logTWN)))
    else
        PDGPU_DISPATCH_LOGQ9(lq, (k_cfft_y_inv<LQ, false><<<grid, 2 * ZT * T, smem, s>>>(e.d_S2, e.d_S1, Ny, Nz, pl.Hx,
                                                                                     ZT, e.d_tw, pl.logTWN)))
}

// 3D K3 in place on S2
void launch_k3_3d(Engine& e, double2* spec, int batch, cudaStream_t s) {
    const Plan& pl = e.plan;
    const int d = pl.dim;
    const int NC = pl.k3_cols;
    const int nh = pl.nh;
    const int lq = pl.logPl - (nh == 2 ? 1 : 0);
    const int T = threads_per_transform(lq, 3);
    dim3 grid(batch, (pl.ncols + NC - 1) / NC);
    const bool zsmem = nh == 2;
    const size_t smem = sizeof(double2) * (size_t)NC * (xbuf_slots(lq) + (zsmem ? 2 * d - 1 : d - 1) * (1 << lq));
    const double* ct = e.d_coltab;
    const int M = e.M, om = e.coltab_oddmask;
    if (e.d_coltab) {
        // per-column coefficient block in SMEM: shrink the column group to fit
        const size_t per_col = smem / NC + sizeof(double) * 6 * (e.M + 1);
        int NCs = NC;
        while (NCs > 1 && per_col * NCs > 225 * 1024) NCs >>= 1;
        dim3 sgrid(batch, (pl.ncols + NCs - 1) / NCs);
        if (nh == 1)
            PDGPU_DISPATCH_LOGQ9(lq, (k_spectral<LQ, 3, true, 3, false, true, 1><<<sgrid, NCs * T, per_col * NCs, s>>>(
                                         spec, spec, e.d_sym, pl.ncols, pl.Nl, NCs, e.d_tw, pl.logTWN, ct, M, om)))
        else
            PDGPU_DISPATCH_LOGQ9(lq, (k_spectral<LQ, 3, true, 3, true, true><<<sgrid, NCs * T, per_col * NCs, s>>>(
                                         spec, spec, e.d_sym, pl.ncols, pl.Nl, NCs, e.d_tw, pl.logTWN, ct, M, om)))
    } else if (e.real_symbol) {
        // 128/256-point periodic columns: 16 points per thread (256 = 16 x 16: one exchange
        // per transform instead of the two of 8 x 8 x 4); PDGPU_K3_3D_R8=1: 8 points per thread
        if (nh == 1 && (lq == 8 || lq == 7) && !getenv("PDGPU_K3_3D_R8")) {
            const int T16 = threads_per_transform(lq, 4);
            if (lq == 8)
                k_spectral<8, 3, true, 4, false, false, 1><<<grid, NC * T16, smem, s>>>(spec, spec, e.d_sym, pl.ncols, pl.Nl,
                                                                                       NC, e.d_tw, pl.logTWN);
            else
                k_spectral<7, 3, true, 4, false, false, 1><<<grid, NC * T16, smem, s>>>(spec, spec, e.d_sym, pl.ncols, pl.Nl,
                                                                                       NC, e.d_tw, pl.logTWN);
        } else if (nh == 1)
            PDGPU_DISPATCH_LOGQ9(lq, (k_spectral<LQ, 3, true, 3, false, false, 1><<<grid, NC * T, smem, s>>>(
                                         spec, spec, e.d_sym, pl.ncols, pl.Nl, NC, e.d_tw, pl.logTWN)))
        else
            PDGPU_DISPATCH_LOGQ9(lq, (k_spectral<LQ, 3, true, 3, true><<<grid, NC * T, smem, s>>>(
                                         spec, spec, e.d_sym, pl.ncols, pl.Nl, NC, e.d_tw, pl.logTWN)))
    } else {
        if (nh == 1)
            PDGPU_DISPATCH_LOGQ9(lq, (k_spectral<LQ, 3, false, 3, false, false, 1><<<grid, NC * T, smem, s>>>(
                                         spec, spec, e.d_sym, pl.ncols, pl.Nl, NC, e.d_tw, pl.logTWN)))
        else
            PDGPU_DISPATCH_LOGQ9(lq, (k_spectral<LQ, 3, false, 3, true><<<grid, NC * T, smem, s>>>(
                                         spec, spec, e.d_sym, pl.ncols, pl.Nl, NC, e.d_tw, pl.logTWN)))
    }
}
#endif

#if defined(PDGPU_ALL_PARTS) || PDGPU_PART == 0
void set_kernel_attributes() {
    static bool done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && done[dev]) return;
    set_attrs_k1();
    set_attrs_k5();
    set_attrs_k3_2d();
    set_attrs_3d();
    if (dev < 64) done[dev] = true;
}

void build_twiddles(Engine& e) {
    const int n = 1 << e.plan.logTWN;
    std::vector<double2> tw(n);
    for (int k = 0; k < n; ++k) {
        const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)k / (long double)n;
        tw[k] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    tw[0] = make_double2(1.0, 0.0);
    if (n >= 4) {
        tw[n / 4] = make_double2(0.0, -1.0);
        tw[n / 2] = make_double2(-1.0, 0.0);
        tw[3 * n / 4] = make_double2(0.0, 1.0);
    }
    if (e.d_tw) cudaFree(e.d_tw);
    check(cudaMalloc(&e.d_tw, sizeof(double2) * n), "alloc twiddles");
    check(cudaMemcpy(e.d_tw, tw.data(), sizeof(double2) * n, cudaMemcpyHostToDevice), "copy twiddles");
}

void build_symbol(Engine& e) {
    const Plan& pl = e.plan;
    const int64_t nfreq = (int64_t)pl.ncols * pl.Pl;
    const size_t elt = e.real_symbol ? sizeof(double) : sizeof(double2);
    // 2D real symbols are stored 4 doubles per frequency (one 32-byte load, symbol_product)
    const int ns = (e.dim == 2 && e.real_symbol) ? 4 : e.np;
    if (e.d_sym) cudaFree(e.d_sym);
    check(cudaMalloc(&e.d_sym, elt * nfreq * ns), "alloc symbol");
    const double scale = 1.0 / ((double)pl.P[0] * (double)pl.P[1] * (double)pl.P[2]);
    const int th = 128;
    const int64_t blocks = (nfreq + th - 1) / th;
    k_build_symbol<<<(unsigned)blocks, th, 0, e.stream>>>(e.d_sym, e.d_K, e.dim, e.M, e.np, e.ss, pl.ncols, pl.Pl,
                                                         pl.P[0], pl.P[1], pl.P[2], e.real_symbol ? 1 : 0, scale, pl.nh, ns,
                                                         0);
    check(cudaGetLastError(), "build_symbol launch");
    check(cudaStreamSynchronize(e.stream), "build_symbol");
    build_symbol_half(e);
}

// Mirror planes of the 2D real symbol for 4096-point periodic columns.  A
// stencil of definite parity along y (the physical kernels: xx and yy even, xy
// odd, kernel.hpp:109-116) has H(kx, Pl - ky) = +-H(kx, ky), so the planes over
// ky in [0, Pl/2] carry the whole column: 24 bytes per two frequencies instead
// of 64, small enough to land in K3's exchange buffer.  The identity is
// checked on the table itself; any other stencil keeps the full table.
__global__ void k_symbol_half(const double* __restrict__ sym, double* __restrict__ symh, int ncols, int Q, int HP,
                              unsigned long long* __restrict__ stat) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int nk = Q / 2 + 1;
    double dmax = 0.0, hmax = 0.0;
    if (i < (int64_t)ncols * nk) {
        const int col = (int)(i / nk), k = (int)(i % nk);
        const double* a = sym + ((int64_t)col * Q + k) * 4;
        const double* m = sym + ((int64_t)col * Q + ((Q - k) & (Q - 1))) * 4;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            const double v = a[p];
            symh[((int64_t)col * 3 + p) * HP + k] = v;
            dmax = fmax(dmax, fabs(m[p] - (p == 1 ? -v : v)));
            hmax = fmax(hmax, fabs(v));
        }
    }
    // non-negative doubles order like their bit patterns
    atomicMax(stat, (unsigned long long)__double_as_longlong(dmax));
    atomicMax(stat + 1, (unsigned long long)__double_as_longlong(hmax));
}

void build_symbol_half(Engine& e) {
    const Plan& pl = e.plan;
    if (e.d_symh) cudaFree(e.d_symh);
    e.d_symh = nullptr;
    e.symh_for = nullptr;
    if (e.dim != 2 || !e.real_symbol || pl.nh != 1 || pl.logPl < 9 || pl.logPl > 12 || getenv("PDGPU_NO_SYMH")) return;
    const int Q = pl.Pl, HP = Q / 2 + 8;
    unsigned long long* d_stat = nullptr;
    check(cudaMalloc(&e.d_symh, sizeof(double) * (size_t)pl.ncols * 3 * HP), "alloc symbol planes");
    check(cudaMalloc(&d_stat, 2 * sizeof(unsigned long long)), "alloc symbol stat");
    check(cudaMemsetAsync(e.d_symh, 0, sizeof(double) * (size_t)pl.ncols * 3 * HP, e.stream), "symbol planes");
    check(cudaMemsetAsync(d_stat, 0, 2 * sizeof(unsigned long long), e.stream), "symbol stat");
    const int64_t n = (int64_t)pl.ncols * (Q / 2 + 1);
    k_symbol_half<<<(unsigned)((n + 255) / 256), 256, 0, e.stream>>>((const double*)e.d_sym, e.d_symh, pl.ncols, Q, HP,
                                                                   d_stat);
    check(cudaGetLastError(), "symbol planes launch");
    unsigned long long h[2];
    check(cudaMemcpyAsync(h, d_stat, sizeof(h), cudaMemcpyDeviceToHost, e.stream), "symbol stat copy");
    check(cudaStreamSynchronize(e.stream), "symbol planes");
    cudaFree(d_stat);
    double dmax, hmax;
    memcpy(&dmax, &h[0], 8);
    memcpy(&hmax, &h[1], 8);
    if (dmax <= 1e-14 * hmax) {
        e.symh_for = e.d_sym;
        e.symh_stride = HP;
    } else {
        cudaFree(e.d_symh);
        e.d_symh = nullptr;
    }
}

// symbol of columns [col0, col0 + pl.ncols) of plan pl (2D distributed FFT)
void build_symbol_cols(Engine& e, const Plan& pl, int col0, void** out) {
    const int64_t nfreq = (int64_t)pl.ncols * pl.Pl;
    const size_t elt = e.real_symbol ? sizeof(double) : sizeof(double2);
    const int ns = e.real_symbol ? 4 : e.np;
    if (*out) cudaFree(*out);
    *out = nullptr;
    check(cudaMalloc(out, elt * std::max<int64_t>(nfreq, 1) * ns), "alloc column symbol");
    const double scale = 1.0 / ((double)pl.P[0] * (double)pl.P[1]);
    const int th = 128;
    k_build_symbol<<<(unsigned)((nfreq + th - 1) / th), th, 0, e.stream>>>(*out, e.d_K, 2, e.M, e.np, e.ss, pl.ncols,
                                                                           pl.Pl, pl.P[0], pl.P[1], 1,
                                                                           e.real_symbol ? 1 : 0, scale, 1, ns, col0);
    check(cudaGetLastError(), "column symbol launch");
    check(cudaStreamSynchronize(e.stream), "column symbol");
}

// K3 of a distributed-FFT rank: its columns (plan col, symbol sym) from in to out
void launch_k3_2d_cols(Engine& e, const Plan& col, void* sym, const double2* in, double2* out, int batch,
                       cudaStream_t s) {
    Plan saved = e.plan;
    void* ssym = e.d_sym;
    double2* sS2 = e.d_S2;
    double* sct = e.d_coltab;
    e.plan.ncols = col.ncols;
    e.plan.Nl = col.Nl;
    e.plan.Pl = col.Pl;
    e.plan.logPl = col.logPl;
    e.plan.nh = 1;
    e.d_sym = sym;
    e.d_S2 = out;
    e.d_coltab = nullptr;
    try {
        launch_k3_2d(e, in, batch, s);
    } catch (...) {
        e.plan = saved;
        e.d_sym = ssym;
        e.d_S2 = sS2;
        e.d_coltab = sct;
        throw;
    }
    e.plan = saved;
    e.d_sym = ssym;
    e.d_S2 = sS2;
    e.d_coltab = sct;
}

void engine_alloc_workspace(Engine& e, int64_t batch) {
    if (batch <= e.cap_batch) return;
    // a captured CG iteration holds the workspace pointers it was recorded with
    touch_state(e);
    if (e.d_S1) cudaFree(e.d_S1);
    if (e.d_S2) cudaFree(e.d_S2);
    e.d_S1 = e.d_S2 = nullptr;
    const Plan& pl = e.plan;
    check(cudaMalloc(&e.d_S1, sizeof(double2) * pl.S1_per_vec * batch), "alloc S1");
    if (pl.S2_per_vec) check(cudaMalloc(&e.d_S2, sizeof(double2) * pl.S2_per_vec * batch), "alloc S2");
    if (e.d_xstrip) cudaFree(e.d_xstrip);
    if (e.d_fx) cudaFree(e.d_fx);
    e.d_xstrip = nullptr;
    e.d_fx = nullptr;
    if (pl.dim == 3 && pl.circ[0]) {  // 4M x-values per (y, z) row and component; 2M x-pass results
        check(cudaMalloc(&e.d_xstrip, sizeof(double) * (size_t)batch * 3 * 4 * e.M * pl.N[1] * pl.N[2]), "alloc strip");
        check(cudaMalloc(&e.d_fx, sizeof(double) * (size_t)batch * 3 * 2 * e.M * pl.N[1] * pl.N[2]), "alloc fx");
    }
    e.cap_batch = batch;
}

void launch_fast_apply(Engine& e, const double* u, double* f, int batch, cudaStream_t s, double scale,
                       const uint8_t* cmask, const double* body) {
    const Plan& pl = e.plan;
    if (e.a2a.G > 0 && !e.a2a_external) {  // distributed FFT arm (transpose.cu), NCCL or one rank
        a2a_phase1(e, u, batch, s);
        a2a_exchange(e, batch, s);
        a2a_phase2(e, batch, s);
        a2a_exchange(e, batch, s);
        a2a_phase3(e, f, batch, s, scale, cmask, body);
        a2a_alias(e, u, batch, s);
        PassTimer pt(e, kPassCorr, s);
        launch_wrap_correction(e, u, f, batch, s, scale, cmask);
        check(cudaGetLastError(), "fast_apply launch");
        return;
    }
    engine_alloc_workspace(e, batch);
    const int d = pl.dim;
    // halo slabs over NCCL: the M rows beyond each interior face travel on the
    // comm stream while K1..K5 run (they read only the owned rows); K6w waits
    const double* halo = halo_exchange_begin(e, u, batch, s);
    if (!halo) {  // the caller's ghost rows (pdgpu_set_ghosts), [batch][dim][2][M][plane]
        const int64_t plane = d == 3 ? (int64_t)pl.N[0] * pl.N[1] : pl.N[0];
        e.ghost_view = e.d_ghost;
        e.ghost_bc_stride = e.user_ghost_bc ? e.user_ghost_bc : 2 * e.M * plane;
        e.ghost_side_stride = e.user_ghost_side ? e.user_ghost_side : e.M * plane;
    }
    {
        PassTimer pt(e, kPassK1, s);
        launch_k1(e, u, batch, s);
    }
    double2* spec = e.d_S1;
    if (d == 3) {
        PassTimer pt(e, kPassK2, s);
        launch_k2_3d(e, batch, s);
        spec = e.d_S2;
    }
    double2* xin = e.d_S1;
    {
        PassTimer pt(e, kPassK3, s);
        if (d == 2) {
            launch_k3_2d(e, spec, batch, s, /*blocked_ok=*/true);
            xin = e.d_S2;
        } else {
            launch_k3_3d(e, spec, batch, s);
        }
    }
    if (d == 3) {
        PassTimer pt(e, kPassK4, s);
        launch_k4_3d(e, batch, s);
    }
    if (d == 3 && (pl.circ_mask || e.ghost_view)) {  // 3D face path: the wrap x pass feeds K5's epilogue
        PassTimer pt(e, kPassCorr, s);
        launch_wrap_xpass(e, u, batch, s, scale, cmask);
    }
    {
        PassTimer pt(e, kPassK5, s);
        launch_k5(e, xin, f, batch, s, scale, cmask, body);
    }
    if (halo) halo_exchange_end(e, s);
    if (pl.circ_mask || e.ghost_view) {  // K6w: wrap correction / slab ghost rows (timed with the corrections)
        PassTimer pt(e, kPassCorr, s);
        launch_wrap_correction(e, u, f, batch, s, scale, cmask);
    }
    check(cudaGetLastError(), "fast_apply launch");
}
#endif

}  // namespace pdgpu
