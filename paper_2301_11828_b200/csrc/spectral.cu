// spectral.cu -- the MSBFM spectral product f = A_hat u on sm_100a.
//
// Replaces FastForce<Dim>::apply (reference convolution.hpp:249-259): d
// forward padded FFTs (forward_field :119-128), the d x d per-frequency
// product with conj(G_hat) (hadamard :135-154) and d inverse FFTs with window
// extraction (inverse_extract :158-172).
//
// Pass structure (one vector; B vectors batch into the grid):
//   K1 rfft_rows   : real rows along x -> half spectrum (Hx = Px/2+1), written
//                    transposed [kx][row] so the next pass reads contiguously.
//   K2 cfft_y_fwd  : (3D) padded y FFT, written transposed [kx][ky][z].
//   K3 spectral    : padded FFT along the last axis, d x d symbol multiply,
//                    inverse FFT, truncation to the window -- fused, one CTA
//                    per column group, all d components resident in SMEM.
//   K4 cfft_y_inv  : (3D) inverse y FFT + truncation, transposed back.
//   K5 irfft_rows  : C2R along x + truncation + epilogue (scale, constraint
//                    mask, body force), written in the reference's node order.
// The symbol (K9, build_symbol) is conj(G_hat)/prod(P) evaluated once by a
// direct DFT of the (2M+1)^d stencil: real for the physical (even) stencils,
// complex for arbitrary ones (the reference's random-stencil tests).
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <stdexcept>

#include "engine.h"
#include "fft.cuh"

namespace pdgpu {

static inline int ilog2(int64_t v) {
    int l = 0;
    while ((int64_t(1) << l) < v) ++l;
    return l;
}

void plan_init(Plan& pl, int dim, const int* dims) {
    pl.dim = dim;
    for (int d = 0; d < 3; ++d) {
        pl.N[d] = d < dim ? dims[d] : 1;
        if (d < dim) {
            const int lp = ilog2(pl.N[d]);
            pl.logP[d] = lp + 1;
            pl.P[d] = 1 << (lp + 1);
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
        pl.S1_per_vec = (int64_t)dim * pl.Hx * pl.N[1];
        pl.S2_per_vec = pl.S1_per_vec;
    } else {
        pl.ncols = pl.Hx * pl.P[1];
        pl.Nl = pl.N[2];
        pl.Pl = pl.P[2];
        pl.logPl = pl.logP[2];
        pl.S1_per_vec = (int64_t)dim * pl.N[2] * pl.Hx * pl.N[1];
        pl.S2_per_vec = (int64_t)dim * pl.Hx * pl.P[1] * pl.N[2];
    }
    pl.logTWN = std::max(pl.logP[0], std::max(pl.logP[1], pl.logP[2]));
    const int64_t row_bytes = (int64_t)(pl.P[0] / 2) * 16;
    pl.k1_rows = (int)std::max<int64_t>(1, std::min<int64_t>(8, 131072 / row_bytes));
    const int64_t col_bytes_both = (int64_t)dim * pl.Pl * 16;
    if (col_bytes_both <= 200 * 1024) {
        pl.k3_halves = 2;
        pl.k3_cols = (int)std::max<int64_t>(1, std::min<int64_t>(8, 98304 / col_bytes_both));
    } else {
        pl.k3_halves = 1;
        pl.k3_cols = 1;
    }
    if (dim == 3) {
        const int64_t yrow = (int64_t)pl.P[1] * 16;
        pl.k2_zt = (int)std::max<int64_t>(1, std::min<int64_t>(8, 65536 / yrow));
        pl.k2_zt = std::min(pl.k2_zt, pl.N[2]);
    }
}

// ------------------------------------------------------------------ K1 ---
template <int IPT>
__global__ void __launch_bounds__(1024) k_rfft_rows(const double* __restrict__ u, double2* __restrict__ S,
                                                    int Nx, int Nrow, int Hx, int logQx, int TR,
                                                    const double2* __restrict__ tw, int logTWN) {
    extern __shared__ double2 sm[];
    const int Qx = 1 << logQx;
    const int slab = blockIdx.y;
    const int row0 = blockIdx.x * TR;
    const int nr = min(TR, Nrow - row0);
    const double* src = u + ((int64_t)slab * Nrow + row0) * Nx;
    const int shE = logTWN - (logQx + 1);  // exp(-2 pi i n / (2Qx))
    for (int idx = threadIdx.x; idx < nr * Qx; idx += blockDim.x) {
        const int r = idx >> logQx, n = idx & (Qx - 1);
        const int i0 = 2 * n;
        const double a = i0 < Nx ? src[(int64_t)r * Nx + i0] : 0.0;
        const double b = i0 + 1 < Nx ? src[(int64_t)r * Nx + i0 + 1] : 0.0;
        const double2 z = make_double2(a, b);
        sm[(r << (logQx + 1)) + n] = z;
        sm[(r << (logQx + 1)) + Qx + n] = cmul(z, __ldg(tw + (n << shE)));
    }
    __syncthreads();
    block_fft<-1, IPT>(sm, 2 * nr, logQx, tw, logTWN);
    const int halfP = 2 * Qx;
    const int shX = logTWN - (logQx + 2);  // exp(-2 pi i k / Px)
    for (int idx = threadIdx.x; idx < nr * Hx; idx += blockDim.x) {
        const int kx = idx / nr, r = idx - kx * nr;
        const int k = kx & (halfP - 1);
        const int k2 = (halfP - kx) & (halfP - 1);
        const double2* Z = sm + (r << (logQx + 1));
        const double2 A = Z[(k & 1) * Qx + (k >> 1)];
        const double2 B = cconj(Z[(k2 & 1) * Qx + (k2 >> 1)]);
        const double2 Fe = cscale(cadd(A, B), 0.5);
        const double2 D = csub(A, B);
        const double2 Fo = make_double2(0.5 * D.y, -0.5 * D.x);
        const double2 W = __ldg(tw + (kx << shX));
        S[((int64_t)slab * Hx + kx) * Nrow + row0 + r] = cadd(Fe, cmul(W, Fo));
    }
}

// ------------------------------------------------------------------ K5 ---
template <int IPT, bool MASK, bool BODY>
__global__ void __launch_bounds__(1024) k_irfft_rows(const double2* __restrict__ S, double* __restrict__ f,
                                                     int Nx, int Nrow, int Nz, int dim, int Hx, int logQx,
                                                     int TR, const double2* __restrict__ tw, int logTWN,
                                                     double scale, const uint8_t* __restrict__ cmask,
                                                     const double* __restrict__ body, int64_t nodes) {
    extern __shared__ double2 sm[];
    const int Qx = 1 << logQx;
    const int halfP = 2 * Qx;
    const int slab = blockIdx.y;
    const int row0 = blockIdx.x * TR;
    const int nr = min(TR, Nrow - row0);
    const int shX = logTWN - (logQx + 2);  // exp(+2 pi i k / Px)
    const double2* src = S + (int64_t)slab * Hx * Nrow + row0;
    // Z[k] = (X[k] + conj X[h-k]) + i e^{+2 pi i k/Px} (X[k] - conj X[h-k]),  h = Px/2
    for (int idx = threadIdx.x; idx < nr * (Qx + 1); idx += blockDim.x) {
        const int k = idx / nr, r = idx - k * nr;
        const int k2 = halfP - k;
        const double2 Xa = src[(int64_t)k * Nrow + r];
        const double2 Xb = src[(int64_t)k2 * Nrow + r];
        double2* Z = sm + (r << (logQx + 1));
        {
            const double2 s = cadd(Xa, cconj(Xb));
            const double2 dd = csub(Xa, cconj(Xb));
            const double2 W = twiddle<1>(tw, k << shX);
            const double2 t = cmul(W, dd);
            const double2 z = make_double2(s.x - t.y, s.y + t.x);
            Z[(k & 1) * Qx + (k >> 1)] = z;
        }
        if (k != 0 && k != Qx) {
            const double2 s = cadd(Xb, cconj(Xa));
            const double2 dd = csub(Xb, cconj(Xa));
            const double2 W = twiddle<1>(tw, k2 << shX);
            const double2 t = cmul(W, dd);
            const double2 z = make_double2(s.x - t.y, s.y + t.x);
            Z[(k2 & 1) * Qx + (k2 >> 1)] = z;
        }
    }
    __syncthreads();
    block_fft<1, IPT>(sm, 2 * nr, logQx, tw, logTWN);
    const int shE = logTWN - (logQx + 1);  // exp(+2 pi i n / (2Qx))
    const int a = (slab / Nz) % dim;
    const int z = slab % Nz;
    double* dst = f + ((int64_t)slab * Nrow + row0) * Nx;
    for (int idx = threadIdx.x; idx < nr * Qx; idx += blockDim.x) {
        const int r = idx >> logQx, n = idx & (Qx - 1);
        const int i0 = 2 * n;
        if (i0 >= Nx) continue;
        const double2* Z = sm + (r << (logQx + 1));
        const double2 zz = cadd(Z[n], cmul(twiddle<1>(tw, n << shE), Z[Qx + n]));
        const int64_t node = ((int64_t)z * Nrow + row0 + r) * Nx + i0;
        double v0 = zz.x * scale, v1 = zz.y * scale;
        if (BODY) {
            v0 += body[(int64_t)a * nodes + node];
            if (i0 + 1 < Nx) v1 += body[(int64_t)a * nodes + node + 1];
        }
        if (MASK) {
            if ((cmask[node] >> a) & 1u) v0 = 0.0;
            if (i0 + 1 < Nx && ((cmask[node + 1] >> a) & 1u)) v1 = 0.0;
        }
        dst[(int64_t)r * Nx + i0] = v0;
        if (i0 + 1 < Nx) dst[(int64_t)r * Nx + i0 + 1] = v1;
    }
}

// ------------------------------------------------------------------ K3 ---
// Columns: in[((b*D + c)*ncols + col)*Nl + n], n < Nl.  Symbol H[(pair*ncols + col)*Pl + k].
// SMEM layout [cc][c][hh][Ql].  NH = 2: both half spectra resident (in-place
// allowed).  NH = 1: the two halves run back to back, the second accumulates
// into `out` (out must not alias in).
template <int D>
__device__ __forceinline__ int pair_of(int a, int b) {
    if (a > b) { const int t = a; a = b; b = t; }
    if (D == 2) return a + b;
    return (a == 0 ? 0 : (a == 1 ? 3 : 5)) + b - a;
}

template <int IPT, int D, bool REAL>
__global__ void __launch_bounds__(1024) k_spectral(const double2* in, double2* out, const void* __restrict__ sym,
                                                   int ncols, int Nl, int logPl, int NC, int NH,
                                                   const double2* __restrict__ tw, int logTWN) {
    extern __shared__ double2 sm[];
    const int logQl = logPl - 1;
    const int Ql = 1 << logQl;
    const int Pl = 1 << logPl;
    const int col0 = blockIdx.x * NC;
    const int nc = min(NC, ncols - col0);
    const int b = blockIdx.y;
    const int shP = logTWN - logPl;  // exp(-+2 pi i n / Pl)
    const int npass = NH == 2 ? 1 : 2;
    for (int pass = 0; pass < npass; ++pass) {
        // load (+ odd-half pre-twiddle)
        for (int idx = threadIdx.x; idx < nc * D * Ql; idx += blockDim.x) {
            const int n = idx & (Ql - 1);
            const int t = idx >> logQl;  // cc*D + c
            const int cc = t / D, c = t - cc * D;
            double2 v = make_double2(0.0, 0.0);
            if (n < Nl) v = in[((int64_t)(b * D + c) * ncols + col0 + cc) * Nl + n];
            if (NH == 2) {
                sm[((t * 2) << logQl) + n] = v;
                sm[((t * 2 + 1) << logQl) + n] = cmul(v, __ldg(tw + (n << shP)));
            } else {
                sm[(t << logQl) + n] = pass ? cmul(v, __ldg(tw + (n << shP))) : v;
            }
        }
        __syncthreads();
        block_fft<-1, IPT>(sm, nc * D * NH, logQl, tw, logTWN);
        // per-frequency d x d product with the symbol
        for (int idx = threadIdx.x; idx < nc * NH * Ql; idx += blockDim.x) {
            const int m = idx & (Ql - 1);
            const int rest = idx >> logQl;  // cc*NH + hh
            const int cc = rest / NH, hh = rest - cc * NH;
            const int h = NH == 2 ? hh : pass;
            const int ky = 2 * m + h;
            const int col = col0 + cc;
            double2 U[D];
#pragma unroll
            for (int c = 0; c < D; ++c) U[c] = sm[(((cc * D + c) * NH + hh) << logQl) + m];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const int64_t si = ((int64_t)pair_of<D>(a, c) * ncols + col) * Pl + ky;
                    if (REAL) {
                        const double g = __ldg((const double*)sym + si);
                        acc.x += g * U[c].x;
                        acc.y += g * U[c].y;
                    } else {
                        acc = cadd(acc, cmul(__ldg((const double2*)sym + si), U[c]));
                    }
                }
                sm[(((cc * D + a) * NH + hh) << logQl) + m] = acc;
            }
        }
        __syncthreads();
        block_fft<1, IPT>(sm, nc * D * NH, logQl, tw, logTWN);
        // combine halves, truncate to the window, store
        for (int idx = threadIdx.x; idx < nc * D * Nl; idx += blockDim.x) {
            const int t = idx / Nl, n = idx - t * Nl;
            const int cc = t / D, a = t - cc * D;
            const int64_t o = ((int64_t)(b * D + a) * ncols + col0 + cc) * Nl + n;
            double2 y;
            if (NH == 2) {
                y = cadd(sm[((t * 2) << logQl) + n],
                         cmul(twiddle<1>(tw, n << shP), sm[((t * 2 + 1) << logQl) + n]));
            } else {
                y = sm[(t << logQl) + n];
                if (pass) y = cadd(out[o], cmul(twiddle<1>(tw, n << shP), y));
            }
            out[o] = y;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------- K2 / K4 (3D) ---
template <int IPT>
__global__ void __launch_bounds__(1024) k_cfft_y_fwd(const double2* __restrict__ S1, double2* __restrict__ S2,
                                                     int Ny, int Nz, int Hx, int logPy, int ZT,
                                                     const double2* __restrict__ tw, int logTWN) {
    extern __shared__ double2 sm[];
    const int logQ = logPy - 1, Q = 1 << logQ, Py = 1 << logPy;
    const int z0 = blockIdx.x * ZT;
    const int nz = min(ZT, Nz - z0);
    const int kx = blockIdx.y;
    const int bd = blockIdx.z;
    const int shP = logTWN - logPy;
    for (int idx = threadIdx.x; idx < nz * Q; idx += blockDim.x) {
        const int zz = idx >> logQ, n = idx & (Q - 1);
        double2 v = make_double2(0.0, 0.0);
        if (n < Ny) v = S1[(((int64_t)bd * Nz + z0 + zz) * Hx + kx) * Ny + n];
        sm[((zz * 2) << logQ) + n] = v;
        sm[((zz * 2 + 1) << logQ) + n] = cmul(v, __ldg(tw + (n << shP)));
    }
    __syncthreads();
    block_fft<-1, IPT>(sm, 2 * nz, logQ, tw, logTWN);
    for (int idx = threadIdx.x; idx < Py * nz; idx += blockDim.x) {
        const int ky = idx / nz, zz = idx - ky * nz;
        S2[(((int64_t)bd * Hx + kx) * Py + ky) * Nz + z0 + zz] = sm[((zz * 2 + (ky & 1)) << logQ) + (ky >> 1)];
    }
}

template <int IPT>
__global__ void __launch_bounds__(1024) k_cfft_y_inv(const double2* __restrict__ S2, double2* __restrict__ S1,
                                                     int Ny, int Nz, int Hx, int logPy, int ZT,
                                                     const double2* __restrict__ tw, int logTWN) {
    extern __shared__ double2 sm[];
    const int logQ = logPy - 1, Py = 1 << logPy;
    const int z0 = blockIdx.x * ZT;
    const int nz = min(ZT, Nz - z0);
    const int kx = blockIdx.y;
    const int bd = blockIdx.z;
    const int shP = logTWN - logPy;
    for (int idx = threadIdx.x; idx < Py * nz; idx += blockDim.x) {
        const int ky = idx / nz, zz = idx - ky * nz;
        sm[((zz * 2 + (ky & 1)) << logQ) + (ky >> 1)] = S2[(((int64_t)bd * Hx + kx) * Py + ky) * Nz + z0 + zz];
    }
    __syncthreads();
    block_fft<1, IPT>(sm, 2 * nz, logQ, tw, logTWN);
    for (int idx = threadIdx.x; idx < nz * Ny; idx += blockDim.x) {
        const int zz = idx / Ny, n = idx - zz * Ny;
        const double2 y = cadd(sm[((zz * 2) << logQ) + n], cmul(twiddle<1>(tw, n << shP), sm[((zz * 2 + 1) << logQ) + n]));
        S1[(((int64_t)bd * Nz + z0 + zz) * Hx + kx) * Ny + n] = y;
    }
}

// ------------------------------------------------------------ symbol K9 --
// H(k) = scale * sum_o K(o) exp(+2 pi i k.o / P) = conj(G_hat(k)) / prod(P)
// (convolution.hpp:107-116 embeds K at wrapped offsets and FFTs; the product
// at :140-153 uses conj(G_hat)).  Direct DFT over the stencil, phases exact.
__global__ void k_build_symbol(void* sym, const double* __restrict__ K, int dim, int M, int np, int64_t ss,
                               int ncols, int Pl, int P0, int P1, int P2, int real, double scale) {
    const int64_t nfreq = (int64_t)ncols * Pl;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nfreq) return;
    const int col = (int)(idx / Pl), kl = (int)(idx % Pl);
    int k0, k1, k2;
    if (dim == 2) { k0 = col; k1 = kl; k2 = 0; }
    else { k0 = col / P1; k1 = col % P1; k2 = kl; }
    const int side = 2 * M + 1;
    double2 ex[17], ey[17], ez[17];
    for (int o = -M; o <= M; ++o) {
        double s, c;
        int m0 = (int)(((int64_t)k0 * (o + P0)) % P0);
        sincospi(2.0 * (double)m0 / (double)P0, &s, &c);
        ex[o + M] = make_double2(c, s);
        int m1 = (int)(((int64_t)k1 * (o + P1)) % P1);
        sincospi(2.0 * (double)m1 / (double)P1, &s, &c);
        ey[o + M] = make_double2(c, s);
        if (dim == 3) {
            int m2 = (int)(((int64_t)k2 * (o + P2)) % P2);
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
    for (int p = 0; p < np; ++p) {
        const int64_t o = (int64_t)p * nfreq + idx;
        if (real) ((double*)sym)[o] = acc[p].x * scale;
        else ((double2*)sym)[o] = make_double2(acc[p].x * scale, acc[p].y * scale);
    }
}

// ------------------------------------------------------------------ host --
static void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

#define PDGPU_SMEM_ATTR(...) \
    check(cudaFuncSetAttribute(__VA_ARGS__, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448), "smem attr")

template <int IPT>
static void set_attrs_ipt() {
    PDGPU_SMEM_ATTR(k_rfft_rows<IPT>);
    PDGPU_SMEM_ATTR(k_irfft_rows<IPT, false, false>);
    PDGPU_SMEM_ATTR(k_irfft_rows<IPT, true, false>);
    PDGPU_SMEM_ATTR(k_irfft_rows<IPT, true, true>);
    PDGPU_SMEM_ATTR(k_irfft_rows<IPT, false, true>);
    PDGPU_SMEM_ATTR(k_spectral<IPT, 2, true>);
    PDGPU_SMEM_ATTR(k_spectral<IPT, 2, false>);
    PDGPU_SMEM_ATTR(k_spectral<IPT, 3, true>);
    PDGPU_SMEM_ATTR(k_spectral<IPT, 3, false>);
    PDGPU_SMEM_ATTR(k_cfft_y_fwd<IPT>);
    PDGPU_SMEM_ATTR(k_cfft_y_inv<IPT>);
}

void set_kernel_attributes() {
    set_attrs_ipt<1>();
    set_attrs_ipt<2>();
    set_attrs_ipt<4>();
    set_attrs_ipt<8>();
}

// threads and items-per-thread for a block FFT with `items` radix-4 work items
static void pick_threads(int64_t items, int& nth, int& ipt) {
    nth = 64;
    while (nth < 1024 && (items + nth - 1) / nth > 4) nth <<= 1;
    int64_t need = (items + nth - 1) / nth;
    ipt = need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : 8;
    if (need > 8) throw std::runtime_error("FFT tile too large for one CTA");
}

#define DISPATCH_IPT(ipt, KCALL)                     \
    switch (ipt) {                                   \
        case 1: { constexpr int I = 1; KCALL; } break; \
        case 2: { constexpr int I = 2; KCALL; } break; \
        case 4: { constexpr int I = 4; KCALL; } break; \
        default: { constexpr int I = 8; KCALL; } break; \
    }

void build_twiddles(Engine& e) {
    const int n = 1 << e.plan.logTWN;
    std::vector<double2> tw(n);
    for (int k = 0; k < n; ++k) {
        // exact-argument evaluation in long double
        const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)k / (long double)n;
        tw[k] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    // enforce exact symmetric values at the quarter points
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
    if (e.d_sym) cudaFree(e.d_sym);
    check(cudaMalloc(&e.d_sym, elt * nfreq * e.np), "alloc symbol");
    const double scale = 1.0 / ((double)pl.P[0] * (double)pl.P[1] * (double)pl.P[2]);
    const int th = 128;
    const int64_t blocks = (nfreq + th - 1) / th;
    k_build_symbol<<<(unsigned)blocks, th, 0, e.stream>>>(e.d_sym, e.d_K, e.dim, e.M, e.np, e.ss, pl.ncols, pl.Pl,
                                                         pl.P[0], pl.P[1], pl.P[2], e.real_symbol ? 1 : 0, scale);
    check(cudaGetLastError(), "build_symbol launch");
    check(cudaStreamSynchronize(e.stream), "build_symbol");
}

void engine_alloc_workspace(Engine& e, int64_t batch) {
    if (batch <= e.cap_batch) return;
    if (e.d_S1) cudaFree(e.d_S1);
    if (e.d_S2) cudaFree(e.d_S2);
    e.d_S1 = e.d_S2 = nullptr;
    const Plan& pl = e.plan;
    check(cudaMalloc(&e.d_S1, sizeof(double2) * pl.S1_per_vec * batch), "alloc S1");
    const bool need_s2 = pl.dim == 3 || pl.k3_halves == 1;
    if (need_s2) check(cudaMalloc(&e.d_S2, sizeof(double2) * pl.S2_per_vec * batch), "alloc S2");
    e.cap_batch = batch;
}

void launch_fast_apply(Engine& e, const double* u, double* f, int batch, cudaStream_t s, double scale,
                       const uint8_t* cmask, const double* body) {
    const Plan& pl = e.plan;
    engine_alloc_workspace(e, batch);
    const int d = pl.dim;
    const int Nx = pl.N[0], Ny = pl.N[1], Nz = pl.N[2];
    const int Qx = 1 << pl.logQx;
    const int nslab = batch * d * Nz;
    // K1
    {
        const int TR = pl.k1_rows;
        int nth, ipt;
        pick_threads((int64_t)2 * TR * Qx / 4 + 1, nth, ipt);
        dim3 grid((Ny + TR - 1) / TR, nslab);
        const size_t smem = sizeof(double2) * (size_t)TR * 2 * Qx;
        DISPATCH_IPT(ipt, (k_rfft_rows<I><<<grid, nth, smem, s>>>(u, e.d_S1, Nx, Ny, pl.Hx, pl.logQx, TR, e.d_tw,
                                                                   pl.logTWN)));
    }
    double2* specIn = e.d_S1;
    double2* specOut = e.d_S1;
    if (d == 3) {
        const int ZT = pl.k2_zt;
        int nth, ipt;
        pick_threads((int64_t)2 * ZT * (pl.P[1] / 2) / 4 + 1, nth, ipt);
        dim3 grid((Nz + ZT - 1) / ZT, pl.Hx, batch * d);
        const size_t smem = sizeof(double2) * (size_t)ZT * pl.P[1];
        DISPATCH_IPT(ipt, (k_cfft_y_fwd<I><<<grid, nth, smem, s>>>(e.d_S1, e.d_S2, Ny, Nz, pl.Hx, pl.logP[1], ZT,
                                                                    e.d_tw, pl.logTWN)));
        specIn = specOut = e.d_S2;
    } else if (pl.k3_halves == 1) {
        specOut = e.d_S2;
    }
    // K3
    {
        const int NC = pl.k3_cols, NH = pl.k3_halves;
        const int Ql = pl.Pl / 2;
        int nth, ipt;
        pick_threads((int64_t)NC * d * NH * Ql / 4 + 1, nth, ipt);
        dim3 grid((pl.ncols + NC - 1) / NC, batch);
        const size_t smem = sizeof(double2) * (size_t)NC * d * NH * Ql;
        if (d == 2) {
            if (e.real_symbol)
                DISPATCH_IPT(ipt, (k_spectral<I, 2, true><<<grid, nth, smem, s>>>(specIn, specOut, e.d_sym, pl.ncols,
                                                                                 pl.Nl, pl.logPl, NC, NH, e.d_tw,
                                                                                 pl.logTWN)))
            else
                DISPATCH_IPT(ipt, (k_spectral<I, 2, false><<<grid, nth, smem, s>>>(specIn, specOut, e.d_sym, pl.ncols,
                                                                                  pl.Nl, pl.logPl, NC, NH, e.d_tw,
                                                                                  pl.logTWN)))
        } else {
            if (e.real_symbol)
                DISPATCH_IPT(ipt, (k_spectral<I, 3, true><<<grid, nth, smem, s>>>(specIn, specOut, e.d_sym, pl.ncols,
                                                                                 pl.Nl, pl.logPl, NC, NH, e.d_tw,
                                                                                 pl.logTWN)))
            else
                DISPATCH_IPT(ipt, (k_spectral<I, 3, false><<<grid, nth, smem, s>>>(specIn, specOut, e.d_sym, pl.ncols,
                                                                                  pl.Nl, pl.logPl, NC, NH, e.d_tw,
                                                                                  pl.logTWN)))
        }
    }
    double2* xIn = specOut;
    if (d == 3) {
        const int ZT = pl.k2_zt;
        int nth, ipt;
        pick_threads((int64_t)2 * ZT * (pl.P[1] / 2) / 4 + 1, nth, ipt);
        dim3 grid((Nz + ZT - 1) / ZT, pl.Hx, batch * d);
        const size_t smem = sizeof(double2) * (size_t)ZT * pl.P[1];
        DISPATCH_IPT(ipt, (k_cfft_y_inv<I><<<grid, nth, smem, s>>>(e.d_S2, e.d_S1, Ny, Nz, pl.Hx, pl.logP[1], ZT,
                                                                    e.d_tw, pl.logTWN)));
        xIn = e.d_S1;
    }
    // K5
    {
        const int TR = pl.k1_rows;
        int nth, ipt;
        pick_threads((int64_t)2 * TR * Qx / 4 + 1, nth, ipt);
        dim3 grid((Ny + TR - 1) / TR, nslab);
        const size_t smem = sizeof(double2) * (size_t)TR * 2 * Qx;
#define K5_ARGS xIn, f, Nx, Ny, Nz, d, pl.Hx, pl.logQx, TR, e.d_tw, pl.logTWN, scale, cmask, body, pl.nodes
        if (cmask && body) DISPATCH_IPT(ipt, (k_irfft_rows<I, true, true><<<grid, nth, smem, s>>>(K5_ARGS)))
        else if (cmask) DISPATCH_IPT(ipt, (k_irfft_rows<I, true, false><<<grid, nth, smem, s>>>(K5_ARGS)))
        else if (body) DISPATCH_IPT(ipt, (k_irfft_rows<I, false, true><<<grid, nth, smem, s>>>(K5_ARGS)))
        else DISPATCH_IPT(ipt, (k_irfft_rows<I, false, false><<<grid, nth, smem, s>>>(K5_ARGS)))
#undef K5_ARGS
    }
    check(cudaGetLastError(), "fast_apply launch");
}

}  // namespace pdgpu
