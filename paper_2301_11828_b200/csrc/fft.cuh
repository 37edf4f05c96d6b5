// fft.cuh -- CTA-cooperative fp64 FFTs in shared memory for sm_100a.
//
// Replaces the FFTW3 C2C executions of the reference (convolution.hpp:114,127,
// 159).  Transforms are unnormalised, forward = exp(-2*pi*i*k*n/Q) like
// FFTW_FORWARD.  Every transform length here is a power of two: the GPU pads
// each axis to P = 2*pow2ceil(N) (>= N+M, so the linear correlation on the
// window is exact).  The zero half of each padded
// input is never transformed: a P-point DFT of data with support < P/2 is two
// P/2-point DFTs (even and odd outputs), which is what the callers do.
//
// Algorithm: Stockham autosort, radix-4 stages (one radix-8 or radix-2 stage
// first when log2 Q is odd), operands staged in shared memory, butterflies in
// registers.  Each stage loads all of its items into registers, barriers,
// then stores, so a single buffer is reused in place.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pdgpu {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// a * (s*i), s = +-1
template <int S>
__device__ __forceinline__ double2 cmul_si(double2 a) { return make_double2(-S * a.y, S * a.x); }

// twiddle exp(S*2*pi*i*idx/TWN) from the forward table tw[k] = exp(-2*pi*i*k/TWN)
template <int S>
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ tw, int idx) {
    double2 w = __ldg(tw + idx);
    if (S > 0) w.y = -w.y;
    return w;
}

// S = -1 forward, +1 inverse
template <int S>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
    double2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <int S>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
    double2 a = cadd(x0, x2), c = csub(x0, x2);
    double2 b = cadd(x1, x3), d = cmul_si<S>(csub(x1, x3));
    x0 = cadd(a, b);
    x2 = csub(a, b);
    x1 = cadd(c, d);
    x3 = csub(c, d);
}

template <int S>
__device__ __forceinline__ void dft8(double2* v) {
    const double r = 0.70710678118654752440084436210484904;
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<S>(e0, e1, e2, e3);
    dft4<S>(o0, o1, o2, o3);
    // W8^1 = (1 + S i)/sqrt2, W8^2 = S i, W8^3 = (-1 + S i)/sqrt2
    double2 t1 = make_double2(r * (o1.x - S * o1.y), r * (o1.y + S * o1.x));
    double2 t2 = cmul_si<S>(o2);
    double2 t3 = make_double2(r * (-o3.x - S * o3.y), r * (-o3.y + S * o3.x));
    v[0] = cadd(e0, o0);
    v[4] = csub(e0, o0);
    v[1] = cadd(e1, t1);
    v[5] = csub(e1, t1);
    v[2] = cadd(e2, t2);
    v[6] = csub(e2, t2);
    v[3] = cadd(e3, t3);
    v[7] = csub(e3, t3);
}

template <int R, int S>
__device__ __forceinline__ void dftR(double2* v) {
    if constexpr (R == 2) dft2<S>(v[0], v[1]);
    else if constexpr (R == 4) dft4<S>(v[0], v[1], v[2], v[3]);
    else dft8<S>(v);
}

// One Stockham stage of radix R over nb transforms of length Q = 2^logQ held
// contiguously in buf.  IPT bounds the items per thread: nb*Q/R <= IPT*nthreads.
template <int R, int S, int IPT>
__device__ __forceinline__ void stockham_stage(double2* buf, int nb, int logQ, int Ns, int logNsR,
                                               const double2* __restrict__ tw, int logTWN) {
    const int Q = 1 << logQ;
    const int logR = R == 2 ? 1 : (R == 4 ? 2 : 3);
    const int QR = Q >> logR;
    const int total = nb * QR;
    const int nth = blockDim.x;
    double2 v[IPT][R];
    int dst[IPT];
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
        const int item = threadIdx.x + it * nth;
        if (item < total) {
            const int t = item >> (logQ - logR);
            const int j = item & (QR - 1);
            const double2* src = buf + (t << logQ) + j;
            const int k = j & (Ns - 1);
#pragma unroll
            for (int r = 0; r < R; ++r) v[it][r] = src[r * QR];
            if (Ns > 1) {
                const int step = k << (logTWN - logNsR);  // k * TWN / (Ns*R)
#pragma unroll
                for (int r = 1; r < R; ++r) v[it][r] = cmul(v[it][r], twiddle<S>(tw, step * r));
            }
            dftR<R, S>(v[it]);
            dst[it] = (t << logQ) + ((j - k) << logR) + k;
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
        const int item = threadIdx.x + it * nth;
        if (item < total) {
#pragma unroll
            for (int r = 0; r < R; ++r) buf[dst[it] + r * Ns] = v[it][r];
        }
    }
    __syncthreads();
}

// Full in-place FFT of nb transforms of length 2^logQ in shared memory.
// Caller must __syncthreads() before (data staged) -- this routine ends with
// a barrier so results are visible to all threads.
// IPT must satisfy nb*Q/4 <= IPT*blockDim (radix-4) and nb*Q/8 for radix-8;
// the radix-2 case only occurs for Q == 2.
template <int S, int IPT>
__device__ void block_fft(double2* buf, int nb, int logQ, const double2* __restrict__ tw, int logTWN) {
    if (logQ == 0) return;
    int Ns = 1, logNs = 0, l = logQ;
    if (l == 1) {
        stockham_stage<2, S, IPT>(buf, nb, logQ, 1, 1, tw, logTWN);
        return;
    }
    if (l & 1) {
        stockham_stage<8, S, IPT>(buf, nb, logQ, 1, 3, tw, logTWN);
        Ns = 8;
        logNs = 3;
        l -= 3;
    }
    while (l >= 2) {
        stockham_stage<4, S, IPT>(buf, nb, logQ, Ns, logNs + 2, tw, logTWN);
        Ns <<= 2;
        logNs += 2;
        l -= 2;
    }
}

}  // namespace pdgpu
