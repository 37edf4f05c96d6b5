// fft.cuh -- register-resident fp64 FFTs for sm_100a.
//
// Replaces the FFTW3 C2C executions of the reference (convolution.hpp:114,127,
// 159).  Transforms are unnormalised, forward = exp(-2*pi*i*k*n/Q) like
// FFTW_FORWARD.  Every transform length is a power of two: the GPU pads each
// axis to P = 2*pow2ceil(N) (>= N+M, exact linear correlation on the window,
// DESIGN.md "Padding"), and the zero half of each padded input is never
// transformed (a P-point DFT of data supported on [0, P/2) is two P/2-point
// DFTs -- even and odd outputs -- which the callers run).
//
// Algorithm: Stockham autosort.  A transform of Q = 2^LOGQ points is owned
// by T = Q/R threads, each holding R points in registers in the "natural"
// layout  v[j] <-> x[t + j*T].  Passes: radix-R passes, the first without
// twiddles, then (when LOGR does not divide LOGQ) one remainder pass of radix
// 2^(LOGQ mod LOGR) with R/r butterflies per thread; between passes
// the data is exchanged once through shared memory (padded one slot every
// 16 so the 16-byte accesses of every quarter-warp hit distinct banks).  The
// last pass lands in the natural layout again, so a forward transform, a
// pointwise product and an inverse transform chain without extra exchanges.
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
// a * (S*i), S = +-1
template <int S>
__device__ __forceinline__ double2 cmul_si(double2 a) { return make_double2(-S * a.y, S * a.x); }

// twiddle exp(S*2*pi*i*idx/TWN) from the forward table tw[k] = exp(-2*pi*i*k/TWN)
template <int S>
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ tw, int idx) {
    double2 w = __ldg(tw + idx);
    if (S > 0) w.y = -w.y;
    return w;
}

// hide a value from loop-invariant code motion (persistent kernels would
// otherwise precompute per-j twiddle products once and spill them)
__device__ __forceinline__ double2 opaque(double2 a) {
    asm volatile("" : "+d"(a.x), "+d"(a.y));
    return a;
}

__device__ __forceinline__ int opaque(int a) {
    asm volatile("" : "+r"(a));
    return a;
}

// padded shared-memory slot
__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int spad_size(int q) { return q + (q >> 4) + 1; }

// ------------------------------------------------------------ butterflies --
// multiply by exp(S*2*pi*i*E/16) with compile-time E
template <int E, int S>
__device__ __forceinline__ double2 tw16(double2 a) {
    constexpr int e = E & 15;
    if constexpr (e == 0) return a;
    else if constexpr (e == 4) return cmul_si<S>(a);
    else if constexpr (e == 8) return make_double2(-a.x, -a.y);
    else if constexpr (e == 12) return cmul_si<-S>(a);
    else {
        constexpr double C[16] = {1.0,
                                  0.92387953251128675613,
                                  0.70710678118654752440,
                                  0.38268343236508977173,
                                  0.0,
                                  -0.38268343236508977173,
                                  -0.70710678118654752440,
                                  -0.92387953251128675613,
                                  -1.0,
                                  -0.92387953251128675613,
                                  -0.70710678118654752440,
                                  -0.38268343236508977173,
                                  0.0,
                                  0.38268343236508977173,
                                  0.70710678118654752440,
                                  0.92387953251128675613};
        constexpr double c = C[e];
        constexpr double s = S * C[(e + 12) & 15];  // sin(2 pi e/16) = cos(2 pi (e-4)/16)
        return make_double2(a.x * c - a.y * s, a.x * s + a.y * c);
    }
}

// multiply by exp(S*2*pi*i*E/32) with compile-time E
template <int E, int S>
__device__ __forceinline__ double2 tw32(double2 a) {
    constexpr int e = E & 31;
    if constexpr ((e & 1) == 0) {
        return tw16<e / 2, S>(a);
    } else {
        constexpr double C[32] = {1.0,
                                  0.98078528040323044913,
                                  0.92387953251128675613,
                                  0.83146961230254523708,
                                  0.70710678118654752440,
                                  0.55557023301960222474,
                                  0.38268343236508977173,
                                  0.19509032201612826785,
                                  0.0,
                                  -0.19509032201612826785,
                                  -0.38268343236508977173,
                                  -0.55557023301960222474,
                                  -0.70710678118654752440,
                                  -0.83146961230254523708,
                                  -0.92387953251128675613,
                                  -0.98078528040323044913,
                                  -1.0,
                                  -0.98078528040323044913,
                                  -0.92387953251128675613,
                                  -0.83146961230254523708,
                                  -0.70710678118654752440,
                                  -0.55557023301960222474,
                                  -0.38268343236508977173,
                                  -0.19509032201612826785,
                                  0.0,
                                  0.19509032201612826785,
                                  0.38268343236508977173,
                                  0.55557023301960222474,
                                  0.70710678118654752440,
                                  0.83146961230254523708,
                                  0.92387953251128675613,
                                  0.98078528040323044913};
        constexpr double c = C[e];
        constexpr double s = S * C[(e + 24) & 31];  // sin(2 pi e/32) = cos(2 pi (e-8)/32)
        return make_double2(a.x * c - a.y * s, a.x * s + a.y * c);
    }
}

// run-time exponent variant of tw32 (folds to constants inside unrolled loops)
template <int S>
__device__ __forceinline__ double2 tw32r(int e, double2 a) {
    switch (e & 31) {
#define PDGPU_TW32_CASE(E) \
    case E:                \
        return tw32<E, S>(a);
        PDGPU_TW32_CASE(0) PDGPU_TW32_CASE(1) PDGPU_TW32_CASE(2) PDGPU_TW32_CASE(3) PDGPU_TW32_CASE(4)
        PDGPU_TW32_CASE(5) PDGPU_TW32_CASE(6) PDGPU_TW32_CASE(7) PDGPU_TW32_CASE(8) PDGPU_TW32_CASE(9)
        PDGPU_TW32_CASE(10) PDGPU_TW32_CASE(11) PDGPU_TW32_CASE(12) PDGPU_TW32_CASE(13) PDGPU_TW32_CASE(14)
        PDGPU_TW32_CASE(15) PDGPU_TW32_CASE(16) PDGPU_TW32_CASE(17) PDGPU_TW32_CASE(18) PDGPU_TW32_CASE(19)
        PDGPU_TW32_CASE(20) PDGPU_TW32_CASE(21) PDGPU_TW32_CASE(22) PDGPU_TW32_CASE(23) PDGPU_TW32_CASE(24)
        PDGPU_TW32_CASE(25) PDGPU_TW32_CASE(26) PDGPU_TW32_CASE(27) PDGPU_TW32_CASE(28) PDGPU_TW32_CASE(29)
        PDGPU_TW32_CASE(30)
#undef PDGPU_TW32_CASE
        default:
            return tw32<31, S>(a);
    }
}

template <int S>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
    const double2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <int S>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
    const double2 a = cadd(x0, x2), c = csub(x0, x2);
    const double2 b = cadd(x1, x3), d = cmul_si<S>(csub(x1, x3));
    x0 = cadd(a, b);
    x2 = csub(a, b);
    x1 = cadd(c, d);
    x3 = csub(c, d);
}

// in-place DFT of 2^LR points, natural order in and out
template <int LR, int S>
__device__ __forceinline__ void dft(double2* v) {
    if constexpr (LR == 0) {
        return;
    } else if constexpr (LR == 1) {
        dft2<S>(v[0], v[1]);
    } else if constexpr (LR == 2) {
        dft4<S>(v[0], v[1], v[2], v[3]);
    } else if constexpr (LR == 3) {
        // 8 = 2 x 4 (DIT): even/odd inputs
        double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
        double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
        dft4<S>(e0, e1, e2, e3);
        dft4<S>(o0, o1, o2, o3);
        o1 = tw16<2, S>(o1);
        o2 = tw16<4, S>(o2);
        o3 = tw16<6, S>(o3);
        v[0] = cadd(e0, o0);
        v[4] = csub(e0, o0);
        v[1] = cadd(e1, o1);
        v[5] = csub(e1, o1);
        v[2] = cadd(e2, o2);
        v[6] = csub(e2, o2);
        v[3] = cadd(e3, o3);
        v[7] = csub(e3, o3);
    } else {
        // 16 = 4 x 4 in place: input m = 4*m1 + m2, output k = k1 + 4*k2.
        // Column DFT4s over m1 leave A[m2][k1] in v[4*k1 + m2]; after the
        // twiddles, row DFT4s over m2 leave X[k1 + 4*k2] in v[4*k1 + k2];
        // the final index permutation is a compile-time register renaming.
#pragma unroll
        for (int m2 = 0; m2 < 4; ++m2) dft4<S>(v[m2], v[4 + m2], v[8 + m2], v[12 + m2]);
        v[5] = tw16<1, S>(v[5]);
        v[9] = tw16<2, S>(v[9]);
        v[13] = tw16<3, S>(v[13]);
        v[6] = tw16<2, S>(v[6]);
        v[10] = tw16<4, S>(v[10]);
        v[14] = tw16<6, S>(v[14]);
        v[7] = tw16<3, S>(v[7]);
        v[11] = tw16<6, S>(v[11]);
        v[15] = tw16<9, S>(v[15]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) dft4<S>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
        // transpose 4x4: X[k1 + 4*k2] = v[4*k1 + k2]
        double2 t;
        t = v[1]; v[1] = v[4]; v[4] = t;
        t = v[2]; v[2] = v[8]; v[8] = t;
        t = v[3]; v[3] = v[12]; v[12] = t;
        t = v[6]; v[6] = v[9]; v[9] = t;
        t = v[7]; v[7] = v[13]; v[13] = t;
        t = v[11]; v[11] = v[14]; v[14] = t;
    }
}

// --------------------------------------------------------------- plans ----
// Threads-per-transform and points-per-thread for a length-2^LOGQ transform
// with at most 2^LOGRMAX points per thread.
template <int LOGQ, int LOGRMAX>
struct FftShape {
    static constexpr int LOGR = LOGQ < LOGRMAX ? LOGQ : LOGRMAX;
    static constexpr int R = 1 << LOGR;
    static constexpr int Q = 1 << LOGQ;
    static constexpr int T = Q / R;
    static constexpr int LOGT = LOGQ - LOGR;
    static constexpr int LOGREM = LOGR == 0 ? 0 : LOGQ % LOGR;
    static constexpr int NFULL = LOGR == 0 ? 0 : LOGQ / LOGR;
    static constexpr int NPASS = NFULL + (LOGREM ? 1 : 0);
    static constexpr int XBUF = spad_size(Q);  // exchange slots per transform
};

// Per-thread twiddle bases: pass P >= 1 multiplies input m of butterfly b
// by w^m, w = exp(-2 pi i k / (Ns r)), k = b mod Ns.  In full-radix passes
// b = t; in the remainder pass (last, radix r < R) b = t + i*T, i < R/r, all
// below Ns, and w_i = w_t * exp(-2 pi i i/R) (compile-time factor).  Only the
// bases are read from the table (once per kernel); the powers are formed in
// registers (depth <= 4 products, a few ulp), keeping the L1 path free for
// the data exchanges.
struct FftTw {
    double2 w[3];
};

template <int LOGQ, int LOGRMAX>
__device__ __forceinline__ FftTw make_fft_tw(int t, const double2* __restrict__ tw, int logTWN) {
    using Sh = FftShape<LOGQ, LOGRMAX>;
    FftTw r;
#pragma unroll
    for (int p = 1; p < 4; ++p) {
        r.w[p - 1] = make_double2(1.0, 0.0);
        if (p < Sh::NPASS) {
            const int logns = p * Sh::LOGR;
            const int lr = (p == Sh::NPASS - 1 && Sh::LOGREM) ? Sh::LOGREM : Sh::LOGR;
            const int k = t & ((1 << logns) - 1);
            r.w[p - 1] = __ldg(tw + (k << (logTWN - logns - lr)));
        }
    }
    return r;
}

// The same bases from shared memory: one compact table per twiddled pass
// (pass p: 2^logns entries, entry k = tw[k << (logTWN - logns - lr)]), laid
// out back to back, so a warp's loads are consecutive 16-byte entries.  (A
// single table of Q / r_last entries read at the pass's stride put pass 1's
// sixteen entries 256 bytes apart -- an eight-way bank conflict per load.)
// Persistent kernels re-derive the bases per transform (registers); reading
// them from SMEM instead of the global table keeps an L2 round trip (the L1
// is mostly carved out for shared memory) off the start of every transform.
template <int LOGQ, int LOGRMAX>
struct FftTwTable {
    using Sh = FftShape<LOGQ, LOGRMAX>;
    // entries of passes 1 .. p-1
    static constexpr int offset(int p) {
        int o = 0;
        for (int q = 1; q < p; ++q) o += 1 << (q * Sh::LOGR);
        return o;
    }
    static constexpr int SIZE = Sh::NPASS > 1 ? offset(Sh::NPASS) : 1;
};

template <int LOGQ, int LOGRMAX>
__device__ __forceinline__ void fill_fft_tw_table(double2* stw, const double2* __restrict__ tw, int logTWN) {
    using Sh = FftShape<LOGQ, LOGRMAX>;
#pragma unroll
    for (int p = 1; p < 4; ++p) {
        if (p < Sh::NPASS) {
            const int logns = p * Sh::LOGR;
            const int lr = (p == Sh::NPASS - 1 && Sh::LOGREM) ? Sh::LOGREM : Sh::LOGR;
            for (int k = threadIdx.x; k < (1 << logns); k += blockDim.x)
                stw[FftTwTable<LOGQ, LOGRMAX>::offset(p) + k] = __ldg(tw + (k << (logTWN - logns - lr)));
        }
    }
}

template <int LOGQ, int LOGRMAX>
__device__ __forceinline__ FftTw make_fft_tw_s(int t, const double2* stw) {
    using Sh = FftShape<LOGQ, LOGRMAX>;
    FftTw r;
#pragma unroll
    for (int p = 1; p < 4; ++p) {
        r.w[p - 1] = make_double2(1.0, 0.0);
        if (p < Sh::NPASS) {
            const int logns = p * Sh::LOGR;
            const int k = t & ((1 << logns) - 1);
            r.w[p - 1] = stw[FftTwTable<LOGQ, LOGRMAX>::offset(p) + k];
        }
    }
    return r;
}

__device__ __forceinline__ double2 csqr(double2 a) {
    return make_double2(a.x * a.x - a.y * a.y, 2.0 * a.x * a.y);
}

// One Stockham pass of radix 2^LR on the R registers of thread t, Ns = 2^LOGNS.
// Passes with LOGNS > 0 are full radix-R passes (one butterfly per thread).
template <int LOGQ, int LOGR, int LR, int LOGNS, int S>
__device__ __forceinline__ void fft_pass(double2 (&v)[1 << LOGR], double2 base) {
    constexpr int R = 1 << LOGR, r = 1 << LR, nb = R / r;
#pragma unroll
    for (int i = 0; i < nb; ++i) {
        double2 w[r];
#pragma unroll
        for (int m = 0; m < r; ++m) w[m] = v[i + m * nb];
        if constexpr (LOGNS > 0) {
            // sequential powers: only the base and the running power stay
            // live (register pressure), error grows to ~r ulp.  Butterfly i
            // of a remainder pass: base * exp(S 2 pi i i/R).
            // opaque: inside persistent loops the optimiser would otherwise
            // hoist all the powers out of the loop and spill them
            const double2 b0 = opaque(S > 0 ? cconj(base) : base);
            const double2 b1 = tw32r<S>(i * (32 / R), b0);
            double2 p = b1;
#pragma unroll
            for (int m = 1; m < r; ++m) {
                w[m] = cmul(w[m], p);
                if (m + 1 < r) p = cmul(p, b1);
            }
        }
        dft<LR, S>(w);
#pragma unroll
        for (int m = 0; m < r; ++m) v[i + m * nb] = w[m];
    }
}

// store after a pass (Stockham destination), barrier, reload natural layout
template <int LOGQ, int LOGR, int LR, int LOGNS, class Bar>
__device__ __forceinline__ void fft_exchange(double2 (&v)[1 << LOGR], int t, double2* xb, Bar bar) {
    constexpr int R = 1 << LOGR, r = 1 << LR, nb = R / r;
    constexpr int T = (1 << LOGQ) / R;
#pragma unroll
    for (int i = 0; i < nb; ++i) {
        const int b = t + i * T;
        const int base = ((b >> LOGNS) << (LOGNS + LR)) + (b & ((1 << LOGNS) - 1));
        // padded slot of base + m*Ns with compile-time strides where the
        // padding is separable (Ns == 1 and r <= 16, or Ns a multiple of 16)
        if constexpr (LOGNS == 0 && LR <= 4) {
            double2* p = xb + spad(base);
#pragma unroll
            for (int m = 0; m < r; ++m) p[m] = v[i + m * nb];
        } else if constexpr (LOGNS >= 4) {
            constexpr int NS = 1 << LOGNS;
            double2* p = xb + spad(base);
#pragma unroll
            for (int m = 0; m < r; ++m) p[m * (NS + NS / 16)] = v[i + m * nb];
        } else {
#pragma unroll
            for (int m = 0; m < r; ++m) xb[spad(base + (m << LOGNS))] = v[i + m * nb];
        }
    }
    bar();
    if constexpr (T % 16 == 0) {
        const double2* p = xb + spad(t);
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = p[j * (T + T / 16)];
    } else {
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = xb[spad(t + j * T)];
    }
    bar();
}

// Split exchange: the same permutation through a buffer of 8-byte slots,
// real parts first, then imaginary parts (half the shared memory of
// fft_exchange -- lets two CTAs share an SM -- for twice the barriers).
// Padding one slot per 16 keeps every half-warp on distinct banks.
template <int LOGQ, int LOGR, int LR, int LOGNS, class Bar>
__device__ __forceinline__ void fft_exchange_split(double2 (&v)[1 << LOGR], int t, double* xd, Bar bar) {
    constexpr int R = 1 << LOGR, r = 1 << LR, nb = R / r;
    constexpr int T = (1 << LOGQ) / R;
#pragma unroll
    for (int part = 0; part < 2; ++part) {
#pragma unroll
        for (int i = 0; i < nb; ++i) {
            const int b = t + i * T;
            const int base = ((b >> LOGNS) << (LOGNS + LR)) + (b & ((1 << LOGNS) - 1));
#pragma unroll
            for (int m = 0; m < r; ++m) {
                const double2 x = v[i + m * nb];
                xd[spad(base + (m << LOGNS))] = part ? x.y : x.x;
            }
        }
        bar();
        if constexpr (T % 16 == 0) {
            const double* p = xd + spad(t);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (part) v[j].y = p[j * (T + T / 16)];
                else v[j].x = p[j * (T + T / 16)];
            }
        } else {
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (part) v[j].y = xd[spad(t + j * T)];
                else v[j].x = xd[spad(t + j * T)];
            }
        }
        bar();
    }
}

// natural-layout slot of element t + j*T (compile-time stride when T % 16 == 0)
template <int T>
__device__ __forceinline__ int nat_slot(int t, int j) {
    if constexpr (T % 16 == 0) return spad(t) + j * (T + T / 16);
    else return spad(t + j * T);
}

// Hook: called once, behind the last exchange's closing barrier -- from there
// on the exchange buffer is free while the last pass runs in registers (the
// caller may start an asynchronous copy into it).
struct NoHook {
    __device__ __forceinline__ void operator()() const {}
};

template <int LOGQ, int LOGR, int S, int P, int LOGNS, bool SPLIT, class Bar, class Hook>
__device__ __forceinline__ void fft_passes(double2 (&v)[1 << LOGR], int t, double2* xb, const FftTw& tws, Bar bar,
                                           Hook hook) {
    using Sh = FftShape<LOGQ, LOGR>;
    if constexpr (P < Sh::NPASS) {
        constexpr int LR = (P == Sh::NPASS - 1 && Sh::LOGREM) ? Sh::LOGREM : LOGR;
        fft_pass<LOGQ, LOGR, LR, LOGNS, S>(v, P > 0 ? tws.w[P > 0 ? P - 1 : 0] : make_double2(1.0, 0.0));
        if constexpr (P + 1 < Sh::NPASS) {
            if constexpr (SPLIT) fft_exchange_split<LOGQ, LOGR, LR, LOGNS>(v, t, reinterpret_cast<double*>(xb), bar);
            else fft_exchange<LOGQ, LOGR, LR, LOGNS>(v, t, xb, bar);
            if constexpr (P + 2 == Sh::NPASS) hook();
            fft_passes<LOGQ, LOGR, S, P + 1, LOGNS + LR, SPLIT>(v, t, xb, tws, bar, hook);
        }
    }
}

// Full transform: v[j] holds x[t + j*T] on entry and X[t + j*T] on exit.
// xb: this transform's exchange buffer (FftShape::XBUF slots); tws: the
// thread's twiddle bases (make_fft_tw, same for forward and inverse); bar():
// a barrier covering every thread of the transform (all groups of a CTA in
// lockstep use __syncthreads).  SPLIT: xb holds XBUF 8-byte slots instead
// (fft_exchange_split).
template <int LOGQ, int LOGRMAX, int S, class Bar, bool SPLIT = false, class Hook = NoHook>
__device__ __forceinline__ void reg_fft(double2 (&v)[1 << FftShape<LOGQ, LOGRMAX>::LOGR], int t, double2* xb,
                                        const FftTw& tws, Bar bar, Hook hook = Hook{}) {
    using Sh = FftShape<LOGQ, LOGRMAX>;
    static_assert(Sh::NPASS <= 4, "at most three twiddled passes");
    fft_passes<LOGQ, Sh::LOGR, S, 0, 0, SPLIT>(v, t, xb, tws, bar, hook);
}

struct BlockBar {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

}  // namespace pdgpu
