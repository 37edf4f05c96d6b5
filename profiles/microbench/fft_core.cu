// Microbenchmark of the register FFT core (fft.cuh) without global I/O:
// each CTA runs `iters` forward+inverse 2^LOGQ-point transforms on register
// data.  Reports time per transform per SM and the fp64 instruction rate.
#include <cstdio>
#include <vector>
#include "../../paper_2301_11828_b200/csrc/fft.cuh"
using namespace pdgpu;

template <int LOGQ, int MINB, bool SPLIT>
__global__ void __launch_bounds__(FftShape<LOGQ, 4>::T * 1, MINB) bench(const double2* tw, int logTWN, int iters,
                                                                         double2* out) {
    using Sh = FftShape<LOGQ, 4>;
    extern __shared__ double2 sm[];
    const int t = threadIdx.x;
    double2 v[Sh::R];
#pragma unroll
    for (int j = 0; j < Sh::R; ++j) v[j] = make_double2(t * 1e-3 + j, j * 1e-2);
    const FftTw tws = make_fft_tw<LOGQ, 4>(t, tw, logTWN);
    for (int i = 0; i < iters; ++i) {
        reg_fft<LOGQ, 4, -1, BlockBar, SPLIT>(v, t, sm, tws, BlockBar{});
        reg_fft<LOGQ, 4, 1, BlockBar, SPLIT>(v, t, sm, tws, BlockBar{});
#pragma unroll
        for (int j = 0; j < Sh::R; ++j) v[j] = cscale(v[j], 1.0 / (1 << LOGQ));
    }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int j = 0; j < Sh::R; ++j) acc = cadd(acc, v[j]);
    out[blockIdx.x * blockDim.x + t] = acc;
}

template <int LOGQ, int MINB, bool SPLIT = false>
void run(const double2* tw, int logTWN, int ctas_per_sm) {
    using Sh = FftShape<LOGQ, 4>;
    const int iters = 200;
    const int grid = 148 * ctas_per_sm;
    const size_t smem = (SPLIT ? sizeof(double) : sizeof(double2)) * Sh::XBUF;
    cudaFuncSetAttribute(bench<LOGQ, MINB, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    double2* out;
    cudaMalloc(&out, sizeof(double2) * grid * Sh::T);
    bench<LOGQ, MINB, SPLIT><<<grid, Sh::T, smem>>>(tw, logTWN, 2, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bench<LOGQ, MINB, SPLIT><<<grid, Sh::T, smem>>>(tw, logTWN, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ffts = 2.0 * iters * grid;
    const double per_sm_us = ms * 1e3 / (ffts / 148);
    printf("split=%d LOGQ=%d T=%d ctas/SM=%d: %.3f ms, %.3f us per transform per SM (%.0f clk @1.965GHz)  err=%s\n", (int)SPLIT, LOGQ,
           Sh::T, ctas_per_sm, ms, per_sm_us, per_sm_us * 1965, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    const int logTWN = 13, n = 1 << logTWN;
    std::vector<double2> h(n);
    for (int k = 0; k < n; ++k) {
        const long double ang = -2.0L * 3.141592653589793238462643383279502884L * k / n;
        h[k] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    double2* tw;
    cudaMalloc(&tw, sizeof(double2) * n);
    cudaMemcpy(tw, h.data(), sizeof(double2) * n, cudaMemcpyHostToDevice);
    run<12, 1>(tw, logTWN, 1);
    run<12, 2>(tw, logTWN, 2);
    run<12, 3>(tw, logTWN, 3);
    run<11, 1>(tw, logTWN, 2);
    run<11, 2>(tw, logTWN, 4);
    run<8, 1>(tw, logTWN, 8);
    run<12, 1, true>(tw, logTWN, 1);
    run<12, 2, true>(tw, logTWN, 2);
    run<11, 2, true>(tw, logTWN, 4);
    return 0;
}
