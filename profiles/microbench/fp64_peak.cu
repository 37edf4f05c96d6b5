// fp64 issue-rate microbenchmark on B200 (sm_100a): DFMA / DADD / DMUL
// throughput per SM, and shared-memory bandwidth (LDS.64 / LDS.128) -- the two
// resources the register FFT (fft.cuh) is bound by.  VERDICT r1 item 12: the
// "fp64-issue bound" reading of K3 needs a measured fp64 peak.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_peak.cu -o fp64_peak
#include <cstdio>

template <int OP>
__global__ void __launch_bounds__(256) k_fp(double* out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (OP == 0) x[j] = fma(x[j], a, b);
            if (OP == 1) x[j] = x[j] + b;
            if (OP == 2) x[j] = x[j] * a;
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int W>
__global__ void __launch_bounds__(256) k_lds(double* out, int iters) {
    __shared__ double sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    double acc = 0;
    const int t = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (W == 8) acc += sm[(t + j * 256 + i) & 4095];
            else {
                const double2 v = reinterpret_cast<const double2*>(sm)[(t + j * 256 + i) & 2047];
                acc += v.x + v.y;
            }
        }
    }
    out[blockIdx.x * blockDim.x + t] = acc;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[3] = {"DFMA", "DADD", "DMUL"};
    for (int op = 0; op < 3; ++op) {
        const int iters = 4000, grid = sms * 8;
        auto launch = [&](int it) {
            if (op == 0) k_fp<0><<<grid, 256>>>(out, it, 1.0000001, 1e-9);
            if (op == 1) k_fp<1><<<grid, 256>>>(out, it, 1.0000001, 1e-9);
            if (op == 2) k_fp<2><<<grid, 256>>>(out, it, 1.0000001, 1e-9);
        };
        launch(10);
        cudaEventRecord(a);
        launch(iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)grid * 256 * iters * 16;
        const double per_sm_clk = ops / sms / (ms * 1e-3 * clk * 1e3);
        printf("%s: %.3f ms, %.2f Gop/s, %.1f lanes/SM/clk at the reported %d MHz (%.1f TFLOP/s%s)\n", names[op], ms,
               ops / ms / 1e6, per_sm_clk, clk / 1000, ops / ms / 1e9 * (op == 0 ? 2 : 1), op == 0 ? " fma=2" : "");
    }
    for (int w = 0; w < 2; ++w) {
        const int iters = 2000, grid = sms * 4;
        auto launch = [&](int it) {
            if (w == 0) k_lds<8><<<grid, 256>>>(out, it);
            else k_lds<16><<<grid, 256>>>(out, it);
        };
        launch(10);
        cudaEventRecord(a);
        launch(iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)grid * 256 * iters * 16 * (w ? 16 : 8);
        printf("LDS.%d: %.3f ms, %.1f B/clk/SM\n", w ? 128 : 64, ms, bytes / sms / (ms * 1e-3 * clk * 1e3));
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
