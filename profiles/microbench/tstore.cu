// Microbenchmark: HBM write bandwidth of the K1 output pattern (S1[slab][kx][row],
// each CTA owning TR consecutive rows, so each kx gets TR*16 contiguous bytes)
// against plain contiguous stores and the K5 gather (read) pattern.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_transposed_store(double2* S, int Nrow, int Hx, int nslab, int TR, int mode) {
    const int groups = Nrow / TR;
    const long long ntiles = (long long)groups * nslab;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        double2* dst = S + (long long)slab * Hx * Nrow + row0;
        const int n = Hx * TR;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int rr = i % TR, kx = i / TR;
            dst[(long long)kx * Nrow + rr] = make_double2(kx, rr);
        }
        if (mode) __syncthreads();
    }
}

__global__ void k_contig_store(double2* S, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        S[i] = make_double2(i, 0);
}

// K5-like gather: each CTA reads TR rows' worth of a [kx][row] array
__global__ void k_gather(const double2* S, double2* out, int Nrow, int Hx, int nslab, int TR) {
    const int groups = Nrow / TR;
    const long long ntiles = (long long)groups * nslab;
    double2 acc = make_double2(0, 0);
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const double2* src = S + (long long)slab * Hx * Nrow + row0;
        const int n = Hx * TR;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int rr = i % TR, kx = i / TR;
            const double2 v = src[(long long)kx * Nrow + rr];
            acc.x += v.x;
            acc.y += v.y;
        }
    }
    if (acc.x == 12345.678) out[0] = acc;
}

int main() {
    const int Nrow = 4096, Hx = 4097, nslab = 32;  // 4096^2, 2 comps x batch 16
    const long long n = (long long)nslab * Hx * Nrow;
    double2* S;
    cudaMalloc(&S, n * sizeof(double2));
    double2* out;
    cudaMalloc(&out, 64);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double gb = n * 16.0 / 1e9;
    auto run = [&](const char* name, auto launch) {
        launch();
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 3;
        printf("%-40s %8.3f ms  %7.0f GB/s  %s\n", name, ms, gb / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    };
    run("contiguous store", [&] { k_contig_store<<<148 * 8, 256>>>(S, n); });
    for (int TR : {1, 2, 4, 8, 16}) {
        for (int thr : {256, 512}) {
            char nm[64];
            snprintf(nm, 64, "transposed store TR=%d thr=%d", TR, thr);
            run(nm, [&] { k_transposed_store<<<148 * (2048 / thr), thr>>>(S, Nrow, Hx, nslab, TR, 0); });
        }
    }
    for (int TR : {1, 2, 4, 8}) {
        char nm[64];
        snprintf(nm, 64, "gather load TR=%d thr=256", TR);
        run(nm, [&] { k_gather<<<148 * 8, 256>>>(S, out, Nrow, Hx, nslab, TR); });
    }
    return 0;
}
