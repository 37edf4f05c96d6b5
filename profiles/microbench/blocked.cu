// Microbenchmark: a kx-blocked spectrum layout S[slab][kx/KB][row][kx%KB]
// (KB consecutive kx contiguous per row) against the column layout
// S[slab][kx][row] the 2D passes use.  Periodic 4096^2 x 16 vectors x 2
// components: Hx = 2049 columns of 4096 rows, 32 slabs (4.3 GB).
//   K1-like: each CTA stores 2 rows x all kx          (blocked: 2*KB*16 B chunks)
//   K3-like: each CTA reads / writes one kx column     (blocked: 16 B at KB*16 B stride;
//            CTAs on the KB columns of a block run together so L2 merges the lines)
//   K5-like: each CTA reads 2 rows x all kx            (blocked: 2*KB*16 B chunks)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o blocked blocked.cu
#include <cstdio>
#include <cuda_runtime.h>

__host__ __device__ inline long long idx_blocked(int slab, int kx, int row, int Nrow, int NB, int KB) {
    return (((long long)slab * NB + kx / KB) * Nrow + row) * KB + kx % KB;
}

__global__ void k_rows_store(double2* S, int Nrow, int Hx, int nslab, int KB) {
    const int NB = (Hx + KB - 1) / KB;
    const long long ntiles = (long long)(Nrow / 2) * nslab;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int slab = (int)(tile / (Nrow / 2)), row0 = (int)(tile % (Nrow / 2)) * 2;
        const int n = NB * KB * 2;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int kk = i % KB, rr = (i / KB) & 1, kb = i / (2 * KB);
            const int kx = kb * KB + kk;
            if (kx < Hx) S[idx_blocked(slab, kx, row0 + rr, Nrow, NB, KB)] = make_double2(kx, rr);
        }
    }
}

__global__ void k_rows_load(const double2* S, double2* out, int Nrow, int Hx, int nslab, int KB) {
    const int NB = (Hx + KB - 1) / KB;
    const long long ntiles = (long long)(Nrow / 2) * nslab;
    double2 acc = make_double2(0, 0);
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int slab = (int)(tile / (Nrow / 2)), row0 = (int)(tile % (Nrow / 2)) * 2;
        const int n = NB * KB * 2;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int kk = i % KB, rr = (i / KB) & 1, kb = i / (2 * KB);
            const int kx = kb * KB + kk;
            if (kx < Hx) {
                const double2 v = S[idx_blocked(slab, kx, row0 + rr, Nrow, NB, KB)];
                acc.x += v.x;
                acc.y += v.y;
            }
        }
    }
    if (acc.x == 12345.678) out[0] = acc;
}

// one column per item; item order: kx fastest (the KB columns of a block together)
template <bool STORE>
__global__ void k_cols(double2* S, double2* out, int Nrow, int Hx, int nslab, int KB) {
    const int NB = (Hx + KB - 1) / KB;
    const long long nitems = (long long)Hx * nslab;
    double2 acc = make_double2(0, 0);
    for (long long it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int slab = (int)(it / Hx), kx = (int)(it % Hx);
        double2 v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int n = threadIdx.x + j * 256;
            const long long a = idx_blocked(slab, kx, n, Nrow, NB, KB);
            if (STORE) S[a] = make_double2(n, kx);
            else v[j] = S[a];
        }
        if (!STORE) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                acc.x += v[j].x;
                acc.y += v[j].y;
            }
        }
    }
    if (acc.x == 12345.678) out[0] = acc;
}

int main() {
    const int Nrow = 4096, Hx = 2049, nslab = 32;
    const long long n = (long long)nslab * (Hx + 16) * Nrow;  // room for the last partial block at KB = 16
    double2* S;
    cudaMalloc(&S, n * sizeof(double2));
    double2* out;
    cudaMalloc(&out, 64);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double gb = (double)nslab * Hx * Nrow * 16.0 / 1e9;
    auto run = [&](const char* name, auto launch) {
        launch();
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 3;
        printf("%-44s %8.3f ms  %7.0f GB/s  %s\n", name, ms, gb / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    };
    for (int KB : {1, 2, 4, 8, 16}) {
        char nm[80];
        // KB = 1 is the column layout S[slab][kx][row]
        snprintf(nm, 80, "KB=%2d K1-like rows store (2 rows/CTA)", KB);
        run(nm, [&] { k_rows_store<<<148 * 4, 256>>>(S, Nrow, Hx, nslab, KB); });
        snprintf(nm, 80, "KB=%2d K5-like rows load  (2 rows/CTA)", KB);
        run(nm, [&] { k_rows_load<<<148 * 4, 256>>>(S, out, Nrow, Hx, nslab, KB); });
        snprintf(nm, 80, "KB=%2d K3-like column load", KB);
        run(nm, [&] { k_cols<false><<<148 * 2, 256>>>(S, out, Nrow, Hx, nslab, KB); });
        snprintf(nm, 80, "KB=%2d K3-like column store", KB);
        run(nm, [&] { k_cols<true><<<148 * 2, 256>>>(S, out, Nrow, Hx, nslab, KB); });
    }
    return 0;
}
