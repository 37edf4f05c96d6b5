// Microbenchmark: HBM write bandwidth of the K1 output pattern (S1[slab][kx][row],
// each CTA owning TR consecutive rows, so each kx gets TR*16 contiguous bytes)
// against plain contiguous stores and the K5 gather (read) pattern.
#include <cstdio>
#include <cuda.h>
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


// TMA variants: S viewed as a 2D tensor of doubles, dim0 = 2*Nrow (contiguous),
// dim1 = Hx*nslab (kx rows); a box {2*TR, 256} moves TR rows x 256 kx.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* smem, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
                 "r"((unsigned)__cvta_generic_to_shared(smem)), "r"(x), "r"(y), "r"(z)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* m, void* smem, unsigned long long* bar, int x, int y,
                                            int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            (unsigned)__cvta_generic_to_shared(smem)),
        "l"(m), "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}

template <int TR>
__global__ void k_tma_store(const __grid_constant__ CUtensorMap tm, int Nrow, int Hx, int nslab) {
    extern __shared__ __align__(128) double2 buf[];  // 2 x [Hx][TR]
    const int groups = Nrow / TR;
    const long long ntiles = (long long)groups * nslab;
    int par = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, par ^= 1) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        double2* b = buf + par * ((Hx + 255) / 256 * 256) * TR;
        // buffer par was last used two tiles ago: allow <= 1 outstanding group reading smem
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        for (int i = threadIdx.x; i < Hx * TR; i += blockDim.x) b[i] = make_double2(i, row0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k0 = 0; k0 < Hx; k0 += 256)
                tma_store_2d(&tm, b + k0 * TR, 2 * row0, k0, slab);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int TR>
__global__ void k_tma_load(const __grid_constant__ CUtensorMap tm, double2* out, int Nrow, int Hx, int nslab) {
    extern __shared__ __align__(128) double2 buf[];  // [Hx][TR]
    __shared__ __align__(8) unsigned long long bar;
    const int groups = Nrow / TR;
    const long long ntiles = (long long)groups * nslab;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double2 acc = make_double2(0, 0);
    unsigned phase = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int slab = (int)(tile / groups), row0 = (int)(tile % groups) * TR;
        const int nbox = (Hx + 255) / 256;
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(&bar)),
                         "r"(nbox * 256 * TR * 16)
                         : "memory");
            for (int k0 = 0; k0 < Hx; k0 += 256) tma_load_2d(&tm, buf + k0 * TR, &bar, 2 * row0, k0, slab);
        }
        // wait
        asm volatile(
            "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
                (unsigned)__cvta_generic_to_shared(&bar)),
            "r"(phase)
            : "memory");
        phase ^= 1;
        for (int i = threadIdx.x; i < Hx * TR; i += blockDim.x) {
            acc.x += buf[i].x;
            acc.y += buf[i].y;
        }
        __syncthreads();
    }
    if (acc.x == 12345.678) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(void* base, int Nrow, int Hx, int nslab, int TR) {
    static EncodeFn enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    }
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)2 * Nrow, (cuuint64_t)Hx, (cuuint64_t)nslab};
    cuuint64_t strides[2] = {(cuuint64_t)Nrow * 16, (cuuint64_t)Hx * Nrow * 16};
    cuuint32_t box[3] = {(cuuint32_t)(2 * TR), 256, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
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
    {
        const CUtensorMap m2 = make_map(S, Nrow, Hx, nslab, 2);
        const CUtensorMap m4 = make_map(S, Nrow, Hx, nslab, 4);
        const CUtensorMap m1 = make_map(S, Nrow, Hx, nslab, 1);
        const size_t sm2 = 2 * (size_t)(Hx + 255) / 256 * 256 * 2 * 16, sm4 = sm2 / 2 * 4 / 2 * 2;
        cudaFuncSetAttribute(k_tma_store<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        cudaFuncSetAttribute(k_tma_store<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        cudaFuncSetAttribute(k_tma_load<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        cudaFuncSetAttribute(k_tma_load<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        cudaFuncSetAttribute(k_tma_load<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        const size_t b1 = (size_t)((Hx + 255) / 256) * 256 * 16;
        auto chk = [](const char* w) { cudaError_t e = cudaGetLastError(); if (e) printf("  [%s] %s\n", w, cudaGetErrorString(e)); };
        chk("before");
        run("TMA store TR=1 (2 bufs, 3 CTA/SM)", [&] { k_tma_store<1><<<148 * 3, 256, 2 * b1>>>(m1, Nrow, Hx, nslab); });
        chk("after store");
        run("TMA load TR=1 (3 CTA/SM)", [&] { k_tma_load<1><<<148 * 3, 256, b1>>>(m1, out, Nrow, Hx, nslab); });
        run("TMA load TR=2 (1 CTA/SM)", [&] { k_tma_load<2><<<148, 256, 2 * b1>>>(m2, out, Nrow, Hx, nslab); });
        (void)sm2; (void)sm4;
    }
    return 0;
}
