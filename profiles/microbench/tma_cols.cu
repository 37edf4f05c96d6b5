// Microbenchmark: moving one spectral column (Nrow rows x 16 B) between SMEM
// and a row-pair-blocked HBM layout S[slab][rp][kx][2 rows] (32 B per
// (rp, kx)) with TMA tensor boxes {2 rows x complex, 1 kx, 256 rp}.  This is
// the access K3 would make if K1 wrote whole row pairs contiguously.
// Compared against the contiguous-column layout (bulk copies of 64 KB).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n W_%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* m, void* dst, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(m),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// each CTA walks columns (slab, kx); loads a whole column (Nrow x 16 B) into SMEM
template <bool BLOCKED, bool STORE>
__global__ void k_cols(const __grid_constant__ CUtensorMap tm, double2* S, int Nrow, int Hx, int nslab, int reps) {
    extern __shared__ __align__(128) double2 buf[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar);
    __syncthreads();
    const long long ncol = (long long)Hx * nslab;
    unsigned ph = 0;
    double acc = 0;
    for (long long c = blockIdx.x; c < ncol; c += gridDim.x) {
        const int slab = (int)(c / Hx), kx = (int)(c % Hx);
        if (!STORE) {
            if (threadIdx.x == 0) {
                mbar_expect_tx(&bar, Nrow * 16);
                if (BLOCKED) {
                    for (int r0 = 0; r0 < Nrow / 2; r0 += 256) tma_load_4d(&tm, buf + 2 * r0, &bar, 0, kx, r0, slab);
                } else {
                    bulk_load(buf, S + ((long long)slab * Hx + kx) * Nrow, Nrow * 16, &bar);
                }
            }
            mbar_wait(&bar, ph);
            ph ^= 1;
            acc += buf[threadIdx.x].x;
            __syncthreads();
        } else {
            if (threadIdx.x == 0) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncthreads();
            for (int i = threadIdx.x; i < Nrow; i += blockDim.x) buf[i] = make_double2(i, kx);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0) {
                if (BLOCKED) {
                    for (int r0 = 0; r0 < Nrow / 2; r0 += 256) tma_store_4d(&tm, buf + 2 * r0, 0, kx, r0, slab);
                } else {
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                     S + ((long long)slab * Hx + kx) * Nrow),
                                 "r"(smem_u32(buf)), "r"(Nrow * 16)
                                 : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (STORE && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (acc == 1234.5) S[0].x = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int Nrow = 4096, Hx = 4097, nslab = 32;
    const long long n = (long long)nslab * Hx * Nrow;
    double2* S;
    cudaMalloc(&S, n * sizeof(double2));
    cudaMemset(S, 0, n * sizeof(double2));
    EncodeFn enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    // S[slab][rp][kx][2 rows][re,im] as doubles: d0 = 4 doubles (2 rows x complex), d1 = kx, d2 = rp, d3 = slab
    CUtensorMap m;
    cuuint64_t dims[4] = {4, (cuuint64_t)Hx, (cuuint64_t)Nrow / 2, (cuuint64_t)nslab};
    cuuint64_t strides[3] = {32, (cuuint64_t)Hx * 32, (cuuint64_t)Hx * 32 * (Nrow / 2)};
    cuuint32_t box[4] = {4, 1, 256, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, S, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    const size_t smem = Nrow * 16;
    cudaFuncSetAttribute(k_cols<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k_cols<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k_cols<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k_cols<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double gb = n * 16.0 / 1e9;
    auto run = [&](const char* nm, auto k, int per_sm) {
        k<<<148 * per_sm, 256, smem>>>(m, S, Nrow, Hx, nslab, 1);
        cudaEventRecord(a);
        k<<<148 * per_sm, 256, smem>>>(m, S, Nrow, Hx, nslab, 1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-44s %8.3f ms %7.0f GB/s %s\n", nm, ms, gb / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    };
    for (int per : {1, 2, 3}) {
        char nm[96];
        snprintf(nm, 96, "column load, blocked rp layout, TMA  %d CTA/SM", per);
        run(nm, k_cols<true, false>, per);
        snprintf(nm, 96, "column load, contiguous, bulk       %d CTA/SM", per);
        run(nm, k_cols<false, false>, per);
        snprintf(nm, 96, "column store, blocked rp layout, TMA %d CTA/SM", per);
        run(nm, k_cols<true, true>, per);
        snprintf(nm, 96, "column store, contiguous, bulk      %d CTA/SM", per);
        run(nm, k_cols<false, true>, per);
    }
    return 0;
}
