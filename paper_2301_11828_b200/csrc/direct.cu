// direct.cu -- K·u by direct stencil summation on the device.
//
// f_a[p] = sum_o sum_b K_ab(o) u_b[p + o], u = 0 outside the lattice: the
// same linear correlation FastForce::apply evaluates through the padded FFT
// (convolution.hpp:130-134,160), computed the way the reference's own
// independent oracle does it (tests/support/oracles.hpp:72-96 tbt_apply_all).
// an on-device cross-check of the MSBFM path that
// needs no host round trip, and the comparison point for its roofline (a
// banded stencil moves ~16 B/DOF against >= 80 B/DOF for the FFT route).
//
// 2D: 32 x 32 node tiles, u tile + M-halo in SMEM, each thread 4 rows of one
// column with a register window of 4 + 2M values per component; offsets are
// compile-time (M template), coefficients uniform loads from the stencil
// table.  3D: thread per node over the in-band offset list (cross-check only).
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "engine.h"

namespace pdgpu {

namespace {

constexpr int kTX = 32, kTY = 32, kRows = 4;  // tile; rows per thread

constexpr int isqrt_c(int v) {
    int r = 0;
    while ((r + 1) * (r + 1) <= v) ++r;
    return r;
}

// K: n_pairs x (2M+1)^2 stencils, storage index (oy+M)*(2M+1) + (ox+M)
template <int M>
__global__ void __launch_bounds__(kTX * (kTY / kRows)) k_direct2d(const double* __restrict__ u, double* __restrict__ f,
                                                                  const double* __restrict__ K, int Nx, int Ny,
                                                                  int64_t nodes, double scale,
                                                                  const uint8_t* __restrict__ cmask) {
    constexpr int W = kTX + 2 * M, H = kTY + 2 * M, SIDE = 2 * M + 1, SS = SIDE * SIDE, WIN = kRows + 2 * M;
    __shared__ double su[2][H][W + 1];
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    const double* ub = u + (int64_t)b * 2 * nodes;
    for (int i = threadIdx.y * kTX + threadIdx.x; i < H * W; i += kTX * (kTY / kRows)) {
        const int yy = i / W, xx = i - yy * W;
        const int gx = x0 + xx - M, gy = y0 + yy - M;
        const bool in = gx >= 0 && gx < Nx && gy >= 0 && gy < Ny;
        const int64_t p = (int64_t)gy * Nx + gx;
        su[0][yy][xx] = in ? ub[p] : 0.0;
        su[1][yy][xx] = in ? ub[nodes + p] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x, ty = threadIdx.y * kRows;
    double acc[kRows][2];
#pragma unroll
    for (int i = 0; i < kRows; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
    for (int dx = -M; dx <= M; ++dx) {
        double w0[WIN], w1[WIN];
#pragma unroll
        for (int r = 0; r < WIN; ++r) {
            w0[r] = su[0][ty + r][tx + M + dx];
            w1[r] = su[1][ty + r][tx + M + dx];
        }
        const int R = isqrt_c(M * M - dx * dx);
#pragma unroll
        for (int dy = -M; dy <= M; ++dy) {
            if (dy < -R || dy > R) continue;
            const int si = (dy + M) * SIDE + (dx + M);
            const double kxx = __ldg(K + si), kxy = __ldg(K + SS + si), kyy = __ldg(K + 2 * SS + si);
#pragma unroll
            for (int i = 0; i < kRows; ++i) {
                const double a0 = w0[i + dy + M], a1 = w1[i + dy + M];
                acc[i][0] = fma(kxx, a0, fma(kxy, a1, acc[i][0]));
                acc[i][1] = fma(kxy, a0, fma(kyy, a1, acc[i][1]));
            }
        }
    }
    const int gx = x0 + tx;
    if (gx >= Nx) return;
    double* fb = f + (int64_t)b * 2 * nodes;
#pragma unroll
    for (int i = 0; i < kRows; ++i) {
        const int gy = y0 + ty + i;
        if (gy >= Ny) continue;
        const int64_t p = (int64_t)gy * Nx + gx;
        const uint8_t cm = cmask ? cmask[p] : 0;  // constrained rows read zero (CG operator)
        fb[p] = (cm & 1u) ? 0.0 : scale * acc[i][0];
        fb[nodes + p] = (cm & 2u) ? 0.0 : scale * acc[i][1];
    }
}

// 3D: thread per node; offs[k] (k < nof) in-band off-centre offsets, koff[k*6 + pair],
// centre coefficients kc[pair]
__global__ void k_direct3d(const double* __restrict__ u, double* __restrict__ f, const int* __restrict__ offs,
                           const double* __restrict__ koff, const double* __restrict__ kc, int nof, int Nx, int Ny,
                           int Nz, int64_t nodes, double scale, const uint8_t* __restrict__ cmask) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (p >= nodes) return;
    const int i = (int)(p % Nx), j = (int)((p / Nx) % Ny), k = (int)(p / ((int64_t)Nx * Ny));
    const double* ub = u + (int64_t)b * 3 * nodes;
    double acc[3];
    {
        const double ux = ub[p], uy = ub[nodes + p], uz = ub[2 * nodes + p];
        acc[0] = kc[0] * ux + kc[1] * uy + kc[2] * uz;
        acc[1] = kc[1] * ux + kc[3] * uy + kc[4] * uz;
        acc[2] = kc[2] * ux + kc[4] * uy + kc[5] * uz;
    }
    for (int o = 0; o < nof; ++o) {
        const int qi = i + offs[3 * o], qj = j + offs[3 * o + 1], qk = k + offs[3 * o + 2];
        if (qi < 0 || qi >= Nx || qj < 0 || qj >= Ny || qk < 0 || qk >= Nz) continue;
        const int64_t q = ((int64_t)qk * Ny + qj) * Nx + qi;
        const double* c = koff + 6 * o;
        const double ux = __ldg(ub + q), uy = __ldg(ub + nodes + q), uz = __ldg(ub + 2 * nodes + q);
        acc[0] += c[0] * ux + c[1] * uy + c[2] * uz;
        acc[1] += c[1] * ux + c[3] * uy + c[4] * uz;
        acc[2] += c[2] * ux + c[4] * uy + c[5] * uz;
    }
    double* fb = f + (int64_t)b * 3 * nodes;
    const uint8_t cm = cmask ? cmask[p] : 0;
    fb[p] = (cm & 1u) ? 0.0 : scale * acc[0];
    fb[nodes + p] = (cm & 2u) ? 0.0 : scale * acc[1];
    fb[2 * nodes + p] = (cm & 4u) ? 0.0 : scale * acc[2];
}

}  // namespace

// 3D centre coefficients (stencil index of o = 0; stencils stored first in
// d_K); allocated outside any graph capture (pdgpu_set_cg_operator)
void direct_prepare(Engine& e) {
    if (e.dim != 3 || e.d_kc) return;
    std::vector<double> kc(6);
    const int o0[3] = {0, 0, 0};
    const int64_t si = assembly::stencil_index(3, e.M, o0);
    for (int pr = 0; pr < 6; ++pr) kc[pr] = e.stencils[(size_t)(pr * e.ss + si)];
    if (cudaMalloc(&e.d_kc, sizeof(double) * 6) != cudaSuccess) throw std::runtime_error("alloc kc");
    cudaMemcpy(e.d_kc, kc.data(), sizeof(double) * 6, cudaMemcpyHostToDevice);
}

void launch_direct_apply(Engine& e, const double* u, double* f, int batch, cudaStream_t s, double scale,
                         const uint8_t* cmask) {
    const Plan& pl = e.plan;
    PassTimer pt(e, kPassVec, s);
    if (e.dim == 2) {
        dim3 grid((pl.N[0] + kTX - 1) / kTX, (pl.N[1] + kTY - 1) / kTY, batch);
        dim3 block(kTX, kTY / kRows);
        switch (e.M) {
            case 1: k_direct2d<1><<<grid, block, 0, s>>>(u, f, e.d_K, pl.N[0], pl.N[1], pl.nodes, scale, cmask); break;
            case 2: k_direct2d<2><<<grid, block, 0, s>>>(u, f, e.d_K, pl.N[0], pl.N[1], pl.nodes, scale, cmask); break;
            case 3: k_direct2d<3><<<grid, block, 0, s>>>(u, f, e.d_K, pl.N[0], pl.N[1], pl.nodes, scale, cmask); break;
            case 4: k_direct2d<4><<<grid, block, 0, s>>>(u, f, e.d_K, pl.N[0], pl.N[1], pl.nodes, scale, cmask); break;
            case 5: k_direct2d<5><<<grid, block, 0, s>>>(u, f, e.d_K, pl.N[0], pl.N[1], pl.nodes, scale, cmask); break;
            default: throw std::runtime_error("direct stencil: 2D horizon M must be 1..5");
        }
    } else {
        direct_prepare(e);
        const double* koff = e.d_K + e.np * e.ss;
        const int th = 256;
        dim3 grid((unsigned)((pl.nodes + th - 1) / th), batch);
        k_direct3d<<<grid, th, 0, s>>>(u, f, e.d_offs, koff, e.d_kc, e.nof, pl.N[0], pl.N[1], pl.N[2], pl.nodes,
                                      scale, cmask);
    }
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw std::runtime_error(std::string("direct launch: ") + cudaGetErrorString(err));
}

}  // namespace pdgpu
