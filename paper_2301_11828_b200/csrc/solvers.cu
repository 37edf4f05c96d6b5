// solvers.cu -- CG vector kernels (fused axpy + dot, deterministic
// warp-shuffle reductions) and the velocity-Verlet elementwise kernels.
//
// CG is new work (the reference has only ADR, timestepping.hpp:79-145);
// VV drift/kick/constraints follow timestepping.hpp:312-334 and
// corrections.hpp:142-160.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "engine.h"

namespace pdgpu {

static void check(cudaError_t e, const char* what);

constexpr int kRedBlocks = 592;  // 4 x 148 SMs, fixed => deterministic order

constexpr int kRedThreads = 256;

// CG reduction grid: one block per SM for small systems (cheaper totals and
// grid barriers), kRedBlocks otherwise.  Every CG kernel of a solve uses the
// same grid, so the fused and the split (multi-rank) steps sum in the same
// order (bit-identical iterates).
static int cg_red_grid(const Engine& e, int64_t n) {
    if (const char* genv = getenv("PDGPU_CG_GRID")) return std::max(1, std::min(kRedBlocks, atoi(genv)));
    return n <= (int64_t)e.num_sms * kRedThreads * 16 ? std::min(e.num_sms, kRedBlocks) : kRedBlocks;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-reduce v into partial[blockIdx.x]; the last block to finish sums the
// partials in index order into *out.  Deterministic for a fixed grid.
__device__ void grid_reduce(double v, double* partial, unsigned int* ticket, double* out) {
    __shared__ double ws[32];
    __shared__ bool last;
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) ws[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double s = lane < (blockDim.x >> 5) ? ws[lane] : 0.0;
        s = warp_sum(s);
        if (lane == 0) {
            partial[blockIdx.x] = s;
            __threadfence();
            const unsigned int t = atomicAdd(ticket, 1u);
            last = (t == gridDim.x - 1);
        }
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double s = 0.0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += ((volatile double*)partial)[i];
        s = warp_sum(s);
        if (lane == 0) ws[wid] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += ws[w];
            *out = tot;
            *ticket = 0u;
        }
    }
}

__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* partial,
                      unsigned int* ticket, double* out) {
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += a[i] * b[i];
    grid_reduce(s, partial, ticket, out);
}

// scal[0] = rr, scal[1] = p.q ; alpha = rr / pq ; x += alpha p ; r -= alpha q ; rr_out = r.r
__global__ void k_cg_update(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                            const double* __restrict__ q, int64_t n, const double* scal, double* partial,
                            unsigned int* ticket, double* rr_out) {
    const double alpha = scal[0] / scal[1];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        s += ri * ri;
    }
    grid_reduce(s, partial, ticket, rr_out);
}

// beta = scal[2] / scal[0] ; p = r + beta p
__global__ void k_cg_direction(double* __restrict__ p, const double* __restrict__ r, int64_t n,
                               const double* scal) {
    const double beta = scal[2] / scal[0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = r[i] + beta * p[i];
}

__global__ void k_rotate(double* scal) { scal[0] = scal[2]; }

// ---- graph-replayable CG step with the convergence test on the device ----
// scal = {rr, p.q, rr_new, tol^2 * rr_0, done, iterations, -, rr_old}
template <class CB>
__device__ void grid_reduce_cb(double v, double* partial, unsigned int* ticket, CB cb) {
    __shared__ double ws[32];
    __shared__ bool last;
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) ws[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double s = lane < (blockDim.x >> 5) ? ws[lane] : 0.0;
        s = warp_sum(s);
        if (lane == 0) {
            partial[blockIdx.x] = s;
            __threadfence();
            const unsigned int t = atomicAdd(ticket, 1u);
            last = (t == gridDim.x - 1);
        }
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double s = 0.0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += ((volatile double*)partial)[i];
        s = warp_sum(s);
        if (lane == 0) ws[wid] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += ws[w];
            cb(tot);
            *ticket = 0u;
        }
    }
}

__global__ void k_cg_update_dev(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                                const double* __restrict__ q, int64_t n, double* scal, double* partial,
                                unsigned int* ticket) {
    if (scal[4] != 0.0) return;
    const double alpha = scal[0] / scal[1];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        s += ri * ri;
    }
    // the last block runs this after every block has read alpha (scal[0]):
    // rotate rr in place (old -> scal[7], new -> scal[0] and scal[2]), so no
    // separate rotation kernel is needed
    grid_reduce_cb(s, partial, ticket, [&](double tot) {
        scal[7] = scal[0];
        scal[0] = tot;
        scal[2] = tot;
        scal[5] += 1.0;
        if (tot <= scal[3] || scal[5] >= scal[6]) scal[4] = 1.0;  // converged, or the iteration cap
    });
}

// multi-rank variant (NCCL): the update writes this rank's r.r to scal[9];
// after the all-reduce of scal[9], k_cg_finish rotates and tests on one thread
__global__ void k_cg_update_local(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                                  const double* __restrict__ q, int64_t n, double* scal, double* partial,
                                  unsigned int* ticket) {
    if (scal[4] != 0.0) return;
    const double alpha = scal[0] / scal[1];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        s += ri * ri;
    }
    grid_reduce_cb(s, partial, ticket, [&](double tot) { scal[9] = tot; });
}

__global__ void k_cg_finish(double* scal) {
    if (scal[4] != 0.0) return;
    const double tot = scal[9];
    scal[7] = scal[0];
    scal[0] = tot;
    scal[2] = tot;
    scal[5] += 1.0;
    if (tot <= scal[3]) scal[4] = 1.0;
}

__global__ void k_cg_direction_dev(double* __restrict__ p, const double* __restrict__ r, int64_t n,
                                   const double* scal) {
    if (scal[4] != 0.0) return;
    const double beta = scal[0] / scal[7];  // rr_new / rr_old, rotated by k_cg_update_dev
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = r[i] + beta * p[i];
}

// ---- one CG step in one cooperative kernel (graph-captured single-GPU CG):
// p.q, the x / r update with r.r, and the new direction, separated by two grid
// barriers instead of three launches.  Every block forms the totals itself from
// the per-block partials in the same fixed order as grid_reduce's last block,
// so the iterates are bit-identical to k_dot + k_cg_update_dev +
// k_cg_direction_dev.
__device__ __forceinline__ void block_partial(double v, double* partial, double* ws) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) ws[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double s = lane < (blockDim.x >> 5) ? ws[lane] : 0.0;
        s = warp_sum(s);
        if (lane == 0) partial[blockIdx.x] = s;
    }
    __syncthreads();
}

__device__ __forceinline__ double block_total(const double* partial, double* ws, double* tot) {
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += __ldcg(partial + i);  // not L1: other SMs wrote it
    s = warp_sum(s);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) ws[wid] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
        *tot = t;
    }
    __syncthreads();
    return *tot;
}

__global__ void __launch_bounds__(kRedThreads) k_cg_fused(double* __restrict__ x, double* __restrict__ r,
                                                         double* __restrict__ p, const double* __restrict__ q,
                                                         int64_t n, double* scal, double* partA, double* partB) {
    namespace cg = cooperative_groups;
    __shared__ double ws[32];
    __shared__ double tot;
    if (scal[4] != 0.0) return;  // converged: every block leaves before any barrier
    const double rr = scal[0], thr = scal[3];
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
    double s = 0.0;
    for (int64_t i = i0; i < n; i += st) s += p[i] * q[i];
    block_partial(s, partA, ws);
    cg::this_grid().sync();
    const double pq = block_total(partA, ws, &tot);
    const double alpha = rr / pq;
    s = 0.0;
    for (int64_t i = i0; i < n; i += st) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        s += ri * ri;
    }
    block_partial(s, partB, ws);
    cg::this_grid().sync();
    const double rrn = block_total(partB, ws, &tot);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        scal[1] = pq;
        scal[7] = rr;
        scal[0] = rrn;
        scal[2] = rrn;
        scal[5] += 1.0;
        if (rrn <= thr || scal[5] >= scal[6]) scal[4] = 1.0;  // converged, or the iteration cap
    }
    if (rrn <= thr) return;
    const double beta = rrn / rr;
    for (int64_t i = i0; i < n; i += st) p[i] = r[i] + beta * p[i];
}

// true when the fused step can run (all kRedBlocks co-resident); launches it
bool launch_cg_fused(Engine& e, double* x, double* r, double* p, const double* q, int64_t n, double* scal,
                     cudaStream_t s) {
    static int ok = -1;
    if (ok < 0) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_fused, kRedThreads, 0);
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, e.device);
        const char* env = getenv("PDGPU_CG_FUSED");
        ok = coop && per_sm * e.num_sms >= kRedBlocks && !(env && env[0] == '0');
    }
    if (!ok) return false;
    cudaLaunchConfig_t cfg = {};
    // small systems: one block per SM (cheaper grid barriers and totals);
    // the reduction order is fixed by the grid, so results are deterministic
    const int grid = cg_red_grid(e, n);
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kRedThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    check(cudaLaunchKernelEx(&cfg, k_cg_fused, x, r, p, q, n, scal, e.d_red, e.d_red + 1024), "cg fused");
    e.launches += 1;
    return true;
}

__global__ void k_mask_rhs(double* out, const double* b, const double* Auc, const uint8_t* cmask, int64_t N,
                           int dim) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * dim) return;
    const int a = (int)(i / N);
    const int64_t p = i - (int64_t)a * N;
    const double v = b[i] + (Auc ? Auc[i] : 0.0);
    out[i] = ((cmask[p] >> a) & 1u) ? 0.0 : v;
}

__global__ void k_vv_drift(double* u, const double* v, const double* f, const uint8_t* cmask, int64_t N, int dim,
                           double dt, double inv_rho) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * dim) return;
    const int a = (int)(i / N);
    const int64_t p = i - (int64_t)a * N;
    if ((cmask[p] >> a) & 1u) return;
    // u += dt*v + 0.5*dt*dt*f*inv_rho   (timestepping.hpp:318-319, same order, no contraction)
    const double t1 = __dmul_rn(dt, v[i]);
    const double t2 = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(0.5, dt), dt), f[i]), inv_rho);
    u[i] = __dadd_rn(u[i], __dadd_rn(t1, t2));
}

__global__ void k_vv_kick(double* v, const double* fprev, const double* f, const uint8_t* cmask, int64_t N, int dim,
                          double dt, double inv_rho) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * dim) return;
    const int a = (int)(i / N);
    const int64_t p = i - (int64_t)a * N;
    if ((cmask[p] >> a) & 1u) return;
    // v += 0.5*dt*(f_prev + f)*inv_rho   (timestepping.hpp:330-331)
    const double t = __dmul_rn(__dmul_rn(__dmul_rn(0.5, dt), __dadd_rn(fprev[i], f[i])), inv_rho);
    v[i] = __dadd_rn(v[i], t);
}

// ------------------------------------------------------------------ ADR --
// AdrIntegrator (timestepping.hpp:79-145).  Damping estimate: num = sum u^2 k
// (k > 0), den = sum u^2 over unconstrained DOFs, k = -(f - f_prev) /
// (m_a dt v_half); deterministic two-value grid reduction (fixed grid, the
// last block sums the partials in index order) that leaves c in *cout.
__global__ void k_adr_damping(const double* __restrict__ u, const double* __restrict__ vh,
                              const double* __restrict__ f, const double* __restrict__ fprev,
                              const uint8_t* __restrict__ cmask, int64_t N, int dim, double m0, double m1, double m2,
                              double dt, double* partial, unsigned int* ticket, double* cout, int raw) {
    __shared__ double ws[2][32];
    __shared__ bool last;
    double num = 0.0, den = 0.0;
    const int64_t tot = N * dim;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int a = (int)(i / N);
        const int64_t p = i - (int64_t)a * N;
        if ((cmask[p] >> a) & 1u) continue;
        const double m = a == 0 ? m0 : (a == 1 ? m1 : m2);
        const double up = u[i], v = vh[i];
        double k = 0.0;
        if (v != 0.0) k = -__ddiv_rn(__dadd_rn(f[i], -fprev[i]), __dmul_rn(__dmul_rn(m, dt), v));
        const double u2 = __dmul_rn(up, up);
        if (k > 0.0) num = __dadd_rn(num, __dmul_rn(u2, k));
        den = __dadd_rn(den, u2);
    }
    num = warp_sum(num);
    den = warp_sum(den);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        ws[0][wid] = num;
        ws[1][wid] = den;
    }
    __syncthreads();
    if (wid == 0) {
        double a = lane < (int)(blockDim.x >> 5) ? ws[0][lane] : 0.0;
        double b = lane < (int)(blockDim.x >> 5) ? ws[1][lane] : 0.0;
        a = warp_sum(a);
        b = warp_sum(b);
        if (lane == 0) {
            partial[2 * blockIdx.x] = a;
            partial[2 * blockIdx.x + 1] = b;
            __threadfence();
            last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double sn = 0.0, sd = 0.0;
        for (int i = 0; i < (int)gridDim.x; ++i) {
            sn += ((volatile double*)partial)[2 * i];
            sd += ((volatile double*)partial)[2 * i + 1];
        }
        if (raw) {  // multi-rank: this rank's sums to cout[2], cout[3]; k_adr_c after the all-reduce
            cout[2] = sn;
            cout[3] = sd;
        } else {
            double c = 0.0;
            if (!(sd <= 0.0 || sn <= 0.0)) c = fmin(2.0 * sqrt(sn / sd), 1.9 / dt);
            *cout = c;
        }
        *ticket = 0u;
    }
}

__global__ void k_adr_c(double* cout, double dt) {
    const double sn = cout[2], sd = cout[3];
    double c = 0.0;
    if (!(sd <= 0.0 || sn <= 0.0)) c = fmin(2.0 * sqrt(sn / sd), 1.9 / dt);
    *cout = c;
}

// first call: v_half = 0.5 dt f / m (unconstrained); else v_half = (lead v_half
// + 2 dt f / m) * trail with c from *cdev (or the fixed damping); then u += dt v_half
__global__ void k_adr_advance(double* __restrict__ u, double* __restrict__ vh, const double* __restrict__ f,
                              const uint8_t* __restrict__ cmask, int64_t N, int dim, double m0, double m1, double m2,
                              double dt, int first, const double* __restrict__ cdev) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * dim) return;
    const int a = (int)(i / N);
    const int64_t p = i - (int64_t)a * N;
    if ((cmask[p] >> a) & 1u) return;
    const double inv_m = __ddiv_rn(1.0, a == 0 ? m0 : (a == 1 ? m1 : m2));
    double v;
    if (first) {
        v = __dmul_rn(__dmul_rn(__dmul_rn(0.5, dt), f[i]), inv_m);
    } else {
        const double c = *cdev;
        const double lead = __dadd_rn(2.0, -__dmul_rn(c, dt));
        const double trail = __ddiv_rn(1.0, __dadd_rn(2.0, __dmul_rn(c, dt)));
        v = __dmul_rn(__dadd_rn(__dmul_rn(lead, vh[i]), __dmul_rn(__dmul_rn(__dmul_rn(2.0, dt), f[i]), inv_m)), trail);
    }
    vh[i] = v;
    u[i] = __dadd_rn(u[i], __dmul_rn(dt, v));
}

__global__ void k_set_scalar(double* dst, double v) { *dst = v; }

__global__ void k_enforce(double* u, double* v, const long long* dofs, const double* val, const int* kind, int64_t n,
                          double t) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t k = dofs[i];
    if (kind[i] == 0) {
        u[k] = val[i];
        v[k] = 0.0;
    } else {
        u[k] = __dmul_rn(val[i], t);
        v[k] = val[i];
    }
}

__global__ void k_scatter(double* y, const long long* ids, const double* val, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[ids[i]] = val[i];
}

__global__ void k_axpy(double* y, const double* x, double a, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] += a * x[i];
}

static void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

static unsigned blocks_for(int64_t n, int th) { return (unsigned)((n + th - 1) / th); }

void launch_dot(Engine& e, const double* a, const double* b, int64_t n, double* out_dev, cudaStream_t s) {
    k_dot<<<cg_red_grid(e, n), kRedThreads, 0, s>>>(a, b, n, e.d_red, e.d_ticket, out_dev);
    check(cudaGetLastError(), "dot");
}

void launch_cg_update(Engine& e, double* x, double* r, const double* p, const double* q, int64_t n,
                      const double* scal, double* rr_out, cudaStream_t s) {
    k_cg_update<<<cg_red_grid(e, n), kRedThreads, 0, s>>>(x, r, p, q, n, scal, e.d_red, e.d_ticket, rr_out);
    check(cudaGetLastError(), "cg_update");
}

void launch_cg_step_dev(Engine& e, double* x, double* r, double* p, const double* q, int64_t n, double* scal,
                        cudaStream_t s) {
    k_cg_update_dev<<<cg_red_grid(e, n), kRedThreads, 0, s>>>(x, r, p, q, n, scal, e.d_red, e.d_ticket);
    k_cg_direction_dev<<<cg_red_grid(e, n), kRedThreads, 0, s>>>(p, r, n, scal);
    e.launches += 2;
    check(cudaGetLastError(), "cg_step_dev");
}

void launch_cg_step_dev_comm(Engine& e, double* x, double* r, double* p, const double* q, int64_t n, double* scal,
                             cudaStream_t s) {
    k_cg_update_local<<<cg_red_grid(e, n), kRedThreads, 0, s>>>(x, r, p, q, n, scal, e.d_red, e.d_ticket);
    comm_allreduce(e, scal + 9, 1, s);
    k_cg_finish<<<1, 1, 0, s>>>(scal);
    k_cg_direction_dev<<<cg_red_grid(e, n), kRedThreads, 0, s>>>(p, r, n, scal);
    e.launches += 3;
    check(cudaGetLastError(), "cg_step_dev_comm");
}

void launch_cg_direction(double* p, const double* r, int64_t n, const double* scal, cudaStream_t s) {
    k_cg_direction<<<kRedBlocks, kRedThreads, 0, s>>>(p, r, n, scal);
    k_rotate<<<1, 1, 0, s>>>(const_cast<double*>(scal));
    check(cudaGetLastError(), "cg_direction");
}

void launch_mask_rhs(double* out, const double* b, const double* Auc, const uint8_t* cmask, int64_t N, int dim,
                     cudaStream_t s) {
    k_mask_rhs<<<blocks_for(N * dim, 256), 256, 0, s>>>(out, b, Auc, cmask, N, dim);
    check(cudaGetLastError(), "mask_rhs");
}

void launch_vv_drift(double* u, const double* v, const double* f, const uint8_t* cmask, int64_t N, int dim, double dt,
                     double inv_rho, cudaStream_t s) {
    k_vv_drift<<<blocks_for(N * dim, 256), 256, 0, s>>>(u, v, f, cmask, N, dim, dt, inv_rho);
    check(cudaGetLastError(), "vv_drift");
}

// kick of step n and drift of step n + 1 in one pass (timestepping.hpp:330-331
// then :318-319 of the next step): the same operations in the same order, so
// v and u are bit-identical to k_vv_kick followed by k_vv_drift; six array
// passes instead of eight
__global__ void k_vv_kick_drift(double* u, double* v, const double* fprev, const double* f, const uint8_t* cmask,
                                int64_t N, int dim, double dt, double inv_rho) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * dim) return;
    const int a = (int)(i / N);
    const int64_t p = i - (int64_t)a * N;
    if ((cmask[p] >> a) & 1u) return;
    const double fi = f[i];
    const double t = __dmul_rn(__dmul_rn(__dmul_rn(0.5, dt), __dadd_rn(fprev[i], fi)), inv_rho);
    const double vn = __dadd_rn(v[i], t);
    v[i] = vn;
    const double t1 = __dmul_rn(dt, vn);
    const double t2 = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(0.5, dt), dt), fi), inv_rho);
    u[i] = __dadd_rn(u[i], __dadd_rn(t1, t2));
}

void launch_vv_kick_drift(double* u, double* v, const double* fprev, const double* f, const uint8_t* cmask, int64_t N,
                          int dim, double dt, double inv_rho, cudaStream_t s) {
    k_vv_kick_drift<<<blocks_for(N * dim, 256), 256, 0, s>>>(u, v, fprev, f, cmask, N, dim, dt, inv_rho);
    check(cudaGetLastError(), "vv_kick_drift");
}

void launch_vv_kick(double* v, const double* fprev, const double* f, const uint8_t* cmask, int64_t N, int dim,
                    double dt, double inv_rho, cudaStream_t s) {
    k_vv_kick<<<blocks_for(N * dim, 256), 256, 0, s>>>(v, fprev, f, cmask, N, dim, dt, inv_rho);
    check(cudaGetLastError(), "vv_kick");
}

void launch_adr_step(Engine& e, bool first, cudaStream_t s) {
    const int64_t N = e.plan.nodes, m = N * e.dim;
    double* cdev = e.d_scal + 10;  // CG uses scal[0..9]; [10] = c, [12..13] = the rank's raw sums
    if (!first) {
        if (e.adr_fixed) {
            k_set_scalar<<<1, 1, 0, s>>>(cdev, e.adr_fixed_c);
        } else {
            const bool multi = comm_attached(e);
            k_adr_damping<<<kRedBlocks, kRedThreads, 0, s>>>(e.d_u, e.d_vh, e.d_f, e.d_fprev, e.d_cmask, N, e.dim,
                                                             e.adr_mass[0], e.adr_mass[1], e.adr_mass[2], e.dt,
                                                             e.d_red, e.d_ticket, cdev, multi ? 1 : 0);
            if (multi) {
                comm_allreduce(e, cdev + 2, 2, s);
                k_adr_c<<<1, 1, 0, s>>>(cdev, e.dt);
                e.launches += 1;
            }
        }
        e.launches += 1;
    }
    k_adr_advance<<<blocks_for(m, 256), 256, 0, s>>>(e.d_u, e.d_vh, e.d_f, e.d_cmask, N, e.dim, e.adr_mass[0],
                                                     e.adr_mass[1], e.adr_mass[2], e.dt, first ? 1 : 0, cdev);
    e.launches += 1;
    check(cudaGetLastError(), "adr step");
}

void launch_enforce(double* u, double* v, const long long* dofs, const double* val, const int* kind, int64_t n,
                    double t, cudaStream_t s) {
    if (n == 0) return;
    k_enforce<<<blocks_for(n, 256), 256, 0, s>>>(u, v, dofs, val, kind, n, t);
    check(cudaGetLastError(), "enforce");
}

// MonitorWriter row: dst[k * dim + d] = u[d * N + nodes[k]]
__global__ void k_monitor_gather(const double* __restrict__ u, const long long* __restrict__ nodes, int n, int dim,
                                 int64_t N, double* __restrict__ dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * dim) return;
    const int k = i / dim, d = i - k * dim;
    dst[i] = u[(int64_t)d * N + nodes[k]];
}

void launch_monitor_gather(const double* u, const long long* nodes, int n, int dim, int64_t N, double* dst,
                           cudaStream_t s) {
    if (n <= 0) return;
    k_monitor_gather<<<(n * dim + 127) / 128, 128, 0, s>>>(u, nodes, n, dim, N, dst);
}

void launch_scatter(double* y, const long long* ids, const double* val, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    k_scatter<<<blocks_for(n, 256), 256, 0, s>>>(y, ids, val, n);
    check(cudaGetLastError(), "scatter");
}

// Simulation::finite() (timestepping.hpp:256-261): *ok = 0 if any entry of u
// is not finite (the caller sets *ok = 1 first)
__global__ void k_finite(const double* __restrict__ u, int64_t n, int* ok) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad = bad || !isfinite(u[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *ok = 0;
}

void launch_finite(const double* u, int64_t n, int* ok, cudaStream_t s) {
    k_finite<<<kRedBlocks, kRedThreads, 0, s>>>(u, n, ok);
    check(cudaGetLastError(), "finite");
}

void launch_axpy(double* y, const double* x, double a, int64_t n, cudaStream_t s) {
    k_axpy<<<blocks_for(n, 256), 256, 0, s>>>(y, x, a, n);
    check(cudaGetLastError(), "axpy");
}

}  // namespace pdgpu
