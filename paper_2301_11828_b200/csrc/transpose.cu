// transpose.cu -- the all-to-all distributed FFT of a 2D lattice over G ranks
// (north_star's "NCCL all-to-all transposes over NVLink inside
// the distributed FFT").  The halo slabs (comm.cpp) are the default multi-GPU
// path; this is the comparison arm.
//
// Rank r owns rows [r0[r], r0[r+1]) of an Nx x Nyg lattice (its engine's
// lattice) and the half-spectrum columns [k0[r], k0[r+1]) of the y pass.
//   K1 (own rows) -> S1[b][c][kx][j]
//   pack:   send[s][b][c][kl < Kmax][j < Rmax] = S1[b][c][k0[s] + kl][j]
//   all-to-all (NCCL grouped send/recv, or device copies in a single process)
//   unpack: C1[b][c][kl][r0[s] + j] = recv[s][b][c][kl][j]      (j < R_s)
//   K3 over the global columns (length Nyg, this rank's symbol) -> C2
//   pack:   send[s][b][c][kl][j] = C2[b][c][kl][r0[s] + j]
//   all-to-all
//   unpack: S2[b][c][k0[s] + kl][j] = recv[s][b][c][kl][j]      (kl < K_s)
//   K5 (own rows) -> f;  wrap correction: x aliases locally, y aliases at the
//   global faces from the opposite end's M rows (ghost entries, subtracted)
// Every peer block is Kmax x Rmax complex per (vector, component), so the
// exchange is a plain all-to-all of equal blocks.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "engine.h"

namespace pdgpu {

void build_symbol_cols(Engine& e, const Plan& pl, int col0, void** out);
void launch_k3_2d_cols(Engine& e, const Plan& col, void* sym, const double2* in, double2* out, int batch,
                       cudaStream_t s);
void launch_k1(Engine& e, const double* u, int batch, cudaStream_t s);
void launch_k5(Engine& e, const double2* xin, double* f, int batch, cudaStream_t s, double scale,
               const uint8_t* cmask, const double* body);
void build_twiddles(Engine& e);
void engine_alloc_workspace(Engine& e, int64_t batch);

namespace {

void check(cudaError_t err, const char* what) {
    if (err != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(err));
}

// elements: (s, bc, kl, j) over G x BC x Kmax x Rmax, j fastest
__global__ void k_a2a_pack_rows(const double2* __restrict__ S1, double2* __restrict__ send, const int* __restrict__ k0,
                                int G, int BC, int Hx, int R, int Kmax, int Rmax) {
    const int64_t n = (int64_t)G * BC * Kmax * Rmax;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i % Rmax);
        int64_t r = i / Rmax;
        const int kl = (int)(r % Kmax);
        r /= Kmax;
        const int bc = (int)(r % BC), s = (int)(r / BC);
        const int kx = k0[s] + kl;
        send[i] = (j < R && kx < k0[s + 1]) ? S1[((int64_t)bc * Hx + kx) * R + j] : make_double2(0.0, 0.0);
    }
}

// recv[s][bc][kl][j] -> C[bc][kl][r0[s] + j]  (kl < ncol, j < R_s)
__global__ void k_a2a_unpack_cols(const double2* __restrict__ recv, double2* __restrict__ C, const int* __restrict__ r0,
                                  int G, int BC, int ncol, int Nyg, int Kmax, int Rmax) {
    const int64_t n = (int64_t)G * BC * Kmax * Rmax;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i % Rmax);
        int64_t r = i / Rmax;
        const int kl = (int)(r % Kmax);
        r /= Kmax;
        const int bc = (int)(r % BC), s = (int)(r / BC);
        if (kl >= ncol || j >= r0[s + 1] - r0[s]) continue;
        C[((int64_t)bc * ncol + kl) * Nyg + r0[s] + j] = recv[i];
    }
}

// C[bc][kl][r0[s] + j] -> send[s][bc][kl][j]
__global__ void k_a2a_pack_cols(const double2* __restrict__ C, double2* __restrict__ send, const int* __restrict__ r0,
                                int G, int BC, int ncol, int Nyg, int Kmax, int Rmax) {
    const int64_t n = (int64_t)G * BC * Kmax * Rmax;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i % Rmax);
        int64_t r = i / Rmax;
        const int kl = (int)(r % Kmax);
        r /= Kmax;
        const int bc = (int)(r % BC), s = (int)(r / BC);
        send[i] = (kl < ncol && j < r0[s + 1] - r0[s]) ? C[((int64_t)bc * ncol + kl) * Nyg + r0[s] + j]
                                                      : make_double2(0.0, 0.0);
    }
}

// recv[s][bc][kl][j] -> S2[bc][k0[s] + kl][j]  (kl < K_s, j < R)
__global__ void k_a2a_unpack_rows(const double2* __restrict__ recv, double2* __restrict__ S2, const int* __restrict__ k0,
                                  int G, int BC, int Hx, int R, int Kmax, int Rmax) {
    const int64_t n = (int64_t)G * BC * Kmax * Rmax;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i % Rmax);
        int64_t r = i / Rmax;
        const int kl = (int)(r % Kmax);
        r /= Kmax;
        const int bc = (int)(r % BC), s = (int)(r / BC);
        if (j >= R || kl >= k0[s + 1] - k0[s]) continue;
        S2[((int64_t)bc * Hx + k0[s] + kl) * R + j] = recv[i];
    }
}

unsigned grid_for(const Engine& e, int64_t n) {
    return (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)e.num_sms * 8);
}

}  // namespace

void a2a_free(Engine& e) {
    A2A& a = e.a2a;
    for (void* p : {(void*)a.d_sym, (void*)a.d_c1, (void*)a.d_c2, (void*)a.d_send, (void*)a.d_recv, (void*)a.d_alias,
                    (void*)a.d_bounds})
        if (p) cudaFree(p);
    a = A2A();
}

int64_t a2a_block(const Engine& e, int batch) {
    return (int64_t)batch * e.dim * e.a2a.Kmax * e.a2a.Rmax;
}

void a2a_setup(Engine& e, int G, int rank, int Nyg, const int* r0, const int* k0) {
    if (e.dim != 2) throw std::runtime_error("the distributed FFT arm is 2D");
    if (G < 1 || rank < 0 || rank >= G) throw std::runtime_error("bad rank");
    if (Nyg < 16 || (Nyg & (Nyg - 1))) throw std::runtime_error("distributed FFT: global rows must be a power of two >= 16");
    const Plan& pl = e.plan;
    if (!pl.circ[0]) throw std::runtime_error("distributed FFT: x must use the periodic embedding");
    if (r0[0] != 0 || r0[G] != Nyg || k0[0] != 0 || k0[G] != pl.Hx)
        throw std::runtime_error("distributed FFT: row / column splits must cover the lattice");
    for (int g = 0; g < G; ++g)
        if (r0[g + 1] < r0[g] || k0[g + 1] < k0[g]) throw std::runtime_error("distributed FFT: decreasing split");
    if (r0[rank + 1] - r0[rank] != pl.N[1]) throw std::runtime_error("distributed FFT: engine rows != its share");
    if (pl.N[1] < 2 * e.M + 1) throw std::runtime_error("distributed FFT: a rank needs at least 2M+1 rows");
    a2a_free(e);
    A2A& a = e.a2a;
    a.G = G;
    a.rank = rank;
    a.Nyg = Nyg;
    a.r0.assign(r0, r0 + G + 1);
    a.k0.assign(k0, k0 + G + 1);
    for (int g = 0; g < G; ++g) {
        a.Rmax = std::max(a.Rmax, r0[g + 1] - r0[g]);
        a.Kmax = std::max(a.Kmax, k0[g + 1] - k0[g]);
    }
    // column plan: this rank's columns, global length Nyg (periodic, one half)
    Plan c = pl;
    c.ncols = k0[rank + 1] - k0[rank];
    c.Nl = c.Pl = Nyg;
    int l = 0;
    while ((1 << l) < Nyg) ++l;
    c.logPl = l;
    c.nh = 1;
    c.P[1] = Nyg;
    a.col = c;
    // twiddles long enough for the global columns
    if (l > e.plan.logTWN) {
        e.plan.logTWN = l;
        build_twiddles(e);
    }
    a.col.logTWN = e.plan.logTWN;
    build_symbol_cols(e, a.col, k0[rank], &a.d_sym);
    // bounds on the device: r0 (G+1) then k0 (G+1), in a small int buffer
    std::vector<int> b(a.r0);
    b.insert(b.end(), a.k0.begin(), a.k0.end());
    check(cudaMalloc(&a.d_bounds, sizeof(int) * b.size()), "alloc bounds");
    check(cudaMemcpy(a.d_bounds, b.data(), sizeof(int) * b.size(), cudaMemcpyHostToDevice), "copy bounds");
    // slab frame: D^e and near-surface flags of the global faces, positions and ids
    e.slab.off = r0[rank];
    e.slab.global = Nyg;
    // the wrap tables in distributed-FFT form
    touch_state(e);
    for (void** p : {(void**)&e.d_wrows, (void**)&e.d_wo0, (void**)&e.d_wK, (void**)&e.d_lidx, (void**)&e.d_loff,
                     (void**)&e.d_lK, (void**)&e.d_sidx, (void**)&e.d_stab, (void**)&e.d_fidx, (void**)&e.d_ftab}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    build_wrap_table(e);
    if (!e.d_stab) throw std::runtime_error("distributed FFT: wrap tables unavailable");
    e.cap_batch = 0;  // workspace re-sized on the next call
}

void a2a_ensure(Engine& e, int batch) {
    A2A& a = e.a2a;
    engine_alloc_workspace(e, batch);
    if (batch <= a.cap) return;
    touch_state(e);
    for (double2** p : {&a.d_c1, &a.d_c2, &a.d_send, &a.d_recv}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    if (a.d_alias) cudaFree(a.d_alias);
    const int64_t cols = (int64_t)batch * e.dim * a.col.ncols * a.Nyg;
    const int64_t blk = (int64_t)a.G * a2a_block(e, batch);
    check(cudaMalloc(&a.d_c1, sizeof(double2) * std::max<int64_t>(cols, 1)), "alloc C1");
    check(cudaMalloc(&a.d_c2, sizeof(double2) * std::max<int64_t>(cols, 1)), "alloc C2");
    check(cudaMalloc(&a.d_send, sizeof(double2) * blk), "alloc send");
    check(cudaMalloc(&a.d_recv, sizeof(double2) * blk), "alloc recv");
    // opposite-end rows: [send|recv][side][batch][dim][M][Nx]
    check(cudaMalloc(&a.d_alias, sizeof(double) * 4 * (size_t)batch * e.dim * e.M * e.plan.N[0]), "alloc alias rows");
    a.cap = batch;
}

void a2a_phase1(Engine& e, const double* u, int batch, cudaStream_t s) {
    A2A& a = e.a2a;
    a2a_ensure(e, batch);
    {
        PassTimer pt(e, kPassK1, s);
        launch_k1(e, u, batch, s);
    }
    const int* bounds = a.d_bounds;
    const int64_t n = (int64_t)a.G * a2a_block(e, batch);
    PassTimer pt(e, kPassHalo, s);
    k_a2a_pack_rows<<<grid_for(e, n), 256, 0, s>>>(e.d_S1, a.d_send, bounds + a.G + 1, a.G, batch * e.dim,
                                                   e.plan.Hx, e.plan.N[1], a.Kmax, a.Rmax);
    check(cudaGetLastError(), "a2a pack rows");
}

void a2a_phase2(Engine& e, int batch, cudaStream_t s) {
    A2A& a = e.a2a;
    const int* bounds = a.d_bounds;
    const int64_t n = (int64_t)a.G * a2a_block(e, batch);
    {
        PassTimer pt(e, kPassHalo, s);
        k_a2a_unpack_cols<<<grid_for(e, n), 256, 0, s>>>(a.d_recv, a.d_c1, bounds, a.G, batch * e.dim, a.col.ncols,
                                                         a.Nyg, a.Kmax, a.Rmax);
        check(cudaGetLastError(), "a2a unpack columns");
    }
    if (a.col.ncols > 0) {
        PassTimer pt(e, kPassK3, s);
        launch_k3_2d_cols(e, a.col, a.d_sym, a.d_c1, a.d_c2, batch, s);
    }
    PassTimer pt(e, kPassHalo, s);
    k_a2a_pack_cols<<<grid_for(e, n), 256, 0, s>>>(a.d_c2, a.d_send, bounds, a.G, batch * e.dim, a.col.ncols, a.Nyg,
                                                   a.Kmax, a.Rmax);
    check(cudaGetLastError(), "a2a pack columns");
}

void a2a_phase3(Engine& e, double* f, int batch, cudaStream_t s, double scale, const uint8_t* cmask,
                const double* body) {
    A2A& a = e.a2a;
    const int* bounds = a.d_bounds;
    const int64_t n = (int64_t)a.G * a2a_block(e, batch);
    {
        PassTimer pt(e, kPassHalo, s);
        k_a2a_unpack_rows<<<grid_for(e, n), 256, 0, s>>>(a.d_recv, e.d_S2, bounds + a.G + 1, a.G, batch * e.dim,
                                                         e.plan.Hx, e.plan.N[1], a.Kmax, a.Rmax);
        check(cudaGetLastError(), "a2a unpack rows");
    }
    PassTimer pt(e, kPassK5, s);
    launch_k5(e, e.d_S2, f, batch, s, scale, cmask, body);
}

double* a2a_alias_recv(Engine& e, int batch) {
    return e.a2a.d_alias + (size_t)2 * batch * e.dim * e.M * e.plan.N[0];
}

// d_send -> d_recv: NCCL all-to-all of equal blocks, or a copy on one rank
void a2a_exchange(Engine& e, int batch, cudaStream_t s) {
    A2A& a = e.a2a;
    PassTimer pt(e, kPassHalo, s);
    if (a.G == 1) {
        check(cudaMemcpyAsync(a.d_recv, a.d_send, sizeof(double2) * a2a_block(e, batch), cudaMemcpyDeviceToDevice, s),
              "a2a self copy");
        return;
    }
    a2a_nccl_exchange(e, batch, s);
}

// the M rows beyond each slab face in the global periodic sense (side 0: the
// rows before the slab, from rank - 1 mod G; side 1: the rows after it, from
// rank + 1 mod G) as ghost rows of the wrap correction: across a global face
// every entry that leaves the slab aliases onto them, across an interior face
// those that also leave along x
void a2a_alias(Engine& e, const double* u, int batch, cudaStream_t s) {
    A2A& a = e.a2a;
    const size_t side = (size_t)batch * e.dim * e.M * e.plan.N[0];
    double* send = a.d_alias;
    double* recv = a2a_alias_recv(e, batch);
    e.ghost_bc_stride = (int64_t)e.M * e.plan.N[0];
    e.ghost_side_stride = (int64_t)side;
    PassTimer pt(e, kPassHalo, s);
    halo_pack(e, u, batch, send, s);  // side 0 = the first M rows, side 1 = the last M
    if (a.G == 1) {                   // both ends are this rank: swap the sides
        check(cudaMemcpyAsync(recv, send + side, sizeof(double) * side, cudaMemcpyDeviceToDevice, s), "alias lo");
        check(cudaMemcpyAsync(recv + side, send, sizeof(double) * side, cudaMemcpyDeviceToDevice, s), "alias hi");
    } else {
        a2a_nccl_alias(e, batch, s);
    }
    e.ghost_view = recv;
}

}  // namespace pdgpu
