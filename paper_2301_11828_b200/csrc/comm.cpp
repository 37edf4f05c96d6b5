// comm.cpp -- multi-GPU halo slabs over NCCL, one process per
// GPU.  Host-side orchestration only: the kernels are the single-GPU ones.
//
// Rank r's engine holds rows [r0, r1) of the slowest axis (pdgpu_set_slab);
// ranks are ordered by slab, so the rows before the slab live on rank - 1 and
// the rows after it on rank + 1.  Every K.u (apply / matvec / evaluate_force)
// exchanges the M rows next to each interior face with those neighbours:
//
//   s:            record ev_fork ----------------- K1 .. K5 ------- wait ev_join -> K6w (reads the received rows)
//   comm_stream:  wait ev_fork -> pack (2 x memcpy2D) -> ncclSend/ncclRecv (grouped) -> record ev_join
//
// so the transfer overlaps the spectral passes, which need only the owned
// rows; only the wrap correction K6w reads the ghost rows.  CG dot products
// are all-reduced in place on the launching stream (capturable into the CG
// graph).  libnccl is dlopen'ed on first use (the one torch already loaded
// when present), so libpdgpu.so has no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "engine.h"

namespace pdgpu {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

NcclApi load_api() {
    NcclApi a;
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
        h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch's copy)
        if (!h) h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) {
        a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
        return a;
    }
    auto sym = [&](const char* n) {
        void* p = dlsym(h, n);
        if (!p) a.error = std::string("libnccl lacks ") + n;
        return p;
    };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    return a;
}

const NcclApi& api() {
    static const NcclApi a = load_api();
    if (!a.error.empty()) throw std::runtime_error(a.error);
    return a;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + api().GetErrorString(r));
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

int64_t plane_of(const Engine& e) {
    return e.dim == 3 ? (int64_t)e.plan.N[0] * e.plan.N[1] : e.plan.N[0];
}

}  // namespace

void comm_unique_id(void* out) {
    ncclUniqueId id;
    nccl_check(api().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    memcpy(out, &id, sizeof(id));
}

void comm_init(Engine& e, int nranks, int rank, const void* id) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank / nranks");
    comm_destroy(e);
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    nccl_check(api().CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
    e.nccl_comm = c;
    e.nranks = nranks;
    e.rank = rank;
    cuda_ok(cudaStreamCreateWithFlags(&e.comm_stream, cudaStreamNonBlocking), "comm stream");
    cuda_ok(cudaEventCreateWithFlags(&e.ev_fork, cudaEventDisableTiming), "event");
    cuda_ok(cudaEventCreateWithFlags(&e.ev_join, cudaEventDisableTiming), "event");
    touch_state(e);
}

void comm_destroy(Engine& e) {
    if (e.comm_stream) cudaStreamSynchronize(e.comm_stream);
    if (e.nccl_comm) api().CommDestroy((ncclComm_t)e.nccl_comm);
    if (e.comm_stream) cudaStreamDestroy(e.comm_stream);
    if (e.ev_fork) cudaEventDestroy(e.ev_fork);
    if (e.ev_join) cudaEventDestroy(e.ev_join);
    if (e.d_halo) cudaFree(e.d_halo);
    if (e.d_face_recv) cudaFree(e.d_face_recv);
    e.d_face_recv = nullptr;
    e.nccl_comm = nullptr;
    e.comm_stream = nullptr;
    e.ev_fork = e.ev_join = nullptr;
    e.d_halo = nullptr;
    e.halo_cap = 0;
    e.nranks = 1;
    e.rank = 0;
}

bool comm_attached(const Engine& e) { return e.nccl_comm != nullptr; }

static bool lo_face(const Engine& e) { return slab_lo_face(e); }
static bool hi_face(const Engine& e) { return slab_hi_face(e); }

// the halo exchange belongs to the halo slabs; the distributed FFT moves
// the spectrum instead (a2a_nccl_exchange) and only the global faces' rows
bool halo_active(const Engine& e) {
    return comm_attached(e) && e.nranks > 1 && slab_has_faces(e) && e.a2a.G == 0;
}

// [send|recv][side][batch][dim][M][plane]; side 0 = the rows before the slab
void ensure_halo(Engine& e, int batch) {
    if (batch <= e.halo_cap) return;
    touch_state(e);
    if (e.d_halo) cudaFree(e.d_halo);
    e.d_halo = nullptr;
    const size_t n = (size_t)2 * 2 * batch * e.dim * e.M * plane_of(e);
    cuda_ok(cudaMalloc(&e.d_halo, sizeof(double) * n), "alloc halo buffers");
    cuda_ok(cudaMemset(e.d_halo, 0, sizeof(double) * n), "zero halo buffers");
    e.halo_cap = batch;
}

void halo_pack(const Engine& e, const double* u, int batch, double* send, cudaStream_t s) {
    const int64_t plane = plane_of(e), N = e.plan.nodes, R = e.plan.N[e.dim - 1];
    const size_t w = sizeof(double) * (size_t)(e.M * plane);
    const size_t side = (size_t)batch * e.dim * e.M * plane;
    // the first M owned rows (to rank - 1) and the last M (to rank + 1), every (vector, component)
    cuda_ok(cudaMemcpy2DAsync(send, w, u, sizeof(double) * N, w, (size_t)batch * e.dim, cudaMemcpyDeviceToDevice, s),
            "pack low rows");
    cuda_ok(cudaMemcpy2DAsync(send + side, w, u + (R - e.M) * plane, sizeof(double) * N, w, (size_t)batch * e.dim,
                              cudaMemcpyDeviceToDevice, s),
            "pack high rows");
}

const double* halo_exchange_begin(Engine& e, const double* u, int batch, cudaStream_t s) {
    if (e.halo_external) return e.ghost_view;  // a group driver placed this call's ghost rows already
    if (!halo_active(e)) return nullptr;
    ensure_halo(e, batch);
    const int64_t plane = plane_of(e);
    const size_t side = (size_t)batch * e.dim * e.M * plane;
    const size_t stride = (size_t)2 * e.halo_cap * e.dim * e.M * plane;  // send block size
    double* send = e.d_halo;
    double* recv = e.d_halo + stride;
    cuda_ok(cudaEventRecord(e.ev_fork, s), "fork");
    cuda_ok(cudaStreamWaitEvent(e.comm_stream, e.ev_fork, 0), "fork wait");
    PassTimer pt(e, kPassHalo, e.comm_stream, 0);  // pack + transfer, on the comm stream (overlapped)
    halo_pack(e, u, batch, send, e.comm_stream);
    const ncclComm_t c = (ncclComm_t)e.nccl_comm;
    nccl_check(api().GroupStart(), "ncclGroupStart");
    if (lo_face(e)) {
        nccl_check(api().Send(send, side, ncclFloat64, e.rank - 1, c, e.comm_stream), "ncclSend low");
        nccl_check(api().Recv(recv, side, ncclFloat64, e.rank - 1, c, e.comm_stream), "ncclRecv low");
    }
    if (hi_face(e)) {
        nccl_check(api().Send(send + side, side, ncclFloat64, e.rank + 1, c, e.comm_stream), "ncclSend high");
        nccl_check(api().Recv(recv + side, side, ncclFloat64, e.rank + 1, c, e.comm_stream), "ncclRecv high");
    }
    nccl_check(api().GroupEnd(), "ncclGroupEnd");
    pt.finish();
    cuda_ok(cudaEventRecord(e.ev_join, e.comm_stream), "join");
    // ghost view of the received rows for K6w: [side][batch][dim][M][plane]
    e.ghost_view = recv;
    e.ghost_bc_stride = e.M * plane;
    e.ghost_side_stride = (int64_t)side;
    return recv;
}

void halo_exchange_end(Engine& e, cudaStream_t s) {
    if (e.halo_external) return;
    cuda_ok(cudaStreamWaitEvent(s, e.ev_join, 0), "join wait");
}

// the u halo of one field now (stream-ordered), for kernels outside a K.u
void halo_exchange_now(Engine& e, const double* u, cudaStream_t s) {
    if (halo_exchange_begin(e, u, 1, s)) halo_exchange_end(e, s);
}

// the ledger words of the last M rows (rank -> rank + 1) after a stretch sweep:
// the lower slab decided every bond crossing the face between them
void ledger_face_buffer(Engine& e) {
    if (e.d_face_recv) return;
    const size_t words = (size_t)e.M * plane_of(e) * e.lw;
    cuda_ok(cudaMalloc(&e.d_face_recv, sizeof(uint32_t) * words), "alloc face ledger");
    cuda_ok(cudaMemset(e.d_face_recv, 0, sizeof(uint32_t) * words), "zero face ledger");
}

const uint32_t* ledger_face_send(const Engine& e) {
    const int64_t R = e.plan.N[e.dim - 1];
    return e.d_ledger + (size_t)(R - e.M) * plane_of(e) * e.lw;
}

void ledger_exchange(Engine& e, cudaStream_t s) {
    if (!halo_active(e) || !e.d_ledger) return;
    ledger_face_buffer(e);
    const size_t words = (size_t)e.M * plane_of(e) * e.lw;
    const ncclComm_t c = (ncclComm_t)e.nccl_comm;
    nccl_check(api().GroupStart(), "ncclGroupStart");
    if (hi_face(e)) nccl_check(api().Send(ledger_face_send(e), words, ncclUint32, e.rank + 1, c, s), "ncclSend ledger");
    if (lo_face(e)) nccl_check(api().Recv(e.d_face_recv, words, ncclUint32, e.rank - 1, c, s), "ncclRecv ledger");
    nccl_check(api().GroupEnd(), "ncclGroupEnd");
    if (lo_face(e)) launch_merge_face(e, e.d_face_recv, s);
}

// distributed FFT: the all-to-all of equal blocks d_send[g] -> rank g's
// d_recv[rank] (grouped send/recv; the own block is a device copy)
void a2a_nccl_exchange(Engine& e, int batch, cudaStream_t s) {
    if (!comm_attached(e) || e.nranks != e.a2a.G || e.rank != e.a2a.rank)
        throw std::runtime_error("distributed FFT: the NCCL communicator does not match the rank layout");
    const int64_t blk = a2a_block(e, batch);
    const size_t n = (size_t)blk * 2;  // doubles
    double* send = reinterpret_cast<double*>(e.a2a.d_send);
    double* recv = reinterpret_cast<double*>(e.a2a.d_recv);
    const ncclComm_t c = (ncclComm_t)e.nccl_comm;
    cuda_ok(cudaMemcpyAsync(recv + (size_t)e.rank * n, send + (size_t)e.rank * n, sizeof(double) * n,
                            cudaMemcpyDeviceToDevice, s),
            "a2a own block");
    nccl_check(api().GroupStart(), "ncclGroupStart");
    for (int g = 0; g < e.a2a.G; ++g) {
        if (g == e.rank) continue;
        nccl_check(api().Send(send + (size_t)g * n, n, ncclFloat64, g, c, s), "ncclSend a2a");
        nccl_check(api().Recv(recv + (size_t)g * n, n, ncclFloat64, g, c, s), "ncclRecv a2a");
    }
    nccl_check(api().GroupEnd(), "ncclGroupEnd");
}

// the ring halo of the distributed FFT (G > 1): my first M rows to rank - 1,
// my last M to rank + 1 (mod G); d_alias holds them packed
// [side][batch][dim][M][Nx], the received rows land in a2a_alias_recv
// (side 0 from rank - 1, side 1 from rank + 1)
void a2a_nccl_alias(Engine& e, int batch, cudaStream_t s) {
    const int G = e.a2a.G;
    const size_t side = (size_t)batch * e.dim * e.M * e.plan.N[0];
    double* send = e.a2a.d_alias;
    double* recv = a2a_alias_recv(e, batch);
    const int lo = (e.rank + G - 1) % G, hi = (e.rank + 1) % G;
    const ncclComm_t c = (ncclComm_t)e.nccl_comm;
    nccl_check(api().GroupStart(), "ncclGroupStart");
    nccl_check(api().Send(send, side, ncclFloat64, lo, c, s), "ncclSend ring low");
    nccl_check(api().Recv(recv + side, side, ncclFloat64, hi, c, s), "ncclRecv ring high");
    nccl_check(api().Send(send + side, side, ncclFloat64, hi, c, s), "ncclSend ring high");
    nccl_check(api().Recv(recv, side, ncclFloat64, lo, c, s), "ncclRecv ring low");
    nccl_check(api().GroupEnd(), "ncclGroupEnd");
}

void comm_allreduce(Engine& e, double* d, int n, cudaStream_t s) {
    if (!comm_attached(e)) return;  // one rank: still a real (identity) all-reduce
    nccl_check(api().AllReduce(d, d, (size_t)n, ncclFloat64, ncclSum, (ncclComm_t)e.nccl_comm, s), "ncclAllReduce");
}

}  // namespace pdgpu
