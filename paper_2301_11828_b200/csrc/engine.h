// engine.h -- internal state of one GPU MSBFM engine (the object behind the
// opaque pdgpu_t handle).  Host-only C++; kernels live in *.cu files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "assembly.h"

namespace pdgpu {

constexpr int kMaxDim = 3;

// Transform geometry.  Two embeddings per axis:
//  - padded:   P = 2*pow2ceil(N) >= N+M, so the circular correlation equals
//              the reference's linear one on the window (convolution.hpp:58-71
//              uses P = 2N, identical for power-of-two N);
//  - periodic: P = N (power of two, N >= max(2M+1, 16)).  The circular
//              correlation then differs from the linear one only on the M
//              node layers at each face of the axis, where stencil offsets
//              leaving the lattice wrap onto the opposite face; those aliased
//              terms are subtracted by the wrap correction (K6w,
//              corrections.cu) -- the same "circulant + sparse boundary
//              correction" split MSBFM already uses for D^e.  A quarter of
//              the padded FFT volume in 2D, an eighth in 3D.
// Default: periodic on every eligible axis; PDGPU_EMBED=padded forces padding.
struct Plan {
    int dim = 2;
    int N[3] = {1, 1, 1};
    int P[3] = {1, 1, 1};
    int logP[3] = {0, 0, 0};
    int circ[3] = {0, 0, 0};  // 1 = periodic embedding along this axis
    int circ_mask = 0;        // bit d = circ[d]
    int nh = 2;               // half-spectra of the last-axis pass: 2 padded, 1 periodic
    int64_t nodes = 0;  // N0*N1*N2
    int Hx = 0;         // R2C half spectrum along x: P0/2 + 1 columns
    int logQx = 0;      // x transforms are Qx = P0/4 points (R2C + zero half)
    // spectral (last-axis) pass: column count, physical length, padded length
    int ncols = 0, Nl = 0, Pl = 0, logPl = 0;
    int64_t S1_per_vec = 0;  // complex elements per vector in S1 (d*Nz*Hx*Ny)
    int64_t S2_per_vec = 0;  // complex elements per vector in S2 (3D: d*Hx*Py*Nz; 2D K3 output)
    int logTWN = 0;          // twiddle table length = max P
    // launch shapes
    int k1_rows = 1;         // rows per CTA in the x passes
    int k3_cols = 1;         // columns per CTA in the spectral pass
    int k3_halves = 2;       // 2 = both half-spectra resident, 1 = two passes
    int k2_zt = 1;           // z rows per CTA in the 3D y passes
};

struct Constraint {
    double lo[3], hi[3];
    uint8_t dir_mask;
    int kind;  // 0 displacement, 1 velocity (grid.hpp:160-166)
    double value;
};

// All-to-all distributed FFT (north_star's transpose scheme; the
// halo slabs are the default multi-GPU path).  Rank `rank` of G owns rows
// [r0[rank], r0[rank+1]) of an Nx x Nyg lattice for the x passes and the
// half-spectrum columns [k0[rank], k0[rank+1]) for the y pass; two all-to-all
// transposes move the spectrum between the layouts (blocks padded to
// Kmax x Rmax so every peer block has one size).  Global y faces: the wrap
// correction subtracts the aliased terms from the opposite end's M rows.
struct A2A {
    int G = 0, rank = 0, Nyg = 0;       // G > 0: on
    std::vector<int> r0, k0;            // G + 1 boundaries each
    int Rmax = 0, Kmax = 0;
    Plan col;                           // this rank's columns: ncols = k0[rank+1]-k0[rank], Nl = Pl = Nyg
    void* d_sym = nullptr;              // symbol of those columns
    double2 *d_c1 = nullptr, *d_c2 = nullptr, *d_send = nullptr, *d_recv = nullptr;
    int64_t cap = 0;                    // batch capacity of the buffers
    int* d_bounds = nullptr;            // r0 (G+1) then k0 (G+1) on the device
    double* d_alias = nullptr;          // [send|recv][side][batch][dim][M][Nx]: opposite-end rows
};

struct Engine {
    int device = 0;
    int num_sms = 148;
    int dim = 2, M = 0, np = 3, nof = 0, lw = 1;
    int64_t ss = 0;  // stencil size (2M+1)^dim
    Plan plan;
    bool real_symbol = true;
    std::vector<double> stencils;  // np * ss, KernelStack storage order (kernel.hpp:50-54)
    std::vector<int> offs;         // nof*3, for_each_offset order (kernel.hpp:71-89)

    // geometry for positions (grid.hpp:15-67) -- needed by fracture/constraints
    double h = 1.0, origin[3] = {0, 0, 0}, delta = 0.0, rho = 1.0;

    cudaStream_t stream = nullptr;  // engine-owned default stream
    cudaStream_t copy_in = nullptr, copy_out = nullptr;  // host-API copy pipeline
    double2* d_tw = nullptr;        // exp(-2 pi i k / TWN)
    void* d_sym = nullptr;          // symbol: real double or double2, np * ncols * Pl
    double* d_K = nullptr;          // stencils on device (np * ss), then koff[nof][np]
    // wrap correction (periodic embedding): nonzero stencil entries grouped in
    // (o2, o1) rows, o0 ascending -- d_wrows[2*row] = first entry, [2*row+1] =
    // end; d_wo0[entry] = o0; d_wK[entry*np + pair] = K
    int* d_wrows = nullptr;
    int* d_wo0 = nullptr;
    double* d_wK = nullptr;
    // per (axis, side, depth) lists of the entries that leave the lattice for a
    // node M or more away from the other faces: d_lidx[(axis*2+side)*M+depth]
    // = first entry (one extra end slot), d_loff[4*entry] = o0, o1, o2, d_lK as d_wK
    int* d_lidx = nullptr;
    int* d_loff = nullptr;
    double* d_lK = nullptr;
    // per-state entry lists (k_wrap_tab): a band node's state is its position
    // class on every axis (interior, depth l from the low face, depth l from
    // the high face: (2M+1)^dim states); d_sidx[state] = first record (one
    // extra end slot); a record {lin (int64), box entry (int32), flags (int32)}
    // says: subtract K(box) u[p + lin] (flag 1, lin already wrapped) and/or add
    // the ghost-row term (flag 2, side bit 2, layer bits 3-7, in-plane offset
    // bits 8-31).  Empty (d_stab null) when an axis is shorter than 2M + 1.
    int* d_sidx = nullptr;
    int4* d_stab = nullptr;
    // 3D face passes (k_wrap_face, every axis periodic, no ghost rows): per
    // (axis, side, depth) the entries whose offset along that axis leaves the
    // lattice, {o_B, o_C, o_A, box entry} with (B, C) the tile axes of the
    // pass; d_fidx[(axis*2+side)*M+depth] = first record (one end slot)
    int* d_fidx = nullptr;
    int4* d_ftab = nullptr;
    int face_rec_max = 0;
    // D^e is the lattice's own (no set_surface_diag / set_regions / slab);
    // fold_surface_next: the caller adds the corrections right after this
    // K.u, so the face passes may take D^e (surface_folded: they did)
    bool surf_default = false, fold_surface_next = false, surface_folded = false;
    A2A a2a;
    bool a2a_external = false;  // a single-process group driver runs the distributed-FFT phases
    bool pdl = false;           // launches of the current capture use programmatic dependent launch
    bool cg_direct = false;     // CG's operator: direct stencil sum instead of MSBFM (pdgpu_set_cg_operator)
    bool xstrip_ready = false;  // K1 of this K.u wrote d_xstrip (3D face passes read it)
    // 3D face passes: the x pass runs before K5 and leaves its per-node result
    // in d_fx ([b][c][slot 2M][z][y]); K5 adds it at the row ends it writes
    double* d_fx = nullptr;
    bool xpass_done = false;
    double* d_kc = nullptr;         // centre coefficients (3D direct stencil)
    double* d_coltab = nullptr;     // separable symbol: per column n_pairs x (M+1) coefficients (2D)
    int coltab_oddmask = 0;         // bit p: pair p odd along the column axis (sin terms)
    double* d_symh = nullptr;       // 2D real symbol mirrored along the column axis: per column the planes
                                    // xx, xy, yy over ky in [0, Pl/2] (symh_stride doubles each); K3 lands a
                                    // column's planes in shared memory by one bulk copy
    const void* symh_for = nullptr;  // the d_sym these planes were cut from
    bool s2_blocked = false;         // 2D: K3 wrote S2 row-blocked, [slab][row / 8][kx][row % 8] (K5 reads it so)
    int symh_stride = 0;
    double2* d_scratch = nullptr;   // per-CTA component park of the two-CTA/SM spectral kernel
    int64_t scratch_cap = 0;
    int* d_offs = nullptr;          // nof*3
    long long* d_disp = nullptr;    // nof: linear node displacement of each offset
    int64_t cap_batch = 0;
    double2* d_S1 = nullptr;
    double2* d_S2 = nullptr;
    double* d_xstrip = nullptr;     // 3D wrap correction: the 2M-wide x-face strips, [b][c][slot][z][y]
    double* d_u_stage = nullptr;    // host-API staging
    double* d_f_stage = nullptr;
    int64_t stage_cap = 0;

    // regions / corrections
    uint8_t* d_cmask = nullptr;        // N, constraint direction mask per node
    std::vector<uint8_t> h_cmask, h_near;
    assembly::SlabFrame slab;          // rows of a larger lattice (pdgpu_set_slab)
    const double* d_ghost = nullptr;   // caller's ghost rows of the interior slab faces (pdgpu_set_ghosts)
    // ghost rows the current K.u reads (K6w): the caller's buffer
    // [batch][dim][2][M][plane] or the NCCL receive buffer [2][batch][dim][M][plane]
    const double* ghost_view = nullptr;
    int64_t ghost_bc_stride = 0, ghost_side_stride = 0;
    int64_t user_ghost_bc = 0, user_ghost_side = 0;  // pdgpu_set_ghosts_strided (0 = default layout)
    // multi-GPU halo slabs over NCCL (comm.cpp)
    void* nccl_comm = nullptr;
    int nranks = 1, rank = 0;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    double* d_halo = nullptr;          // [send|recv][side][batch][dim][M][plane]
    int64_t halo_cap = 0;
    bool halo_external = false;        // ghost rows placed by a single-process group driver (abi.cu)
    uint32_t* d_face_recv = nullptr;   // ledger words of the lower neighbour's last M rows
    int64_t n_surf = 0;
    long long* d_surf_rows = nullptr;  // surface node ids
    double* d_surf_de = nullptr;       // n_surf * np
    uint32_t* d_ledger = nullptr;      // N * lw bit set over offsets
    long long* d_bond_rows = nullptr;  // rows with >=1 broken bond (unordered)
    int* d_listed = nullptr;           // N flags: row already in d_bond_rows
    unsigned long long* d_counters = nullptr;  // [0] = #bond rows, [1] = #new pairs, [2] = breaks since read
    int64_t n_bond_rows = 0;           // host mirror
    bool bond_rows_on_device = false;  // [0] may be ahead of n_bond_rows (unsynchronised sim_step)
    int64_t total_broken = 0;
    long long* d_new_pairs = nullptr;  // update_bonds output buffer (p, k) pairs
    int64_t new_pairs_cap = 0;
    std::vector<int64_t> last_pairs;   // (p, q) pairs of the last pdgpu_update_bonds sweep, visiting order
    bool sim_swept = false;            // the last sim_step ran the stretch test (pdgpu_sim_newly_broken)

    // constraints / loads / simulation state
    std::vector<Constraint> constraints;
    std::vector<double> h_body;          // dim * N (lazily)
    double* d_body = nullptr;
    long long* d_cdofs = nullptr;        // constrained dof ids (a*N + p), last-writer-wins order
    double* d_cval = nullptr;            // value per constrained dof
    int* d_ckind = nullptr;              // kind per constrained dof
    long long* d_uc_ids = nullptr;       // CG: dofs with a nonzero prescribed displacement
    double* d_uc_val = nullptr;
    int64_t n_uc = 0;
    int64_t n_cdofs = 0;
    double *d_u = nullptr, *d_v = nullptr, *d_f = nullptr, *d_fprev = nullptr;
    double t = 0.0, dt = 0.0;
    int integrator = 0;                  // 0 velocity Verlet, 1 ADR (SolverOptions, timestepping.hpp:53)
    double* d_vh = nullptr;              // ADR staggered velocity v_half
    double adr_mass[3] = {1.0, 1.0, 1.0};  // adr_mass (timestepping.hpp:150-162)
    bool adr_fixed = false;
    double adr_fixed_c = 0.0;
    int64_t step = 0;
    bool force_ready = false;
    bool drift_done = false;  // VV: the next step's drift ran fused with this step's kick (k_vv_kick_drift)
    // MonitorWriter nodes (output.hpp:45-72): u at these nodes is gathered on
    // the device after every step into rows [row][node][dim]; the host keeps
    // (step, t) per row and drains them with pdgpu_sim_monitor_read
    long long* d_mon_nodes = nullptr;
    int n_mon = 0;
    double* d_mon_rows = nullptr;
    int mon_cap = 0, mon_dev_rows = 0;
    std::vector<int64_t> mon_step;
    std::vector<double> mon_t, mon_spill;  // spill: rows moved off the device when its buffer filled
    bool any_cmask = false;              // constraint mask set directly (set_regions)
    double* d_cg = nullptr;              // CG work vectors r, p, q, u_c
    int64_t cg_cap = 0;
    cudaGraphExec_t cg_graph = nullptr;  // one captured CG iteration (keyed by x, stream, state version)
    const double* cg_graph_x = nullptr;
    cudaStream_t cg_graph_stream = nullptr;
    // Bumped by every change a captured launch sequence bakes in by value or
    // by pointer: surface rows / D^e (re)uploads, bond-row count (breaks,
    // ledger replacement), ghost buffer, slab frame, workspace growth.  A
    // captured graph is valid only for the version it was recorded at.
    uint64_t state_version = 0;
    uint64_t cg_graph_version = ~0ull;
    int64_t cg_graph_launches = 0;       // kernels in one captured CG iteration
    // reductions scratch
    double* d_red = nullptr;           // partial sums
    double* d_scal = nullptr;          // device scalars
    unsigned int* d_ticket = nullptr;

    // per-pass device timing (CUDA events on the launching stream) and the
    // number of kernels launched -- read by bench.py for the roofline
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<int> mark_pass;
    std::vector<cudaEvent_t> mark_a, mark_b;
    int64_t launches = 0;
    cudaEvent_t next_event() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t ev;
            cudaEventCreate(&ev);
            ev_pool.push_back(ev);
        }
        return ev_pool[ev_used++];
    }
};

// Programmatic dependent launch (CUDA graphs of small CG iterations): the
// kernel is launched with programmatic stream serialization, so its CTAs are
// scheduled while the previous kernel drains; pdl_entry() at the top of the
// kernels that take part waits for the previous grid's results
// (griddepcontrol.wait) and lets the next kernel be scheduled
// (griddepcontrol.launch_dependents).  Both are no-ops in plain launches.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_maybe_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t s, Args&&... args) {
    if (!pdl) {
        kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
#endif

// halo slabs: this engine's lattice has an interior face below / above
inline bool slab_lo_face(const Engine& e) { return e.slab.global >= 0 && e.slab.off > 0; }
inline bool slab_hi_face(const Engine& e) {
    return e.slab.global >= 0 && e.slab.off + e.plan.N[e.dim - 1] < e.slab.global;
}
inline bool slab_has_faces(const Engine& e) { return slab_lo_face(e) || slab_hi_face(e); }

// Invalidate every captured launch sequence (see Engine::state_version).
inline void touch_state(Engine& e) {
    ++e.state_version;
    if (e.cg_graph) {
        cudaGraphExecDestroy(e.cg_graph);
        e.cg_graph = nullptr;
    }
    e.cg_graph_x = nullptr;
}

enum PassId { kPassK1 = 0, kPassK2 = 1, kPassK3 = 2, kPassK4 = 3, kPassK5 = 4, kPassCorr = 5, kPassBonds = 6,
              kPassVec = 7, kPassHalo = 8, kNumPass = 9 };

// RAII bracket of one pass with events when e.timing is on
struct PassTimer {
    Engine& e;
    int id;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    PassTimer(Engine& e_, int id_, cudaStream_t s_, int nlaunch = 1) : e(e_), id(id_), s(s_) {
        e.launches += nlaunch;
        if (e.timing) {
            a = e.next_event();
            cudaEventRecord(a, s);
        }
    }
    // close the bracket early (before work that must not be timed in it)
    void finish() {
        if (e.timing && !done) {
            cudaEvent_t b = e.next_event();
            cudaEventRecord(b, s);
            e.mark_pass.push_back(id);
            e.mark_a.push_back(a);
            e.mark_b.push_back(b);
        }
        done = true;
    }
    ~PassTimer() { finish(); }
    bool done = false;
};

// spectral.cu
void plan_init(Plan& pl, int dim, const int* dims, int M);
void engine_alloc_workspace(Engine& e, int64_t batch);
void build_twiddles(Engine& e);
void build_symbol(Engine& e);
void build_symbol_half(Engine& e);
void launch_fast_apply(Engine& e, const double* u, double* f, int batch, cudaStream_t s,
                       double scale, const uint8_t* cmask, const double* body);
void set_kernel_attributes();

// direct.cu
void direct_prepare(Engine& e);
void launch_direct_apply(Engine& e, const double* u, double* f, int batch, cudaStream_t s, double scale,
                         const uint8_t* cmask = nullptr);

// transpose.cu (all-to-all distributed FFT)
void a2a_setup(Engine& e, int G, int rank, int Nyg, const int* r0, const int* k0);
void a2a_free(Engine& e);
void a2a_ensure(Engine& e, int batch);
int64_t a2a_block(const Engine& e, int batch);  // complex elements per peer block
void a2a_phase1(Engine& e, const double* u, int batch, cudaStream_t s);  // K1 + pack -> d_send
void a2a_phase2(Engine& e, int batch, cudaStream_t s);                   // unpack + K3 + pack -> d_send
void a2a_phase3(Engine& e, double* f, int batch, cudaStream_t s, double scale, const uint8_t* cmask,
                const double* body);                                       // unpack + K5
void a2a_exchange(Engine& e, int batch, cudaStream_t s);                 // d_send -> d_recv (NCCL, or G = 1)
void a2a_alias(Engine& e, const double* u, int batch, cudaStream_t s);   // opposite-end rows -> ghost_view
double* a2a_alias_recv(Engine& e, int batch);                            // where the opposite-end rows land
void a2a_nccl_exchange(Engine& e, int batch, cudaStream_t s);
void a2a_nccl_alias(Engine& e, int batch, cudaStream_t s);

// corrections.cu
void build_wrap_table(Engine& e);
void launch_wrap_correction(Engine& e, const double* u, double* f, int batch, cudaStream_t s, double scale,
                            const uint8_t* cmask);
bool launch_wrap_xpass(Engine& e, const double* u, int batch, cudaStream_t s, double scale, const uint8_t* cmask);
void launch_corrections(Engine& e, const double* u, double* f, int batch, cudaStream_t s,
                        double scale);
void launch_merge_face(Engine& e, const uint32_t* recv, cudaStream_t s);
int64_t launch_update_bonds(Engine& e, const double* u, double s0, const double* watch,
                            cudaStream_t s, bool sync = true);

// comm.cpp
void comm_unique_id(void* out);
void comm_init(Engine& e, int nranks, int rank, const void* id);
void comm_destroy(Engine& e);
bool comm_attached(const Engine& e);
bool halo_active(const Engine& e);
void ensure_halo(Engine& e, int batch);
void halo_pack(const Engine& e, const double* u, int batch, double* send, cudaStream_t s);
const double* halo_exchange_begin(Engine& e, const double* u, int batch, cudaStream_t s);
void halo_exchange_end(Engine& e, cudaStream_t s);
void halo_exchange_now(Engine& e, const double* u, cudaStream_t s);
void ledger_face_buffer(Engine& e);
const uint32_t* ledger_face_send(const Engine& e);
void ledger_exchange(Engine& e, cudaStream_t s);
void comm_allreduce(Engine& e, double* d, int n, cudaStream_t s);

// solvers.cu
void launch_dot(Engine& e, const double* a, const double* b, int64_t n, double* out_dev,
                cudaStream_t s);
void launch_cg_update(Engine& e, double* x, double* r, const double* p, const double* q, int64_t n,
                      const double* scal, double* rr_out, cudaStream_t s);
void launch_cg_step_dev_comm(Engine& e, double* x, double* r, double* p, const double* q, int64_t n, double* scal,
                             cudaStream_t s);
void launch_cg_direction(double* p, const double* r, int64_t n, const double* scal, cudaStream_t s);
void launch_cg_step_dev(Engine& e, double* x, double* r, double* p, const double* q, int64_t n, double* scal,
                        cudaStream_t s);
bool launch_cg_fused(Engine& e, double* x, double* r, double* p, const double* q, int64_t n, double* scal,
                     cudaStream_t s);
void launch_mask_rhs(double* out, const double* b, const double* Auc, const uint8_t* cmask,
                     int64_t N, int dim, cudaStream_t s);
void launch_vv_drift(double* u, const double* v, const double* f, const uint8_t* cmask, int64_t N,
                     int dim, double dt, double inv_rho, cudaStream_t s);
void launch_vv_kick_drift(double* u, double* v, const double* fprev, const double* f, const uint8_t* cmask, int64_t N,
                          int dim, double dt, double inv_rho, cudaStream_t s);
void launch_vv_kick(double* v, const double* fprev, const double* f, const uint8_t* cmask,
                    int64_t N, int dim, double dt, double inv_rho, cudaStream_t s);
void launch_adr_step(Engine& e, bool first, cudaStream_t s);
void launch_enforce(double* u, double* v, const long long* dofs, const double* val, const int* kind,
                    int64_t n, double t, cudaStream_t s);
void launch_axpy(double* y, const double* x, double a, int64_t n, cudaStream_t s);
void launch_finite(const double* u, int64_t n, int* ok, cudaStream_t s);
void launch_scatter(double* y, const long long* ids, const double* val, int64_t n, cudaStream_t s);
void launch_monitor_gather(const double* u, const long long* nodes, int n, int dim, int64_t N, double* dst,
                           cudaStream_t s);

}  // namespace pdgpu
