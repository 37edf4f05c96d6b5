/*
 * pdgpu.h -- C ABI of the B200 MSBFM engine (libpdgpu.so).
 *
 * Drop-in boundary for the reference library `pdfast` (header-only C++20,
 * proj/include/pdfast/).  Every entry point names the reference interface it
 * replaces as <file>:<line>.  Plain pointers and sizes only; no CUDA or torch
 * types cross this boundary (streams are passed as void*, NULL = the engine's
 * own stream).  The C++ wrapper include/pdgpu.hpp maps these calls back onto
 * the reference's class shapes and exception types.
 *
 * Data layout (shared with the reference): node p = (k*Ny + j)*Nx + i
 * (grid.hpp:30-36), fields are component-major SoA  u[c*N + p]
 * (VecField, field.hpp:14-16).  Batched device entries take
 * [batch][dim][N] fp64.
 *
 * Errors: every int-returning call returns PDGPU_OK (0) or one of the codes
 * below; pdgpu_last_error() returns the thread-local message of the last
 * failure.  The three pdfast exceptions of the hot path keep distinct codes.
 */
#ifndef PDGPU_H
#define PDGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDGPU_OK 0
#define PDGPU_ERR_HORIZON_TOO_LARGE 1 /* pdfast::HorizonTooLargeForGrid, convolution.hpp:61-62 */
#define PDGPU_ERR_SHAPE_MISMATCH 2    /* pdfast::ShapeMismatch, convolution.hpp:120-121 */
#define PDGPU_ERR_LEDGER_OUT_OF_BAND 3 /* pdfast::LedgerOutOfBand, corrections.hpp:99-100 */
#define PDGPU_ERR_INVALID_ARGUMENT 4
#define PDGPU_ERR_CUDA 5
#define PDGPU_ERR_OUT_OF_MEMORY 6
#define PDGPU_ERR_NOT_SUPPORTED 7
#define PDGPU_ERR_IO 8                /* pdfast::IoError, errors.hpp:33-35 */

typedef struct pdgpu_engine* pdgpu_t;

const char* pdgpu_last_error(void);
const char* pdgpu_version(void);

/* ---------------------------------------------------------------- engine --
 * FastForce<Dim>(grid, hz, K)   convolution.hpp:239-246
 *   dims[dim]: lattice nodes per axis; M: band half-width (Horizon::M);
 *   stencils: n_pairs x (2M+1)^dim doubles in KernelStack storage order
 *   (KernelStack::component(pair), kernel.hpp:50-54,72).  Builds the
 *   spectral symbol on `device`.  Fails with PDGPU_ERR_HORIZON_TOO_LARGE
 *   when some dims[d] < M+1, like PadTransform's ctor. */
int pdgpu_create(int dim, const int* dims, int M, const double* stencils, int device, pdgpu_t* out);
void pdgpu_destroy(pdgpu_t h);

/* Grid::h / Grid::origin (grid.hpp:15-20), Horizon::delta (grid.hpp:114-116),
 * Material::rho (material.hpp:33-37): needed by positions (update_bonds,
 * crack seeding, constraints) and by the VV step.  For a slab engine
 * (pdgpu_set_slab) the origin is the global lattice's: positions are
 * computed from global node coordinates, as the reference does. */
int pdgpu_set_geometry(pdgpu_t h, double spacing, const double* origin, double delta, double rho);

/* FastForce::apply(u, f)   convolution.hpp:249-259 -- f = A_hat u, the
 * uncorrected spectral force; f is overwritten.  Device pointers,
 * [batch][dim][N], stream-ordered. */
int pdgpu_apply(pdgpu_t h, const double* u, double* f, int batch, void* stream);
/* Same with host vectors; n_nodes is the caller's field length and must
 * equal the lattice size (ShapeMismatch, convolution.hpp:120-121). */
int pdgpu_apply_host(pdgpu_t h, const double* u, double* f, int64_t n_nodes, int batch);

/* FastForce::last_imag_residue()  convolution.hpp:261.  The R2C pipeline
 * produces real fields by construction: always 0. */
/* FastForce::apply (no corrections) by direct stencil summation on the
 * device -- the reference's independent oracle tbt_apply_all
 * (tests/support/oracles.hpp:72-96) -- as a cross-check of pdgpu_apply and
 * its comparison point.  Same layout and contract as
 * pdgpu_apply. */
int pdgpu_apply_direct(pdgpu_t h, const double* u, double* f, int batch, void* stream);
double pdgpu_last_imag_residue(pdgpu_t h);
/* FastForce::footprint_bytes()  convolution.hpp:263-266 (device bytes held). */
size_t pdgpu_footprint_bytes(pdgpu_t h);
int64_t pdgpu_n_nodes(pdgpu_t h);
int pdgpu_symbol_is_real(pdgpu_t h);
/* 0 complex symbol table, 1 real symbol table, 2 separable per-column
 * symbol (physical stencils of definite parity per axis). */
int pdgpu_symbol_mode(pdgpu_t h);
/* Bytes of symbol table the 2D spectral pass streams per launch: the full
 * table, or -- 4096-point periodic columns of a stencil with definite parity
 * along y -- its mirror planes over ky in [0, Pl/2] (build_symbol_half). */
size_t pdgpu_symbol_stream_bytes(pdgpu_t h);
/* Transform embedding per axis, bit d set = periodic (P_d = N_d, aliased
 * boundary terms removed by the wrap correction), clear = zero-padded to
 * P_d = 2 pow2ceil(N_d) like PadTransform (convolution.hpp:58-71).  Both give
 * the reference's linear correlation; PDGPU_EMBED=padded at create time forces
 * padding on every axis. */
int pdgpu_embedding(pdgpu_t h);

/* ----------------------------------------------------------- corrections --
 * Regions (grid.hpp:172-209): per-node constraint direction mask (bit d =
 * direction d).  near_surface may be NULL (recomputed from the geometry). */
int pdgpu_set_regions(pdgpu_t h, const uint8_t* near_surface, const uint8_t* constraint_mask);
/* Slab (halo) decomposition: this engine's lattice is rows
 * [row_offset, row_offset + dims[dim-1]) of a lattice with global_rows rows
 * along the slowest axis (rows j in 2D, planes k in 3D; grid.hpp:30-36).
 * Rebuilds the near-surface flags and D^e (grid.hpp:181-189,
 * corrections.hpp:24-42) against the global faces: slab faces interior to
 * the global lattice are not surfaces.  The caller supplies M ghost rows on
 * each interior face and keeps only the owned rows of K.u. */
int pdgpu_set_slab(pdgpu_t h, int global_rows, int row_offset);
/* Halo slabs without ghost rows in the lattice: the engine's lattice is the
 * owned rows only (a power-of-two count keeps the slowest axis on the
 * periodic embedding), and the M rows beyond each interior face come from
 * `ghosts`, device [batch][dim][2][M][plane] fp64 (side 0 = the M rows
 * before the slab, side 1 = the M rows after it; plane = Nx (2D) or Nx*Ny
 * (3D)), read by every following apply / mat-vec until reset with NULL.  The
 * wrap correction adds their stencil terms to the rows within M of the face.
 * Requires pdgpu_set_slab; the caller refreshes the buffer's contents before
 * each mat-vec (stream-ordered). */
int pdgpu_set_ghosts(pdgpu_t h, const double* ghosts);
/* Same with an explicit layout: ghost row `layer` of side `side` for vector
 * b, component c at ghosts[(b*dim + c)*vec_comp_stride + side*side_stride +
 * layer*plane + i] (pdgpu_set_ghosts is vec_comp_stride = 2*M*plane,
 * side_stride = M*plane; pdgpu_halo_pack's send layout is vec_comp_stride =
 * M*plane, side_stride = batch*dim*M*plane). */
int pdgpu_set_ghosts_strided(pdgpu_t h, const double* ghosts, int64_t vec_comp_stride, int64_t side_stride);
/* The rows a slab sends to its neighbours before a K.u: send[side][batch][dim]
 * [M][plane] <- the first (side 0, to the rank before) and last (side 1, to the
 * rank after) M owned rows of u ([batch][dim][N] device).  Stream-ordered.
 * Used by the built-in NCCL exchange and by callers that move halos with
 * their own transport. */
int pdgpu_halo_pack(pdgpu_t h, const double* u, int batch, double* send, void* stream);

/* ---------------------------------------------------- multi-GPU (NCCL) --
 * Halo slabs across GPUs, one process per GPU (the reference is
 * single-process).  Rank r's engine is created on its own rows
 * [r0, r1) of the slowest axis (pdgpu_slab_rows) and told its place with
 * pdgpu_set_slab(h, global_rows, r0); pdgpu_comm_init then attaches an NCCL
 * communicator (rank - 1 / rank + 1 hold the neighbouring slabs).  From then on
 * every apply / matvec / evaluate_force exchanges the M rows next to each
 * interior face on a side stream, overlapped with the spectral passes, and
 * pdgpu_cg_solve / the ADR damping all-reduce their dot products (inside the
 * captured CG iteration).  libnccl.so.2 is loaded at first use. */
#define PDGPU_COMM_ID_BYTES 128
/* ncclGetUniqueId on one rank; the caller broadcasts the 128 bytes. */
int pdgpu_comm_unique_id(void* id_out);
int pdgpu_comm_init(pdgpu_t h, int nranks, int rank, const void* id);
/* Balanced contiguous split: rows [*row_begin, *row_end) of rank. */
int pdgpu_slab_rows(int global_rows, int nranks, int rank, int* row_begin, int* row_end);

/* Constraint state as the CG driver uses it (timestepping.hpp:306-309,
 * corrections.hpp:142-160): mask[N] = constrained direction bits per node,
 * uc[dim*N] = prescribed displacement values (0 where free or velocity-driven).
 * Either pointer may be NULL.  Used by multi-rank drivers that run CG over
 * slabs. */
int pdgpu_constraint_values(pdgpu_t h, uint8_t* mask, double* uc);
/* SurfaceDiag raw storage (corrections.hpp:20-62): de is n_pairs x N, rows
 * with near_surface set are used.  By default the engine builds it itself
 * from the stencils (build_de, corrections.hpp:65-68). */
int pdgpu_set_surface_diag(pdgpu_t h, const double* de);
/* BondLedger (ledger.hpp:13-57) as CSR: row_start[N+1], partners sorted per
 * row and symmetric.  Replaces the device ledger.  LedgerOutOfBand if a
 * partner is not an in-band lattice neighbour. */
int pdgpu_set_ledger(pdgpu_t h, const int64_t* row_start, const int64_t* partners);
/* BondLedger::break_bond for n pairs (p,q) (ledger.hpp:21-26). */
int pdgpu_break_bonds(pdgpu_t h, const int64_t* pairs, int64_t n);
/* Broken bonds as sorted (p,q) pairs, p < q; *count = total (may exceed cap).
 * Global node ids: a slab engine lists the pairs whose lower node it holds
 * (q may lie in the next slab), so the ranks' lists together are the ledger. */
int pdgpu_ledger_pairs(pdgpu_t h, int64_t* out_pairs, int64_t cap, int64_t* count);
/* apply_corrections(f, u, de, regions, ledger, K, grid)  corrections.hpp:76-110
 * f += De u (surface rows) + sum_q K(q-p)(u_p - u_q) (fracture rows), rows
 * constrained in the output direction untouched.  Device pointers. */
int pdgpu_apply_corrections(pdgpu_t h, const double* u, double* f, int batch, void* stream);
/* Same on host fields ([batch][dim][N]); f is updated in place. */
int pdgpu_apply_corrections_host(pdgpu_t h, const double* u, double* f, int64_t n_nodes, int batch);
/* K.u as the reference's tests and Simulation compute it:
 * FastForce::apply + apply_corrections (e.g. tests/test_corrections.cpp:107-110). */
int pdgpu_matvec(pdgpu_t h, const double* u, double* f, int batch, void* stream);
int pdgpu_matvec_host(pdgpu_t h, const double* u, double* f, int64_t n_nodes, int batch);
/* Simulation::evaluate_force (timestepping.hpp:295-310): f = A u + body,
 * then zero every constrained (node, dir).  Device pointers, one field. */
int pdgpu_evaluate_force(pdgpu_t h, const double* u, double* f, void* stream);
/* Same on host fields (dim x N); n_nodes as in pdgpu_apply_host. */
int pdgpu_evaluate_force_host(pdgpu_t h, const double* u, double* f, int64_t n_nodes);

/* --------------------------------------------------------------- problem --
 * Problem<Dim> setup (timestepping.hpp:40-52).  Boxes are closed, cell
 * centres tested (geometry.hpp:53-63); lo/hi have dim entries. */
/* Constraint (grid.hpp:160-166): kind 0 = displacement, 1 = velocity. */
int pdgpu_add_constraint(pdgpu_t h, const double* lo, const double* hi, int dir_mask, int kind, double value);
/* Load (timestepping.hpp:26-30): body force density on a box. */
int pdgpu_add_load(pdgpu_t h, const double* lo, const double* hi, const double* value);
/* Body force field directly (dim x N, host). */
int pdgpu_set_body(pdgpu_t h, const double* body);
/* seed_cracks (fracture.hpp:164-198): segment {ax, ay, bx, by, width}
 * (CrackSpec<2>::Segment) / notch {axis, plane, width, lo0, lo1, lo2, hi0,
 * hi1, hi2} (CrackSpec<3>::Notch).  *added = bonds newly broken. */
int pdgpu_seed_segment(pdgpu_t h, const double* seg, int64_t* added);
int pdgpu_seed_notch(pdgpu_t h, const double* notch, int64_t* added);

/* ------------------------------------------------------------- fracture --
 * update_bonds(grid, hz, u, ledger, s0, watch)  fracture.hpp:204-231.
 * u on the device ([dim][N]); watch = {lo[dim], hi[dim]} or NULL.
 * Newly broken bonds are returned as (p, q) pairs in the reference's
 * visiting order (p ascending, then offset order); *count = total. */
int pdgpu_update_bonds(pdgpu_t h, const double* u, double s0, const double* watch, int64_t* out_pairs, int64_t cap,
                       int64_t* count);
/* Same with u a host field (dim x N, n_nodes = lattice size, else ShapeMismatch). */
int pdgpu_update_bonds_host(pdgpu_t h, const double* u, int64_t n_nodes, double s0, const double* watch,
                            int64_t* out_pairs, int64_t cap, int64_t* count);
/* All (p, q) pairs of the last pdgpu_update_bonds[_host] sweep (visiting
 * order), e.g. when that call's cap was smaller than its count. */
int pdgpu_last_new_pairs(pdgpu_t h, int64_t* out_pairs, int64_t cap, int64_t* count);

/* ------------------------------------------------------------ CG solver --
 * New static solver (the reference has ADR only): Hestenes-Stiefel CG on
 * K := -A restricted to free DOFs, rhs = mask .* (b + A u_c) with u_c the
 * prescribed displacement values.  b, x device [dim][N]; on return x holds
 * the full displacement (free solution + prescribed values).  Stops at
 * ||r|| <= tol ||rhs||. */
int pdgpu_cg_solve(pdgpu_t h, const double* b, double* x, double tol, int maxit, int* iters, double* relres,
                   void* stream);
/* Host-vector variant; hist (optional, nhist x dim x N) receives the first
 * nhist iterates x_1..x_nhist (free part, before prescribed values). */
int pdgpu_cg_solve_host(pdgpu_t h, const double* b, double* x, double tol, int maxit, int* iters, double* relres,
                        double* hist, int nhist);

/* ------------------------------------------------------ velocity Verlet --
 * Simulation<Dim> with Integrator::Vv (timestepping.hpp:167-351).
 * sim_init zeroes u, v (optional initial velocity field), applies
 * constraints at t = 0 (timestepping.hpp:201). */
int pdgpu_sim_init(pdgpu_t h, double dt, const double* v0);
/* n_steps of Simulation::step (timestepping.hpp:209-241); s0 < 0 disables
 * fracture; watch as in update_bonds.  *broken = bonds broken in these steps. */
int pdgpu_sim_step(pdgpu_t h, int n_steps, double s0, const double* watch, int64_t* broken);
/* Halo slabs in one process: n engines holding consecutive row slabs of one
 * lattice (each with pdgpu_set_slab, no communicator; one or several
 * devices) advanced together by n_steps of Simulation::step.  Halo rows and
 * the ledger words of bonds broken across a face move by device-to-device
 * copies between the phases of each step (the NCCL path does the same
 * inside pdgpu_sim_step).  *broken = bonds broken over all slabs. */
int pdgpu_group_sim_step(pdgpu_t* engines, int n, int n_steps, double s0, const double* watch, int64_t* broken);

/* ----------------------------------------------- distributed FFT (2D) --
 * The all-to-all transpose arm of SURVEY §8e (north_star's distributed FFT;
 * the halo slabs above are the default multi-GPU path).  Engine `rank` of
 * `nranks` is created on its rows [row_bounds[rank], row_bounds[rank+1]) of
 * an Nx x global_rows lattice (global_rows a power of two, Nx periodic) and
 * also owns the half-spectrum columns [col_bounds[rank], col_bounds[rank+1])
 * (col_bounds[nranks] = Nx/2 + 1).  Every K.u then runs K1 on its rows, an
 * all-to-all transpose (NCCL grouped send/recv of equal padded blocks after
 * pdgpu_comm_init; a copy for one rank), the y pass over the global columns
 * with this rank's symbol, the reverse transpose and K5; the wrap correction
 * takes the x aliases locally and the y aliases at the global faces from the
 * opposite end's M rows.  D^e and the near-surface flags follow the global
 * lattice.  Cross-face broken bonds are not supported in this arm.
 * pdgpu_group_matvec_transpose: the same K.u for n engines of one process
 * (rank r = engines[r]) with device copies for the transposes. */
int pdgpu_set_transpose(pdgpu_t h, int nranks, int rank, int global_rows, const int* row_bounds,
                        const int* col_bounds);
int pdgpu_group_matvec_transpose(pdgpu_t* engines, int n, const double* const* u, double* const* f, int batch);
/* Simulation<Dim> with Integrator::Adr (AdrIntegrator, timestepping.hpp:79-145;
 * adr_mass :150-162): the reference's quasi-static solver.  Same state and
 * constraints as sim_init (v0 = 0); fixed_damping NaN = adaptive Rayleigh-
 * quotient damping (SolverOptions::fixed_damping = std::nullopt).
 * pdgpu_sim_step then advances ADR steps (the stretch test runs after each
 * step when s0 >= 0, as in Simulation::step). */
int pdgpu_sim_init_adr(pdgpu_t h, double dt, double fixed_damping);
/* Simulation::adr_damping() (timestepping.hpp:271): damping c of the last step. */
int pdgpu_sim_adr_damping(pdgpu_t h, double* c);
/* Copies of the state (host, dim x N each, any may be NULL). */
int pdgpu_sim_get(pdgpu_t h, double* u, double* v, double* f, double* t);
/* SimState::f_prev and ::v_half (timestepping.hpp:55-61), host, either may be NULL. */
int pdgpu_sim_get_aux(pdgpu_t h, double* f_prev, double* v_half);
/* InitialVelocity (timestepping.hpp:33-37, applied in the Simulation ctor
 * :194-197): overwrite v (dim x N host) and re-apply the constraints at the
 * current time (enforce_constraints, corrections.hpp:142-160). */
int pdgpu_sim_set_velocity(pdgpu_t h, const double* v);
/* Simulation::newly_broken() (timestepping.hpp:273): the (p, q) pairs broken
 * by the stretch test of the last step of the last pdgpu_sim_step call, in
 * the reference's visiting order; *count = 0 when that call had s0 < 0. */
int pdgpu_sim_newly_broken(pdgpu_t h, int64_t* out_pairs, int64_t cap, int64_t* count);
/* Simulation::finite() (timestepping.hpp:256-261): *ok = 1 iff every entry of
 * u is finite (device reduction, no copy of u). */
int pdgpu_sim_finite(pdgpu_t h, int* ok);

/* ---------------------------------------------------------- diagnostics --
 * Per-pass device timing with CUDA events on the launching stream (pass ids:
 * 0 K1 x-forward, 1 K2 y-forward (3D), 2 K3 spectral, 3 K4 y-inverse (3D),
 * 4 K5 x-inverse, 5 surface correction, 6 fracture correction, 7 vector
 * ops, 8 halo exchange on the comm stream -- overlapped with 0..4).  timing_read synchronises, returns the summed milliseconds and
 * launch counts per pass since the last read, and resets them. */
int pdgpu_timing_enable(pdgpu_t h, int on);
int pdgpu_timing_read(pdgpu_t h, double* ms_per_pass, int64_t* count_per_pass, int npass);
/* Number of kernels this engine has launched (all entry points). */
int64_t pdgpu_launch_count(pdgpu_t h);

/* ------------------------------------------------------------- assembly --
 * Host-side restatements of the reference's setup routines, so a caller
 * without the reference can assemble a problem. */
/* build_kernel (kernel.hpp:99-127): out n_pairs x (2M+1)^dim */
int pdgpu_build_kernel(int dim, double spacing, double delta, int M, double E, double thickness, double* out);
/* Regions near-surface flags (grid.hpp:181-189): out N bytes */
int pdgpu_near_surface(int dim, const int* dims, int M, uint8_t* out);

/* ------------------------------------------------------------ snapshots --
 * write_snapshot_dat / read_snapshot_dat (output.hpp:74-154): the
 * reference's plain-text, bit-exact trajectory format ("dir/snap_%07d.dat",
 * %.17g values, node ids from 1).  u is dim x N host SoA; damage may be NULL
 * (written as 0).  Host-only (no handle, no device).  The reader fills the
 * header fields; pass u = NULL first to learn dims, then buffers of dim*N
 * (and N for damage). */
int pdgpu_write_snapshot(int dim, const int* dims, double spacing, const double* origin, const double* u,
                         const double* damage, int64_t step, double t, const char* dir, char* path_out, int path_cap);
int pdgpu_read_snapshot(const char* path, int dim, int* dims, double* spacing, double* origin, int64_t* step,
                        double* t, double* u, double* damage);

/* CG's operator (new work, the reference has no CG): 0 = MSBFM (default),
 * 1 = the direct stencil sum of the same operator (the reference's own
 * independent oracle form, tests/support/oracles.hpp:72-96) plus the same
 * corrections -- at M = 3 it moves fewer bytes; MSBFM's advantage is
 * asymptotic in the horizon.  Slab engines always use MSBFM. */
int pdgpu_set_cg_operator(pdgpu_t h, int direct);

/* ------------------------------------------------------------- monitors --
 * MonitorWriter (output.hpp:45-72) and nearest_node (output.hpp:33-41): the
 * reference's tab-separated monitor file ("# step\tt\tnode\tu_x\tu_y[\tu_z]",
 * then one row per point and append: step, %.17g t, node id from 1, %.17g
 * components), flushed after every append.  pdgpu_monitor_open with path ""
 * or NULL only resolves nodes; an unwritable path fails with PDGPU_ERR_IO
 * (the reference throws IoError).  pdgpu_monitor_append takes one row of
 * values [point][component].
 * pdgpu_sim_monitor registers nodes with an engine: after every step of
 * pdgpu_sim_step u at those nodes is gathered on the device (one tiny kernel,
 * no field download); pdgpu_sim_monitor_read drains the recorded rows
 * (steps[count], t[count], values[count][n][dim]); pass NULL buffers to learn
 * count.  This is the CLI's per-step monitor.append (tools/pdfast_cli.cpp:76)
 * without a per-step host round trip. */
typedef struct pdgpu_monitor* pdgpu_monitor_t;
int pdgpu_monitor_open(const char* path, int dim, const int* dims, double spacing, const double* origin,
                       const double* points, int npts, pdgpu_monitor_t* out);
int pdgpu_monitor_nodes(int dim, const int* dims, double spacing, const double* origin, const double* points, int npts,
                        int64_t* nodes);
int pdgpu_monitor_append(pdgpu_monitor_t m, int64_t step, double t, const double* values);
void pdgpu_monitor_close(pdgpu_monitor_t m);
int pdgpu_sim_monitor(pdgpu_t h, const int64_t* nodes, int n);
int pdgpu_sim_monitor_read(pdgpu_t h, int64_t* steps, double* t, double* values, int64_t cap, int64_t* count);

#ifdef __cplusplus
}
#endif

#endif /* PDGPU_H */
