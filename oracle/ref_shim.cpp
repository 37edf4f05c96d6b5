// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers
// (/root/reference/proj/include/pdfast, compiled in place, never copied)
// linked against oracle/fftw_cpu.  Output: oracle/_ref/libpdref.so.
//
// TEST INFRASTRUCTURE ONLY: used by oracle/gen_golden.py (golden vectors),
// by tests/ to pin the C restatement oracle/oracle.c, and by bench.py's
// reference arm / cpu_baseline leg (the reference's own FastForce::apply +
// apply_corrections timed on the host cores).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <random>
#include <thread>
#include <vector>

#include "pdfast/convolution.hpp"
#include "pdfast/corrections.hpp"
#include "pdfast/fracture.hpp"
#include "pdfast/reference.hpp"
#include "pdfast/timestepping.hpp"
#include "support/oracles.hpp"

using namespace pdfast;

namespace {

struct RefProblem {
    int dim;
    IVec<3> dims{};
    double h, delta, E, thickness, rho, nu;
    int M;
    Vec<3> origin{};
    std::vector<double> stencils;  // optional override (np x ss)
    std::vector<std::array<double, 6>> con_lo_hi;
    std::vector<int> con_mask, con_kind;
    std::vector<double> con_val;
    std::vector<std::array<double, 9>> cracks;  // 2D: 5 used, 3D notch: 9
    std::vector<std::pair<index_t, index_t>> extra_bonds;
    std::vector<std::array<double, 9>> loads;  // lo(3) hi(3) value(3)
    // built objects (one of the two dims is live)
    std::unique_ptr<void, void (*)(void*)> impl{nullptr, [](void*) {}};
};

template <int Dim>
struct Built {
    Grid<Dim> grid;
    Horizon hz;
    Material mat;
    KernelStack<Dim> K;
    Regions<Dim> regions;
    SurfaceDiag<Dim> de;
    BondLedger ledger;
    std::unique_ptr<FastForce<Dim>> engine;
    std::vector<Constraint<Dim>> constraints;
    std::vector<Load<Dim>> loads;
    CrackSpec<Dim> cracks;
    std::unique_ptr<Simulation<Dim>> sim;
};

template <int Dim>
Built<Dim>* build(RefProblem& P) {
    auto* B = new Built<Dim>();
    B->grid.h = P.h;
    for (int d = 0; d < Dim; ++d) {
        B->grid.dims[d] = P.dims[d];
        B->grid.origin[d] = P.origin[d];
    }
    B->grid.thickness = P.thickness;
    B->hz = Horizon{P.delta, P.M};
    B->mat = Material{P.E, P.nu, P.rho, std::nullopt, std::nullopt, PlaneMode::Stress};
    if (P.stencils.empty()) {
        B->K = build_kernel(B->grid, B->hz, B->mat);
    } else {
        B->K = KernelStack<Dim>(P.M, P.h);
        const size_t ss = B->K.stencil_size();
        const int side = 2 * P.M + 1;
        for (size_t i = 0; i < ss; ++i) {
            IVec<Dim> off{};
            size_t rem = i;
            for (int d = 0; d < Dim; ++d) {  // axis 0 fastest (kernel.hpp:50-54)
                off[d] = (int)(rem % side) - P.M;
                rem /= side;
            }
            for (int a = 0; a < Dim; ++a)
                for (int b = a; b < Dim; ++b) B->K.at(a, b, off) = P.stencils[pair_index<Dim>(a, b) * ss + i];
        }
    }
    for (size_t c = 0; c < P.con_mask.size(); ++c) {
        Constraint<Dim> cs;
        for (int d = 0; d < Dim; ++d) {
            cs.box.lo[d] = P.con_lo_hi[c][d];
            cs.box.hi[d] = P.con_lo_hi[c][3 + d];
        }
        cs.dir_mask = (std::uint8_t)P.con_mask[c];
        cs.kind = P.con_kind[c] ? ConstraintKind::Velocity : ConstraintKind::Displacement;
        cs.value = P.con_val[c];
        B->constraints.push_back(cs);
    }
    for (const auto& l : P.loads) {
        Load<Dim> ld;
        for (int d = 0; d < Dim; ++d) {
            ld.box.lo[d] = l[d];
            ld.box.hi[d] = l[3 + d];
            ld.value[d] = l[6 + d];
        }
        B->loads.push_back(ld);
    }
    B->regions = classify_regions<Dim>(B->grid, B->hz, B->constraints);
    B->de = build_de(B->grid, B->hz, B->regions, B->K);
    if constexpr (Dim == 2) {
        for (const auto& c : P.cracks) B->cracks.segments.push_back({{c[0], c[1]}, {c[2], c[3]}, c[4]});
    } else {
        for (const auto& c : P.cracks) {
            typename CrackSpec<3>::Notch n;
            n.axis = (int)c[0];
            n.plane = c[1];
            n.width = c[2];
            n.lo = {c[3], c[4], c[5]};
            n.hi = {c[6], c[7], c[8]};
            B->cracks.notches.push_back(n);
        }
    }
    B->ledger = seed_cracks(B->cracks, B->grid, B->hz);
    for (auto& pq : P.extra_bonds) B->ledger.break_bond(pq.first, pq.second);
    B->engine = std::make_unique<FastForce<Dim>>(B->grid, B->hz, B->K);
    return B;
}

template <int Dim>
Built<Dim>* get(RefProblem* P) {
    return static_cast<Built<Dim>*>(P->impl.get());
}

template <int Dim>
void to_field(const double* u, VecField<Dim>& f, index_t n) {
    f.resize(n);
    for (int d = 0; d < Dim; ++d) std::memcpy(f.c[d].data(), u + d * n, sizeof(double) * n);
}

template <int Dim>
void from_field(const VecField<Dim>& f, double* out, index_t n) {
    for (int d = 0; d < Dim; ++d) std::memcpy(out + d * n, f.c[d].data(), sizeof(double) * n);
}

template <int Dim>
void matvec_t(Built<Dim>* B, const double* u, double* f, bool corrected) {
    const index_t n = B->grid.n_nodes();
    VecField<Dim> U, F(n);
    to_field<Dim>(u, U, n);
    B->engine->apply(U, F);
    if (corrected) apply_corrections(F, U, B->de, B->regions, B->ledger, B->K, B->grid);
    from_field<Dim>(F, f, n);
}

template <int Dim>
int64_t pairs_t(const BondLedger& L, int64_t* out, int64_t cap) {
    int64_t c = 0;
    for (index_t p = 0; p < L.n_nodes(); ++p)
        for (index_t q : L.broken_partners(p)) {
            if (q <= p) continue;
            if (out && c < cap) {
                out[2 * c] = p;
                out[2 * c + 1] = q;
            }
            ++c;
        }
    return c;
}

#define DISPATCH(P, CALL) ((P)->dim == 2 ? CALL<2> : CALL<3>)

}  // namespace

extern "C" {

// ---------------------------------------------------------------- RNG ---
void* ref_rng_new(uint32_t seed) { return new std::mt19937(seed); }
void ref_rng_free(void* r) { delete static_cast<std::mt19937*>(r); }
uint32_t ref_rng_next(void* r) { return (uint32_t)(*static_cast<std::mt19937*>(r))(); }
// tests/support/oracles.hpp:113-119 semantics (one distribution, component-major)
void ref_rng_uniform(void* r, int64_t n, double a, double b, double* out) {
    std::uniform_real_distribution<double> dist(a, b);
    for (int64_t i = 0; i < n; ++i) out[i] = dist(*static_cast<std::mt19937*>(r));
}

// ------------------------------------------------------------ problem ---
void* ref_new(int dim, const int* dims, double h, const double* origin, double thickness, double delta, int M,
              double E, double rho) {
    auto* P = new RefProblem();
    P->dim = dim;
    for (int d = 0; d < dim; ++d) {
        P->dims[d] = dims[d];
        P->origin[d] = origin ? origin[d] : 0.0;
    }
    P->h = h;
    P->thickness = thickness;
    P->delta = delta;
    P->M = M;
    P->E = E;
    P->rho = rho;
    P->nu = dim == 2 ? 1.0 / 3.0 : 0.25;
    return P;
}

void ref_free(void* vp) {
    auto* P = static_cast<RefProblem*>(vp);
    if (P->impl) {
        if (P->dim == 2) delete get<2>(P);
        else delete get<3>(P);
        P->impl.release();
    }
    delete P;
}

void ref_set_stencils(void* vp, const double* K, int64_t count) {
    static_cast<RefProblem*>(vp)->stencils.assign(K, K + count);
}
void ref_add_constraint(void* vp, const double* lo, const double* hi, int mask, int kind, double value) {
    auto* P = static_cast<RefProblem*>(vp);
    std::array<double, 6> b{};
    for (int d = 0; d < P->dim; ++d) {
        b[d] = lo[d];
        b[3 + d] = hi[d];
    }
    P->con_lo_hi.push_back(b);
    P->con_mask.push_back(mask);
    P->con_kind.push_back(kind);
    P->con_val.push_back(value);
}
void ref_add_load(void* vp, const double* lo, const double* hi, const double* value) {
    auto* P = static_cast<RefProblem*>(vp);
    std::array<double, 9> l{};
    for (int d = 0; d < P->dim; ++d) {
        l[d] = lo[d];
        l[3 + d] = hi[d];
        l[6 + d] = value[d];
    }
    P->loads.push_back(l);
}
void ref_add_crack(void* vp, const double* geom, int n) {
    std::array<double, 9> c{};
    for (int i = 0; i < n && i < 9; ++i) c[i] = geom[i];
    static_cast<RefProblem*>(vp)->cracks.push_back(c);
}
void ref_add_bond(void* vp, int64_t p, int64_t q) { static_cast<RefProblem*>(vp)->extra_bonds.push_back({p, q}); }

// build: kernels, regions, De, seeded ledger (+ extra bonds), FastForce
int ref_finalize(void* vp) {
    auto* P = static_cast<RefProblem*>(vp);
    try {
        if (P->dim == 2) P->impl = std::unique_ptr<void, void (*)(void*)>(build<2>(*P), [](void*) {});
        else P->impl = std::unique_ptr<void, void (*)(void*)>(build<3>(*P), [](void*) {});
    } catch (const HorizonTooLargeForGrid&) {
        return 1;
    } catch (const std::exception&) {
        return 4;
    }
    return 0;
}

void ref_get_kernel(void* vp, double* out) {
    auto* P = static_cast<RefProblem*>(vp);
    auto copy = [&](auto* B) {
        const size_t ss = B->K.stencil_size();
        const int np = P->dim * (P->dim + 1) / 2;
        for (int p = 0; p < np; ++p) std::memcpy(out + p * ss, B->K.component(p).data(), sizeof(double) * ss);
    };
    if (P->dim == 2) copy(get<2>(P));
    else copy(get<3>(P));
}

void ref_get_regions(void* vp, uint8_t* near, uint8_t* cmask, double* de) {
    auto* P = static_cast<RefProblem*>(vp);
    auto copy = [&](auto* B, auto dimc) {
        constexpr int Dim = decltype(dimc)::value;
        const index_t n = B->grid.n_nodes();
        for (index_t p = 0; p < n; ++p) {
            if (near) near[p] = B->regions.near_surface(p) ? 1 : 0;
            if (cmask) cmask[p] = B->regions.constraint_mask(p);
            if (de)
                for (int a = 0; a < Dim; ++a)
                    for (int b = a; b < Dim; ++b) de[pair_index<Dim>(a, b) * n + p] = B->de.raw(a, b, p);
        }
    };
    if (P->dim == 2) copy(get<2>(P), std::integral_constant<int, 2>{});
    else copy(get<3>(P), std::integral_constant<int, 3>{});
}

// FastForce::apply (corrected = 0) or + apply_corrections (corrected = 1).
// Returns 0, or 3 on LedgerOutOfBand.
int ref_matvec(void* vp, const double* u, double* f, int corrected) {
    auto* P = static_cast<RefProblem*>(vp);
    try {
        if (P->dim == 2) matvec_t<2>(get<2>(P), u, f, corrected != 0);
        else matvec_t<3>(get<3>(P), u, f, corrected != 0);
    } catch (const LedgerOutOfBand&) {
        return 3;
    }
    return 0;
}

double ref_imag_residue(void* vp) {
    auto* P = static_cast<RefProblem*>(vp);
    return P->dim == 2 ? get<2>(P)->engine->last_imag_residue() : get<3>(P)->engine->last_imag_residue();
}

// dense_force (reference.hpp:100-127)
void ref_dense(void* vp, const double* u, double* f) {
    auto* P = static_cast<RefProblem*>(vp);
    auto run = [&](auto* B, auto dimc) {
        constexpr int Dim = decltype(dimc)::value;
        const index_t n = B->grid.n_nodes();
        VecField<Dim> U, F(n);
        to_field<Dim>(u, U, n);
        auto table = build_neighbor_table(B->grid, B->hz);
        dense_force(F, U, B->grid, B->hz, B->mat, table, B->ledger);
        from_field<Dim>(F, f, n);
    };
    if (P->dim == 2) run(get<2>(P), std::integral_constant<int, 2>{});
    else run(get<3>(P), std::integral_constant<int, 3>{});
}

int64_t ref_ledger_pairs(void* vp, int64_t* out, int64_t cap) {
    auto* P = static_cast<RefProblem*>(vp);
    if (P->dim == 2) return pairs_t<2>(get<2>(P)->sim ? get<2>(P)->sim->ledger() : get<2>(P)->ledger, out, cap);
    return pairs_t<3>(get<3>(P)->sim ? get<3>(P)->sim->ledger() : get<3>(P)->ledger, out, cap);
}

// update_bonds (fracture.hpp:204-231) on the problem's ledger
int64_t ref_update_bonds(void* vp, const double* u, double s0, const double* watch, int64_t* out, int64_t cap) {
    auto* P = static_cast<RefProblem*>(vp);
    auto run = [&](auto* B, auto dimc) -> int64_t {
        constexpr int Dim = decltype(dimc)::value;
        const index_t n = B->grid.n_nodes();
        VecField<Dim> U;
        to_field<Dim>(u, U, n);
        std::optional<Box<Dim>> w;
        if (watch) {
            Box<Dim> b;
            for (int d = 0; d < Dim; ++d) {
                b.lo[d] = watch[d];
                b.hi[d] = watch[Dim + d];
            }
            w = b;
        }
        auto br = update_bonds<Dim>(B->grid, B->hz, U, B->ledger, s0, w);
        for (int64_t i = 0; i < (int64_t)br.size() && i < cap; ++i) {
            out[2 * i] = br[i].first;
            out[2 * i + 1] = br[i].second;
        }
        return (int64_t)br.size();
    };
    if (P->dim == 2) return run(get<2>(P), std::integral_constant<int, 2>{});
    return run(get<3>(P), std::integral_constant<int, 3>{});
}

// bond_stretch (fracture.hpp:17-29)
double ref_bond_stretch(int dim, const double* xp, const double* xq, const double* up, const double* uq) {
    if (dim == 2)
        return bond_stretch<2>({xp[0], xp[1]}, {xq[0], xq[1]}, {up[0], up[1]}, {uq[0], uq[1]});
    return bond_stretch<3>({xp[0], xp[1], xp[2]}, {xq[0], xq[1], xq[2]}, {up[0], up[1], up[2]}, {uq[0], uq[1], uq[2]});
}

// --------------------------------------------------------- CG (new) ------
// Hestenes-Stiefel CG over the reference mat-vec: K := -A on free dofs,
// rhs = mask (b + A u_c); identical definition to oracle.c orc_cg.
int ref_cg(void* vp, const double* b, double* x, double tol, int maxit, int* iters, double* relres, double* hist,
           int nhist) {
    auto* P = static_cast<RefProblem*>(vp);
    auto run = [&](auto* B, auto dimc) {
        constexpr int Dim = decltype(dimc)::value;
        const index_t n = B->grid.n_nodes();
        const index_t m = Dim * n;
        auto masked = [&](std::vector<double>& v) {
            for (int d = 0; d < Dim; ++d)
                for (index_t p = 0; p < n; ++p)
                    if (B->regions.constrained(p, d)) v[d * n + p] = 0.0;
        };
        std::vector<double> uc(m, 0.0), Auc(m), r(m), p(m), q(m);
        for (const auto& cs : B->constraints) {
            if (cs.kind != ConstraintKind::Displacement) continue;
            for (index_t i = 0; i < n; ++i)
                if (cs.box.contains(B->grid.pos(i)))
                    for (int d = 0; d < Dim; ++d)
                        if ((cs.dir_mask >> d) & 1u) uc[d * n + i] = cs.value;
        }
        matvec_t<Dim>(B, uc.data(), Auc.data(), true);
        for (index_t i = 0; i < m; ++i) r[i] = b[i] + Auc[i];
        masked(r);
        std::fill(x, x + m, 0.0);
        p = r;
        double rr = 0;
        for (index_t i = 0; i < m; ++i) rr += r[i] * r[i];
        const double bnorm = std::sqrt(rr);
        int k = 0;
        double rel = bnorm > 0 ? 1.0 : 0.0;
        while (bnorm > 0 && k < maxit) {
            matvec_t<Dim>(B, p.data(), q.data(), true);
            for (index_t i = 0; i < m; ++i) q[i] = -q[i];
            masked(q);
            double pq = 0;
            for (index_t i = 0; i < m; ++i) pq += p[i] * q[i];
            const double alpha = rr / pq;
            double rr1 = 0;
            for (index_t i = 0; i < m; ++i) {
                x[i] += alpha * p[i];
                r[i] -= alpha * q[i];
                rr1 += r[i] * r[i];
            }
            ++k;
            if (hist && k <= nhist) std::memcpy(hist + (size_t)(k - 1) * m, x, sizeof(double) * m);
            rel = std::sqrt(rr1) / bnorm;
            if (rel <= tol) break;
            const double beta = rr1 / rr;
            for (index_t i = 0; i < m; ++i) p[i] = r[i] + beta * p[i];
            rr = rr1;
        }
        for (index_t i = 0; i < m; ++i) x[i] += uc[i];
        *iters = k;
        *relres = rel;
    };
    if (P->dim == 2) run(get<2>(P), std::integral_constant<int, 2>{});
    else run(get<3>(P), std::integral_constant<int, 3>{});
    return 0;
}

// ----------------------------------------------------------- VV (sim) ----
int ref_sim_init(void* vp, double dt, double s0, const double* watch) {
    auto* P = static_cast<RefProblem*>(vp);
    auto run = [&](auto* B, auto dimc) {
        constexpr int Dim = decltype(dimc)::value;
        Problem<Dim> prob;
        prob.grid = B->grid;
        prob.horizon = B->hz;
        prob.material = B->mat;
        prob.constraints = B->constraints;
        prob.loads = B->loads;
        prob.cracks = B->cracks;
        if (s0 >= 0) prob.s0 = s0;
        if (watch) {
            Box<Dim> b;
            for (int d = 0; d < Dim; ++d) {
                b.lo[d] = watch[d];
                b.hi[d] = watch[Dim + d];
            }
            prob.watch = b;
        }
        B->sim = std::make_unique<Simulation<Dim>>(prob, SolverOptions{Method::Fast, Integrator::Vv, dt, std::nullopt});
    };
    if (P->dim == 2) run(get<2>(P), std::integral_constant<int, 2>{});
    else run(get<3>(P), std::integral_constant<int, 3>{});
    return 0;
}

// Simulation with Integrator::Adr (timestepping.hpp:79-162); fixed NaN = adaptive damping
int ref_sim_init_adr(void* vp, double dt, double s0, const double* watch, double fixed) {
    auto* P = static_cast<RefProblem*>(vp);
    auto run = [&](auto* B, auto dimc) {
        constexpr int Dim = decltype(dimc)::value;
        Problem<Dim> prob;
        prob.grid = B->grid;
        prob.horizon = B->hz;
        prob.material = B->mat;
        prob.constraints = B->constraints;
        prob.loads = B->loads;
        prob.cracks = B->cracks;
        if (s0 >= 0) prob.s0 = s0;
        if (watch) {
            Box<Dim> b;
            for (int d = 0; d < Dim; ++d) {
                b.lo[d] = watch[d];
                b.hi[d] = watch[Dim + d];
            }
            prob.watch = b;
        }
        std::optional<double> fd;
        if (fixed == fixed) fd = fixed;
        B->sim = std::make_unique<Simulation<Dim>>(prob, SolverOptions{Method::Fast, Integrator::Adr, dt, fd});
    };
    if (P->dim == 2) run(get<2>(P), std::integral_constant<int, 2>{});
    else run(get<3>(P), std::integral_constant<int, 3>{});
    return 0;
}

double ref_sim_adr_damping(void* vp) {
    auto* P = static_cast<RefProblem*>(vp);
    return P->dim == 2 ? get<2>(P)->sim->adr_damping() : get<3>(P)->sim->adr_damping();
}

int64_t ref_sim_step(void* vp, int n) {
    auto* P = static_cast<RefProblem*>(vp);
    int64_t nb = 0;
    for (int i = 0; i < n; ++i) {
        if (P->dim == 2) {
            get<2>(P)->sim->step();
            nb += (int64_t)get<2>(P)->sim->newly_broken().size();
        } else {
            get<3>(P)->sim->step();
            nb += (int64_t)get<3>(P)->sim->newly_broken().size();
        }
    }
    return nb;
}

void ref_sim_get(void* vp, double* u, double* v, double* f, double* t) {
    auto* P = static_cast<RefProblem*>(vp);
    auto run = [&](auto* B, auto dimc) {
        constexpr int Dim = decltype(dimc)::value;
        const auto& st = B->sim->state();
        const index_t n = B->grid.n_nodes();
        if (u) from_field<Dim>(st.u, u, n);
        if (v) from_field<Dim>(st.v, v, n);
        if (f) from_field<Dim>(st.f, f, n);
        if (t) *t = st.t;
    };
    if (P->dim == 2) run(get<2>(P), std::integral_constant<int, 2>{});
    else run(get<3>(P), std::integral_constant<int, 3>{});
}

// ------------------------------------------------------------- timing ----
// The reference hot path (FastForce::apply + apply_corrections) over
// n_vec vectors with `threads` independent FastForce instances (allowed by
// convolution.hpp:53-54), inputs u (n_vec x dim x N).  Returns wall seconds.
double ref_bench(void* vp, const double* u, int64_t n_vec, int threads) {
    auto* P = static_cast<RefProblem*>(vp);
    auto run = [&](auto* B, auto dimc) -> double {
        constexpr int Dim = decltype(dimc)::value;
        const index_t n = B->grid.n_nodes();
        std::vector<std::unique_ptr<FastForce<Dim>>> eng;
        for (int t = 0; t < threads; ++t) eng.push_back(std::make_unique<FastForce<Dim>>(B->grid, B->hz, B->K));
        std::vector<VecField<Dim>> U(n_vec), F(threads);
        for (int64_t v = 0; v < n_vec; ++v) to_field<Dim>(u + v * Dim * n, U[v], n);
        for (int t = 0; t < threads; ++t) F[t].resize(n);
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                for (int64_t v = t; v < n_vec; v += threads) {
                    eng[t]->apply(U[v], F[t]);
                    apply_corrections(F[t], U[v], B->de, B->regions, B->ledger, B->K, B->grid);
                }
            });
        for (auto& th : pool) th.join();
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    if (P->dim == 2) return run(get<2>(P), std::integral_constant<int, 2>{});
    return run(get<3>(P), std::integral_constant<int, 3>{});
}

}  // extern "C"

// ------------------------------------------- reference test-suite oracles --
// tests/support/oracles.hpp (compiled in place): random_kernel :99-110,
// random_field :113-119, random_ledger :123-137, tbt_apply_all :72-96.
extern "C" {

void ref_random_kernel(void* rng, int dim, int M, double h, double* out) {
    auto& r = *static_cast<std::mt19937*>(rng);
    auto copy = [&](const auto& K, int np) {
        const size_t ss = K.stencil_size();
        for (int p = 0; p < np; ++p) std::memcpy(out + p * ss, K.component(p).data(), sizeof(double) * ss);
    };
    if (dim == 2) copy(oracle::random_kernel<2>(M, h, r), 3);
    else copy(oracle::random_kernel<3>(M, h, r), 6);
}

void ref_random_field(void* rng, int dim, int64_t n, double amp, double* out) {
    auto& r = *static_cast<std::mt19937*>(rng);
    if (dim == 2) from_field<2>(oracle::random_field<2>(n, r, amp), out, n);
    else from_field<3>(oracle::random_field<3>(n, r, amp), out, n);
}

int64_t ref_random_ledger(void* rng, int dim, const int* dims, int M, int tries, int64_t* out, int64_t cap) {
    auto& r = *static_cast<std::mt19937*>(rng);
    if (dim == 2) {
        Grid<2> g;
        g.dims = {dims[0], dims[1]};
        g.h = 1.0;
        return pairs_t<2>(oracle::random_ledger<2>(g, M, tries, r), out, cap);
    }
    Grid<3> g;
    g.dims = {dims[0], dims[1], dims[2]};
    g.h = 1.0;
    return pairs_t<3>(oracle::random_ledger<3>(g, M, tries, r), out, cap);
}

void ref_tbt_apply_all(void* vp, const double* u, double* f) {
    auto* P = static_cast<RefProblem*>(vp);
    auto run = [&](auto* B, auto dimc) {
        constexpr int Dim = decltype(dimc)::value;
        const index_t n = B->grid.n_nodes();
        VecField<Dim> U;
        to_field<Dim>(u, U, n);
        from_field<Dim>(oracle::tbt_apply_all<Dim>(B->grid, B->K, U), f, n);
    };
    if (P->dim == 2) run(get<2>(P), std::integral_constant<int, 2>{});
    else run(get<3>(P), std::integral_constant<int, 3>{});
}



}  // extern "C"
