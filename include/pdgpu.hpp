// pdgpu.hpp -- C++ drop-in wrappers over the C ABI (pdgpu.h) with the
// reference library's class shapes.  Header-only.
//
// Operator level (duck-typed on the reference's types, compiles without pdfast):
//
//   pdfast::FastForce<Dim>(grid, hz, K)        -> pdgpu::FastForce<Dim>(grid, hz, K)
//   engine.apply(u, f)                          (convolution.hpp:249-259)
//   pdfast::apply_corrections(f,u,de,regions,ledger,K,grid)
//                                              -> pdgpu::apply_corrections(engine, f, u, regions, ledger)
//   pdfast::update_bonds(grid,hz,u,ledger,s0,watch)
//                                              -> pdgpu::update_bonds(engine, u, ledger, s0, watch)
//
// Solver level (needs the reference's types: define PDGPU_WITH_PDFAST after
// including pdfast):
//
//   pdfast::Simulation<Dim>(problem, options)  -> pdgpu::Simulation<Dim>(problem, options)
//     step / run / finite / state / ledger / newly_broken / adr_damping /
//     damage / footprint_bytes as in timestepping.hpp:167-351, with the
//     state resident on the device; plus evaluate_force (timestepping.hpp:
//     295-310) and solve_static (CG on K := -A over the free DOFs).
//
// With PDGPU_WITH_PDFAST, errors map back onto the reference's exception
// types (errors.hpp:8-59).
#pragma once
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pdgpu.h"

namespace pdgpu {

#ifdef PDGPU_WITH_PDFAST
[[noreturn]] inline void raise(int code) {
    const std::string msg = pdgpu_last_error();
    switch (code) {
        case PDGPU_ERR_HORIZON_TOO_LARGE: throw pdfast::HorizonTooLargeForGrid(msg);
        case PDGPU_ERR_SHAPE_MISMATCH: throw pdfast::ShapeMismatch(msg);
        case PDGPU_ERR_LEDGER_OUT_OF_BAND: throw pdfast::LedgerOutOfBand(msg);
        default: throw pdfast::Error(msg);
    }
}
#else
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void raise(int code) { throw Error(code, pdgpu_last_error()); }
#endif

inline void check(int code) {
    if (code != PDGPU_OK) raise(code);
}

using Pairs = std::vector<std::pair<int64_t, int64_t>>;

inline Pairs to_pairs(const std::vector<int64_t>& flat, int64_t n) {
    Pairs out;
    out.reserve((size_t)n);
    for (int64_t i = 0; i < n; ++i) out.emplace_back(flat[(size_t)(2 * i)], flat[(size_t)(2 * i + 1)]);
    return out;
}

// VecField<Dim> (field.hpp:14-47) <-> the ABI's component-major [dim][N] buffer
template <int Dim, class FieldT>
void pack_field(const FieldT& u, std::vector<double>& b) {
    const int64_t n = (int64_t)u.c[0].size();
    b.resize((size_t)(Dim * n));
    for (int d = 0; d < Dim; ++d)
        for (int64_t p = 0; p < n; ++p) b[(size_t)(d * n + p)] = u.c[d][(size_t)p];
}
template <int Dim, class FieldT>
void unpack_field(const std::vector<double>& b, FieldT& f) {
    const int64_t n = (int64_t)b.size() / Dim;
    for (int d = 0; d < Dim; ++d) {
        f.c[d].resize((size_t)n);
        for (int64_t p = 0; p < n; ++p) f.c[d][(size_t)p] = b[(size_t)(d * n + p)];
    }
}

template <int Dim>
class FastForce {
  public:
    static constexpr int n_pairs = Dim * (Dim + 1) / 2;

    // FastForce(const Grid<Dim>&, const Horizon&, const KernelStack<Dim>&), convolution.hpp:239
    template <class GridT, class HorizonT, class KernelT>
    FastForce(const GridT& grid, const HorizonT& hz, const KernelT& K, int device = 0, double rho = 1.0) {
        int dims[3] = {1, 1, 1};
        for (int d = 0; d < Dim; ++d) dims[d] = grid.dims[d];
        std::vector<double> st;
        for (int p = 0; p < n_pairs; ++p) {
            const auto& c = K.component(p);
            st.insert(st.end(), c.begin(), c.end());
        }
        check(pdgpu_create(Dim, dims, hz.M, st.data(), device, &h_));
        double origin[3] = {0, 0, 0};
        for (int d = 0; d < Dim; ++d) origin[d] = grid.origin[d];
        check(pdgpu_set_geometry(h_, grid.h, origin, hz.delta, rho));
        n_ = 1;
        for (int d = 0; d < Dim; ++d) n_ *= dims[d];
    }
    FastForce(const FastForce&) = delete;
    FastForce& operator=(const FastForce&) = delete;
    ~FastForce() { pdgpu_destroy(h_); }

    // f = A_hat u over all components (the uncorrected force), host VecField
    template <class FieldT>
    void apply(const FieldT& u, FieldT& f) {
        std::vector<double> ub, fb;
        pack_field<Dim>(u, ub);
        fb.resize(ub.size());
        check(pdgpu_apply_host(h_, ub.data(), fb.data(), (int64_t)u.c[0].size(), 1));
        unpack_field<Dim>(fb, f);
    }

    // FastForce::apply + apply_corrections in one call (host fields)
    template <class FieldT>
    void matvec(const FieldT& u, FieldT& f) {
        std::vector<double> ub, fb;
        pack_field<Dim>(u, ub);
        fb.resize(ub.size());
        check(pdgpu_matvec_host(h_, ub.data(), fb.data(), (int64_t)u.c[0].size(), 1));
        unpack_field<Dim>(fb, f);
    }

    double last_imag_residue() const { return pdgpu_last_imag_residue(h_); }
    std::size_t footprint_bytes() const { return pdgpu_footprint_bytes(h_); }

    // Regions (grid.hpp:172-209) and BondLedger (ledger.hpp:13-57) uploads
    template <class RegionsT>
    void set_regions(const RegionsT& regions) {
        std::vector<uint8_t> ns((size_t)n_), cm((size_t)n_);
        for (int64_t p = 0; p < n_; ++p) {
            ns[(size_t)p] = regions.near_surface(p) ? 1 : 0;
            cm[(size_t)p] = regions.constraint_mask(p);
        }
        check(pdgpu_set_regions(h_, ns.data(), cm.data()));
    }
    template <class LedgerT>
    void set_ledger(const LedgerT& ledger) {
        std::vector<int64_t> rs((size_t)n_ + 1, 0), pt;
        for (int64_t p = 0; p < n_; ++p) {
            const auto& v = ledger.broken_partners(p);
            pt.insert(pt.end(), v.begin(), v.end());
            rs[(size_t)p + 1] = (int64_t)pt.size();
        }
        if (pt.empty()) pt.push_back(0);
        check(pdgpu_set_ledger(h_, rs.data(), pt.data()));
    }

    // update_bonds (fracture.hpp:204-231) against the engine's device ledger:
    // returns the newly broken (p, q) pairs in the reference's visiting order.
    // u_dev: device-resident [Dim][N]; watch_lo_hi = {lo[Dim], hi[Dim]} or null.
    Pairs update_bonds(const double* u_dev, double s0, const double* watch_lo_hi = nullptr) {
        int64_t cnt = 0;
        check(pdgpu_update_bonds(h_, u_dev, s0, watch_lo_hi, nullptr, 0, &cnt));
        return last_new_pairs();
    }
    // same with a host VecField
    template <class FieldT>
    Pairs update_bonds_host(const FieldT& u, double s0, const double* watch_lo_hi = nullptr) {
        std::vector<double> ub;
        pack_field<Dim>(u, ub);
        int64_t cnt = 0;
        check(pdgpu_update_bonds_host(h_, ub.data(), (int64_t)u.c[0].size(), s0, watch_lo_hi, nullptr, 0, &cnt));
        return last_new_pairs();
    }

    Pairs ledger_pairs() const {
        int64_t cnt = 0;
        check(pdgpu_ledger_pairs(h_, nullptr, 0, &cnt));
        std::vector<int64_t> buf((size_t)(2 * cnt + 2));
        check(pdgpu_ledger_pairs(h_, buf.data(), cnt, &cnt));
        return to_pairs(buf, cnt);
    }

    pdgpu_t handle() const { return h_; }
    int64_t n_nodes() const { return n_; }

  private:
    Pairs last_new_pairs() const {
        int64_t cnt = 0;
        check(pdgpu_last_new_pairs(h_, nullptr, 0, &cnt));
        std::vector<int64_t> buf((size_t)(2 * cnt + 2));
        check(pdgpu_last_new_pairs(h_, buf.data(), cnt, &cnt));
        return to_pairs(buf, cnt);
    }
    pdgpu_t h_ = nullptr;
    int64_t n_ = 0;
};

// apply_corrections(f, u, de, regions, ledger, K, grid), corrections.hpp:76-110:
// the engine is given the same regions / ledger (set_regions / set_ledger).
template <int Dim, class FieldT, class RegionsT, class LedgerT>
void apply_corrections(FastForce<Dim>& eng, FieldT& f, const FieldT& u, const RegionsT& regions,
                       const LedgerT& ledger) {
    eng.set_regions(regions);
    eng.set_ledger(ledger);
    std::vector<double> ub, fb;
    pack_field<Dim>(u, ub);
    pack_field<Dim>(f, fb);
    check(pdgpu_apply_corrections_host(eng.handle(), ub.data(), fb.data(), (int64_t)u.c[0].size(), 1));
    unpack_field<Dim>(fb, f);
}

// update_bonds(grid, hz, u, ledger, s0, watch), fracture.hpp:204-231: the
// stretch test on the device against `ledger` (uploaded first), the new
// pairs inserted into `ledger` (BondLedger::break_bond, ledger.hpp:21-26) and
// returned in the reference's visiting order.  `watch` is any object with
// lo/hi arrays (Box<Dim>, geometry.hpp:53-63) or nullptr.
template <int Dim, class FieldT, class LedgerT, class BoxT = std::nullptr_t>
Pairs update_bonds(FastForce<Dim>& eng, const FieldT& u, LedgerT& ledger, double s0, const BoxT* watch = nullptr) {
    eng.set_ledger(ledger);
    double w[6] = {0, 0, 0, 0, 0, 0};
    if constexpr (!std::is_same_v<BoxT, std::nullptr_t>) {
        if (watch)
            for (int d = 0; d < Dim; ++d) {
                w[d] = watch->lo[d];
                w[Dim + d] = watch->hi[d];
            }
    }
    Pairs out = eng.update_bonds_host(u, s0, watch ? w : nullptr);
    for (const auto& pq : out) ledger.break_bond(pq.first, pq.second);
    return out;
}

#ifdef PDGPU_WITH_PDFAST
struct CgResult {
    int iterations = 0;
    double relative_residual = 0.0;
};

// Simulation<Dim> (timestepping.hpp:167-351) on the device: the same
// constructor (Problem + SolverOptions) and public interface.  Assembly of
// the host-side objects (stencils, regions) uses the reference's own
// functions; the state, constraints, ledger and every step live on the GPU.
// Method::Dense is the reference's meshfree comparison path and is not
// offered (pdfast::Error).
template <int Dim>
class Simulation {
  public:
    Simulation(pdfast::Problem<Dim> problem, pdfast::SolverOptions options, int device = 0)
        : prob_(std::move(problem)), opts_(options) {
        const auto t0 = clock_t::now();
        if (opts_.method != pdfast::Method::Fast)
            throw pdfast::Error("pdgpu::Simulation runs the fast (MSBFM) method only");
        kernels_ = pdfast::build_kernel(prob_.grid, prob_.horizon, prob_.material);
        regions_ = pdfast::classify_regions(prob_.grid, prob_.horizon, prob_.constraints);
        engine_ = std::make_unique<FastForce<Dim>>(prob_.grid, prob_.horizon, kernels_, device, prob_.material.rho);
        const pdgpu_t h = engine_->handle();
        for (const auto& cs : prob_.constraints)
            check(pdgpu_add_constraint(h, cs.box.lo.data(), cs.box.hi.data(), cs.dir_mask,
                                       cs.kind == pdfast::ConstraintKind::Velocity ? 1 : 0, cs.value));
        for (const auto& ld : prob_.loads) check(pdgpu_add_load(h, ld.box.lo.data(), ld.box.hi.data(), ld.value.data()));
        // seed_cracks (fracture.hpp:164-198); the ledger is a set, so seeding
        // crack by crack gives the same bonds as the reference's single pass
        int64_t added = 0;
        if constexpr (Dim == 2) {
            for (const auto& sg : prob_.cracks.segments) {
                const double g[5] = {sg.a[0], sg.a[1], sg.b[0], sg.b[1], sg.width};
                check(pdgpu_seed_segment(h, g, &added));
            }
        } else {
            for (const auto& nt : prob_.cracks.notches) {
                const double g[9] = {(double)nt.axis, nt.plane, nt.width, nt.lo[0], nt.lo[1], nt.lo[2],
                                     nt.hi[0], nt.hi[1], nt.hi[2]};
                check(pdgpu_seed_notch(h, g, &added));
            }
        }
        const int64_t n = prob_.grid.n_nodes();
        std::vector<double> v0((size_t)(Dim * n), 0.0);
        bool any_v0 = false;
        for (const auto& iv : prob_.initial_velocities)
            for (int64_t p = 0; p < n; ++p)
                if (iv.box.contains(prob_.grid.pos(p)))
                    for (int d = 0; d < Dim; ++d) {
                        v0[(size_t)(d * n + p)] = iv.value[d];
                        any_v0 = true;
                    }
        if (opts_.integrator == pdfast::Integrator::Adr) {
            check(pdgpu_sim_init_adr(h, opts_.dt, opts_.fixed_damping ? *opts_.fixed_damping : std::nan("")));
            if (any_v0) check(pdgpu_sim_set_velocity(h, v0.data()));
        } else {
            check(pdgpu_sim_init(h, opts_.dt, any_v0 ? v0.data() : nullptr));
        }
        if (prob_.watch) {
            for (int d = 0; d < Dim; ++d) {
                watch_[d] = prob_.watch->lo[d];
                watch_[Dim + d] = prob_.watch->hi[d];
            }
        }
        ledger_ = pdfast::BondLedger(n);
        for (auto* fld : {&state_.u, &state_.v, &state_.f, &state_.f_prev, &state_.v_half}) fld->resize(n);
        dirty_ = true;
        timers_.assembly_s = seconds_since(t0);
    }

    void step() {
        const auto t0 = clock_t::now();
        int64_t broken = 0;
        check(pdgpu_sim_step(engine_->handle(), 1, prob_.s0 ? *prob_.s0 : -1.0, prob_.watch ? watch_ : nullptr,
                             &broken));
        ++step_;
        dirty_ = true;
        timers_.stepping_s += seconds_since(t0);  // fracture sweep included (one device pass per step)
    }
    void run(int64_t n_steps) {
        for (int64_t i = 0; i < n_steps; ++i) step();
    }
    template <class Callback>
    void run(int64_t n_steps, Callback&& cb) {
        for (int64_t i = 0; i < n_steps; ++i) {
            step();
            cb(*this);
        }
    }

    bool finite() const {
        int ok = 0;
        check(pdgpu_sim_finite(engine_->handle(), &ok));
        return ok != 0;
    }

    const pdfast::SimState<Dim>& state() const {
        sync();
        return state_;
    }
    const pdfast::Grid<Dim>& grid() const { return prob_.grid; }
    const pdfast::Horizon& horizon() const { return prob_.horizon; }
    const pdfast::Regions<Dim>& regions() const { return regions_; }
    const pdfast::KernelStack<Dim>& kernels() const { return kernels_; }
    const pdfast::PhaseTimers& timers() const { return timers_; }
    const pdfast::BondLedger& ledger() const {
        sync();
        return ledger_;
    }
    const std::vector<std::pair<pdfast::index_t, pdfast::index_t>>& newly_broken() const {
        sync();
        return newly_broken_;
    }
    double adr_damping() const {
        if (opts_.integrator != pdfast::Integrator::Adr) return 0.0;
        double c = 0.0;
        check(pdgpu_sim_adr_damping(engine_->handle(), &c));
        return c;
    }
    std::vector<double> damage() const { return pdfast::damage_field(prob_.grid, prob_.horizon, ledger()); }
    std::size_t footprint_bytes() const {
        return engine_->footprint_bytes() + (size_t)prob_.grid.n_nodes() * Dim * sizeof(double) * 6;
    }

    // Simulation::evaluate_force (timestepping.hpp:295-310) on a given field:
    // f = A u + body, zero on constrained (node, dir)
    void evaluate_force(const pdfast::VecField<Dim>& u, pdfast::VecField<Dim>& f) const {
        std::vector<double> ub, fb;
        pack_field<Dim>(u, ub);
        fb.resize(ub.size());
        check(pdgpu_evaluate_force_host(engine_->handle(), ub.data(), fb.data(), (int64_t)u.c[0].size()));
        unpack_field<Dim>(fb, f);
    }

    // Static solve K_ff u_f = b_f + (A u_c)_f with the problem's prescribed
    // displacements (CG, the reference's ADR alternative); x = the full
    // displacement field.
    CgResult solve_static(const pdfast::VecField<Dim>& b, pdfast::VecField<Dim>& x, double tol = 1e-10,
                          int maxit = 100000) const {
        std::vector<double> bb, xb;
        pack_field<Dim>(b, bb);
        xb.resize(bb.size());
        CgResult r;
        check(pdgpu_cg_solve_host(engine_->handle(), bb.data(), xb.data(), tol, maxit, &r.iterations,
                                  &r.relative_residual, nullptr, 0));
        unpack_field<Dim>(xb, x);
        return r;
    }

    FastForce<Dim>& engine() { return *engine_; }

  private:
    using clock_t = std::chrono::steady_clock;
    static double seconds_since(clock_t::time_point t0) {
        return std::chrono::duration<double>(clock_t::now() - t0).count();
    }

    // device -> host mirror of the state, ledger and last breaks, on demand
    void sync() const {
        if (!dirty_) return;
        const pdgpu_t h = engine_->handle();
        const int64_t n = prob_.grid.n_nodes();
        std::vector<double> u((size_t)(Dim * n)), v(u.size()), f(u.size()), fp(u.size()), vh(u.size());
        double t = 0.0;
        check(pdgpu_sim_get(h, u.data(), v.data(), f.data(), &t));
        check(pdgpu_sim_get_aux(h, fp.data(), vh.data()));
        unpack_field<Dim>(u, state_.u);
        unpack_field<Dim>(v, state_.v);
        unpack_field<Dim>(f, state_.f);
        unpack_field<Dim>(fp, state_.f_prev);
        unpack_field<Dim>(vh, state_.v_half);
        state_.t = t;
        state_.step = step_;
        ledger_ = pdfast::BondLedger(n);
        for (const auto& pq : engine_->ledger_pairs()) ledger_.break_bond(pq.first, pq.second);
        int64_t cnt = 0;
        check(pdgpu_sim_newly_broken(h, nullptr, 0, &cnt));
        std::vector<int64_t> buf((size_t)(2 * cnt + 2));
        check(pdgpu_sim_newly_broken(h, buf.data(), cnt, &cnt));
        newly_broken_.clear();
        for (int64_t i = 0; i < cnt; ++i) newly_broken_.emplace_back(buf[(size_t)(2 * i)], buf[(size_t)(2 * i + 1)]);
        dirty_ = false;
    }

    pdfast::Problem<Dim> prob_;
    pdfast::SolverOptions opts_;
    pdfast::KernelStack<Dim> kernels_;
    pdfast::Regions<Dim> regions_;
    std::unique_ptr<FastForce<Dim>> engine_;
    double watch_[6] = {0, 0, 0, 0, 0, 0};
    int64_t step_ = 0;
    pdfast::PhaseTimers timers_;
    mutable bool dirty_ = true;
    mutable pdfast::SimState<Dim> state_;
    mutable pdfast::BondLedger ledger_;
    mutable std::vector<std::pair<pdfast::index_t, pdfast::index_t>> newly_broken_;
};
#endif  // PDGPU_WITH_PDFAST

}  // namespace pdgpu
