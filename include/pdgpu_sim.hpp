// pdgpu_sim.hpp -- solver-level C++ drop-in: pdgpu::Simulation<Dim>.
//
//   pdfast::Simulation<Dim>(problem, options)  -> pdgpu::Simulation<Dim>(problem, options)
//     step / run / finite / state / ledger / newly_broken / adr_damping /
//     damage / footprint_bytes as in timestepping.hpp:167-351, with the
//     state resident on the device; plus evaluate_force (timestepping.hpp:
//     295-310) and solve_static (CG on K := -A over the free DOFs).
//
// Uses the reference's own types (Problem, SolverOptions, SimState,
// BondLedger, ...) and its host-side assembly (build_kernel,
// classify_regions); everything per step runs through libpdgpu.so.
#pragma once
#include "pdfast/output.hpp"
#include "pdfast/timestepping.hpp"
#ifndef PDGPU_WITH_PDFAST
#define PDGPU_WITH_PDFAST
#endif
#include "pdgpu.hpp"

namespace pdgpu {

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

// MonitorWriter<Dim> (output.hpp:45-72) on libpdgpu's writer: the same
// constructor, nodes() and append(step, t, u) (host field), byte-identical
// rows; append_recorded(sim) writes the rows a Simulation recorded on the
// device since the last call (Simulation::monitor), i.e. the CLI's per-step
// monitor.append (tools/pdfast_cli.cpp:76) without a field download per step.
template <int Dim>
class MonitorWriter {
  public:
    MonitorWriter() = default;
    MonitorWriter(const std::string& path, const pdfast::Grid<Dim>& grid, const std::vector<pdfast::Vec<Dim>>& points) {
        std::vector<double> pts;
        for (const auto& x : points) pts.insert(pts.end(), x.begin(), x.end());
        int dims[Dim];
        for (int d = 0; d < Dim; ++d) dims[d] = grid.dims[d];
        nodes64_.resize(points.size());
        check(pdgpu_monitor_nodes(Dim, dims, grid.h, grid.origin.data(), pts.data(), (int)points.size(),
                                  nodes64_.data()));
        nodes_.assign(nodes64_.begin(), nodes64_.end());
        const int rc = pdgpu_monitor_open(path.c_str(), Dim, dims, grid.h, grid.origin.data(), pts.data(),
                                          (int)points.size(), &m_);
        if (rc == PDGPU_ERR_IO) throw pdfast::IoError(pdgpu_last_error());
        check(rc);
    }
    MonitorWriter(const MonitorWriter&) = delete;
    MonitorWriter& operator=(const MonitorWriter&) = delete;
    ~MonitorWriter() { pdgpu_monitor_close(m_); }

    const std::vector<pdfast::index_t>& nodes() const { return nodes_; }

    void append(pdfast::index_t step, double t, const pdfast::VecField<Dim>& u) {
        std::vector<double> row;
        for (pdfast::index_t p : nodes_)
            for (int d = 0; d < Dim; ++d) row.push_back(u.c[d][p]);
        if (!m_) return;
        check(pdgpu_monitor_append(m_, step, t, row.data()));
    }

    // rows recorded on the device by sim (after sim.engine() monitors nodes())
    int64_t append_recorded(Simulation<Dim>& sim) {
        const pdgpu_t h = sim.engine().handle();
        int64_t cnt = 0;
        check(pdgpu_sim_monitor_read(h, nullptr, nullptr, nullptr, 0, &cnt));
        std::vector<int64_t> steps((size_t)cnt + 1);
        std::vector<double> t((size_t)cnt + 1), vals((size_t)(cnt * nodes_.size() * Dim) + 1);
        check(pdgpu_sim_monitor_read(h, steps.data(), t.data(), vals.data(), cnt, &cnt));
        for (int64_t r = 0; r < cnt && m_; ++r)
            check(pdgpu_monitor_append(m_, steps[(size_t)r], t[(size_t)r], vals.data() + (size_t)r * nodes_.size() * Dim));
        return cnt;
    }
    // register this writer's nodes with the simulation's per-step device record
    void watch(Simulation<Dim>& sim) const {
        check(pdgpu_sim_monitor(sim.engine().handle(), nodes64_.data(), (int)nodes64_.size()));
    }

  private:
    pdgpu_monitor_t m_ = nullptr;
    std::vector<int64_t> nodes64_;
    std::vector<pdfast::index_t> nodes_;
};

}  // namespace pdgpu
