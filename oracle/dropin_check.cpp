// dropin_check.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Runs the C++ drop-in (include/pdgpu.hpp over libpdgpu.so) side by side with
// the reference's own C++ path on the reference's own types: the unmodified
// pdfast headers (compiled here against oracle/fftw_cpu) are the checker.
// Built by oracle/Makefile into oracle/_ref/dropin_check when the reference
// tree is present; run on the GPU box by tests/test_gpu_cpp_dropin.py.
// Prints one JSON object per check.
//
// Call sites mirrored:
//   FastForce::apply + apply_corrections    tests/test_corrections.cpp:107-110, 320-323
//   update_bonds                            fracture.hpp:204-231
//   Simulation (VV + fracture, ADR)         timestepping.hpp:167-351, acceptance_main.cpp:197-219
//   the three hot-path exceptions           errors.hpp:21-29
#include <fftw3.h>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <random>
#include <string>

#include "pdfast/scenario.hpp"
#include "pdfast/timestepping.hpp"
#include "support/oracles.hpp"
#include "pdgpu_sim.hpp"

using namespace pdfast;

namespace {

int g_fail = 0;

void report(const char* name, bool pass, const std::string& detail) {
    std::printf("{\"check\": \"%s\", \"pass\": %s, %s}\n", name, pass ? "true" : "false", detail.c_str());
    std::fflush(stdout);
    if (!pass) ++g_fail;
}

template <int Dim>
double rel_l2(const VecField<Dim>& a, const VecField<Dim>& b) {
    double num = 0.0, den = 0.0;
    for (int d = 0; d < Dim; ++d)
        for (size_t i = 0; i < a.c[d].size(); ++i) {
            const double e = a.c[d][i] - b.c[d][i];
            num += e * e;
            den += b.c[d][i] * b.c[d][i];
        }
    return std::sqrt(num / (den > 0 ? den : 1.0));
}

template <int Dim>
VecField<Dim> random_field(index_t n, std::mt19937& rng, double amp = 1.0) {
    std::uniform_real_distribution<double> U(-amp, amp);
    VecField<Dim> u(n);
    for (int d = 0; d < Dim; ++d)
        for (auto& x : u.c[d]) x = U(rng);
    return u;
}

const Material kUnit{1.0, 0.25, 1.0, {}, {}, PlaneMode::Stress};

// FastForce::apply + apply_corrections with constraints and a random crack
// ledger, pdfast vs pdgpu on the same objects
template <int Dim>
void check_matvec(IVec<Dim> dims, const char* name) {
    Grid<Dim> g;
    g.h = 1.0 / dims[0];
    g.dims = dims;
    g.thickness = 1.0;
    const Horizon hz{3.015 * g.h, 3};
    const auto K = build_kernel(g, hz, kUnit);
    Constraint<Dim> cs;
    for (int d = 0; d < Dim; ++d) cs.box.hi[d] = g.extent(d);
    cs.box.hi[0] = 3.015 * g.h;
    cs.dir_mask = 1;
    const auto regions = classify_regions<Dim>(g, hz, {cs});
    const auto de = build_de(g, hz, regions, K);
    std::mt19937 rng(Dim * 101);
    const BondLedger ledger = oracle::random_ledger<Dim>(g, hz.M, 200, rng);
    const auto u = random_field<Dim>(g.n_nodes(), rng);

    VecField<Dim> f_ref(g.n_nodes()), f_gpu(g.n_nodes());
    FastForce<Dim> ref(g, hz, K);
    ref.apply(u, f_ref);
    apply_corrections(f_ref, u, de, regions, ledger, K, g);

    pdgpu::FastForce<Dim> gpu(g, hz, K);  // was: FastForce<Dim> engine(g, hz, K)
    gpu.apply(u, f_gpu);                  // same call
    pdgpu::apply_corrections(gpu, f_gpu, u, regions, ledger);
    const double err = rel_l2<Dim>(f_gpu, f_ref);
    char buf[200];
    std::snprintf(buf, sizeof buf, "\"rel_l2\": %.3e, \"bonds\": %lld, \"tol\": 1e-11", err,
                  (long long)ledger.total_broken());
    report(name, err <= 1e-11, buf);
}

// update_bonds: the same pairs in the same order, and equal ledgers
void check_update_bonds() {
    Grid<2> g;
    g.h = 1.0 / 64;
    g.dims = {64, 48};
    g.thickness = 1.0;
    const Horizon hz{3.015 * g.h, 3};
    const auto K = build_kernel(g, hz, kUnit);
    std::mt19937 rng(7);
    BondLedger l_ref(g.n_nodes()), l_gpu(g.n_nodes());
    pdgpu::FastForce<2> gpu(g, hz, K);
    Box<2> watch{{0.1, 0.05}, {0.9, 0.7}};
    bool same = true;
    long long total = 0;
    for (int round = 0; round < 4; ++round) {
        const auto u = random_field<2>(g.n_nodes(), rng, 2e-3 * g.h * (round + 1));
        const Box<2>* w = round % 2 ? &watch : nullptr;
        const auto a = update_bonds(g, hz, u, l_ref, 1e-3, w ? std::optional<Box<2>>(*w) : std::nullopt);
        const auto b = pdgpu::update_bonds(gpu, u, l_gpu, 1e-3, w);
        same = same && a.size() == b.size();
        for (size_t i = 0; same && i < a.size(); ++i) same = a[i].first == b[i].first && a[i].second == b[i].second;
        total += (long long)a.size();
    }
    const bool eq = l_ref == l_gpu;
    char buf[160];
    std::snprintf(buf, sizeof buf, "\"pairs_identical\": %s, \"ledgers_equal\": %s, \"broken\": %lld",
                  same ? "true" : "false", eq ? "true" : "false", total);
    report("update_bonds", same && eq && total > 0, buf);
}

// Simulation<2> VV with fracture: the criterion-5 problem (acceptance_main.cpp:197-219)
void check_simulation_vv() {
    auto cfg = preset("precracked_plate", 0.05 / 100.0);
    auto prob = make_problem<2>(cfg);
    const SolverOptions opts{Method::Fast, Integrator::Vv, cfg.dt, std::nullopt};
    Simulation<2> ref(prob, opts);
    pdgpu::Simulation<2> gpu(prob, opts);  // was: Simulation<2> sim(prob, opts)
    double worst = 0.0;
    bool breaks_equal = true, ledgers_equal = true;
    for (int n = 0; n < 200; ++n) {
        ref.step();
        gpu.step();
        breaks_equal = breaks_equal && ref.newly_broken() == gpu.newly_broken();
        if (n % 20 == 19) ledgers_equal = ledgers_equal && ref.ledger() == gpu.ledger();
        const double scale = ref.state().u.max_abs();
        double diff = 0.0;
        for (int d = 0; d < 2; ++d)
            for (size_t i = 0; i < ref.state().u.c[d].size(); ++i)
                diff = std::max(diff, std::abs(ref.state().u.c[d][i] - gpu.state().u.c[d][i]));
        if (scale > 0) worst = std::max(worst, diff / scale);
    }
    const bool t_equal = ref.state().t == gpu.state().t && ref.state().step == gpu.state().step;
    const bool fin = gpu.finite() && ref.finite();
    const auto dref = ref.damage(), dgpu = gpu.damage();
    const bool dmg = dref == dgpu;
    char buf[320];
    std::snprintf(buf, sizeof buf,
                  "\"max_rel_u\": %.3e, \"tol\": 1e-8, \"newly_broken_equal\": %s, \"ledgers_equal\": %s, "
                  "\"bonds\": %lld, \"t_equal\": %s, \"finite\": %s, \"damage_equal\": %s",
                  worst, breaks_equal ? "true" : "false", ledgers_equal ? "true" : "false",
                  (long long)gpu.ledger().total_broken(), t_equal ? "true" : "false", fin ? "true" : "false",
                  dmg ? "true" : "false");
    report("simulation_vv_fracture", worst <= 1e-8 && breaks_equal && ledgers_equal && t_equal && fin && dmg, buf);
}

// Simulation<2> with Integrator::Adr on a loaded, clamped plate
void check_simulation_adr() {
    Problem<2> prob;
    prob.grid.h = 1.0 / 64;
    prob.grid.dims = {64, 64};
    prob.grid.thickness = 1.0;
    prob.horizon = Horizon{3.015 * prob.grid.h, 3};
    prob.material = kUnit;
    Constraint<2> clamp;
    clamp.box.lo = {0.0, 0.0};
    clamp.box.hi = {3.015 * prob.grid.h, 1.0};
    clamp.dir_mask = 3;
    prob.constraints.push_back(clamp);
    Load<2> load;
    load.box.lo = {0.5, 0.0};
    load.box.hi = {1.0, 1.0};
    load.value = {1e-3, -2e-3};
    prob.loads.push_back(load);
    const SolverOptions opts{Method::Fast, Integrator::Adr, 1.0, std::nullopt};
    Simulation<2> ref(prob, opts);
    pdgpu::Simulation<2> gpu(prob, opts);
    for (int n = 0; n < 60; ++n) {
        ref.step();
        gpu.step();
    }
    const double err = rel_l2<2>(gpu.state().u, ref.state().u);
    const double dc = std::abs(gpu.adr_damping() - ref.adr_damping()) / std::max(std::abs(ref.adr_damping()), 1e-300);
    char buf[160];
    std::snprintf(buf, sizeof buf, "\"rel_l2_u\": %.3e, \"damping_rel\": %.3e, \"tol\": 1e-9", err, dc);
    report("simulation_adr", err <= 1e-9 && dc <= 1e-9, buf);
}

// evaluate_force and the CG static solve, graded by the reference's operator
void check_static_solve() {
    Problem<2> prob;
    prob.grid.h = 1.0 / 128;
    prob.grid.dims = {128, 128};
    prob.grid.thickness = 1.0;
    prob.horizon = Horizon{3.015 * prob.grid.h, 3};
    prob.material = kUnit;
    const double dl = 3.015 * prob.grid.h;
    for (int ax = 0; ax < 2; ++ax)
        for (int side = 0; side < 2; ++side) {
            Constraint<2> cs;
            cs.box.lo = {0.0, 0.0};
            cs.box.hi = {1.0, 1.0};
            if (side == 0) cs.box.hi[ax] = dl;
            else cs.box.lo[ax] = 1.0 - dl;
            cs.dir_mask = 3;
            cs.value = ax == 1 && side == 1 ? 1e-3 : 0.0;  // one prescribed non-zero layer
            prob.constraints.push_back(cs);
        }
    prob.cracks.segments.push_back({{0.3, 0.5}, {0.7, 0.5}, 0.0});
    const SolverOptions opts{Method::Fast, Integrator::Vv, 1.0, std::nullopt};
    Simulation<2> ref(prob, opts);  // reference evaluate_force path (timestepping.hpp:295-310)
    pdgpu::Simulation<2> gpu(prob, opts);
    const bool ledger_eq = ref.ledger() == gpu.ledger();
    const index_t n = prob.grid.n_nodes();
    std::mt19937 rng(11);
    const auto u = random_field<2>(n, rng);
    // the reference's operator on the same objects: FastForce + apply_corrections
    const auto& K = ref.kernels();
    const auto& regions = ref.regions();
    const auto de = build_de(prob.grid, prob.horizon, regions, K);
    FastForce<2> eng(prob.grid, prob.horizon, K);
    auto refop = [&](const VecField<2>& x, VecField<2>& f) {
        eng.apply(x, f);
        apply_corrections(f, x, de, regions, ref.ledger(), K, prob.grid);
    };
    VecField<2> f_ref(n), f_gpu(n);
    refop(u, f_ref);
    for (int d = 0; d < 2; ++d)
        for (index_t p = 0; p < n; ++p)
            if (regions.constrained(p, d)) f_ref.c[d][p] = 0.0;
    gpu.evaluate_force(u, f_gpu);
    const double ef = rel_l2<2>(f_gpu, f_ref);
    // CG: K u = b on the free DOFs with the prescribed layer
    const auto b = random_field<2>(n, rng);
    VecField<2> x(n);
    const auto res = gpu.solve_static(b, x, 1e-10, 50000);
    VecField<2> Ax(n);
    refop(x, Ax);
    double num = 0.0, den = 0.0;
    VecField<2> uc(n), Auc(n);
    for (const auto& cs : prob.constraints)
        for (index_t p = 0; p < n; ++p)
            if (cs.box.contains(prob.grid.pos(p)))
                for (int d = 0; d < 2; ++d)
                    if ((cs.dir_mask >> d) & 1u) uc.c[d][p] = cs.value;
    refop(uc, Auc);
    for (int d = 0; d < 2; ++d)
        for (index_t p = 0; p < n; ++p) {
            if (regions.constrained(p, d)) continue;
            const double r = Ax.c[d][p] + b.c[d][p];
            const double bf = b.c[d][p] + Auc.c[d][p];
            num += r * r;
            den += bf * bf;
        }
    const double relres = std::sqrt(num / den);
    char buf[240];
    std::snprintf(buf, sizeof buf,
                  "\"evaluate_force_rel_l2\": %.3e, \"cg_iterations\": %d, \"cg_relres_gpu\": %.3e, "
                  "\"cg_relres_reference_operator\": %.3e, \"ledger_equal\": %s",
                  ef, res.iterations, res.relative_residual, relres, ledger_eq ? "true" : "false");
    report("evaluate_force_and_cg", ef <= 1e-11 && relres <= 1e-10 * (1 + 1e-3) && ledger_eq, buf);
}

// the reference's exception types come back through the C ABI
void check_errors() {
    bool horizon = false, shape = false, band = false;
    Grid<2> g;
    g.h = 1.0;
    g.dims = {3, 3};
    g.thickness = 1.0;
    const Horizon hz{3.0, 3};
    const auto K = build_kernel(g, hz, kUnit);
    try {
        pdgpu::FastForce<2> e(g, hz, K);
    } catch (const HorizonTooLargeForGrid&) {
        horizon = true;  // convolution.hpp:61-62
    }
    g.dims = {16, 16};
    const auto K2 = build_kernel(g, hz, kUnit);
    pdgpu::FastForce<2> e2(g, hz, K2);
    VecField<2> u(10), f(10);
    try {
        e2.apply(u, f);
    } catch (const ShapeMismatch&) {
        shape = true;  // convolution.hpp:120-121
    }
    BondLedger far(g.n_nodes());
    far.break_bond(0, 200);  // 12 rows apart: outside the band
    VecField<2> u2(g.n_nodes()), f2(g.n_nodes());
    const auto regions = classify_regions<2>(g, hz, {});
    try {
        pdgpu::apply_corrections(e2, f2, u2, regions, far);
    } catch (const LedgerOutOfBand&) {
        band = true;  // corrections.hpp:99-100
    }
    char buf[160];
    std::snprintf(buf, sizeof buf, "\"horizon_too_large\": %s, \"shape_mismatch\": %s, \"ledger_out_of_band\": %s",
                  horizon ? "true" : "false", shape ? "true" : "false", band ? "true" : "false");
    report("exceptions", horizon && shape && band, buf);
}

}  // namespace

// MonitorWriter (output.hpp:45-72): the reference writer fed every step from
// the reference Simulation vs pdgpu::MonitorWriter fed from the rows the GPU
// Simulation recorded on the device; same nodes, steps and times, values to the
// trajectory tolerance; IoError on an unwritable path from both
void check_monitor() {
    auto cfg = preset("precracked_plate", 0.05 / 100.0);
    auto prob = make_problem<2>(cfg);
    const SolverOptions opts{Method::Fast, Integrator::Vv, cfg.dt, std::nullopt};
    Simulation<2> ref(prob, opts);
    pdgpu::Simulation<2> gpu(prob, opts);
    const std::vector<Vec<2>> pts = {{0.0255, 0.0125}, {0.01, 0.04}, {-1.0, 9.0}};
    const std::string pr = "/tmp/pdgpu_mon_ref.tsv", pg = "/tmp/pdgpu_mon_gpu.tsv";
    bool ok = true;
    {
        MonitorWriter<2> mref(pr, prob.grid, pts);
        pdgpu::MonitorWriter<2> mgpu(pg, prob.grid, pts);
        ok = ok && mref.nodes() == mgpu.nodes();
        mgpu.watch(gpu);
        for (int n = 0; n < 60; ++n) {
            ref.step();
            mref.append(ref.state().step, ref.state().t, ref.state().u);
        }
        gpu.run(60);
        ok = ok && mgpu.append_recorded(gpu) == 60;
    }
    auto rows = [](const std::string& path) {
        std::ifstream in(path);
        std::string line;
        std::vector<std::vector<double>> out;
        std::getline(in, line);
        while (std::getline(in, line)) {
            std::istringstream ss(line);
            std::vector<double> v;
            double x;
            while (ss >> x) v.push_back(x);
            out.push_back(v);
        }
        return out;
    };
    const auto a = rows(pr), b = rows(pg);
    double worst = 0.0, scale = 0.0;
    ok = ok && a.size() == b.size() && a.size() == 60 * pts.size();
    for (size_t r = 0; ok && r < a.size(); ++r) {
        ok = ok && a[r][0] == b[r][0] && a[r][1] == b[r][1] && a[r][2] == b[r][2];
        for (int d = 3; d < 5; ++d) {
            worst = std::max(worst, std::abs(a[r][d] - b[r][d]));
            scale = std::max(scale, std::abs(a[r][d]));
        }
    }
    const double rel = scale > 0 ? worst / scale : worst;
    bool ioerr_ref = false, ioerr_gpu = false;
    try {
        MonitorWriter<2>("/nonexistent_dir/m.tsv", prob.grid, pts);
    } catch (const IoError&) {
        ioerr_ref = true;
    }
    try {
        pdgpu::MonitorWriter<2>("/nonexistent_dir/m.tsv", prob.grid, pts);
    } catch (const IoError&) {
        ioerr_gpu = true;
    }
    char buf[200];
    std::snprintf(buf, sizeof buf, "\"rows\": %zu, \"max_rel_u\": %.3e, \"tol\": 1e-8, \"io_error\": %s", b.size(), rel,
                  ioerr_ref && ioerr_gpu ? "true" : "false");
    report("monitor", ok && rel <= 1e-8 && ioerr_ref && ioerr_gpu, buf);
}

int main() {
    check_matvec<2>({128, 96}, "matvec_2d");
    check_matvec<3>({24, 20, 16}, "matvec_3d");
    check_update_bonds();
    check_simulation_vv();
    check_simulation_adr();
    check_static_solve();
    check_errors();
    check_monitor();
    return g_fail;
}
