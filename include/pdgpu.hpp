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
// Solver level: include/pdgpu_sim.hpp (pdgpu::Simulation<Dim>).
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


}  // namespace pdgpu
