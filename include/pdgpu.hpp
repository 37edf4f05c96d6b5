// pdgpu.hpp -- C++ drop-in wrappers over the C ABI (pdgpu.h) with the
// reference library's class shapes.  Header-only; duck-typed on the
// reference's types so it compiles against pdfast without including it:
//
//   pdfast::FastForce<Dim>(grid, hz, K)        -> pdgpu::FastForce<Dim>(grid, hz, K)
//   engine.apply(u, f)                          (convolution.hpp:249-259)
//   pdfast::apply_corrections(f,u,de,regions,ledger,K,grid)
//                                              -> pdgpu::apply_corrections(engine, f, u, regions, ledger)
//   pdfast::update_bonds(grid,hz,u,ledger,s0,watch)
//                                              -> engine.update_bonds(u, s0, watch)
//
// Errors map back onto the reference's exception types when the caller
// defines PDGPU_WITH_PDFAST before including this header (after pdfast).
#pragma once
#include <cstdint>
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

template <int Dim>
class FastForce {
  public:
    static constexpr int n_pairs = Dim * (Dim + 1) / 2;

    // FastForce(const Grid<Dim>&, const Horizon&, const KernelStack<Dim>&), convolution.hpp:239
    template <class GridT, class HorizonT, class KernelT>
    FastForce(const GridT& grid, const HorizonT& hz, const KernelT& K, int device = 0) {
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
        check(pdgpu_set_geometry(h_, grid.h, origin, hz.delta, 1.0));
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
        pack(u, ub);
        fb.resize(ub.size());
        check(pdgpu_apply_host(h_, ub.data(), fb.data(), (int64_t)u.c[0].size(), 1));
        unpack(fb, f);
    }

    // FastForce::apply + apply_corrections in one call (host fields)
    template <class FieldT>
    void matvec(const FieldT& u, FieldT& f) {
        std::vector<double> ub, fb;
        pack(u, ub);
        fb.resize(ub.size());
        check(pdgpu_matvec_host(h_, ub.data(), fb.data(), (int64_t)u.c[0].size(), 1));
        unpack(fb, f);
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

    // update_bonds (fracture.hpp:204-231) on device-resident u ([Dim][N] doubles)
    std::vector<std::pair<int64_t, int64_t>> update_bonds(const double* u_dev, double s0,
                                                          const double* watch_lo_hi = nullptr) {
        int64_t cnt = 0;
        check(pdgpu_update_bonds(h_, u_dev, s0, watch_lo_hi, nullptr, 0, &cnt));
        return {};  // counts only; use ledger_pairs() for the set
    }

    std::vector<std::pair<int64_t, int64_t>> ledger_pairs() const {
        int64_t cnt = 0;
        check(pdgpu_ledger_pairs(h_, nullptr, 0, &cnt));
        std::vector<int64_t> buf((size_t)(2 * cnt + 2));
        check(pdgpu_ledger_pairs(h_, buf.data(), cnt, &cnt));
        std::vector<std::pair<int64_t, int64_t>> out;
        for (int64_t i = 0; i < cnt; ++i) out.emplace_back(buf[(size_t)(2 * i)], buf[(size_t)(2 * i + 1)]);
        return out;
    }

    pdgpu_t handle() const { return h_; }

  private:
    template <class FieldT>
    void pack(const FieldT& u, std::vector<double>& b) const {
        const int64_t n = (int64_t)u.c[0].size();
        b.resize((size_t)(Dim * n));
        for (int d = 0; d < Dim; ++d)
            for (int64_t p = 0; p < n; ++p) b[(size_t)(d * n + p)] = u.c[d][(size_t)p];
    }
    template <class FieldT>
    void unpack(const std::vector<double>& b, FieldT& f) const {
        const int64_t n = (int64_t)b.size() / Dim;
        for (int d = 0; d < Dim; ++d) {
            f.c[d].resize((size_t)n);
            for (int64_t p = 0; p < n; ++p) f.c[d][(size_t)p] = b[(size_t)(d * n + p)];
        }
    }
    pdgpu_t h_ = nullptr;
    int64_t n_ = 0;
};

// apply_corrections(f, u, de, regions, ledger, K, grid), corrections.hpp:76-110:
// the engine must carry the same regions/ledger (set_regions / set_ledger).
template <int Dim, class FieldT, class RegionsT, class LedgerT>
void apply_corrections(FastForce<Dim>& eng, FieldT& f, const FieldT& u, const RegionsT& regions,
                       const LedgerT& ledger) {
    eng.set_regions(regions);
    eng.set_ledger(ledger);
    const int64_t n = (int64_t)u.c[0].size();
    std::vector<double> ub((size_t)(Dim * n)), fb((size_t)(Dim * n));
    for (int d = 0; d < Dim; ++d)
        for (int64_t p = 0; p < n; ++p) {
            ub[(size_t)(d * n + p)] = u.c[d][(size_t)p];
            fb[(size_t)(d * n + p)] = f.c[d][(size_t)p];
        }
    check(pdgpu_apply_corrections_host(eng.handle(), ub.data(), fb.data(), n, 1));
    for (int d = 0; d < Dim; ++d)
        for (int64_t p = 0; p < n; ++p) f.c[d][(size_t)p] = fb[(size_t)(d * n + p)];
}

}  // namespace pdgpu
