// snap_writer.cpp -- TEST INFRASTRUCTURE: runs the reference's own
// write_snapshot_dat (output.hpp:76-102, unmodified headers compiled in place)
// on raw fp64 inputs, to produce the golden snapshot files under
// tests/golden/snap*d/ (oracle/gen_golden.py).  Output: oracle/_ref/snap_writer.
//   snap_writer dim N0 N1 [N2] h o0 o1 [o2] step t dir u.raw damage.raw
// and the reference's MonitorWriter (output.hpp:45-72) for the monitor goldens:
//   snap_writer mon dim N0 N1 [N2] h o0 o1 [o2] path points.raw npts rows.raw nrows
//   (points: npts x dim doubles; rows: nrows x (step, t, u[dim][n]) doubles)
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "pdfast/output.hpp"

using namespace pdfast;

template <int Dim>
static int run(char** a) {
    Grid<Dim> g;
    int i = 0;
    for (int d = 0; d < Dim; ++d) g.dims[d] = std::atoi(a[i++]);
    g.h = std::strtod(a[i++], nullptr);
    for (int d = 0; d < Dim; ++d) g.origin[d] = std::strtod(a[i++], nullptr);
    const index_t step = std::atoll(a[i++]);
    const double t = std::strtod(a[i++], nullptr);
    const char* dir = a[i++];
    const index_t n = g.n_nodes();
    VecField<Dim> u(n);
    std::vector<double> damage((size_t)n);
    FILE* fu = std::fopen(a[i++], "rb");
    FILE* fd = std::fopen(a[i++], "rb");
    if (!fu || !fd) return 2;
    for (int d = 0; d < Dim; ++d)
        if (std::fread(u.c[d].data(), sizeof(double), (size_t)n, fu) != (size_t)n) return 3;
    if (std::fread(damage.data(), sizeof(double), (size_t)n, fd) != (size_t)n) return 3;
    std::fclose(fu);
    std::fclose(fd);
    std::printf("%s\n", write_snapshot_dat<Dim>(dir, g, u, damage, step, t).c_str());
    return 0;
}

template <int Dim>
static int run_monitor(char** a) {
    Grid<Dim> g;
    int i = 0;
    for (int d = 0; d < Dim; ++d) g.dims[d] = std::atoi(a[i++]);
    g.h = std::strtod(a[i++], nullptr);
    for (int d = 0; d < Dim; ++d) g.origin[d] = std::strtod(a[i++], nullptr);
    const char* path = a[i++];
    FILE* fp = std::fopen(a[i++], "rb");
    const int npts = std::atoi(a[i++]);
    FILE* fr = std::fopen(a[i++], "rb");
    const int nrows = std::atoi(a[i++]);
    if (!fp || !fr) return 2;
    std::vector<Vec<Dim>> pts((size_t)npts);
    for (auto& x : pts)
        if (std::fread(x.data(), sizeof(double), Dim, fp) != (size_t)Dim) return 3;
    MonitorWriter<Dim> mon(path, g, pts);
    const index_t n = g.n_nodes();
    VecField<Dim> u(n);
    for (int r = 0; r < nrows; ++r) {
        double st[2];
        if (std::fread(st, sizeof(double), 2, fr) != 2) return 3;
        for (int d = 0; d < Dim; ++d)
            if (std::fread(u.c[d].data(), sizeof(double), (size_t)n, fr) != (size_t)n) return 3;
        mon.append((index_t)st[0], st[1], u);
    }
    for (index_t p : mon.nodes()) std::printf("%lld\n", (long long)p);
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 2) return 1;
    if (std::string(argv[1]) == "mon") {
        const int dim = std::atoi(argv[2]);
        return dim == 2 ? run_monitor<2>(argv + 3) : run_monitor<3>(argv + 3);
    }
    const int dim = std::atoi(argv[1]);
    return dim == 2 ? run<2>(argv + 2) : run<3>(argv + 2);
}
