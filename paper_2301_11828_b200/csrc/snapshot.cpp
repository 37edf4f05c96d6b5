// snapshot.cpp -- the reference's plain-text snapshot format (output.hpp:74-154)
// for trajectory dumps of GPU runs: "# key value" header lines (dim, dims, h,
// origin, step, t, columns), then one row per node "id u_x u_y [u_z] damage"
// with ids from 1 and every double printed %.17g, so the file round-trips
// bit-exactly and compares byte for byte with the reference's own writer.
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <sys/stat.h>

#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

namespace pdgpu {
namespace snapshot {

static std::string g17(double v) {
    char buf[40];
    snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

static bool make_dirs(const std::string& dir) {
    std::string cur;
    std::stringstream ss(dir);
    std::string part;
    if (!dir.empty() && dir[0] == '/') cur = "/";
    while (std::getline(ss, part, '/')) {
        if (part.empty()) continue;
        cur += part + "/";
        if (mkdir(cur.c_str(), 0755) != 0 && errno != EEXIST) return false;
    }
    return true;
}

// write_snapshot_dat (output.hpp:76-102); returns the path ("" on failure)
std::string write(const std::string& dir, int dim, const int* dims, double h, const double* origin,
                  const double* u, const double* damage, int64_t step, double t) {
    if (!make_dirs(dir)) return "";
    char tag[16];
    snprintf(tag, sizeof tag, "%07lld", (long long)step);
    const std::string path = dir + "/snap_" + tag + ".dat";
    FILE* fp = fopen(path.c_str(), "w");
    if (!fp) return "";
    std::string head = "# pdfast snapshot\n# dim " + std::to_string(dim) + "\n# dims";
    for (int d = 0; d < dim; ++d) head += " " + std::to_string(dims[d]);
    head += "\n# h " + g17(h) + "\n# origin";
    for (int d = 0; d < dim; ++d) head += " " + g17(origin[d]);
    head += "\n# step " + std::to_string((long long)step) + "\n# t " + g17(t) + "\n";
    head += std::string("# columns node u_x u_y ") + (dim == 3 ? "u_z damage" : "damage") + "\n";
    fputs(head.c_str(), fp);
    int64_t n = 1;
    for (int d = 0; d < dim; ++d) n *= dims[d];
    std::string row;
    for (int64_t p = 0; p < n; ++p) {
        row = std::to_string((long long)(p + 1));
        for (int d = 0; d < dim; ++d) row += " " + g17(u[(int64_t)d * n + p]);
        row += " " + g17(damage ? damage[p] : 0.0) + "\n";
        fputs(row.c_str(), fp);
    }
    const bool ok = ferror(fp) == 0;
    fclose(fp);
    return ok ? path : "";
}

// read_snapshot_dat (output.hpp:116-154).  With u == nullptr only the header
// fields are filled (call once for dims, then again with buffers).
bool read(const std::string& path, int dim, int* dims, double* h, double* origin, int64_t* step, double* t,
          double* u, double* damage, std::string& err) {
    std::ifstream in(path);
    if (!in) {
        err = "cannot open snapshot file: " + path;
        return false;
    }
    std::string line;
    int64_t n = 0;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        if (line[0] == '#') {
            std::istringstream is(line.substr(1));
            std::string key;
            is >> key;
            if (key == "dims") {
                n = 1;
                for (int d = 0; d < dim; ++d) {
                    is >> dims[d];
                    n *= dims[d];
                }
                if (u)
                    for (int64_t i = 0; i < (int64_t)dim * n; ++i) u[i] = 0.0;
                if (damage)
                    for (int64_t i = 0; i < n; ++i) damage[i] = 0.0;
            } else if (key == "h") {
                is >> *h;
            } else if (key == "origin") {
                for (int d = 0; d < dim; ++d) is >> origin[d];
            } else if (key == "step") {
                long long s = 0;
                is >> s;
                *step = s;
            } else if (key == "t") {
                is >> *t;
            }
            continue;
        }
        if (!u) break;  // header only
        std::istringstream is(line);
        long long id = 0;
        is >> id;
        if (id < 1 || id > n) {
            err = "snapshot row id out of range in " + path;
            return false;
        }
        for (int d = 0; d < dim; ++d) is >> u[(int64_t)d * n + id - 1];
        double dmg = 0.0;
        is >> dmg;
        if (damage) damage[id - 1] = dmg;
        if (!is) {
            err = "malformed snapshot row in " + path;
            return false;
        }
    }
    return true;
}

// ---- MonitorWriter (output.hpp:45-72): tab-separated rows "step t node u..."
// with node ids from 1 and %.17g values, one header line, flushed per append.
// nearest_node (output.hpp:33-41): floor((x - origin) / h) clamped per axis.
int64_t nearest_node(int dim, const int* dims, double h, const double* origin, const double* x) {
    int64_t p = 0, stride = 1;
    for (int d = 0; d < dim; ++d) {
        int i = (int)std::floor((x[d] - origin[d]) / h);
        i = std::min(std::max(i, 0), dims[d] - 1);
        p += stride * i;
        stride *= dims[d];
    }
    return p;
}

struct Monitor {
    FILE* fp = nullptr;
    int dim = 0;
    std::vector<int64_t> nodes;
};

Monitor* monitor_open(const char* path, int dim, const int* dims, double h, const double* origin, const double* pts,
                      int npts, std::string& err) {
    Monitor* m = new Monitor();
    m->dim = dim;
    for (int k = 0; k < npts; ++k) m->nodes.push_back(nearest_node(dim, dims, h, origin, pts + (size_t)k * dim));
    if (path && path[0]) {
        m->fp = fopen(path, "w");
        if (!m->fp) {
            err = std::string("cannot open monitor file: ") + path;
            delete m;
            return nullptr;
        }
        fputs(dim == 3 ? "# step\tt\tnode\tu_x\tu_y\tu_z\n" : "# step\tt\tnode\tu_x\tu_y\n", m->fp);
    }
    return m;
}

// vals: this row's monitored values [node][component]
void monitor_append(Monitor* m, int64_t step, double t, const double* vals) {
    if (!m->fp) return;
    std::string out;
    const std::string ts = g17(t);
    for (size_t k = 0; k < m->nodes.size(); ++k) {
        out += std::to_string((long long)step) + "\t" + ts + "\t" + std::to_string((long long)(m->nodes[k] + 1));
        for (int d = 0; d < m->dim; ++d) out += "\t" + g17(vals[k * m->dim + d]);
        out += "\n";
    }
    fputs(out.c_str(), m->fp);
    fflush(m->fp);
}

void monitor_close(Monitor* m) {
    if (m->fp) fclose(m->fp);
    delete m;
}

}  // namespace snapshot
}  // namespace pdgpu
