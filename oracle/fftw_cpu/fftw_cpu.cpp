// fftw_cpu.cpp -- CPU implementation of the fftw3.h subset (TEST
// INFRASTRUCTURE ONLY; see fftw3.h).  Mixed-radix Stockham autosort with
// per-stage twiddle tables; multi-dimensional transforms are done axis by
// axis, strided axes in cache-friendly blocks of columns.  Plans are
// immutable after creation; execution uses thread-local scratch, so distinct
// plans/buffers may execute concurrently (the reference's contract,
// convolution.hpp:53-54).
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <complex>
#include <vector>

namespace {

using cd = std::complex<double>;

struct Stage {
    int R;                 // radix
    int Ns;                // product of previous radices
    std::vector<cd> tw;    // Ns x R twiddles exp(sign 2 pi i k r / (Ns R))
    std::vector<cd> root;  // R x R DFT matrix (generic radices)
};

struct Plan1D {
    int n = 1;
    int sign = -1;
    std::vector<Stage> stages;
};

void make_plan1d(Plan1D& p, int n, int sign) {
    p.n = n;
    p.sign = sign;
    p.stages.clear();
    int rem = n, Ns = 1;
    while (rem > 1) {
        int R;
        if (rem % 4 == 0) R = 4;
        else if (rem % 2 == 0) R = 2;
        else if (rem % 3 == 0) R = 3;
        else if (rem % 5 == 0) R = 5;
        else if (rem % 7 == 0) R = 7;
        else {
            R = rem;
            for (int f = 11; f * f <= rem; f += 2)
                if (rem % f == 0) { R = f; break; }
        }
        Stage s;
        s.R = R;
        s.Ns = Ns;
        s.tw.resize((size_t)Ns * R);
        for (int k = 0; k < Ns; ++k)
            for (int r = 0; r < R; ++r) {
                const long double a = (long double)sign * 2.0L * 3.141592653589793238462643383279502884L *
                                      (long double)k * r / ((long double)Ns * R);
                s.tw[(size_t)k * R + r] = cd((double)cosl(a), (double)sinl(a));
            }
        if (R != 2 && R != 4) {
            s.root.resize((size_t)R * R);
            for (int a = 0; a < R; ++a)
                for (int b = 0; b < R; ++b) {
                    const long double ang = (long double)sign * 2.0L * 3.141592653589793238462643383279502884L *
                                            (long double)((a * b) % R) / R;
                    s.root[(size_t)a * R + b] = cd((double)cosl(ang), (double)sinl(ang));
                }
        }
        p.stages.push_back(std::move(s));
        Ns *= R;
        rem /= R;
    }
}

// transform one contiguous vector x (length n) using scratch y; result in x
void exec1d(const Plan1D& p, cd* x, cd* y) {
    const int n = p.n;
    cd* in = x;
    cd* out = y;
    cd v[64];
    for (const Stage& s : p.stages) {
        const int R = s.R, Ns = s.Ns, L = n / R;
        for (int j = 0; j < L; ++j) {
            const int k = j % Ns;
            const cd* tw = &s.tw[(size_t)k * R];
            if (R <= 64) {
                for (int r = 0; r < R; ++r) v[r] = in[j + r * L] * tw[r];
            }
            const int base = (j / Ns) * Ns * R + k;
            if (R == 2) {
                out[base] = v[0] + v[1];
                out[base + Ns] = v[0] - v[1];
            } else if (R == 4) {
                const cd a = v[0] + v[2], c = v[0] - v[2];
                const cd b = v[1] + v[3];
                const cd d0 = v[1] - v[3];
                const cd d = p.sign < 0 ? cd(d0.imag(), -d0.real()) : cd(-d0.imag(), d0.real());
                out[base] = a + b;
                out[base + Ns] = c + d;
                out[base + 2 * Ns] = a - b;
                out[base + 3 * Ns] = c - d;
            } else if (R <= 64) {
                for (int a = 0; a < R; ++a) {
                    cd acc = 0.0;
                    for (int b = 0; b < R; ++b) acc += s.root[(size_t)a * R + b] * v[b];
                    out[base + a * Ns] = acc;
                }
            } else {  // large prime radix: direct, reading straight from `in`
                for (int a = 0; a < R; ++a) {
                    cd acc = 0.0;
                    for (int b = 0; b < R; ++b) acc += s.root[(size_t)a * R + b] * (in[j + b * L] * tw[b]);
                    out[base + a * Ns] = acc;
                }
            }
        }
        cd* t = in;
        in = out;
        out = t;
    }
    if (in != x) memcpy(x, in, sizeof(cd) * (size_t)n);
}

}  // namespace

struct fftw_plan_s {
    int rank;
    std::vector<int> n;
    int sign;
    std::vector<Plan1D> axes;  // axes[d] plans dimension n[d] (n[0] slowest)
    fftw_complex* in;
    fftw_complex* out;
};

extern "C" {

fftw_complex* fftw_alloc_complex(size_t n) {
    void* p = nullptr;
    if (posix_memalign(&p, 64, sizeof(fftw_complex) * (n ? n : 1)) != 0) return nullptr;
    return (fftw_complex*)p;
}

void fftw_free(void* p) { free(p); }

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags) {
    (void)flags;
    fftw_plan p = new fftw_plan_s;
    p->rank = rank;
    p->n.assign(n, n + rank);
    p->sign = sign;
    p->axes.resize(rank);
    for (int d = 0; d < rank; ++d) make_plan1d(p->axes[d], n[d], sign);
    p->in = in;
    p->out = out;
    return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    size_t total = 1;
    for (int d = 0; d < p->rank; ++d) total *= (size_t)p->n[d];
    if (in != out) memcpy(out, in, sizeof(fftw_complex) * total);
    cd* data = reinterpret_cast<cd*>(out);
    thread_local std::vector<cd> scratch, block;
    for (int d = p->rank - 1; d >= 0; --d) {
        const int len = p->n[d];
        size_t stride = 1;
        for (int e = d + 1; e < p->rank; ++e) stride *= (size_t)p->n[e];
        const size_t outer = total / (stride * len);
        if (scratch.size() < (size_t)len) scratch.resize(len);
        if (stride == 1) {
            for (size_t o = 0; o < outer; ++o) exec1d(p->axes[d], data + o * len, scratch.data());
        } else {
            const size_t B = 16;
            if (block.size() < B * len) block.resize(B * len);
            for (size_t o = 0; o < outer; ++o) {
                cd* base = data + o * stride * len;
                for (size_t c0 = 0; c0 < stride; c0 += B) {
                    const size_t nb = stride - c0 < B ? stride - c0 : B;
                    for (int i = 0; i < len; ++i)
                        for (size_t c = 0; c < nb; ++c) block[c * len + i] = base[(size_t)i * stride + c0 + c];
                    for (size_t c = 0; c < nb; ++c) exec1d(p->axes[d], block.data() + c * len, scratch.data());
                    for (int i = 0; i < len; ++i)
                        for (size_t c = 0; c < nb; ++c) base[(size_t)i * stride + c0 + c] = block[c * len + i];
                }
            }
        }
    }
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
