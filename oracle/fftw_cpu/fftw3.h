/*
 * fftw3.h -- minimal CPU provider of the FFTW3 API subset the reference uses.
 *
 * TEST INFRASTRUCTURE ONLY (oracle).  FFTW3 itself is not installed in this
 * image and is not vendored by the reference (proj/CMakeLists.txt:12-13,
 * unpinned `find_library(fftw3)`); this header + fftw_cpu.cpp implement
 * exactly the calls the reference makes (convolution.hpp:27,33,44,69-70,
 * 77-78,114,127,159) with FFTW's published semantics: unnormalised
 * complex DFTs, FFTW_FORWARD = exp(-2*pi*i*j*k/n), row-major multi-dim
 * arrays with the slowest axis first, new-array execute on any buffer of
 * the planned shape.  Mixed radix (2,3,4,5,7, generic odd primes).
 */
#ifndef ORACLE_FFTW3_H
#define ORACLE_FFTW3_H
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_MEASURE (0U)

fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
#endif
