/*
 * oracle/fftw3.h -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * FFTW3 is not installed in this image; the reference's
 * frontend.cpp / signals.cpp include <fftw3.h>.  This header declares exactly the
 * FFTW surface those two files use (grep-complete: 6 functions, 2 types,
 * 3 constants -- SURVEY.md §8(c)), so the UNMODIFIED reference sources compile
 * against oracle/fftw_shim.c.  Call sites: proj/src/frontend.cpp:54-60,71-80,139
 * and proj/src/signals.cpp:83-95.
 */
#ifndef ORACLE_FFTW3_SHIM_H
#define ORACLE_FFTW3_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct oracle_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);
fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
