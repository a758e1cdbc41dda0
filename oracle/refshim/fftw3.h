// fftw3.h stand-in -- TEST INFRASTRUCTURE ONLY (oracle/_ref build of the reference).
//
// FFTW is not installed in this image.  The reference touches it in one place
// (/root/reference/proj/src/nufft.cpp:17-55: fftw_plan_dft with
// FFTW_ESTIMATE | FFTW_UNALIGNED, fftw_execute_dft, fftw_destroy_plan), so this
// header declares exactly that surface and fftw3_standin.cpp implements it
// with a table-twiddle mixed-radix Cooley-Tukey (unnormalised, sign as FFTW
// defines it: FFTW_FORWARD = exp(-2 pi i jk/n)).  Written from scratch.
#pragma once

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_standin_plan* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
