/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.  Canonical fp64 FFT used by the FFTW-API
 * shim (fwshim.c) and by the C restatement (oracle/fw_oracle.c).
 *
 * This is an independent CPU implementation of the transform definition that
 * DESIGN.md §3 ("canonical FFT") pins down: power-of-two Stockham passes with
 * radices 16/8/4/2, fixed in-register DFT kernels, host-computed twiddle tables,
 * explicit fma() in complex products and no other contraction
 * (-ffp-contract=off).  Real-input / Hermitian-input transforms use the
 * half-length packing formulation (R2C / C2R).  The CUDA kernels implement the
 * same definition independently, so identical inputs give identical bits; the
 * canonical FFT is itself checked against numpy's pocketfft and against the
 * reference's own FFT tests (test_grid.cpp:33-98) in tests/.
 */
#ifndef FWCANON_H
#define FWCANON_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double re, im;
} fwc_cd;

/* cos(2*pi*t/n), sin(2*pi*t/n) with quadrant/octant reduction (exact at
 * multiples of pi/2). */
void fwc_twiddle(long t, long n, double* c, double* s);

typedef struct {
  int n;          /* power of two >= 1 */
  int npass;
  int radix[16];
  fwc_cd* tw;     /* n entries: (cos, sin)(2 pi t / n) */
} fwc_plan1d;

int fwc_is_pow2(long n);
void fwc_plan1d_init(fwc_plan1d* p, int n);
void fwc_plan1d_free(fwc_plan1d* p);
/* canonical radix sequence for n */
int fwc_radices(int n, int* radix);

/* In-place C2C of length p->n on x, scratch must hold n entries.  dir = -1
 * forward (e^{-i}), +1 backward, unnormalized. */
void fwc_c2c(const fwc_plan1d* p, fwc_cd* x, fwc_cd* scratch, int dir);

/* R2C of n = 2*half->n reals -> n/2+1 bins.  twn: n-entry table (fwc_plan1d
 * of length n supplies it).  scratch: n/2 entries. */
void fwc_r2c(const fwc_plan1d* half, const fwc_cd* twn, const double* x, fwc_cd* X,
             fwc_cd* scratch);
/* C2R (unnormalized backward) of n/2+1 Hermitian bins -> n reals; only the
 * real parts of X[0] and X[n/2] are used.  scratch: n/2 entries. */
void fwc_c2r(const fwc_plan1d* half, const fwc_cd* twn, const fwc_cd* X, double* x,
             fwc_cd* scratch);

/* Multi-dimensional real transforms on row-major grids (axis 0 slowest), the
 * half spectrum stored as [n0]..[n_{d-2}][n_{d-1}/2+1].
 * forward: R2C along the last axis, then C2C along axes d-2 .. 0.
 * backward: C2C along axes 0 .. d-2, then C2R along the last axis.
 * All dims must be powers of two, last >= 4. */
typedef struct {
  int d;
  int n[3];
  fwc_plan1d ax[3];   /* per-axis C2C plans (the last axis' table feeds R2C/C2R) */
  fwc_plan1d half;    /* length n[d-1]/2 */
} fwc_realnd;

int fwc_realnd_init(fwc_realnd* p, int d, const int* n);
void fwc_realnd_free(fwc_realnd* p);
size_t fwc_realnd_nhalf(const fwc_realnd* p);
void fwc_realnd_forward(const fwc_realnd* p, const double* x, fwc_cd* H);
/* H is destroyed.  If imag0/imagh are non-null they receive, per row, the
 * imaginary parts of the p = 0 and p = n/2 bins after the axis passes (the
 * anti-Hermitian remainder; see fwshim.c). */
void fwc_realnd_backward(const fwc_realnd* p, fwc_cd* H, double* x, double* imag0,
                         double* imagh);

#ifdef __cplusplus
}
#endif

#endif
