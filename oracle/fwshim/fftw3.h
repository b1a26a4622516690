/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product path.
 *
 * Minimal FFTW3-compatible declarations so the reference sources under
 * /root/reference/proj/src compile unmodified.  FFTW3 itself is a third-party
 * dependency of the reference (proj/CMakeLists.txt:13-14, version unpinned) that
 * is absent from this image; oracle/fwshim/fwshim.c restates the transform it
 * computes (the unnormalized multi-dimensional DFT, FFTW's documented
 * definition: sign -1 = forward e^{-2 pi i jk/n}, +1 = backward).
 *
 * Only the subset the reference uses is declared (call sites: grid.cpp:25-31,
 * 85-89, 134-137; flap.cpp:270-279).
 */
#ifndef FWSHIM_FFTW3_H
#define FWSHIM_FFTW3_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fwshim_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out,
                        int sign, unsigned flags);
fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

/* shim-only diagnostics (not FFTW API): how many executes took the real-input /
 * Hermitian-input fast paths vs the general complex path. */
void fwshim_stats(long* real_fwd, long* herm_bwd, long* general);

#ifdef __cplusplus
}
#endif

#endif
