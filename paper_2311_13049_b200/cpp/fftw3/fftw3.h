/*
 * fftw3.h — the FFTW3 API subset the reference calls (grid.cpp:25-31, 85-89, 134-137;
 * flap.cpp:270-279), served by the B200 backend in the drop-in build
 * (paper_2311_13049_b200/cpp/fftw_gpu.cpp: every execute is an unnormalised DFT on the device,
 * fw_grid_dft).  Declarations follow FFTW's documented interface: fftw_complex = double[2],
 * sign FFTW_FORWARD = -1 (e^{-2 pi i jk/n}), FFTW_BACKWARD = +1, row-major multi-dimensional
 * arrays; planner flags are accepted and ignored (there is one device algorithm).
 */
#ifndef FW_DROPIN_FFTW3_H
#define FW_DROPIN_FFTW3_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fw_dropin_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
