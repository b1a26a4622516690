/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the checker.
 *
 * Plain-C restatement of the reference's hot path (fracwave, /root/reference/proj):
 * the M-term matrix-free apply of (-Delta)^{s(x)}, the viscoacoustic seismic
 * stepper and the TSFP2 time-splitting step.  Expansion tables are streamed
 * term by term with the reference's own recurrences (bit-identical to
 * build_expansion, flap.cpp:96-135) so memory is O(N) instead of O(MN).
 * FFTs use the canonical fp64 FFT in fwshim/fwcanon.c (the FFTW3 restatement).
 *
 * Parity pin: tests/test_oracle_pins.py checks every function here bit-for-bit
 * against the reference itself (oracle/_ref, the unmodified reference sources
 * built against fwshim), and checks fwcanon against numpy's pocketfft and the
 * reference's FFT known-answer tests.
 */
#ifndef FW_ORACLE_H
#define FW_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes (same values as include/fw_capi.h) */
enum {
  FWO_OK = 0,
  FWO_E_ARG = 1,
  FWO_E_GRID_MISMATCH = 2,
  FWO_E_NEGATIVE_M = 3,
  FWO_E_ORDER_RANGE = 4,
  FWO_E_DEVIATION = 5,
  FWO_E_GAMMA_RANGE = 6,
  FWO_E_BLOWUP = 7,
  FWO_E_ODD_SIZE = 8,
  FWO_E_EMPTY_INTERVAL = 9,
  FWO_E_DIM_RANGE = 10,
  FWO_E_UNSUPPORTED = 13
};

const char* fwo_last_error(void);

/* |mu_k|^2 over the full grid, row-major (grid.cpp:60-80) */
int fwo_mu2(int d, const int* J, const double* lo, const double* hi, double* mu2);

/* OrderField statistics (orderfield.cpp:10-36, is_constant orderfield.cpp:55-57) */
int fwo_order_stats(const double* s, size_t N, const double* s0_override, double* s0,
                    double* smin, double* smax, int* constant_order);

/* apply_expansion (flap.cpp:38-92) with build_expansion tables (flap.cpp:96-135)
 * regenerated term by term.  m_first = 0: apply_matrix_free; 1: the m >= 1
 * perturbation (apply_perturbation, flap.cpp:161-168). */
int fwo_apply(int d, const int* J, const double* lo, const double* hi, const double* s,
              const double* s0_override, int M, int m_first, const double* u, double* out,
              double* imag_residue);

/* apply_constant_order (flap.cpp:137-149) */
int fwo_constant_order(int d, const int* J, const double* lo, const double* hi,
                       const double* u, double s, double* out);

/* derive_medium coefficient fields (seismic.cpp:11-44) */
int fwo_medium(int d, const int* J, const double* gamma, const double* c0, double omega0,
               double* c, double* eta, double* tau_coef);

/* SeismicStepper construction + nsteps step() (seismic.cpp:85-133).  Returns
 * FWO_E_BLOWUP with *n_out = offending step on blow-up. */
int fwo_seismic(int d, const int* J, const double* lo, const double* hi, const double* gamma,
                const double* c0, double omega0, int M, const double* phi, const double* psi,
                double tau, double blowup_factor, int nsteps, double* cur_out, double* prev_out,
                double* atten_prev_out, long* n_out);

/* Stepper TSFP2 (stepping.cpp:106-131, 266-304), f = none (0) or cubic (1) */
int fwo_tsfp2(int d, const int* J, const double* lo, const double* hi, const double* s, int M,
              double kappa, int cubic, const double* phi, const double* psi, double tau,
              int nsteps, double* u_out, double* v_out);

/* canonical half-spectrum transforms (for tests): forward real -> N_h complex
 * (interleaved), and backward Hermitian half -> real */
int fwo_rfftn(int d, const int* J, const double* x, double* H);
int fwo_irfftn(int d, const int* J, const double* H, double* x);

#ifdef __cplusplus
}
#endif

#endif
