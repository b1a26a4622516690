// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// extern "C" entry points into the *reference itself* (the unmodified sources
// under /root/reference/proj/src, compiled by oracle/Makefile against the FFTW
// shim) so pytest can run the reference on arbitrary seeded inputs through
// ctypes.  This TU #includes proj/src/seismic.cpp so the reference's
// anonymous-namespace derive_medium (seismic.cpp:11-44) can be reached with
// numeric gamma/c0 fields (the reference's Expr language has no atan/sigmoid,
// expr.cpp:20-29); seismic.cpp is therefore not linked separately.
#include "src/seismic.cpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <typeinfo>
#include <vector>

#include "fracwave/errors.hpp"
#include "fracwave/flap.hpp"
#include "fracwave/grid.hpp"
#include "fracwave/harness.hpp"
#include "fracwave/orderfield.hpp"
#include "fracwave/seismic.hpp"
#include "fracwave/stepping.hpp"

using namespace fwave;

namespace {

thread_local std::string g_err;

// error codes shared with include/fw_capi.h
int code_of(const std::exception& e) {
  if (dynamic_cast<const GridMismatch*>(&e)) return 2;
  if (dynamic_cast<const NegativeM*>(&e)) return 3;
  if (dynamic_cast<const OrderOutOfRange*>(&e)) return 4;
  if (dynamic_cast<const DeviationTooLarge*>(&e)) return 5;
  if (dynamic_cast<const GammaOutOfRange*>(&e)) return 6;
  if (dynamic_cast<const BlowupDetected*>(&e)) return 7;
  if (dynamic_cast<const OddSize*>(&e)) return 8;
  if (dynamic_cast<const EmptyInterval*>(&e)) return 9;
  if (dynamic_cast<const DimOutOfRange*>(&e)) return 10;
  if (dynamic_cast<const PicardDiverged*>(&e)) return 15;
  if (dynamic_cast<const CgStagnated*>(&e)) return 16;
  return 99;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

Grid make_grid(int d, const int* J, const double* lo, const double* hi) {
  std::vector<std::pair<double, double>> b;
  std::vector<int> s;
  for (int m = 0; m < d; ++m) {
    b.emplace_back(lo[m], hi[m]);
    s.push_back(J[m]);
  }
  return Grid(b, s);
}

std::vector<double> vec(const double* p, std::size_t n) { return std::vector<double>(p, p + n); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// apply_matrix_free / _serial / apply_perturbation (flap.cpp:151-168)
// mode: 0 = apply_matrix_free, 1 = apply_matrix_free_serial, 2 = apply_perturbation
int ref_apply(int d, const int* J, const double* lo, const double* hi, const double* s,
              const double* s0_override, int M, int mode, const double* u, double* out,
              double* residue, double* s0_out, int* constant_out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    OrderField of = s0_override ? OrderField(g, vec(s, N), *s0_override) : OrderField(g, vec(s, N));
    ExpansionOperator op = build_expansion(of, M);
    Field uf(g, vec(u, N));
    Field r = mode == 0   ? apply_matrix_free(op, uf, residue)
              : mode == 1 ? apply_matrix_free_serial(op, uf, residue)
                          : apply_perturbation(op, uf, residue);
    std::memcpy(out, r.values().data(), N * sizeof(double));
    if (s0_out) *s0_out = op.order.s0();
    if (constant_out) *constant_out = op.constant_order ? 1 : 0;
  });
}

// build_expansion tables (flap.cpp:96-135): base (N), log_weights (M*N), dev (M*N)
int ref_tables(int d, const int* J, const double* lo, const double* hi, const double* s, int M,
               double* mu2, double* base, double* lw, double* dev, double* s0_out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    ExpansionOperator op = build_expansion(OrderField(g, vec(s, N)), M);
    if (mu2) std::memcpy(mu2, g.mu_abs2().data(), N * sizeof(double));
    if (base) std::memcpy(base, op.base_symbol.data(), N * sizeof(double));
    for (int m = 0; m < M; ++m) {
      if (lw) std::memcpy(lw + m * N, op.log_weights[m].data(), N * sizeof(double));
      if (dev) std::memcpy(dev + m * N, op.deviation_powers[m].data(), N * sizeof(double));
    }
    if (s0_out) *s0_out = op.order.s0();
  });
}

// apply_constant_order (flap.cpp:137-149)
int ref_constant_order(int d, const int* J, const double* lo, const double* hi, const double* u,
                       double s, double* out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    Field r = apply_constant_order(Field(g, vec(u, g.total())), s);
    std::memcpy(out, r.values().data(), g.total() * sizeof(double));
  });
}

// Grid::forward / Grid::inverse (grid.cpp:171-197) on a real field
int ref_forward(int d, const int* J, const double* lo, const double* hi, const double* u,
                double* spec_interleaved) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    Spectrum sp = forward(Field(g, vec(u, g.total())));
    std::memcpy(spec_interleaved, sp.coeffs().data(), g.total() * 2 * sizeof(double));
  });
}

// assemble_dense + apply_dense (flap.cpp:170-243): entries (N x N, nullable) and A u
int ref_dense(int d, const int* J, const double* lo, const double* hi, const double* s, const double* u,
              double* entries, double* out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    DenseOperator op = assemble_dense(OrderField(g, vec(s, N)));
    if (entries) std::memcpy(entries, op.entries.data(), N * N * sizeof(double));
    Field o = apply_dense(op, Field(g, vec(u, N)));
    std::memcpy(out, o.values().data(), N * sizeof(double));
  });
}

// apply_toeplitz (flap.cpp:245-285)
int ref_toeplitz(int d, const int* J, const double* lo, const double* hi, const double* s, const double* u,
                 double* out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    Field o = apply_toeplitz(OrderField(g, vec(s, N)), Field(g, vec(u, N)));
    std::memcpy(out, o.values().data(), N * sizeof(double));
  });
}

// truncation_indicator (flap.cpp:287-294)
int ref_truncation_indicator(int M, double mu_abs, double s0, double* out) {
  return guard([&] { *out = truncation_indicator(M, mu_abs, s0); });
}

// ricker_initial (seismic.cpp:70-83)
int ref_ricker(int d, const int* J, const double* lo, const double* hi, double nu0, const double* xc,
               double* out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    Field f = ricker_initial(nu0, std::vector<double>(xc, xc + d), g);
    std::memcpy(out, f.values().data(), g.total() * sizeof(double));
  });
}

// derive_medium (seismic.cpp:11-44)
int ref_medium(int d, const int* J, const double* lo, const double* hi, const double* gamma,
               const double* c0, double omega0, int M, double* c, double* eta, double* tau_coef,
               double* s0_disp, double* s0_atten) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    SeismicMedium m = derive_medium(g, vec(gamma, N), vec(c0, N), omega0, M);
    std::memcpy(c, m.c.values().data(), N * sizeof(double));
    std::memcpy(eta, m.eta.values().data(), N * sizeof(double));
    std::memcpy(tau_coef, m.tau_coef.values().data(), N * sizeof(double));
    *s0_disp = m.disp_op.order.s0();
    *s0_atten = m.atten_op.order.s0();
  });
}

// SeismicStepper (seismic.cpp:85-142): construct, then `nsteps` step() calls.
// cur_out gets current() after the last step; *n_out = n().  On BlowupDetected
// the code is 7 and *n_out is the step count reached.
int ref_seismic(int d, const int* J, const double* lo, const double* hi, const double* gamma,
                const double* c0, double omega0, int M, const double* phi, const double* psi,
                double tau, double blowup_factor, int nsteps, double* cur_out, long* n_out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    SeismicMedium m = derive_medium(g, vec(gamma, N), vec(c0, N), omega0, M);
    SeismicStepper st(m, Field(g, vec(phi, N)), Field(g, vec(psi, N)), tau, blowup_factor);
    try {
      for (int i = 0; i < nsteps; ++i) st.step();
    } catch (...) {
      *n_out = st.n();
      std::memcpy(cur_out, st.current().values().data(), N * sizeof(double));
      throw;
    }
    *n_out = st.n();
    std::memcpy(cur_out, st.current().values().data(), N * sizeof(double));
  });
}

// Stepper TSFP2 (stepping.cpp:119-138, 266-304); f = none (0) or cubic (1)
int ref_tsfp2(int d, const int* J, const double* lo, const double* hi, const double* s, int M,
              double kappa, int cubic, const double* phi, const double* psi, double tau,
              int nsteps, double* u_out, double* v_out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    WaveProblem p;
    p.grid = g;
    p.order = OrderField(g, vec(s, N));
    p.kappa = kappa;
    p.f = cubic ? Nonlinearity::cubic() : Nonlinearity::none();
    p.phi = Field(g, vec(phi, N));
    p.psi = Field(g, vec(psi, N));
    p.M = M;
    StepperConfig cfg;
    cfg.method = Method::TSFP2;
    cfg.tau = tau;
    Stepper st(p, cfg);
    for (int i = 0; i < nsteps; ++i) st.step();
    std::memcpy(u_out, st.current().values().data(), N * sizeof(double));
    std::memcpy(v_out, st.velocity().values().data(), N * sizeof(double));
  });
}

// LFFP (stepping.cpp:170-181) for the classical-limit comparison (test_seismic.cpp:67-95)
int ref_lffp(int d, const int* J, const double* lo, const double* hi, const double* s, int M,
             double kappa, const double* phi, const double* psi, double tau, int nsteps,
             double* u_out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    WaveProblem p;
    p.grid = g;
    p.order = OrderField(g, vec(s, N));
    p.kappa = kappa;
    p.f = Nonlinearity::none();
    p.phi = Field(g, vec(phi, N));
    p.psi = Field(g, vec(psi, N));
    p.M = M;
    StepperConfig cfg;
    cfg.method = Method::LFFP;
    cfg.tau = tau;
    Stepper st(p, cfg);
    for (int i = 0; i < nsteps; ++i) st.step();
    std::memcpy(u_out, st.current().values().data(), N * sizeof(double));
  });
}

// Stepper with Method::LFFP (0) / CNFP (1) / TSFP2 (2) (stepping.cpp:119-138, 170-304), f none (0) or
// cubic (1), the StepperConfig fields as given.  After `nsteps` step() calls (or the one
// that threw) cur_out = current(), *n_out = n(), *picard_out = total_picard_iterations().
int ref_wave(int method, int d, const int* J, const double* lo, const double* hi, const double* s, int M,
             double kappa, int cubic, const double* phi, const double* psi, double tau, double picard_tol,
             int picard_max_iters, double inner_cg_tol, int cg_max_iters, double blowup_factor, int nsteps,
             double* cur_out, long* n_out, long* picard_out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    WaveProblem p;
    p.grid = g;
    p.order = OrderField(g, vec(s, N));
    p.kappa = kappa;
    p.f = cubic ? Nonlinearity::cubic() : Nonlinearity::none();
    p.phi = Field(g, vec(phi, N));
    p.psi = Field(g, vec(psi, N));
    p.M = M;
    StepperConfig cfg;
    cfg.method = method == 0 ? Method::LFFP : (method == 1 ? Method::CNFP : Method::TSFP2);
    cfg.tau = tau;
    cfg.picard_tol = picard_tol;
    cfg.picard_max_iters = picard_max_iters;
    cfg.inner_cg_tol = inner_cg_tol;
    cfg.cg_max_iters = cg_max_iters;
    cfg.blowup_factor = blowup_factor;
    Stepper st(p, cfg);
    auto out = [&] {
      std::memcpy(cur_out, st.current().values().data(), N * sizeof(double));
      *n_out = st.n();
      *picard_out = st.total_picard_iterations();
    };
    try {
      for (int i = 0; i < nsteps; ++i) st.step();
    } catch (...) {
      out();
      throw;
    }
    out();
  });
}

// CPU-baseline timers, following the reference's own drivers: best-of-`repeats`
// steady_clock around apply_matrix_free (bench_kernels.cpp:22-31,
// harness.cpp:407-415) and the mean per step over SeismicStepper::step() after
// construction (construction = 3 applies, untimed).
int ref_time_apply(int d, const int* J, const double* lo, const double* hi, const double* s, int M,
                   const double* u, int repeats, double* best_seconds) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    ExpansionOperator op = build_expansion(OrderField(g, vec(s, N)), M);
    Field uf(g, vec(u, N));
    double best = 1e300;
    for (int r = 0; r < repeats; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      Field out = apply_matrix_free(op, uf);
      const auto t1 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    }
    *best_seconds = best;
  });
}

int ref_time_seismic(int d, const int* J, const double* lo, const double* hi, const double* gamma,
                     const double* c0, double omega0, int M, const double* phi, const double* psi,
                     double tau, int warmup, int steps, double* per_step_seconds, double* cur_out) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    const std::size_t N = g.total();
    SeismicMedium m = derive_medium(g, vec(gamma, N), vec(c0, N), omega0, M);
    SeismicStepper st(m, Field(g, vec(phi, N)), Field(g, vec(psi, N)), tau);
    for (int i = 0; i < warmup; ++i) st.step();
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < steps; ++i) st.step();
    const auto t1 = std::chrono::steady_clock::now();
    *per_step_seconds = std::chrono::duration<double>(t1 - t0).count() / std::max(steps, 1);
    if (cur_out) std::memcpy(cur_out, st.current().values().data(), N * sizeof(double));
  });
}

// write_snapshot (harness.cpp:541-557): FWS1 files written by the reference itself
int ref_write_snapshot(int d, const int* J, const double* lo, const double* hi, const double* values,
                       double time, const char* path) {
  return guard([&] {
    Grid g = make_grid(d, J, lo, hi);
    write_snapshot(Field(g, vec(values, g.total())), time, path);
  });
}

}  // extern "C"
