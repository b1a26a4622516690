// stepper_gpu.hpp — fwave::gpu::Stepper: the reference's Stepper public API
// (proj/include/fracwave/stepping.hpp:72-94) with the state resident on the B200.
// LFFP / CNFP run on fw_wave_* (levels, Picard iterates and CG vectors in HBM, the
// operator served by the hot-path apply), TSFP2 on fw_tsfp2_*.
//
// Same constructor arguments (WaveProblem, StepperConfig) and members; current()
// and velocity() copy back to the host.  Not offered (out of scope):
// cfg.use_dense and an expression-valued Nonlinearity (Kind::Custom) -> fwave::Error.
#pragma once

#include <cmath>
#include <string>

#include "fracwave/errors.hpp"
#include "fracwave/grid.hpp"
#include "fracwave/stepping.hpp"
#include "fw_capi.h"

namespace fwave {
namespace gpu {

class Stepper {
 public:
  Stepper(const WaveProblem& p, const StepperConfig& cfg, int device = 0)
      : method_(cfg.method), tau_(cfg.tau), cur_(p.grid, 0.0), vel_(p.grid, 0.0) {
    if (cfg.use_dense) throw Error("B200 backend: the dense operator is not offered (use_dense)");
    if (p.f.kind == Nonlinearity::Kind::Custom)
      throw Error("B200 backend: expression-valued nonlinearities are not offered (none / cubic)");
    check(fw_ctx_create(device, &ctx_));
    const Grid& g = p.grid;
    int J[3] = {1, 1, 1};
    double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
    for (int m = 0; m < g.dim(); ++m) {
      J[m] = g.size(m);
      lo[m] = g.lo(m);
      hi[m] = g.hi(m);
    }
    const int f = p.f.kind == Nonlinearity::Kind::Cubic ? 1 : 0;
    if (method_ == Method::TSFP2) {
      check(fw_tsfp2_create(ctx_, g.dim(), J, lo, hi, p.order.values().data(), p.M, p.kappa, f,
                            p.phi.values().data(), p.psi.values().data(), cfg.tau, cfg.blowup_factor, &ts_));
    } else {
      check(fw_wave_create(ctx_, method_ == Method::LFFP ? 0 : 1, g.dim(), J, lo, hi, p.order.values().data(),
                           p.M, p.kappa, f, p.phi.values().data(), p.psi.values().data(), cfg.tau, cfg.picard_tol,
                           cfg.picard_max_iters, cfg.inner_cg_tol, cfg.cg_max_iters, cfg.blowup_factor, &wv_));
    }
  }
  ~Stepper() {
    if (wv_) fw_wave_destroy(wv_);
    if (ts_) fw_tsfp2_destroy(ts_);
    fw_ctx_destroy(ctx_);
  }
  Stepper(const Stepper&) = delete;
  Stepper& operator=(const Stepper&) = delete;

  void step() { advance(1); }
  void advance(int steps) { check(ts_ ? fw_tsfp2_step(ts_, steps) : fw_wave_step(wv_, steps)); }
  void advance_to(double t_final) {  // stepping.cpp:165-168
    const long target = std::lround(t_final / tau_);
    while (n() < target) step();
  }
  const Field& current() {
    if (ts_)
      check(fw_tsfp2_get(ts_, cur_.values().data(), nullptr, nullptr));
    else
      check(fw_wave_get(wv_, cur_.values().data(), nullptr, nullptr, nullptr));
    return cur_;
  }
  const Field& velocity() {  // TSFP2 only (stepping.cpp:144)
    if (ts_) check(fw_tsfp2_get(ts_, nullptr, vel_.values().data(), nullptr));
    return vel_;
  }
  double time() { return n() * tau_; }
  long n() {
    long n = 0;
    check(ts_ ? fw_tsfp2_get(ts_, nullptr, nullptr, &n) : fw_wave_get(wv_, nullptr, nullptr, &n, nullptr));
    return n;
  }
  long total_picard_iterations() {
    if (ts_) return 0;
    long pt = 0;
    check(fw_wave_get(wv_, nullptr, nullptr, nullptr, &pt));
    return pt;
  }

 private:
  static void check(int rc) {
    if (rc == FW_OK) return;
    const std::string msg = std::string("B200 backend: ") + fw_last_error();
    switch (rc) {
      case FW_E_BLOWUP: throw BlowupDetected(msg);
      case FW_E_PICARD_DIVERGED: throw PicardDiverged(msg);
      case FW_E_CG_STAGNATED: throw CgStagnated(msg);
      case FW_E_NEGATIVE_M: throw NegativeM(msg);
      case FW_E_ORDER_RANGE: throw OrderOutOfRange(msg);
      case FW_E_DEVIATION: throw DeviationTooLarge(msg);
      case FW_E_GRID_MISMATCH: throw GridMismatch(msg);
      default: throw Error(msg);
    }
  }
  Method method_;
  double tau_;
  Field cur_, vel_;
  fw_ctx ctx_ = nullptr;
  fw_wave wv_ = nullptr;
  fw_tsfp2 ts_ = nullptr;
};

}  // namespace gpu
}  // namespace fwave
