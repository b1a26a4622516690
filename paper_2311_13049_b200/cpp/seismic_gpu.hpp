// seismic_gpu.hpp — fwave::gpu::SeismicStepper: the reference's SeismicStepper
// public API (proj/include/fracwave/seismic.hpp:36-46) with the state resident on
// the B200 and each step() one fused launch (fw_seis_* in include/fw_capi.h).
//
// The reference class holds `const SeismicMedium&` and private host Fields, so it
// cannot be re-targeted in place; this class takes the same constructor arguments
// and exposes the same members.  current() copies the wavefield back to the host
// (the reference returns a host Field reference).
#pragma once

#include <cmath>
#include <string>
#include <vector>

#include "fracwave/errors.hpp"
#include "fracwave/grid.hpp"
#include "fracwave/seismic.hpp"
#include "fw_capi.h"

namespace fwave {
namespace gpu {

class SeismicStepper {
 public:
  SeismicStepper(const SeismicMedium& medium, const Field& phi, const Field& psi, double tau,
                 double blowup_factor = 1e8, int device = 0)
      : grid_(medium.grid), tau_(tau), cur_(medium.grid, 0.0) {
    check(fw_ctx_create(device, &ctx_));
    const Grid& g = medium.grid;
    int J[3] = {1, 1, 1};
    double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
    for (int m = 0; m < g.dim(); ++m) {
      J[m] = g.size(m);
      lo[m] = g.lo(m);
      hi[m] = g.hi(m);
    }
    // derive_medium is re-evaluated from gamma and c0 on the way in (seismic.cpp:11-44)
    check(fw_seis_create(ctx_, g.dim(), J, lo, hi, medium.gamma.values().data(), medium.c0.values().data(),
                         medium.omega0, medium.disp_op.M, phi.values().data(), psi.values().data(), tau,
                         blowup_factor, &st_));
  }
  ~SeismicStepper() {
    fw_seis_destroy(st_);
    fw_ctx_destroy(ctx_);
  }
  SeismicStepper(const SeismicStepper&) = delete;
  SeismicStepper& operator=(const SeismicStepper&) = delete;

  void step() { check(fw_seis_step(st_, 1)); }
  void advance(int steps) { check(fw_seis_step(st_, steps)); }
  void advance_to(double t_final) {
    const long target = std::lround(t_final / tau_);  // seismic.cpp:139-142
    const long k = target - n();
    if (k > 0) advance(static_cast<int>(k));
  }
  const Field& current() {
    long n = 0;
    check(fw_seis_get(st_, cur_.values().data(), nullptr, nullptr, &n));
    return cur_;
  }
  double time() { return n() * tau_; }
  long n() {
    long n = 0;
    check(fw_seis_get(st_, nullptr, nullptr, nullptr, &n));
    return n;
  }

 private:
  static void check(int rc) {
    if (rc == FW_OK) return;
    const std::string msg = std::string("B200 backend: ") + fw_last_error();
    switch (rc) {
      case FW_E_BLOWUP: throw BlowupDetected(msg);
      case FW_E_GAMMA_RANGE: throw GammaOutOfRange(msg);
      case FW_E_NEGATIVE_M: throw NegativeM(msg);
      case FW_E_ORDER_RANGE: throw OrderOutOfRange(msg);
      case FW_E_DEVIATION: throw DeviationTooLarge(msg);
      case FW_E_GRID_MISMATCH: throw GridMismatch(msg);
      default: throw Error(msg);
    }
  }
  Grid grid_;
  double tau_;
  Field cur_;
  fw_ctx ctx_ = nullptr;
  fw_seis st_ = nullptr;
};

}  // namespace gpu
}  // namespace fwave
