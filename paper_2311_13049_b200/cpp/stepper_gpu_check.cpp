// Reference-side check of fwave::gpu::Stepper against the reference's own Stepper
// (stepping.cpp) on the same WaveProblem, both inside the drop-in build: LFFP bit for bit
// (the same device apply on both sides), TSFP2 to relative L2 1e-12 (the reference's
// oscillator flows call Grid::dft, which the drop-in serves with the device's full complex
// DFT, while fw_tsfp2 uses the real transforms), CNFP (device CG with tree-order dot
// products) to 1e-10, with the same step and Picard counts, and the reference's
// exceptions (BlowupDetected, PicardDiverged).  Bitwise pins against the reference built
// on the oracle's canonical FFT: tests/test_gpu_wave.py.
#include <cmath>
#include <cstdio>

#include "fracwave/stepping.hpp"
#include "stepper_gpu.hpp"

using namespace fwave;

namespace {

WaveProblem problem(bool cubic) {
  Grid g = build_grid({{-16.0, 16.0}}, {256});
  WaveProblem p;
  p.grid = g;
  std::vector<double> s(g.total()), phi(g.total());
  for (std::size_t j = 0; j < g.total(); ++j) {
    const double x = g.point(j)[0];
    s[j] = 1.5 + 0.3 * std::tanh(x);  // the s1-like profile of test_stepping.cpp
    phi[j] = std::exp(-x * x);
  }
  p.order = OrderField(g, s);
  p.kappa = 1.0;
  p.f = cubic ? Nonlinearity::cubic() : Nonlinearity::none();
  p.phi = Field(g, phi);
  p.psi = Field(g, 0.0);
  p.M = 15;
  return p;
}

double rel(const Field& a, const Field& b) {
  double num = 0.0, den = 0.0;
  for (std::size_t j = 0; j < a.size(); ++j) {
    num += (a[j] - b[j]) * (a[j] - b[j]);
    den += b[j] * b[j];
  }
  return std::sqrt(num / (den > 0 ? den : 1.0));
}

}  // namespace

int main() {
  int fails = 0;
  struct Case {
    Method m;
    bool cubic;
    double tau;
    int steps;
  } cases[] = {{Method::LFFP, false, 1e-3, 40}, {Method::LFFP, true, 1e-3, 40}, {Method::TSFP2, true, 1e-3, 30},
               {Method::CNFP, false, 1e-2, 12}, {Method::CNFP, true, 1e-2, 8}};
  for (const Case& c : cases) {
    const WaveProblem p = problem(c.cubic);
    StepperConfig cfg;
    cfg.method = c.m;
    cfg.tau = c.tau;
    Stepper ref(p, cfg);
    gpu::Stepper dev(p, cfg);
    ref.advance(c.steps);
    dev.advance(c.steps);
    const double e = rel(dev.current(), ref.current());
    const double tol = c.m == Method::LFFP ? 0.0 : (c.m == Method::TSFP2 ? 1e-12 : 1e-10);
    const bool ok = e <= tol && dev.n() == ref.n() &&
                    dev.total_picard_iterations() == ref.total_picard_iterations();
    std::printf("method %d f=%s: rel L2 %.3e, n %ld/%ld, picard %ld/%ld %s\n", (int)c.m, c.cubic ? "cubic" : "none",
                e, dev.n(), ref.n(), dev.total_picard_iterations(), ref.total_picard_iterations(),
                ok ? "ok" : "FAIL");
    if (!ok) ++fails;
  }
  {  // blow-up: same exception, same n, same pre-step state
    const WaveProblem p = problem(false);
    StepperConfig cfg;
    cfg.method = Method::LFFP;
    cfg.tau = 0.9;
    Stepper ref(p, cfg);
    gpu::Stepper dev(p, cfg);
    bool rt = false, dt = false;
    try {
      ref.advance(400);
    } catch (const BlowupDetected&) {
      rt = true;
    }
    try {
      dev.advance(400);
    } catch (const BlowupDetected&) {
      dt = true;
    }
    const bool ok = rt && dt && ref.n() == dev.n() && rel(dev.current(), ref.current()) == 0.0;
    std::printf("LFFP blow-up: reference n %ld, device n %ld %s\n", ref.n(), dev.n(), ok ? "ok" : "FAIL");
    if (!ok) ++fails;
  }
  {  // Picard cap
    const WaveProblem p = problem(true);
    StepperConfig cfg;
    cfg.method = Method::CNFP;
    cfg.tau = 5e-2;
    cfg.picard_max_iters = 1;
    gpu::Stepper dev(p, cfg);
    bool thrown = false;
    try {
      dev.step();
    } catch (const PicardDiverged&) {
      thrown = true;
    }
    std::printf("CNFP Picard cap: PicardDiverged %s\n", thrown ? "ok" : "FAIL");
    if (!thrown) ++fails;
  }
  std::printf(fails ? "[FAIL] %d\n" : "[PASS]\n", fails);
  return fails ? 1 : 0;
}
