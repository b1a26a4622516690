// Reference-side check of fwave::gpu::SeismicStepper: the reference's own
// classical-limit test (test_seismic.cpp:67-95 / acceptance 8, 1D part) and a
// variable-gamma run compared with the reference SeismicStepper class (its host-side update loop calling the drop-in applies).
#include <cmath>
#include <cstdio>

#include "fracwave/seismic.hpp"
#include "fracwave/stepping.hpp"
#include "seismic_gpu.hpp"

using namespace fwave;

int main() {
  int fails = 0;
  {  // gamma = 0 vs classical LFFP, 100 steps, per-step sup diff <= 1e-12
    Grid g = build_grid({{-16.0, 16.0}}, {256});
    const double c0 = 0.9, tau = 1e-3;
    SeismicMedium m = build_medium_constant(0.0, c0, 1.0, g, 10);
    Field phi(g), psi(g, 0.0);
    for (std::size_t j = 0; j < g.total(); ++j) phi[j] = std::exp(-g.point(j)[0] * g.point(j)[0]);
    gpu::SeismicStepper seis(m, phi, psi, tau);
    WaveProblem p;
    p.grid = g;
    p.order = sample_order(1.0, g);
    p.kappa = c0 * c0;
    p.f = Nonlinearity::none();
    p.phi = phi;
    p.psi = psi;
    Stepper classic(p, {Method::LFFP, tau});
    double worst = 0.0;
    for (int n = 0; n < 100; ++n) {
      seis.step();
      classic.step();
      const Field& a = seis.current();
      for (std::size_t j = 0; j < g.total(); ++j) worst = std::fmax(worst, std::fabs(a[j] - classic.current()[j]));
    }
    std::printf("gamma=0 GPU stepper vs classical LFFP: worst per-step diff %.3e\n", worst);
    if (!(worst <= 1e-12)) ++fails;
  }
  {  // variable gamma: GPU stepper vs the reference CPU stepper, bitwise
    Grid g = build_grid({{-8.0, 8.0}, {-8.0, 8.0}}, {64, 64});
    SeismicMedium m = build_medium(parse("0.01+0.005*tanh(y)"), parse("1"), 1.0, g, 12);
    Field phi = ricker_initial(1.0, {0.0, 0.0}, g), psi(g, 0.0);
    gpu::SeismicStepper a(m, phi, psi, 1e-3);
    SeismicStepper b(m, phi, psi, 1e-3);
    a.advance(25);
    b.advance(25);
    double diff = 0.0;
    for (std::size_t j = 0; j < g.total(); ++j) diff = std::fmax(diff, std::fabs(a.current()[j] - b.current()[j]));
    std::printf("variable-gamma 2D, 25 steps: fused GPU stepper vs reference SeismicStepper (host update, drop-in applies) max |diff| = %.3e (n %ld vs %ld)\n", diff,
                a.n(), b.n());
    if (!(diff == 0.0) || a.n() != b.n()) ++fails;
  }
  std::printf("%s\n", fails ? "[FAIL] seismic_gpu_check" : "[PASS] seismic_gpu_check");
  return fails ? 1 : 0;
}
