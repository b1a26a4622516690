// Reference-side check of the slab-decomposed stepper of the C-ABI (fw_slab_seis_*), as a C++
// host of the reference would drive it on a C3/C4-style 3D grid: one process per GPU, rank and
// world size from FW_RANK / FW_WORLD (default 0 / 1), the NCCL unique id made by rank 0 and handed
// over through the file FW_NCCL_ID_FILE.  Every rank compares its planes with the reference's own
// SeismicStepper (seismic.cpp:85-142, host update, drop-in applies) after 6 steps: max |diff|
// <= 1e-12 (the stepping formula is the reference's; the applies agree to the fp64 floor).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include <map>

#include "dropin_ctx.hpp"
#include "fracwave/expr.hpp"
#include "fracwave/seismic.hpp"
#include "fw_capi.h"

using namespace fwave;

static int env_int(const char* k, int d) {
  const char* v = std::getenv(k);
  return v ? std::atoi(v) : d;
}

int main() {
  const int P = env_int("FW_WORLD", 1), rank = env_int("FW_RANK", 0);
  const std::vector<std::pair<double, double>> bounds = {{-4.0, 4.0}, {-4.0, 4.0}, {-1.0, 1.0}};
  Grid g = build_grid(bounds, {256, 256, 8});
  const std::size_t N = g.total();
  // the medium as the reference's expression language evaluates it (build_medium, seismic.cpp:48-60)
  const Expr gexpr = parse("0.02 + 0.015*sin(x)*cos(0.5*y)"), cexpr = parse("1");
  std::vector<double> gamma(N), c0(N), phi(N), psi(N, 0.0);
  std::map<std::string, double> env;
  for (std::size_t j = 0; j < N; ++j) {
    const auto x = g.point(j);
    env["x"] = x[0];
    env["y"] = x[1];
    env["z"] = x[2];
    gamma[j] = gexpr.eval(env);
    c0[j] = cexpr.eval(env);
    phi[j] = std::exp(-(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]) / 0.5);
  }
  unsigned char id[128] = {0};
  if (P > 1) {
    const char* path = std::getenv("FW_NCCL_ID_FILE");
    if (!path) {
      std::fprintf(stderr, "FW_NCCL_ID_FILE is needed for FW_WORLD > 1\n");
      return 2;
    }
    if (rank == 0) {
      if (fw_nccl_unique_id(id) != FW_OK) {
        std::fprintf(stderr, "%s\n", fw_last_error());
        return 2;
      }
      std::ofstream(std::string(path) + ".tmp", std::ios::binary).write((const char*)id, 128);
      std::rename((std::string(path) + ".tmp").c_str(), path);
    } else {
      for (;;) {
        std::ifstream f(path, std::ios::binary);
        if (f && f.read((char*)id, 128)) break;
        std::this_thread::sleep_for(std::chrono::milliseconds(20));
      }
    }
  }
  int J[3] = {256, 256, 8};
  double lo[3] = {-4.0, -4.0, -1.0}, hi[3] = {4.0, 4.0, 1.0};
  fw_ctx ctx = gpu_dropin::context();
  fw_slab_seis s = nullptr;
  if (fw_slab_seis_create(ctx, id, P, rank, J, lo, hi, gamma.data(), c0.data(), 1.0, 6, phi.data(), psi.data(), 1e-3,
                          1e8, &s) != FW_OK ||
      fw_slab_seis_step(s, 6) != FW_OK) {
    std::fprintf(stderr, "slab stepper: %s\n", fw_last_error());
    return 1;
  }
  const std::size_t nloc = N / P;
  std::vector<double> cur(nloc);
  long n = 0;
  size_t tb = 0;
  fw_slab_seis_get(s, cur.data(), nullptr, nullptr, &n);
  fw_slab_seis_info(s, &tb, nullptr, nullptr);
  // the reference's own stepper (host update loop; its applies are the drop-in's)
  SeismicMedium m = build_medium(gexpr, cexpr, 1.0, g, 6);
  SeismicStepper ref(m, Field(g, phi), Field(g, psi), 1e-3);
  ref.advance(6);
  double diff = 0.0;
  for (std::size_t j = 0; j < nloc; ++j) diff = std::fmax(diff, std::fabs(cur[j] - ref.current()[rank * nloc + j]));
  std::printf("rank %d/%d: slab stepper vs reference SeismicStepper after 6 steps: max |diff| = %.3e, n %ld vs %ld, "
              "table bytes on this rank %zu\n",
              rank, P, diff, n, ref.n(), tb);
  fw_slab_seis_destroy(s);
  const bool ok = diff <= 1e-12 && n == ref.n();
  std::printf("%s\n", ok ? "[PASS] slab_seis_check" : "[FAIL] slab_seis_check");
  return ok ? 0 : 1;
}
