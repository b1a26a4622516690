// fftw_gpu.cpp — the FFTW3 entry points the reference calls, on the B200 backend.
//
// In the drop-in build the reference's Grid (grid.cpp:82-90, 134-137) and apply_toeplitz
// (flap.cpp:270-279) plan and execute FFTW transforms; here a plan records the rank, the
// dimensions and the sign, and every execute is one device DFT through the C-ABI
// (fw_grid_dft: the canonical power-of-two Stockham plan, Bluestein for other lengths), on the
// drop-in's device context and under its lock (the reference executes plans from OpenMP
// threads, e.g. assemble_dense, flap.cpp:192-201).  Out-of-place executes copy `in` to `out`
// first.  There is no CPU FFT in the drop-in library: a transform the device cannot serve is
// reported on stderr and aborts (FFTW's API has no error channel).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "dropin_ctx.hpp"
#include "fftw3.h"
#include "fw_capi.h"

struct fw_dropin_plan_s {
  int rank = 0;
  int n[3] = {1, 1, 1};
  int sign = FFTW_FORWARD;
  fftw_complex* in = nullptr;
  fftw_complex* out = nullptr;
  size_t total = 0;
};

namespace {

void execute(const fw_dropin_plan_s* p, fftw_complex* in, fftw_complex* out) {
  if (!p) return;
  if (in != out) std::memmove(out, in, p->total * sizeof(fftw_complex));
  std::lock_guard<std::mutex> lock(fwave::gpu_dropin::mutex());
  const int rc = fw_grid_dft(fwave::gpu_dropin::context(), p->rank, p->n, reinterpret_cast<double*>(out), p->sign);
  if (rc != FW_OK) {
    std::fprintf(stderr, "fftw_execute on the B200 backend failed: %s\n", fw_last_error());
    std::abort();
  }
}

}  // namespace

extern "C" {

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign, unsigned) {
  if (rank < 1 || rank > 3 || !n) return nullptr;
  fw_dropin_plan_s* p = new fw_dropin_plan_s();
  p->rank = rank;
  p->total = 1;
  for (int m = 0; m < rank; ++m) {
    p->n[m] = n[m];
    p->total *= (size_t)n[m];
  }
  p->sign = sign < 0 ? FFTW_FORWARD : FFTW_BACKWARD;
  p->in = in;
  p->out = out;
  return p;
}

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags) {
  return fftw_plan_dft(1, &n, in, out, sign, flags);
}

void fftw_execute(const fftw_plan p) {
  if (p) execute(p, p->in, p->out);
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) { execute(p, in, out); }

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
