// fw_capi.cu — implementation of include/fw_capi.h.
//
// Host-side setup restates the reference's table construction exactly
// (Grid |mu|^2 grid.cpp:60-80, OrderField s0 orderfield.cpp:10-36,
// build_expansion flap.cpp:96-135, derive_medium seismic.cpp:11-44) with the
// same glibc pow/log/cos/sin calls, so the device tables are bit-identical to
// the reference's.  Transcendentals are evaluated on the host once per
// operator on the Hermitian half; the M-fold recurrences run on the device
// (IEEE mul/div: bit-identical).  There is no CPU compute fallback: every
// apply runs the sm_100a kernels in fw_kernels.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/fw_capi.h"
#include "fw_fft.cuh"
#include "fw_internal.h"
#include "fw_step2d.h"

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define FW_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      return set_err(e_ == cudaErrorMemoryAllocation ? FW_E_OOM : FW_E_CUDA,           \
                     std::string(#call) + ": " + cudaGetErrorString(e_));             \
    }                                                                                   \
  } while (0)

// every entry point that allocates or launches first makes its context's device current
// (another context on another device may have switched it in this thread)
#define FW_SETDEV(ctxp)                                      \
  do {                                                       \
    if (ctxp) FW_CUDA(cudaSetDevice((ctxp)->device));        \
  } while (0)

#define FW_TRY(expr)               \
  do {                             \
    int rc_ = (expr);              \
    if (rc_ != FW_OK) return rc_;  \
  } while (0)

// ---- twiddles: same definition as oracle/fwshim/fwcanon.c fwc_twiddle ----
void twiddle(long t, long n, double* c, double* s) {
  t %= n;
  if (t < 0) t += n;
  if (t == 0) {
    *c = 1.0;
    *s = 0.0;
    return;
  }
  const long quarter = n / 4;
  const long q = t / quarter;
  const long tq = t - q * quarter;
  double cc, ss;
  if (tq == 0) {
    cc = 1.0;
    ss = 0.0;
  } else if (8 * tq <= n) {
    const double ang = (2.0 * M_PI) * ((double)tq / (double)n);
    cc = cos(ang);
    ss = sin(ang);
  } else {
    const long tr = quarter - tq;
    const double ang = (2.0 * M_PI) * ((double)tr / (double)n);
    cc = sin(ang);
    ss = cos(ang);
  }
  switch (q) {
    case 0: *c = cc; *s = ss; break;
    case 1: *c = -ss; *s = cc; break;
    case 2: *c = -cc; *s = -ss; break;
    default: *c = ss; *s = -cc; break;
  }
}

bool is_pow2(long n) { return n >= 1 && (n & (n - 1)) == 0; }

// Grid::Grid validation (grid.cpp:35-58) + this backend's size support
// Grid::Grid validation (grid.cpp:35-58) and the geometry
int check_grid_ref(int dim, const int* J, const double* lo, const double* hi, fw::GridGeom* g) {
  if (!J) return set_err(FW_E_ARG, "null size array");
  if (dim < 1 || dim > 3) return set_err(FW_E_DIM_RANGE, "dimension must be 1, 2 or 3, got " + std::to_string(dim));
  for (int m = 0; m < dim; ++m) {
    if (J[m] < 4 || J[m] % 2 != 0)
      return set_err(FW_E_ODD_SIZE, "axis " + std::to_string(m) + ": point count " + std::to_string(J[m]) +
                                        " must be even and >= 4");
    if (lo && hi && !(hi[m] > lo[m])) return set_err(FW_E_EMPTY_INTERVAL, "axis " + std::to_string(m) + ": empty interval");
  }
  g->d = dim;
  g->N = 1;
  for (int m = 0; m < 3; ++m) g->J[m] = m < dim ? J[m] : 1;
  for (int m = 0; m < dim; ++m) g->N *= (size_t)J[m];
  g->nl = J[dim - 1];
  g->hp1 = g->nl / 2 + 1;
  g->rows = g->N / (size_t)g->nl;
  g->Nh = g->rows * (size_t)g->hp1;
  return FW_OK;
}

// ... plus the device transforms: full = some axis is not a power of two (served by the
// full-spectrum C2C path, fw_dft.cu); lengths past the device transforms' reach: FW_E_UNSUPPORTED
int plan_grid(int dim, const int* J, const double* lo, const double* hi, fw::GridGeom* g, bool* full) {
  FW_TRY(check_grid_ref(dim, J, lo, hi, g));
  *full = false;
  for (int m = 0; m < dim; ++m) {
    if (!fw::dft_length_supported(J[m]))
      return set_err(FW_E_UNSUPPORTED, "axis " + std::to_string(m) + ": length " + std::to_string(J[m]) +
                                           " beyond the device transforms (powers of two <= 4096, other even "
                                           "lengths <= 2048)");
    if (!is_pow2(J[m])) *full = true;
  }
  return FW_OK;
}

// the table geometry of the full-spectrum path: every bin of the last axis
fw::GridGeom full_geom(fw::GridGeom g) {
  g.hp1 = g.nl;
  g.Nh = g.N;
  return g;
}

// ... plus what the canonical real-transform pipeline serves
int check_grid(int dim, const int* J, const double* lo, const double* hi, fw::GridGeom* g) {
  FW_TRY(check_grid_ref(dim, J, lo, hi, g));
  for (int m = 0; m < dim; ++m)
    if (!is_pow2(J[m]) || J[m] > 4096)
      return set_err(FW_E_UNSUPPORTED, "axis " + std::to_string(m) + ": this backend needs a power of two in [4, 4096], got " +
                                           std::to_string(J[m]));
  return FW_OK;
}

// |mu|^2 on the Hermitian half, summed m = d-1 .. 0 (grid.cpp:60-80)
std::vector<double> half_mu2(const fw::GridGeom& g, const double* lo, const double* hi) {
  std::vector<std::vector<double>> ax(g.d);
  for (int m = 0; m < g.d; ++m) {
    ax[m].resize(g.J[m]);
    const double base = 2.0 * M_PI / (hi[m] - lo[m]);
    for (int p = 0; p < g.J[m]; ++p) {
      const int k = (p < g.J[m] / 2) ? p : p - g.J[m];
      ax[m][p] = (base * k) * (base * k);
    }
  }
  std::vector<double> out(g.Nh);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)g.Nh; ++i) {
    int idx[3] = {0, 0, 0};
    idx[g.d - 1] = (int)(i % g.hp1);
    long long rem = i / g.hp1;
    for (int m = g.d - 2; m >= 0; --m) {
      idx[m] = (int)(rem % g.J[m]);
      rem /= g.J[m];
    }
    double v = 0.0;
    for (int m = g.d - 1; m >= 0; --m) v += ax[m][idx[m]];
    out[i] = v;
  }
  return out;
}

// OrderField (orderfield.cpp:10-36) + is_constant (orderfield.cpp:55-57)
int order_stats(const double* s, size_t N, const double* s0_override, double* s0, double* smin, double* smax,
                int* constant) {
  if (!s) return set_err(FW_E_ARG, "null order values");
  double mn = s[0], mx = s[0];
  for (size_t i = 1; i < N; ++i) {
    if (s[i] < mn) mn = s[i];
    if (mx < s[i]) mx = s[i];
  }
  if (!(mn > 0.0) || !(mx < 2.0)) {
    char b[160];
    snprintf(b, sizeof b, "order range [%f, %f] outside (0, 2)", mn, mx);
    return set_err(FW_E_ORDER_RANGE, b);
  }
  double z;
  if (s0_override) {
    z = *s0_override;
  } else if (mn == mx) {
    z = mn;
  } else {
    double sum = 0.0;
    for (size_t i = 0; i < N; ++i) sum += s[i];
    z = sum / (double)N;
  }
  const double dev = std::max(std::fabs(mn - z), std::fabs(mx - z));
  if (dev >= 1.0) {
    char b[160];
    snprintf(b, sizeof b, "max |s(x) - s0| = %f >= 1; expansion would diverge", dev);
    return set_err(FW_E_DEVIATION, b);
  }
  *s0 = z;
  *smin = mn;
  *smax = mx;
  *constant = (mx - mn <= 1e-14) ? 1 : 0;
  return FW_OK;
}

template <class T>
int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(FW_E_OOM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed: " +
                                 cudaGetErrorString(e));
  }
  return FW_OK;
}

}  // namespace

// ===========================================================================

struct fw_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  double2* master = nullptr;
  long long launches = 0;
  // grow-only scratch slots (single stream: ops on one ctx run in order)
  void* scratch[12] = {};
  size_t scratch_bytes[12] = {};
  double* residue = nullptr;  // device scalar
  int nsm = 148;
  bool force_generic = false;                 // FW_FORCE_GENERIC=1: multi-pass kernels only
  int dbg = 0;                                // FW_STEP2D_DBG: timing experiments only (wrong results)
  int steps_per_launch = 0;                   // FW_STEPS_PER_LAUNCH: seismic steps per persistent launch (0 = all)
  bool step2d_tm = false;                     // FW_STEP2D_TM=1: time-multiplexed persistent kernel (A/B)
  int batch_fields = 0;                       // FW_BATCH_FIELDS: fields per batched pipeline (0 = all that fit)
  int batch_l2_mb = 0;                        // FW_BATCH_L2_MB: term spectra a batched chunk keeps in L2 (0 = no term chunks, the
                                              // default: measured slower at every chunk size)
  int batch_group = 8;                        // FW_BATCH_GROUP: fields per L2-resident chunk
  unsigned long long* counters = nullptr;     // persistent-kernel counters (2 sets)
  unsigned long long* trace = nullptr;        // FW_TRACE=1: persistent-kernel watchdog records (device view)
  unsigned long long* trace_host = nullptr;   //   ... the same buffer, mapped host memory (survives a trap)
  int cset = 0;
  bool generic_lines = false;                 // FW_GENERIC_LINES=1: shared-memory line FFTs only (tests)
  fw::ChirpCache chirps;                      // Bluestein chirps of the non-power-of-two axes (fw_dft.cu)
  fw::LaunchCtx L() { return fw::LaunchCtx{stream, master, &launches, generic_lines}; }
  int get_scratch(int slot, size_t bytes, void** out) {
    if (scratch_bytes[slot] < bytes) {
      if (scratch[slot]) cudaFree(scratch[slot]);
      scratch[slot] = nullptr;
      scratch_bytes[slot] = 0;
      cudaError_t e = cudaMalloc(&scratch[slot], bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(FW_E_OOM, "scratch allocation of " + std::to_string(bytes) + " bytes failed");
      }
      scratch_bytes[slot] = bytes;
    }
    *out = scratch[slot];
    return FW_OK;
  }
};

enum {
  SLOT_UH = 0, SLOT_T = 1, SLOT_U = 2, SLOT_OUT = 3, SLOT_TMP = 4, SLOT_UH2 = 5, SLOT_Y2D = 6, SLOT_T2D = 7,
  SLOT_BUH = 8, SLOT_BT = 9, SLOT_BTAB = 10  // batched multi-field pipeline
};

struct fw_op_s {
  fw_ctx ctx = nullptr;
  fw::GridGeom g;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  int M = 0;
  int constant_order = 0;
  double s0 = 0, smin = 0, smax = 0;
  double* w = nullptr;     // (M+1) x Nh
  double* dev1 = nullptr;  // N
  double* w2d = nullptr;   // persistent 2D kernel: [M+1][groups][J0][4] weights
  double* devt = nullptr;  // persistent 2D kernel: [M][N] deviation powers (s-s0)^m
  size_t bytes = 0;
  bool step2d = false;
  bool full = false;       // non-power-of-two axes: full-spectrum tables, C2C apply (fw_dft.cu)
  bool slab = false;       // fw_op_create_slab: tables of one rank's slab only (stage entry points)
};

extern "C" {

const char* fw_last_error(void) { return g_err.c_str(); }
int fw_version(void) { return FW_CAPI_VERSION; }

int fw_ctx_create(int device, fw_ctx* out) {
  if (!out) return set_err(FW_E_ARG, "null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return set_err(FW_E_CUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
  }
  if (device < 0 || device >= n) return set_err(FW_E_ARG, "device index out of range");
  FW_CUDA(cudaSetDevice(device));
  fw_ctx c = new fw_ctx_s();
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return set_err(FW_E_CUDA, "stream creation failed");
  }
  std::vector<double2> tw(fw::kTwMaster);
  for (int t = 0; t < fw::kTwMaster; ++t) twiddle(t, fw::kTwMaster, &tw[t].x, &tw[t].y);
  if (dalloc(&c->master, tw.size()) || dalloc(&c->residue, 1)) {
    fw_ctx_destroy(c);
    return FW_E_OOM;
  }
  FW_CUDA(cudaMemcpy(c->master, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  const char* fg = getenv("FW_FORCE_GENERIC");
  c->force_generic = fg && fg[0] == '1';
  const char* gl = getenv("FW_GENERIC_LINES");
  c->generic_lines = gl && gl[0] == '1';
  const char* dg = getenv("FW_STEP2D_DBG");
  c->dbg = dg ? atoi(dg) : 0;
  const char* bf = getenv("FW_BATCH_FIELDS");
  c->batch_fields = bf ? std::max(0, atoi(bf)) : 0;
  const char* bl2 = getenv("FW_BATCH_L2_MB");
  if (bl2) c->batch_l2_mb = std::max(0, atoi(bl2));
  const char* bgr = getenv("FW_BATCH_GROUP");
  if (bgr) c->batch_group = std::max(1, atoi(bgr));
  const char* tm = getenv("FW_STEP2D_TM");
  c->step2d_tm = tm && tm[0] == '1';
  const char* spl = getenv("FW_STEPS_PER_LAUNCH");
  c->steps_per_launch = spl ? std::max(0, atoi(spl)) : 0;
  if (dalloc(&c->counters, 2 * (size_t)fw::kStep2dCStride)) {
    fw_ctx_destroy(c);
    return FW_E_OOM;
  }
  FW_CUDA(cudaMemset(c->counters, 0, 2 * (size_t)fw::kStep2dCStride * sizeof(unsigned long long)));
  const char* tr = getenv("FW_TRACE");
  if (tr && tr[0] == '1') {
    const size_t n = (size_t)fw::kTraceAlloc;
    if (cudaHostAlloc((void**)&c->trace_host, n * sizeof(unsigned long long), cudaHostAllocMapped) == cudaSuccess) {
      memset(c->trace_host, 0, n * sizeof(unsigned long long));
      if (cudaHostGetDevicePointer((void**)&c->trace, c->trace_host, 0) != cudaSuccess) c->trace = nullptr;
    } else {
      cudaGetLastError();
      c->trace_host = nullptr;
    }
  }
  fw::init_kernels();
  *out = c;
  return FW_OK;
}

void fw_ctx_destroy(fw_ctx c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : c->scratch)
    if (p) cudaFree(p);
  c->chirps.release();
  if (c->master) cudaFree(c->master);
  if (c->residue) cudaFree(c->residue);
  if (c->counters) cudaFree(c->counters);
  if (c->trace_host) cudaFreeHost(c->trace_host);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int fw_ctx_sync(fw_ctx c) {
  FW_SETDEV(c);
  if (!c) return set_err(FW_E_ARG, "null ctx");
  FW_CUDA(cudaStreamSynchronize(c->stream));
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

void* fw_ctx_stream(fw_ctx c) { return c ? (void*)c->stream : nullptr; }
int fw_ctx_device(fw_ctx c) { return c ? c->device : -1; }

// the thread-local error of the C-ABI, for the library's other translation units (fw_slab.cu)
int fw_internal_set_error(int code, const char* msg) { return set_err(code, msg ? msg : ""); }

/* diagnostics: the persistent kernel's watchdog records (kTraceWords u64: per CTA 8 words = site, thread,
   counter value seen, target, term, globaltimer), readable even after the kernel trapped; FW_E_ARG if
   FW_TRACE=1 was not set at context creation */
int fw_ctx_trace(fw_ctx c, unsigned long long* out) {
  if (!c || !c->trace_host || !out) return set_err(FW_E_ARG, "tracing disabled (set FW_TRACE=1 before fw_ctx_create)");
  if (c->stream) cudaStreamSynchronize(c->stream);  // a trapped kernel leaves a sticky error: ignored here
  memcpy(out, c->trace_host, (size_t)fw::kTraceAlloc * sizeof(unsigned long long));
  return FW_OK;
}
long long fw_ctx_launches(fw_ctx c) { return c ? c->launches : 0; }

}  // extern "C"

namespace {

int op_alloc_common(fw_ctx ctx, const fw::GridGeom& g, const double* lo, const double* hi, int M, fw_op* out,
                    fw_op_s** o, bool full = false) {
  if (M < 0) return set_err(FW_E_NEGATIVE_M, "truncation count M must be >= 0");
  fw_op_s* op = new fw_op_s();
  op->ctx = ctx;
  op->g = g;
  op->full = full;
  const fw::GridGeom gw = full ? full_geom(g) : g;  // table geometry
  for (int m = 0; m < g.d; ++m) {
    op->lo[m] = lo[m];
    op->hi[m] = hi[m];
  }
  op->M = M;
  if (dalloc(&op->w, (size_t)(M + 1) * gw.Nh) || dalloc(&op->dev1, g.N)) {
    fw_op_destroy(op);
    return FW_E_OOM;
  }
  op->bytes = ((size_t)(M + 1) * gw.Nh + g.N) * sizeof(double);
  if (!full && g.d == 2 && fw::step2d_supported(g.J[0], g.J[1], ctx->nsm) && M <= 64) {
    const size_t nw = (size_t)(M + 1) * fw::step2d_col_groups(g.J[1]) * g.J[0] * fw::kStep2dCG;
    if (dalloc(&op->w2d, nw) || dalloc(&op->devt, (size_t)std::max(M, 1) * g.N)) {
      fw_op_destroy(op);
      return FW_E_OOM;
    }
    op->bytes += (nw + (size_t)M * g.N) * sizeof(double);
    op->step2d = true;
  }
  *o = op;
  (void)out;
  return FW_OK;
}

int op_create_internal(fw_ctx ctx, const fw::GridGeom& g0, const double* lo, const double* hi, const double* s,
                       const double* s0_override, int M, fw_op* out, bool full = false) {
  double s0, smin, smax;
  int constant;
  FW_TRY(order_stats(s, g0.N, s0_override, &s0, &smin, &smax, &constant));
  fw_op_s* op = nullptr;
  FW_TRY(op_alloc_common(ctx, g0, lo, hi, M, out, &op, full));
  const fw::GridGeom g = full ? full_geom(g0) : g0;  // table geometry (N bins when full)
  op->s0 = s0;
  op->smin = smin;
  op->smax = smax;
  op->constant_order = constant;
  // flap.cpp:108-122 transcendentals on the host half spectrum
  std::vector<double> mu2 = half_mu2(g, lo, hi);
  std::vector<double> base(g.Nh), logm(g.Nh);
#pragma omp parallel for schedule(static)
  for (long long k = 0; k < (long long)g.Nh; ++k) {
    base[k] = mu2[k] > 0.0 ? pow(mu2[k], s0) : 0.0;
    logm[k] = mu2[k] > 0.0 ? log(mu2[k]) : 0.0;
  }
  auto L = ctx->L();
  double *d_mu2 = nullptr, *d_base = nullptr, *d_logm = nullptr, *d_s = nullptr;
  int rc = FW_OK;
  if ((rc = dalloc(&d_mu2, g.Nh)) || (rc = dalloc(&d_base, g.Nh)) || (rc = dalloc(&d_logm, g.Nh)) ||
      (rc = dalloc(&d_s, g.N))) {
    cudaFree(d_mu2); cudaFree(d_base); cudaFree(d_logm); cudaFree(d_s);
    fw_op_destroy(op);
    return rc;
  }
  cudaMemcpyAsync(d_mu2, mu2.data(), g.Nh * 8, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(d_base, base.data(), g.Nh * 8, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(d_logm, logm.data(), g.Nh * 8, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(d_s, s, g.N * 8, cudaMemcpyHostToDevice, ctx->stream);
  fw::launch_build_weights(L, g.Nh, M, d_mu2, d_base, d_logm, op->w);
  fw::launch_dev1(L, g.N, d_s, s0, op->dev1);
  if (op->step2d) {
    fw::launch_w_to_2d(ctx->stream, g.J[0], g.J[1], M, op->w, op->w2d);
    fw::launch_dev_tables(ctx->stream, g.N, M, op->dev1, op->devt);
  }
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d_mu2); cudaFree(d_base); cudaFree(d_logm); cudaFree(d_s);
  if (e != cudaSuccess) {
    fw_op_destroy(op);
    return set_err(FW_E_CUDA, std::string("table construction: ") + cudaGetErrorString(e));
  }
  *out = op;
  return FW_OK;
}

// persistent single-launch 2D kernel (fw_step2d.cu); ops[0..nops) share grid and M
int launch_persistent(fw_ctx ctx, fw_op const* ops, int nops, int m_first, const double* u, double* const* outs,
                      double* residue, fw::Step2DParams* extra) {
  const fw::GridGeom& g = ops[0]->g;
  const int m_last = ops[0]->constant_order ? 0 : ops[0]->M;
  void *Y = nullptr, *T = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_Y2D, g.Nh * sizeof(double2), &Y));
  FW_TRY(ctx->get_scratch(SLOT_T2D, (size_t)fw::kStep2dRing * g.Nh * sizeof(double2), &T));
  fw::Step2DParams p = extra ? *extra : fw::Step2DParams{};
  if (p.nsteps < 1) p.nsteps = 1;
  p.J0 = g.J[0];
  p.J1 = g.J[1];
  p.M = m_last;
  p.m_first = m_first;
  p.nops = nops;
  p.nterms_total = nops * (m_last + 1 - m_first);
  p.u = u;
  p.Y = (double2*)Y;
  p.T = (double2*)T;
  for (int o = 0; o < nops; ++o) {
    p.w[o] = ops[o]->w2d;
    p.dev[o] = ops[o]->devt;
    p.out[o] = outs[o];
  }
  p.residue = residue;
  p.master = ctx->master;
  p.wcols = fw::step2d_wcols(g.J[1]);
  p.counters = ctx->counters;
  p.trace = ctx->trace;
  p.dbg = ctx->dbg;
  p.cset = ctx->cset;
  p.cstride = fw::kStep2dCStride;
  cudaError_t e = ctx->step2d_tm ? fw::launch_step2d_tm(p, ctx->stream, ctx->nsm)
                                 : fw::launch_step2d(p, ctx->stream, ctx->nsm);
  if (e != cudaSuccess) {
    // only a running kernel zeroes the other counter set: after a failed launch both sets are
    // reset so that the next launch cannot find its spin targets already met
    cudaGetLastError();
    cudaMemsetAsync(ctx->counters, 0, 2 * (size_t)fw::kStep2dCStride * sizeof(unsigned long long), ctx->stream);
    return set_err(FW_E_CUDA, std::string("persistent 2D launch: ") + cudaGetErrorString(e));
  }
  ctx->cset ^= 1;  // the launched kernel zeroes the other set for the next launch
  ctx->launches += 1;
  return FW_OK;
}

bool use_persistent(fw_op op) { return op->step2d && !op->ctx->force_generic; }

// out = A(u) for device pointers, enqueued
int apply_device(fw_op op, const double* u, double* out, int m_first, double* residue, const int* guard,
                 const double2* Uh_pre = nullptr) {
  fw_ctx ctx = op->ctx;
  const fw::GridGeom& g = op->g;
  if (m_first < 0 || m_first > 1) return set_err(FW_E_ARG, "m_first must be 0 or 1");
  const int m_last = op->constant_order ? 0 : op->M;
  auto L = ctx->L();
  if (m_first > m_last) {  // perturbation of a constant-order operator: exact zero (flap.cpp:163-166)
    FW_CUDA(cudaMemsetAsync(out, 0, g.N * sizeof(double), ctx->stream));
    return FW_OK;
  }
  if (op->slab) return set_err(FW_E_ARG, "slab operator: its tables cover one rank's slab (use the stage entry points)");
  if (op->full) {  // non-power-of-two axes: the C2C form (fw_dft.cu)
    void *uh = nullptr, *buf = nullptr, *devm = nullptr;
    FW_TRY(ctx->get_scratch(SLOT_UH, g.N * sizeof(double2), &uh));
    FW_TRY(ctx->get_scratch(SLOT_T, g.N * sizeof(double2), &buf));
    FW_TRY(ctx->get_scratch(SLOT_TMP, g.N * sizeof(double), &devm));
    cudaError_t e = fw::launch_full_forward(L, ctx->chirps, g.d, g.J, (long long)g.N, u, (double2*)uh, true);
    if (e == cudaSuccess) {
      fw::FullApplyArgs a{(const double2*)uh, op->w, op->dev1, (double*)devm, (double2*)buf, out, m_first, m_last,
                          residue, guard};
      e = fw::launch_full_apply(L, ctx->chirps, g.d, g.J, (long long)g.N, a);
    }
    if (e != cudaSuccess) return set_err(FW_E_CUDA, std::string("full-spectrum apply: ") + cudaGetErrorString(e));
    return FW_OK;
  }
  if (!Uh_pre && !guard && use_persistent(op)) {
    fw_op ops[1] = {op};
    double* outs[1] = {out};
    return launch_persistent(ctx, ops, 1, m_first, u, outs, residue, nullptr);
  }
  void* uh = nullptr;
  const double2* Uh = Uh_pre;
  if (!Uh) {
    FW_TRY(ctx->get_scratch(SLOT_UH, g.Nh * sizeof(double2), &uh));
    fw::launch_forward(L, g, u, (double2*)uh, true);
    Uh = (const double2*)uh;
  }
  void* T = nullptr;
  if (g.d >= 2)
    FW_TRY(ctx->get_scratch(SLOT_T, (size_t)(m_last - m_first + 1) * fw::term_elems(L, g) * sizeof(double2), &T));
  fw::InverseArgs a{Uh, op->w, op->dev1, (double2*)T, out, m_first, m_last, residue, guard};
  fw::launch_inverse(L, g, a);
  return FW_OK;
}

}  // namespace

extern "C" {

int fw_op_create(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                 const double* order_values, const double* s0_override, int M, fw_op* out) {
  if (!ctx || !out || !lo || !hi) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  bool full = false;
  FW_TRY(plan_grid(dim, J, lo, hi, &g, &full));
  FW_CUDA(cudaSetDevice(ctx->device));
  return op_create_internal(ctx, g, lo, hi, order_values, s0_override, M, out, full);
}

// One rank's tables of a slab-decomposed 3D grid (slab.py): w_m on the rank's spectral columns
// [J0][J1/P][H] (axis-1 bins [rank J1/P, (rank+1) J1/P)), s - s0 on its planes [J0/P][J1][J2]; s0 and
// the OrderField checks from the GLOBAL order values (orderfield.cpp:10-36), so every rank's tables
// equal the corresponding slices of the single-device operator's (bit for bit).
int fw_op_create_slab(fw_ctx ctx, const int* J, const double* lo, const double* hi, const double* order_values,
                      const double* s0_override, int M, int P, int rank, fw_op* out) {
  FW_SETDEV(ctx);
  if (!ctx || !out || !lo || !hi || !order_values) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  FW_TRY(check_grid(3, J, lo, hi, &g));
  if (P < 1 || rank < 0 || rank >= P || J[0] % P || J[1] % P)
    return set_err(FW_E_ARG, "slab: axes 0 and 1 must be divisible by P and 0 <= rank < P");
  double s0, smin, smax;
  int constant;
  FW_TRY(order_stats(order_values, g.N, s0_override, &s0, &smin, &smax, &constant));
  if (M < 0) return set_err(FW_E_NEGATIVE_M, "truncation count M must be >= 0");
  const int J1l = J[1] / P, J0l = J[0] / P, H = g.hp1;
  const size_t nw = (size_t)J[0] * J1l * H;       // spectral bins of the rank's columns
  const size_t nd = (size_t)J0l * J[1] * J[2];    // the rank's planes
  fw_op_s* op = new fw_op_s();
  op->ctx = ctx;
  op->g = g;
  for (int m = 0; m < 3; ++m) {
    op->lo[m] = lo[m];
    op->hi[m] = hi[m];
  }
  op->M = M;
  op->slab = true;
  op->s0 = s0;
  op->smin = smin;
  op->smax = smax;
  op->constant_order = constant;
  if (dalloc(&op->w, (size_t)(M + 1) * nw) || dalloc(&op->dev1, nd)) {
    fw_op_destroy(op);
    return FW_E_OOM;
  }
  op->bytes = ((size_t)(M + 1) * nw + nd) * sizeof(double);
  // |mu|^2 at (k0, k1 in the rank's columns, k2 < H), summed m = 2..0 as grid.cpp:71-79
  std::vector<double> ax[3];
  for (int m = 0; m < 3; ++m) {
    ax[m].resize(J[m]);
    const double base = 2.0 * M_PI / (hi[m] - lo[m]);
    for (int p = 0; p < J[m]; ++p) {
      const int k = (p < J[m] / 2) ? p : p - J[m];
      ax[m][p] = (base * k) * (base * k);
    }
  }
  std::vector<double> mu2(nw), base(nw), logm(nw);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)nw; ++i) {
    const int k2 = (int)(i % H);
    const int k1 = rank * J1l + (int)((i / H) % J1l);
    const int k0 = (int)(i / ((size_t)H * J1l));
    double v = 0.0;
    v += ax[2][k2];
    v += ax[1][k1];
    v += ax[0][k0];
    mu2[i] = v;
    base[i] = v > 0.0 ? pow(v, s0) : 0.0;  // flap.cpp:108-110
    logm[i] = v > 0.0 ? log(v) : 0.0;      // flap.cpp:119
  }
  double *d_mu2 = nullptr, *d_base = nullptr, *d_logm = nullptr, *d_s = nullptr;
  int rc = FW_OK;
  if ((rc = dalloc(&d_mu2, nw)) || (rc = dalloc(&d_base, nw)) || (rc = dalloc(&d_logm, nw)) || (rc = dalloc(&d_s, nd))) {
    cudaFree(d_mu2); cudaFree(d_base); cudaFree(d_logm); cudaFree(d_s);
    fw_op_destroy(op);
    return rc;
  }
  auto L = ctx->L();
  cudaMemcpyAsync(d_mu2, mu2.data(), nw * 8, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(d_base, base.data(), nw * 8, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(d_logm, logm.data(), nw * 8, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(d_s, order_values + (size_t)rank * nd, nd * 8, cudaMemcpyHostToDevice, ctx->stream);
  fw::launch_build_weights(L, nw, M, d_mu2, d_base, d_logm, op->w);
  fw::launch_dev1(L, nd, d_s, s0, op->dev1);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d_mu2); cudaFree(d_base); cudaFree(d_logm); cudaFree(d_s);
  if (e != cudaSuccess) {
    fw_op_destroy(op);
    return set_err(FW_E_CUDA, std::string("slab tables: ") + cudaGetErrorString(e));
  }
  *out = op;
  return FW_OK;
}

int fw_op_create_from_tables(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi, int M,
                             double s0, int constant_order, const double* base_symbol,
                             const double* const* log_weights, const double* const* deviation_powers,
                             fw_op* out) {
  if (!ctx || !out || !lo || !hi || !base_symbol) return set_err(FW_E_ARG, "null argument");
  if (M > 0 && (!log_weights || !deviation_powers)) return set_err(FW_E_ARG, "null table rows");
  fw::GridGeom g0;
  bool full = false;
  FW_TRY(plan_grid(dim, J, lo, hi, &g0, &full));
  FW_CUDA(cudaSetDevice(ctx->device));
  fw_op_s* op = nullptr;
  FW_TRY(op_alloc_common(ctx, g0, lo, hi, M, out, &op, full));
  const fw::GridGeom g = full ? full_geom(g0) : g0;  // table geometry
  op->s0 = s0;
  op->constant_order = constant_order ? 1 : 0;
  // gather the Hermitian half of the spectral tables (row r, bin q -> full index r*nl + q)
  std::vector<double> base(g.Nh), lw((size_t)std::max(M, 1) * g.Nh);
  for (size_t r = 0; r < g.rows; ++r)
    for (int q = 0; q < g.hp1; ++q) {
      const size_t hi_ = r * g.hp1 + q, fi = r * (size_t)g.nl + q;
      base[hi_] = base_symbol[fi];
      for (int m = 0; m < M; ++m) lw[(size_t)m * g.Nh + hi_] = log_weights[m][fi];
    }
  double *d_base = nullptr, *d_lw = nullptr;
  int rc = FW_OK;
  if ((rc = dalloc(&d_base, g.Nh)) || (rc = dalloc(&d_lw, lw.size()))) {
    cudaFree(d_base); cudaFree(d_lw);
    fw_op_destroy(op);
    return rc;
  }
  auto L = ctx->L();
  cudaMemcpyAsync(d_base, base.data(), g.Nh * 8, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(d_lw, lw.data(), lw.size() * 8, cudaMemcpyHostToDevice, ctx->stream);
  fw::launch_weights_from_lw(L, g.Nh, M, d_base, d_lw, op->w);
  if (M > 0) {
    cudaMemcpyAsync(op->dev1, deviation_powers[0], g.N * 8, cudaMemcpyHostToDevice, ctx->stream);
  } else {
    cudaMemsetAsync(op->dev1, 0, g.N * 8, ctx->stream);
  }
  if (op->step2d) {
    fw::launch_w_to_2d(ctx->stream, g.J[0], g.J[1], M, op->w, op->w2d);
    fw::launch_dev_tables(ctx->stream, g.N, M, op->dev1, op->devt);
  }
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d_base); cudaFree(d_lw);
  if (e != cudaSuccess) {
    fw_op_destroy(op);
    return set_err(FW_E_CUDA, std::string("table upload: ") + cudaGetErrorString(e));
  }
  op->smin = op->smax = NAN;
  *out = op;
  return FW_OK;
}

void fw_op_destroy(fw_op op) {
  if (op && op->ctx) cudaSetDevice(op->ctx->device);
  if (!op) return;
  if (op->w) cudaFree(op->w);
  if (op->dev1) cudaFree(op->dev1);
  if (op->w2d) cudaFree(op->w2d);
  if (op->devt) cudaFree(op->devt);
  delete op;
}

int fw_op_info(fw_op op, fw_op_info_t* info) {
  if (!op || !info) return set_err(FW_E_ARG, "null argument");
  memset(info, 0, sizeof(*info));
  info->dim = op->g.d;
  for (int m = 0; m < 3; ++m) {
    info->J[m] = op->g.J[m];
    info->lo[m] = op->lo[m];
    info->hi[m] = op->hi[m];
  }
  info->M = op->M;
  info->constant_order = op->constant_order;
  info->s0 = op->s0;
  info->smin = op->smin;
  info->smax = op->smax;
  info->N = op->g.N;
  info->N_half = op->g.Nh;
  info->device_bytes = op->bytes;
  return FW_OK;
}

int fw_op_path(fw_op op) {
  if (!op) {
    set_err(FW_E_ARG, "null op");
    return -1;
  }
  return use_persistent(op) ? FW_PATH_PERSISTENT_2D : FW_PATH_MULTIPASS;
}

int fw_apply(fw_op op, const double* u_host, double* out_host, int m_first, double* imag_residue) {
  if (!op || !u_host || !out_host) return set_err(FW_E_ARG, "null argument");
  if (m_first < 0 || m_first > 1) return set_err(FW_E_ARG, "m_first must be 0 or 1");
  fw_ctx ctx = op->ctx;
  FW_CUDA(cudaSetDevice(ctx->device));
  const fw::GridGeom& g = op->g;
  void *du = nullptr, *dout = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_U, g.N * 8, &du));
  FW_TRY(ctx->get_scratch(SLOT_OUT, g.N * 8, &dout));
  FW_CUDA(cudaMemcpyAsync(du, u_host, g.N * 8, cudaMemcpyHostToDevice, ctx->stream));
  FW_CUDA(cudaMemsetAsync(ctx->residue, 0, sizeof(double), ctx->stream));
  FW_TRY(apply_device(op, (const double*)du, (double*)dout, m_first, imag_residue ? ctx->residue : nullptr, nullptr));
  FW_CUDA(cudaMemcpyAsync(out_host, dout, g.N * 8, cudaMemcpyDeviceToHost, ctx->stream));
  double res = 0.0;
  if (imag_residue) FW_CUDA(cudaMemcpyAsync(&res, ctx->residue, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  FW_CUDA(cudaStreamSynchronize(ctx->stream));
  FW_CUDA(cudaGetLastError());
  if (imag_residue) *imag_residue = res;
  return FW_OK;
}

int fw_apply_device(fw_op op, const double* u_dev, double* out_dev, int m_first, double* imag_residue_dev) {
  if (!op || !u_dev || !out_dev) return set_err(FW_E_ARG, "null argument");
  FW_CUDA(cudaSetDevice(op->ctx->device));
  FW_TRY(apply_device(op, u_dev, out_dev, m_first, imag_residue_dev, nullptr));
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

int fw_apply_batch_device(fw_op const* ops, int nfields, const double* const* u_dev, double* const* out_dev) {
  FW_SETDEV((ops && nfields > 0 && ops[0] ? ops[0]->ctx : nullptr));
  if (!ops || !u_dev || !out_dev || nfields < 0) return set_err(FW_E_ARG, "null argument");
  for (int f = 0; f < nfields; ++f)
    if (!ops[f]) return set_err(FW_E_ARG, "null op in batch");
  if (nfields == 0) return FW_OK;
  // one batched pipeline (grid.z = field) when every field shares grid, context and term range and
  // the grid is not served by the persistent single-launch kernel; else one apply per field
  const fw_op o0 = ops[0];
  bool batch = nfields > 1 && o0->g.d >= 2 && !use_persistent(o0) && !o0->full;
  for (int f = 1; f < nfields && batch; ++f) {
    const fw_op o = ops[f];
    batch = o->ctx == o0->ctx && o->g.d == o0->g.d && o->g.N == o0->g.N && o->M == o0->M &&
            o->constant_order == o0->constant_order && !use_persistent(o) && !o->full;
    for (int a = 0; a < o0->g.d && batch; ++a) batch = o->g.J[a] == o0->g.J[a];
  }
  if (!batch) {
    for (int f = 0; f < nfields; ++f) FW_TRY(apply_device(ops[f], u_dev[f], out_dev[f], 0, nullptr, nullptr));
    FW_CUDA(cudaGetLastError());
    return FW_OK;
  }
  fw_ctx ctx = o0->ctx;
  const fw::GridGeom& g = o0->g;
  const int m_last = o0->constant_order ? 0 : o0->M;
  // L2-resident chunks (FW_BATCH_L2_MB > 0; off by default): the all-terms spectra of the whole
  // batch (64 x 17 x 2.1 MB at C5) make a round trip through HBM between the axis-0 pass and the
  // row C2R.  In this mode a group of fields runs the two kernels over a few terms at a time,
  // sized so that the chunk's spectra (written once, read once, the scratch reused by the next
  // chunk) stay in the 126 MB L2; the row C2R resumes the ascending-m recombination from the
  // partial sums of the earlier chunks (same order of additions, same bits).  Measured at C5
  // (M = 16): 1.72 ms unchunked against 2.2 - 5.4 ms for 56 - 400 MB chunks -- the small launches
  // lose more (per-block set-up amortised over 1-3 terms instead of 17, partial waves) than the
  // HBM round trip costs, so the batch-wide pipeline stays the default.
  const size_t term_bytes = fw::term_elems(ctx->L(), g) * sizeof(double2);
  if (ctx->batch_l2_mb > 0 && ctx->batch_fields == 0 && m_last >= 1 && fw::rows_resumable(ctx->L(), g) &&
      (size_t)nfields * (size_t)(m_last + 1) * term_bytes > ((size_t)ctx->batch_l2_mb << 20)) {
    const int Fg = std::min(nfields, ctx->batch_group);
    const int Tc = (int)std::max<size_t>(1, std::min<size_t>((size_t)(m_last + 1),
                                                              ((size_t)ctx->batch_l2_mb << 20) / ((size_t)Fg * term_bytes)));
    const int nchunk = (m_last + Tc) / Tc;
    void *uh = nullptr, *T = nullptr, *tab = nullptr;
    FW_TRY(ctx->get_scratch(SLOT_BUH, (size_t)Fg * g.Nh * sizeof(double2), &uh));
    FW_TRY(ctx->get_scratch(SLOT_BT, (size_t)Fg * Tc * term_bytes, &T));
    const int ngroup = (nfields + Fg - 1) / Fg;
    const size_t per_group = (size_t)(4 + nchunk) * Fg;  // R2C, forward C2C, axes 1.., C2R, axis 0 per chunk
    FW_TRY(ctx->get_scratch(SLOT_BTAB, (size_t)ngroup * per_group * sizeof(fw::BatchLine), &tab));
    fw::BatchLine* dt = static_cast<fw::BatchLine*>(tab);
    std::vector<fw::BatchLine> h((size_t)ngroup * per_group);
    for (int gi = 0; gi < ngroup; ++gi) {
      const int f0 = gi * Fg, F = std::min(Fg, nfields - f0);
      fw::BatchLine* hg = h.data() + (size_t)gi * per_group;
      for (int i = 0; i < F; ++i) {
        const fw_op o = ops[f0 + i];
        double2* Uh = static_cast<double2*>(uh) + (size_t)i * g.Nh;
        double2* Ti = reinterpret_cast<double2*>(static_cast<char*>(T) + (size_t)i * Tc * term_bytes);
        hg[0 * Fg + i] = {u_dev[f0 + i], Uh, nullptr, nullptr, nullptr};       // R2C
        hg[1 * Fg + i] = {Uh, Uh, nullptr, nullptr, nullptr};                  // forward C2C
        hg[2 * Fg + i] = {Ti, Ti, nullptr, nullptr, nullptr};                  // inverse axes 1..d-2
        hg[3 * Fg + i] = {Ti, nullptr, nullptr, o->dev1, out_dev[f0 + i]};    // C2R + recombination
        for (int c = 0; c < nchunk; ++c)                                       // inverse axis 0 (x w_m) of chunk c
          hg[(size_t)(4 + c) * Fg + i] = {Uh, Ti, o->w + (size_t)c * Tc * g.Nh, nullptr, nullptr};
      }
    }
    FW_CUDA(cudaMemcpyAsync(dt, h.data(), h.size() * sizeof(fw::BatchLine), cudaMemcpyHostToDevice, ctx->stream));
    auto L = ctx->L();
    for (int gi = 0; gi < ngroup; ++gi) {
      const int F = std::min(Fg, nfields - gi * Fg);
      const fw::BatchLine* dg = dt + (size_t)gi * per_group;
      fw::launch_forward_batch(L, g, F, dg, dg + Fg, true);
      for (int c = 0; c < nchunk; ++c) {
        const int m0 = c * Tc, m1 = std::min(m_last, m0 + Tc - 1);
        fw::launch_inverse_batch(L, g, F, m0, m1, dg + (size_t)(4 + c) * Fg, dg + 2 * Fg, dg + 3 * Fg, nullptr, c > 0);
      }
    }
    FW_CUDA(cudaGetLastError());
    return FW_OK;
  }
  const size_t per_field = (size_t)(m_last + 1) * term_bytes;
  // fields per batched pipeline: the all-terms spectra of a chunk live in scratch (up to 16 GiB of
  // the 180 GB HBM); chunks are balanced (64 fields at M = 16 fit in one chunk; an unbalanced
  // 59 + 5 split under a 2 GiB cap left the GPU idle in the small chunk)
  size_t cap = std::max<size_t>(1, std::min<size_t>((size_t)nfields, ((size_t)16 << 30) / per_field));
  if (ctx->batch_fields > 0) cap = std::min<size_t>(cap, (size_t)ctx->batch_fields);  // FW_BATCH_FIELDS (A/B)
  const size_t nchunk = ((size_t)nfields + cap - 1) / cap;
  const int Fc = (int)(((size_t)nfields + nchunk - 1) / nchunk);
  void *uh = nullptr, *T = nullptr, *tab = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_BUH, (size_t)Fc * g.Nh * sizeof(double2), &uh));
  FW_TRY(ctx->get_scratch(SLOT_BT, (size_t)Fc * per_field, &T));
  FW_TRY(ctx->get_scratch(SLOT_BTAB, (size_t)5 * Fc * sizeof(fw::BatchLine), &tab));
  fw::BatchLine* dt = static_cast<fw::BatchLine*>(tab);
  for (int f0 = 0; f0 < nfields; f0 += Fc) {
    const int F = std::min(Fc, nfields - f0);
    std::vector<fw::BatchLine> h((size_t)5 * Fc);
    for (int i = 0; i < F; ++i) {
      const fw_op o = ops[f0 + i];
      double2* Uh = static_cast<double2*>(uh) + (size_t)i * g.Nh;
      double2* Ti = reinterpret_cast<double2*>(static_cast<char*>(T) + (size_t)i * per_field);
      h[0 * Fc + i] = {u_dev[f0 + i], Uh, nullptr, nullptr, nullptr};             // R2C
      h[1 * Fc + i] = {Uh, Uh, nullptr, nullptr, nullptr};                        // forward C2C
      h[2 * Fc + i] = {Uh, Ti, o->w, nullptr, nullptr};                           // inverse axis 0 (x w_m)
      h[3 * Fc + i] = {Ti, Ti, nullptr, nullptr, nullptr};                        // inverse axes 1..d-2
      h[4 * Fc + i] = {Ti, nullptr, nullptr, o->dev1, out_dev[f0 + i]};          // C2R + recombination
    }
    FW_CUDA(cudaMemcpyAsync(dt, h.data(), h.size() * sizeof(fw::BatchLine), cudaMemcpyHostToDevice, ctx->stream));
    auto L = ctx->L();
    fw::launch_forward_batch(L, g, F, dt, dt + Fc, true);
    fw::launch_inverse_batch(L, g, F, 0, m_last, dt + 2 * Fc, dt + 3 * Fc, dt + 4 * Fc);
  }
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

// ---- Grid::dft / forward / inverse and apply_constant_order on the device (fw_dft.cu)
namespace {
int plan_dft(fw_ctx ctx, int dim, const int* J, fw::GridGeom* g) {
  if (!ctx) return set_err(FW_E_ARG, "null ctx");
  bool full = false;
  return plan_grid(dim, J, nullptr, nullptr, g, &full);
}
}  // namespace

int fw_grid_dft_device(fw_ctx ctx, int dim, const int* J, double* data_dev, int sign) {
  FW_SETDEV(ctx);
  fw::GridGeom g;
  FW_TRY(plan_dft(ctx, dim, J, &g));
  if (!data_dev || (sign != -1 && sign != 1)) return set_err(FW_E_ARG, "null data or sign not -1 / +1");
  cudaError_t e = fw::launch_dft(ctx->L(), ctx->chirps, g.d, g.J, sign, (double2*)data_dev);
  if (e != cudaSuccess) return set_err(FW_E_CUDA, std::string("grid dft: ") + cudaGetErrorString(e));
  return FW_OK;
}

int fw_grid_dft(fw_ctx ctx, int dim, const int* J, double* data_host, int sign) {
  FW_SETDEV(ctx);
  fw::GridGeom g;
  FW_TRY(plan_dft(ctx, dim, J, &g));
  if (!data_host) return set_err(FW_E_ARG, "null data");
  void* d = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_UH, g.N * sizeof(double2), &d));
  FW_CUDA(cudaMemcpyAsync(d, data_host, g.N * 16, cudaMemcpyHostToDevice, ctx->stream));
  FW_TRY(fw_grid_dft_device(ctx, dim, J, (double*)d, sign));
  FW_CUDA(cudaMemcpyAsync(data_host, d, g.N * 16, cudaMemcpyDeviceToHost, ctx->stream));
  FW_CUDA(cudaStreamSynchronize(ctx->stream));
  return FW_OK;
}

int fw_grid_forward(fw_ctx ctx, int dim, const int* J, const double* u_host, double* spec_host) {
  FW_SETDEV(ctx);
  fw::GridGeom g;
  FW_TRY(plan_dft(ctx, dim, J, &g));
  if (!u_host || !spec_host) return set_err(FW_E_ARG, "null argument");
  void *du = nullptr, *ds = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_U, g.N * 8, &du));
  FW_TRY(ctx->get_scratch(SLOT_UH, g.N * 16, &ds));
  FW_CUDA(cudaMemcpyAsync(du, u_host, g.N * 8, cudaMemcpyHostToDevice, ctx->stream));
  cudaError_t e = fw::launch_full_forward(ctx->L(), ctx->chirps, g.d, g.J, (long long)g.N, (const double*)du,
                                          (double2*)ds, true);
  if (e != cudaSuccess) return set_err(FW_E_CUDA, std::string("grid forward: ") + cudaGetErrorString(e));
  FW_CUDA(cudaMemcpyAsync(spec_host, ds, g.N * 16, cudaMemcpyDeviceToHost, ctx->stream));
  FW_CUDA(cudaStreamSynchronize(ctx->stream));
  return FW_OK;
}

int fw_grid_inverse(fw_ctx ctx, int dim, const int* J, const double* spec_host, double* u_host,
                    double* imag_residue) {
  FW_SETDEV(ctx);
  fw::GridGeom g;
  FW_TRY(plan_dft(ctx, dim, J, &g));
  if (!u_host || !spec_host) return set_err(FW_E_ARG, "null argument");
  void *du = nullptr, *ds = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_OUT, g.N * 8, &du));
  FW_TRY(ctx->get_scratch(SLOT_UH, g.N * 16, &ds));
  FW_CUDA(cudaMemcpyAsync(ds, spec_host, g.N * 16, cudaMemcpyHostToDevice, ctx->stream));
  FW_CUDA(cudaMemsetAsync(ctx->residue, 0, sizeof(double), ctx->stream));
  cudaError_t e = fw::launch_dft(ctx->L(), ctx->chirps, g.d, g.J, +1, (double2*)ds);
  if (e == cudaSuccess) e = fw::launch_real_part(ctx->L(), (long long)g.N, (const double2*)ds, (double*)du, ctx->residue);
  if (e != cudaSuccess) return set_err(FW_E_CUDA, std::string("grid inverse: ") + cudaGetErrorString(e));
  FW_CUDA(cudaMemcpyAsync(u_host, du, g.N * 8, cudaMemcpyDeviceToHost, ctx->stream));
  double res = 0.0;
  FW_CUDA(cudaMemcpyAsync(&res, ctx->residue, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  FW_CUDA(cudaStreamSynchronize(ctx->stream));
  if (imag_residue) *imag_residue = res;
  return FW_OK;
}

// flap.cpp:13-16
static int check_order(double s) {
  if (!(s > 0.0) || !(s < 2.0)) {
    char b[96];
    snprintf(b, sizeof b, "order s = %f outside (0, 2)", s);
    return set_err(FW_E_ORDER_RANGE, b);
  }
  return FW_OK;
}

int fw_apply_constant_order(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                            const double* u_host, double s, double* out_host, double* imag_residue) {
  FW_SETDEV(ctx);
  if (!ctx || !lo || !hi || !u_host || !out_host) return set_err(FW_E_ARG, "null argument");
  FW_TRY(check_order(s));
  fw::GridGeom g;
  bool full = false;
  FW_TRY(plan_grid(dim, J, lo, hi, &g, &full));
  // inverse(|mu|^{2s} .* forward(u)) (flap.cpp:146-149) is the m = 0 term of a constant-order
  // operator: base symbol pow(mu2, s) on the device tables, the same forward / multiply / inverse
  std::vector<double> sv(g.N, s);
  fw_op op = nullptr;
  FW_TRY(op_create_internal(ctx, g, lo, hi, sv.data(), nullptr, 0, &op, full));
  const int rc = fw_apply(op, u_host, out_host, 0, imag_residue);
  fw_op_destroy(op);
  return rc;
}

int fw_apply_constant_order_spectrum(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                                     const double* spec_host, double s, double* out_host) {
  FW_SETDEV(ctx);
  if (!ctx || !lo || !hi || !spec_host || !out_host) return set_err(FW_E_ARG, "null argument");
  FW_TRY(check_order(s));
  fw::GridGeom g;
  bool full = false;
  FW_TRY(plan_grid(dim, J, lo, hi, &g, &full));
  std::vector<double> f = half_mu2(full_geom(g), lo, hi);  // every bin (grid.cpp:60-80)
  for (size_t k = 0; k < f.size(); ++k) f[k] = f[k] > 0.0 ? pow(f[k], s) : 0.0;  // flap.cpp:143-144
  void *ds = nullptr, *df = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_UH, g.N * 16, &ds));
  FW_TRY(ctx->get_scratch(SLOT_OUT, g.N * 8, &df));
  FW_CUDA(cudaMemcpyAsync(ds, spec_host, g.N * 16, cudaMemcpyHostToDevice, ctx->stream));
  FW_CUDA(cudaMemcpyAsync(df, f.data(), g.N * 8, cudaMemcpyHostToDevice, ctx->stream));
  cudaError_t e = fw::launch_spectrum_mul(ctx->L(), (long long)g.N, (const double*)df, (double2*)ds);
  if (e != cudaSuccess) return set_err(FW_E_CUDA, std::string("constant-order spectrum: ") + cudaGetErrorString(e));
  FW_CUDA(cudaMemcpyAsync(out_host, ds, g.N * 16, cudaMemcpyDeviceToHost, ctx->stream));
  FW_CUDA(cudaStreamSynchronize(ctx->stream));
  return FW_OK;
}

}  // extern "C"

// ---- the dense verification operator (flap.cpp:170-243) and the Toeplitz fast path (flap.cpp:245-285)
struct fw_dense_s {
  fw_ctx ctx = nullptr;
  fw::GridGeom g;
  double* A = nullptr;  // N x N row-major, device-resident
};

extern "C" {

int fw_dense_create(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                    const double* order_values, unsigned long long memory_budget, fw_dense* out) {
  FW_SETDEV(ctx);
  if (!ctx || !lo || !hi || !order_values || !out) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  bool full = false;
  FW_TRY(plan_grid(dim, J, lo, hi, &g, &full));
  double s0, smin, smax;
  int constant;
  FW_TRY(order_stats(order_values, g.N, nullptr, &s0, &smin, &smax, &constant));  // the OrderField
  const unsigned long long required = (unsigned long long)g.N * (unsigned long long)g.N * sizeof(double);
  if (required >= memory_budget) {  // flap.cpp:174-176 (strict bound) with MemoryBudgetExceeded's message
    char b[160];
    snprintf(b, sizeof b, "dense operator needs %llu bytes, budget is %llu", required, memory_budget);
    return set_err(FW_E_MEMORY_BUDGET, b);
  }
  fw_dense d = new fw_dense_s();
  d->ctx = ctx;
  d->g = g;
  std::vector<double> mu2 = half_mu2(full_geom(g), lo, hi);  // every bin (grid.cpp:60-80)
  const long long rows = std::max<long long>(1, std::min<long long>((long long)g.N, (256ll << 20) / (16ll * (long long)g.N)));
  double *dmu2 = nullptr, *ds = nullptr;
  void* G = nullptr;
  int rc = dalloc(&d->A, g.N * g.N);
  if (rc == FW_OK) rc = dalloc(&dmu2, g.N);
  if (rc == FW_OK) rc = dalloc(&ds, g.N);
  if (rc == FW_OK) rc = ctx->get_scratch(SLOT_T, (size_t)rows * g.N * sizeof(double2), &G);
  if (rc == FW_OK) {
    cudaMemcpyAsync(dmu2, mu2.data(), g.N * 8, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(ds, order_values, g.N * 8, cudaMemcpyHostToDevice, ctx->stream);
    cudaError_t e = fw::launch_dense_assemble(ctx->L(), ctx->chirps, g.d, g.J, (long long)g.N, dmu2, ds, (double2*)G,
                                              rows, d->A);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = set_err(FW_E_CUDA, std::string("dense assembly: ") + cudaGetErrorString(e));
  }
  cudaFree(dmu2);
  cudaFree(ds);
  if (rc != FW_OK) {
    fw_dense_destroy(d);
    return rc;
  }
  *out = d;
  return FW_OK;
}

void fw_dense_destroy(fw_dense d) {
  if (!d) return;
  if (d->ctx) cudaSetDevice(d->ctx->device);
  if (d->A) cudaFree(d->A);
  delete d;
}

int fw_dense_apply(fw_dense d, const double* u_host, double* out_host) {
  FW_SETDEV(d ? d->ctx : nullptr);
  if (!d || !u_host || !out_host) return set_err(FW_E_ARG, "null argument");
  fw_ctx ctx = d->ctx;
  void *du = nullptr, *dout = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_U, d->g.N * 8, &du));
  FW_TRY(ctx->get_scratch(SLOT_OUT, d->g.N * 8, &dout));
  FW_CUDA(cudaMemcpyAsync(du, u_host, d->g.N * 8, cudaMemcpyHostToDevice, ctx->stream));
  cudaError_t e = fw::launch_dense_matvec(ctx->L(), (long long)d->g.N, d->A, (const double*)du, (double*)dout);
  if (e != cudaSuccess) return set_err(FW_E_CUDA, std::string("dense apply: ") + cudaGetErrorString(e));
  FW_CUDA(cudaMemcpyAsync(out_host, dout, d->g.N * 8, cudaMemcpyDeviceToHost, ctx->stream));
  FW_CUDA(cudaStreamSynchronize(ctx->stream));
  return FW_OK;
}

int fw_dense_entries(fw_dense d, double* entries_host) {
  FW_SETDEV(d ? d->ctx : nullptr);
  if (!d || !entries_host) return set_err(FW_E_ARG, "null argument");
  FW_CUDA(cudaMemcpyAsync(entries_host, d->A, d->g.N * d->g.N * 8, cudaMemcpyDeviceToHost, d->ctx->stream));
  FW_CUDA(cudaStreamSynchronize(d->ctx->stream));
  return FW_OK;
}

int fw_apply_toeplitz(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                      const double* order_values, const double* u_host, double* out_host) {
  FW_SETDEV(ctx);
  if (!ctx || !lo || !hi || !order_values || !u_host || !out_host) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  bool full = false;
  FW_TRY(plan_grid(dim, J, lo, hi, &g, &full));
  double s0, smin, smax;
  int constant;
  FW_TRY(order_stats(order_values, g.N, nullptr, &s0, &smin, &smax, &constant));
  if (!constant) return set_err(FW_E_NOT_CONSTANT, "toeplitz fast path requires a constant order");  // flap.cpp:247
  if (dim != 1) return set_err(FW_E_DIM_UNSUPPORTED, "toeplitz fast path is one-dimensional");       // flap.cpp:249
  const int n = 2 * J[0];
  if (!fw::dft_length_supported(n)) return set_err(FW_E_UNSUPPORTED, "circulant embedding length beyond the device DFT");
  std::vector<double> mu2 = half_mu2(full_geom(g), lo, hi);
  std::vector<double2> t(J[0]);
  for (int k = 0; k < J[0]; ++k) t[k] = make_double2(mu2[k] > 0.0 ? pow(mu2[k], s0) : 0.0, 0.0);  // flap.cpp:257-258
  void *dt = nullptr, *dc = nullptr, *dx = nullptr, *du = nullptr, *dout = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_UH, (size_t)J[0] * sizeof(double2), &dt));
  FW_TRY(ctx->get_scratch(SLOT_T, (size_t)n * sizeof(double2), &dc));
  FW_TRY(ctx->get_scratch(SLOT_TMP, (size_t)n * sizeof(double2), &dx));
  FW_TRY(ctx->get_scratch(SLOT_U, g.N * 8, &du));
  FW_TRY(ctx->get_scratch(SLOT_OUT, g.N * 8, &dout));
  FW_CUDA(cudaMemcpyAsync(dt, t.data(), t.size() * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  FW_CUDA(cudaMemcpyAsync(du, u_host, g.N * 8, cudaMemcpyHostToDevice, ctx->stream));
  cudaError_t e = fw::launch_toeplitz(ctx->L(), ctx->chirps, J[0], (double2*)dt, (const double*)du, (double2*)dc,
                                      (double2*)dx, (double*)dout);
  if (e != cudaSuccess) return set_err(FW_E_CUDA, std::string("toeplitz: ") + cudaGetErrorString(e));
  FW_CUDA(cudaMemcpyAsync(out_host, dout, g.N * 8, cudaMemcpyDeviceToHost, ctx->stream));
  FW_CUDA(cudaStreamSynchronize(ctx->stream));
  return FW_OK;
}

int fw_truncation_indicator(int M, double mu_abs, double s0, double* out) {
  if (!out) return set_err(FW_E_ARG, "null argument");
  if (!(mu_abs > 0.0)) return set_err(FW_E_NONPOSITIVE_FREQ, "truncation indicator requires |mu| > 0");
  const double l = 2.0 * log(mu_abs);
  double term = pow(mu_abs, 2.0 * s0);
  for (int m = 1; m <= M; ++m) term *= l / m;
  *out = term;
  return FW_OK;
}

int fw_rfftn(fw_ctx ctx, int dim, const int* J, const double* x_host, double* H_host) {
  FW_SETDEV(ctx);
  if (!ctx || !x_host || !H_host) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  FW_TRY(check_grid(dim, J, nullptr, nullptr, &g));
  void *dx = nullptr, *dH = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_U, g.N * 8, &dx));
  FW_TRY(ctx->get_scratch(SLOT_UH, g.Nh * 16, &dH));
  FW_CUDA(cudaMemcpyAsync(dx, x_host, g.N * 8, cudaMemcpyHostToDevice, ctx->stream));
  fw::launch_forward(ctx->L(), g, (const double*)dx, (double2*)dH, false);
  FW_CUDA(cudaMemcpyAsync(H_host, dH, g.Nh * 16, cudaMemcpyDeviceToHost, ctx->stream));
  FW_CUDA(cudaStreamSynchronize(ctx->stream));
  return FW_OK;
}

int fw_irfftn(fw_ctx ctx, int dim, const int* J, const double* H_host, double* x_host) {
  FW_SETDEV(ctx);
  if (!ctx || !x_host || !H_host) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  FW_TRY(check_grid(dim, J, nullptr, nullptr, &g));
  void *dx = nullptr, *dH = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_OUT, g.N * 8, &dx));
  FW_TRY(ctx->get_scratch(SLOT_UH, g.Nh * 16, &dH));
  FW_CUDA(cudaMemcpyAsync(dH, H_host, g.Nh * 16, cudaMemcpyHostToDevice, ctx->stream));
  fw::launch_irfft(ctx->L(), g, (double2*)dH, (double*)dx);
  FW_CUDA(cudaMemcpyAsync(x_host, dx, g.N * 8, cudaMemcpyDeviceToHost, ctx->stream));
  FW_CUDA(cudaStreamSynchronize(ctx->stream));
  return FW_OK;
}

}  // extern "C"

// ===========================================================================
// SeismicStepper

struct fw_seis_s {
  fw_ctx ctx = nullptr;
  fw::GridGeom g;
  fw_op A1 = nullptr, A2 = nullptr;  // dispersion (1+gamma), attenuation (1/2+gamma)
  double tau = 0, thr = 0;
  double *c = nullptr, *eta = nullptr, *tc = nullptr;
  double* ubuf[3] = {nullptr, nullptr, nullptr};
  double* abuf[2] = {nullptr, nullptr};
  double* l1 = nullptr;
  int* flag = nullptr;
  // multi-pass step: both operators' inverses batched (grid.z = operator); device tables for the
  // two parities of the L2 output buffer, rebuilt when the scratch they point into moves
  fw::BatchLine* btab = nullptr;
  const void* btab_uh = nullptr;
  const void* btab_T = nullptr;
  long n = 0;    // reported step count (SeismicStepper::n)
  long lvl = 0;  // index of the current level for buffer rotation
  double* pending_out = nullptr;  // host destination of a pending fw_seis_step_io_async
  double* cur() { return ubuf[lvl % 3]; }
  double* prev() { return ubuf[(lvl + 2) % 3]; }
  double* ap() { return abuf[(lvl + 1) % 2]; }
};

namespace {

void seis_free(fw_seis s) {
  if (!s) return;
  fw_op_destroy(s->A1);
  fw_op_destroy(s->A2);
  for (double* p : {s->c, s->eta, s->tc, s->ubuf[0], s->ubuf[1], s->ubuf[2], s->abuf[0], s->abuf[1], s->l1})
    if (p) cudaFree(p);
  if (s->flag) cudaFree(s->flag);
  if (s->btab) cudaFree(s->btab);
  delete s;
}

// one SeismicStepper::step (seismic.cpp:111-133), enqueued
bool seis_persistent(fw_seis s) {
  return use_persistent(s->A1) && use_persistent(s->A2) && s->A1->constant_order == s->A2->constant_order;
}

// nsteps seismic steps in ONE persistent launch (the kernel rotates the state buffers by level)
int seis_enqueue_persistent(fw_seis s, int nsteps) {
  fw::Step2DParams x{};
  x.seismic = 1;
  x.prev = s->prev();
  x.ap = s->ap();
  x.c = s->c;
  x.eta = s->eta;
  x.tc = s->tc;
  x.next = s->ubuf[(s->lvl + 1) % 3];
  x.tau = s->tau;
  x.thr = s->thr;
  x.step = (int)(s->n + 1);
  x.flag = s->flag;
  x.nsteps = nsteps;
  for (int i = 0; i < 3; ++i) x.ub[i] = s->ubuf[i];
  for (int i = 0; i < 2; ++i) x.ab[i] = s->abuf[i];
  x.lvl0 = s->lvl;
  fw_op ops[2] = {s->A1, s->A2};
  double* outs[2] = {s->l1, s->abuf[s->lvl % 2]};
  FW_TRY(launch_persistent(s->ctx, ops, 2, 0, s->cur(), outs, nullptr, &x));
  s->n += nsteps;
  s->lvl += nsteps;
  return FW_OK;
}

int seis_enqueue_step(fw_seis s) {
  fw_ctx ctx = s->ctx;
  const fw::GridGeom& g = s->g;
  auto L = ctx->L();
  double* cur = s->cur();
  double* l2 = s->abuf[s->lvl % 2];
  double* next = s->ubuf[(s->lvl + 1) % 3];
  if (use_persistent(s->A1) && use_persistent(s->A2) && s->A1->constant_order == s->A2->constant_order) {
    fw::Step2DParams x{};
    x.seismic = 1;
    x.prev = s->prev();
    x.ap = s->ap();
    x.c = s->c;
    x.eta = s->eta;
    x.tc = s->tc;
    x.next = next;
    x.tau = s->tau;
    x.thr = s->thr;
    x.step = (int)(s->n + 1);
    x.flag = s->flag;
    fw_op ops[2] = {s->A1, s->A2};
    double* outs[2] = {s->l1, l2};
    FW_TRY(launch_persistent(ctx, ops, 2, 0, cur, outs, nullptr, &x));
    s->n += 1;
    s->lvl += 1;
    return FW_OK;
  }
  if (s->A1->full) {  // non-power-of-two axes: two C2C applies (each with its own forward DFT)
    FW_TRY(apply_device(s->A1, cur, s->l1, 0, nullptr, nullptr));
    FW_TRY(apply_device(s->A2, cur, l2, 0, nullptr, s->flag));
    fw::launch_seis_update(L, g.N, s->tau, cur, s->prev(), s->ap(), s->l1, l2, s->c, s->eta, s->tc, next, s->thr,
                           (int)(s->n + 1), s->flag);
    s->n += 1;
    s->lvl += 1;
    return FW_OK;
  }
  void* uh = nullptr;
  FW_TRY(ctx->get_scratch(SLOT_UH2, g.Nh * sizeof(double2), &uh));
  // shared forward transform of cur for both operators
  fw::launch_forward(L, g, cur, (double2*)uh, true);
  if (g.d >= 2 && s->A1->M == s->A2->M && s->A1->constant_order == s->A2->constant_order) {
    // both inverses in one batched pipeline (grid.z = operator): twice the blocks per launch
    const int m_last = s->A1->constant_order ? 0 : s->A1->M;
    const size_t per_op = (size_t)(m_last + 1) * fw::term_elems(L, g) * sizeof(double2);
    void* T = nullptr;
    FW_TRY(ctx->get_scratch(SLOT_BT, 2 * per_op, &T));
    if (!s->btab) FW_TRY(dalloc(&s->btab, 12));
    if (s->btab_uh != uh || s->btab_T != T) {
      std::vector<fw::BatchLine> h(12);
      fw_op ops[2] = {s->A1, s->A2};
      for (int par = 0; par < 2; ++par)
        for (int o = 0; o < 2; ++o) {
          double2* To = reinterpret_cast<double2*>(static_cast<char*>(T) + (size_t)o * per_op);
          double* out = o == 0 ? s->l1 : s->abuf[par];
          h[par * 6 + 0 + o] = {uh, To, ops[o]->w, nullptr, nullptr};        // inverse axis 0 (x w_m)
          h[par * 6 + 2 + o] = {To, To, nullptr, nullptr, nullptr};          // axes 1..d-2
          h[par * 6 + 4 + o] = {To, nullptr, nullptr, ops[o]->dev1, out};   // C2R + recombination
        }
      FW_CUDA(cudaMemcpyAsync(s->btab, h.data(), h.size() * sizeof(fw::BatchLine), cudaMemcpyHostToDevice,
                              ctx->stream));
      s->btab_uh = uh;
      s->btab_T = T;
    }
    const fw::BatchLine* t = s->btab + (s->lvl % 2) * 6;
    fw::launch_inverse_batch(L, g, 2, 0, m_last, t, t + 2, t + 4, s->flag);
  } else {
    FW_TRY(apply_device(s->A1, cur, s->l1, 0, nullptr, nullptr, (const double2*)uh));
    FW_TRY(apply_device(s->A2, cur, l2, 0, nullptr, s->flag, (const double2*)uh));
  }
  fw::launch_seis_update(L, g.N, s->tau, cur, s->prev(), s->ap(), s->l1, l2, s->c, s->eta, s->tc, next, s->thr,
                         (int)(s->n + 1), s->flag);
  s->n += 1;
  s->lvl += 1;
  return FW_OK;
}

int seis_check(fw_seis s) {
  int flag = fw::kNoBlowup;
  FW_CUDA(cudaMemcpyAsync(&flag, s->flag, sizeof(int), cudaMemcpyDeviceToHost, s->ctx->stream));
  FW_CUDA(cudaStreamSynchronize(s->ctx->stream));
  FW_CUDA(cudaGetLastError());
  if (flag != fw::kNoBlowup) {
    // state is the one before the offending step; n() is the offending step
    const long steps_after = s->n - flag;  // steps enqueued after the offending one (no-ops)
    s->lvl -= steps_after + 1;
    s->n = flag;
    const int none = fw::kNoBlowup;
    FW_CUDA(cudaMemcpyAsync(s->flag, &none, sizeof(int), cudaMemcpyHostToDevice, s->ctx->stream));
    // launches skipped by the flag did not clear their counter sets: reset both
    FW_CUDA(cudaMemsetAsync(s->ctx->counters, 0, 2 * (size_t)fw::kStep2dCStride * sizeof(unsigned long long),
                            s->ctx->stream));
    FW_CUDA(cudaStreamSynchronize(s->ctx->stream));
    char b[160];
    snprintf(b, sizeof b, "sup|u| > %g at step %d", s->thr, flag);
    return set_err(FW_E_BLOWUP, b);
  }
  return FW_OK;
}

}  // namespace

extern "C" {

int fw_seis_create(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi, const double* gamma,
                   const double* c0, double omega0, int M, const double* phi, const double* psi, double tau,
                   double blowup_factor, fw_seis* out) {
  if (!ctx || !out || !lo || !hi || !gamma || !c0 || !phi || !psi) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  bool full = false;
  FW_TRY(plan_grid(dim, J, lo, hi, &g, &full));
  FW_CUDA(cudaSetDevice(ctx->device));
  const size_t N = g.N;
  for (size_t j = 0; j < N; ++j)  // seismic.cpp:14-19
    if (!(gamma[j] >= 0.0) || !(gamma[j] < 0.5)) {
      char b[128];
      snprintf(b, sizeof b, "gamma = %f outside [0, 0.5)", gamma[j]);
      return set_err(FW_E_GAMMA_RANGE, b);
    }
  std::vector<double> c(N), eta(N), tc(N), ord1(N), ord2(N);
  for (size_t j = 0; j < N; ++j) {  // seismic.cpp:30-39
    const double gj = gamma[j];
    const double cg = c0[j];
    const double scale = pow(cg, 2.0 * gj) * pow(omega0, -2.0 * gj);
    c[j] = cg * cos(0.5 * M_PI * gj);
    eta[j] = -scale * cos(M_PI * gj);
    tc[j] = -(scale / cg) * sin(M_PI * gj);
    ord1[j] = 1.0 + gj;
    ord2[j] = 0.5 + gj;
  }
  fw_seis s = new fw_seis_s();
  s->ctx = ctx;
  s->g = g;
  s->tau = tau;
  int rc = op_create_internal(ctx, g, lo, hi, ord1.data(), nullptr, M, &s->A1, full);
  if (rc == FW_OK) rc = op_create_internal(ctx, g, lo, hi, ord2.data(), nullptr, M, &s->A2, full);
  for (double** p : {&s->c, &s->eta, &s->tc, &s->ubuf[0], &s->ubuf[1], &s->ubuf[2], &s->abuf[0], &s->abuf[1], &s->l1})
    if (rc == FW_OK) rc = dalloc(p, N);
  if (rc == FW_OK) rc = dalloc(&s->flag, 1);
  if (rc != FW_OK) {
    seis_free(s);
    return rc;
  }
  auto L = ctx->L();
  cudaStream_t st = ctx->stream;
  cudaMemcpyAsync(s->c, c.data(), N * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(s->eta, eta.data(), N * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(s->tc, tc.data(), N * 8, cudaMemcpyHostToDevice, st);
  const int none = fw::kNoBlowup;
  cudaMemcpyAsync(s->flag, &none, sizeof(int), cudaMemcpyHostToDevice, st);
  // constructor (seismic.cpp:85-109): prev = phi; cur = Taylor start; atten_prev = A2(phi); n = 1
  double sup = 0.0;
  for (size_t j = 0; j < N; ++j) sup = std::max(sup, std::fabs(phi[j]));
  s->thr = blowup_factor * std::max(sup, 1e-300);
  s->lvl = 1;
  s->n = 1;
  double* d_phi = s->prev();    // ubuf[0]
  double* d_psi = s->ubuf[2];   // temporary
  double* d_l2psi = s->abuf[1]; // temporary
  cudaMemcpyAsync(d_phi, phi, N * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_psi, psi, N * 8, cudaMemcpyHostToDevice, st);
  rc = apply_device(s->A1, d_phi, s->l1, 0, nullptr, nullptr);
  if (rc == FW_OK) rc = apply_device(s->A2, d_psi, d_l2psi, 0, nullptr, nullptr);
  if (rc == FW_OK) {
    fw::launch_seis_start(L, N, tau, d_phi, d_psi, s->c, s->eta, s->tc, s->l1, d_l2psi, s->cur());
    rc = apply_device(s->A2, d_phi, s->ap(), 0, nullptr, nullptr);
  }
  if (rc == FW_OK) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = set_err(FW_E_CUDA, std::string("seismic start: ") + cudaGetErrorString(e));
  }
  if (rc != FW_OK) {
    seis_free(s);
    return rc;
  }
  *out = s;
  return FW_OK;
}

void fw_seis_destroy(fw_seis s) {
  if (s && s->ctx) cudaSetDevice(s->ctx->device);
  if (s && s->ctx) cudaStreamSynchronize(s->ctx->stream);
  seis_free(s);
}

int fw_seis_enqueue(fw_seis s, int nsteps) {
  FW_SETDEV((s ? s->ctx : nullptr));
  if (!s || nsteps < 0) return set_err(FW_E_ARG, "bad argument");
  if (seis_persistent(s) && nsteps > 0) {
    const int per = s->ctx->steps_per_launch > 0 ? s->ctx->steps_per_launch : nsteps;
    for (int done = 0; done < nsteps;) {
      const int k = std::min(per, nsteps - done);
      FW_TRY(seis_enqueue_persistent(s, k));
      done += k;
    }
    FW_CUDA(cudaGetLastError());
    return FW_OK;
  }
  for (int i = 0; i < nsteps; ++i) FW_TRY(seis_enqueue_step(s));
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

int fw_seis_step(fw_seis s, int nsteps) {
  FW_SETDEV((s ? s->ctx : nullptr));
  FW_TRY(fw_seis_enqueue(s, nsteps));
  return seis_check(s);
}

int fw_seis_get(fw_seis s, double* cur_host, double* prev_host, double* atten_prev_host, long* n) {
  FW_SETDEV((s ? s->ctx : nullptr));
  if (!s) return set_err(FW_E_ARG, "null stepper");
  FW_TRY(seis_check(s));
  const size_t N = s->g.N;
  cudaStream_t st = s->ctx->stream;
  if (cur_host) FW_CUDA(cudaMemcpyAsync(cur_host, s->cur(), N * 8, cudaMemcpyDeviceToHost, st));
  if (prev_host) FW_CUDA(cudaMemcpyAsync(prev_host, s->prev(), N * 8, cudaMemcpyDeviceToHost, st));
  if (atten_prev_host) FW_CUDA(cudaMemcpyAsync(atten_prev_host, s->ap(), N * 8, cudaMemcpyDeviceToHost, st));
  FW_CUDA(cudaStreamSynchronize(st));
  if (n) *n = s->n;
  return FW_OK;
}

int fw_seis_set_current(fw_seis s, const double* cur_host) {
  FW_SETDEV((s ? s->ctx : nullptr));
  if (!s || !cur_host) return set_err(FW_E_ARG, "null argument");
  FW_CUDA(cudaMemcpyAsync(s->cur(), cur_host, s->g.N * 8, cudaMemcpyHostToDevice, s->ctx->stream));
  return FW_OK;
}

int fw_seis_step_io_async(fw_seis s, const double* cur_in_host, int nsteps, double* cur_out_host) {
  FW_SETDEV((s ? s->ctx : nullptr));
  if (!s) return set_err(FW_E_ARG, "null stepper");
  const size_t N = s->g.N;
  cudaStream_t st = s->ctx->stream;
  if (cur_in_host) FW_CUDA(cudaMemcpyAsync(s->cur(), cur_in_host, N * 8, cudaMemcpyHostToDevice, st));
  FW_TRY(fw_seis_enqueue(s, nsteps));
  // the new wavefield comes back behind the steps, in stream order; no host synchronisation here
  if (cur_out_host) FW_CUDA(cudaMemcpyAsync(cur_out_host, s->cur(), N * 8, cudaMemcpyDeviceToHost, st));
  s->pending_out = cur_out_host;
  return FW_OK;
}

int fw_seis_wait(fw_seis s) {
  FW_SETDEV((s ? s->ctx : nullptr));
  if (!s) return set_err(FW_E_ARG, "null stepper");
  double* out = s->pending_out;
  s->pending_out = nullptr;
  const int rc = seis_check(s);  // the one host synchronisation: everything enqueued has landed
  if (rc == FW_E_BLOWUP && out) {  // the state was rolled back to before the offending step
    cudaStream_t st = s->ctx->stream;
    FW_CUDA(cudaMemcpyAsync(out, s->cur(), s->g.N * 8, cudaMemcpyDeviceToHost, st));
    FW_CUDA(cudaStreamSynchronize(st));
  }
  return rc;
}

int fw_seis_step_io(fw_seis s, const double* cur_in_host, int nsteps, double* cur_out_host) {
  FW_TRY(fw_seis_step_io_async(s, cur_in_host, nsteps, cur_out_host));
  return fw_seis_wait(s);
}

const double* fw_seis_current_device(fw_seis s) { return s ? s->cur() : nullptr; }

int fw_seis_ops(fw_seis s, fw_op* disp, fw_op* atten) {
  if (!s) return set_err(FW_E_ARG, "null stepper");
  if (disp) *disp = s->A1;
  if (atten) *atten = s->A2;
  return FW_OK;
}

int fw_seis_medium(fw_seis s, double* c, double* eta, double* tau_coef) {
  FW_SETDEV((s ? s->ctx : nullptr));
  if (!s) return set_err(FW_E_ARG, "null stepper");
  const size_t N = s->g.N;
  cudaStream_t st = s->ctx->stream;
  if (c) FW_CUDA(cudaMemcpyAsync(c, s->c, N * 8, cudaMemcpyDeviceToHost, st));
  if (eta) FW_CUDA(cudaMemcpyAsync(eta, s->eta, N * 8, cudaMemcpyDeviceToHost, st));
  if (tau_coef) FW_CUDA(cudaMemcpyAsync(tau_coef, s->tc, N * 8, cudaMemcpyDeviceToHost, st));
  FW_CUDA(cudaStreamSynchronize(st));
  return FW_OK;
}

}  // extern "C"

// ===========================================================================
// TSFP2 (stepping.cpp:119-138, 266-304)

struct fw_tsfp2_s {
  fw_ctx ctx = nullptr;
  fw::GridGeom g;
  fw_op A = nullptr;
  double tau = 0, kappa = 1, thr = 0;
  int cubic = 0;
  double *u = nullptr, *v = nullptr, *pert = nullptr;
  double *w = nullptr, *cw = nullptr, *sw = nullptr;
  double2 *uh = nullptr, *vh = nullptr;
  int* flag = nullptr;
  long n = 0;
};

namespace {

void tsfp2_free(fw_tsfp2 t) {
  if (!t) return;
  fw_op_destroy(t->A);
  for (double* p : {t->u, t->v, t->pert, t->w, t->cw, t->sw})
    if (p) cudaFree(p);
  if (t->uh) cudaFree(t->uh);
  if (t->vh) cudaFree(t->vh);
  if (t->flag) cudaFree(t->flag);
  delete t;
}

void osc_flow(fw_tsfp2 t) {  // oscillator_flow(tau/2), stepping.cpp:271-291
  auto L = t->ctx->L();
  fw::launch_forward(L, t->g, t->u, t->uh, true);
  fw::launch_forward(L, t->g, t->v, t->vh, true);
  fw::launch_osc_rotate(L, t->g.Nh, t->w, t->cw, t->sw, 0.5 * t->tau, t->uh, t->vh);
  // guarded: after a flagged step the later steps of the same call leave (u, v) untouched
  fw::launch_irfft(L, t->g, t->uh, t->u, t->flag);
  fw::launch_irfft(L, t->g, t->vh, t->v, t->flag);
}

}  // namespace

extern "C" {

int fw_tsfp2_create(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                    const double* order_values, int M, double kappa, int f_kind, const double* phi,
                    const double* psi, double tau, double blowup_factor, fw_tsfp2* out) {
  if (!ctx || !out || !lo || !hi || !phi || !psi) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  FW_TRY(check_grid(dim, J, lo, hi, &g));
  FW_CUDA(cudaSetDevice(ctx->device));
  fw_tsfp2 t = new fw_tsfp2_s();
  t->ctx = ctx;
  t->g = g;
  t->tau = tau;
  t->kappa = kappa;
  t->cubic = f_kind == 1 ? 1 : 0;
  int rc = op_create_internal(ctx, g, lo, hi, order_values, nullptr, M, &t->A);
  for (double** p : {&t->u, &t->v, &t->pert})
    if (rc == FW_OK) rc = dalloc(p, g.N);
  for (double** p : {&t->w, &t->cw, &t->sw})
    if (rc == FW_OK) rc = dalloc(p, g.Nh);
  if (rc == FW_OK) rc = dalloc(&t->uh, g.Nh);
  if (rc == FW_OK) rc = dalloc(&t->vh, g.Nh);
  if (rc == FW_OK) rc = dalloc(&t->flag, 1);
  if (rc != FW_OK) {
    tsfp2_free(t);
    return rc;
  }
  // osc_w (stepping.cpp:125-131) and the per-bin rotation for dt = tau/2 on the host (glibc cos/sin)
  std::vector<double> mu2 = half_mu2(g, lo, hi);
  std::vector<double> w(g.Nh), cw(g.Nh), sw(g.Nh);
  const double dt = 0.5 * tau;
  for (size_t k = 0; k < g.Nh; ++k) {
    w[k] = mu2[k] > 0.0 ? sqrt(kappa) * pow(mu2[k], 0.5 * t->A->s0) : 0.0;
    cw[k] = cos(w[k] * dt);
    sw[k] = sin(w[k] * dt);
  }
  double sup = 0.0;
  for (size_t j = 0; j < g.N; ++j) sup = std::max(sup, std::fabs(phi[j]));
  t->thr = blowup_factor * std::max(sup, 1e-300);  // stepping.cpp:121
  cudaStream_t st = ctx->stream;
  cudaMemcpyAsync(t->w, w.data(), g.Nh * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(t->cw, cw.data(), g.Nh * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(t->sw, sw.data(), g.Nh * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(t->u, phi, g.N * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(t->v, psi, g.N * 8, cudaMemcpyHostToDevice, st);
  const int none = fw::kNoBlowup;
  cudaMemcpyAsync(t->flag, &none, sizeof(int), cudaMemcpyHostToDevice, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    tsfp2_free(t);
    return set_err(FW_E_CUDA, std::string("tsfp2 setup: ") + cudaGetErrorString(e));
  }
  *out = t;
  return FW_OK;
}

void fw_tsfp2_destroy(fw_tsfp2 t) {
  if (t && t->ctx) cudaSetDevice(t->ctx->device);
  if (t && t->ctx) cudaStreamSynchronize(t->ctx->stream);
  tsfp2_free(t);
}

int fw_tsfp2_step(fw_tsfp2 t, int nsteps) {
  FW_SETDEV((t ? t->ctx : nullptr));
  if (!t || nsteps < 0) return set_err(FW_E_ARG, "bad argument");
  auto L = t->ctx->L();
  const bool kick = !(t->A->constant_order && !t->cubic);  // stepping.cpp:295
  for (int i = 0; i < nsteps; ++i) {
    osc_flow(t);
    if (kick) {
      FW_TRY(apply_device(t->A, t->u, t->pert, 1, nullptr, nullptr));
      fw::launch_tsfp2_kick(L, t->g.N, t->tau, t->kappa, t->cubic, t->u, t->pert, t->v, t->flag);
    }
    osc_flow(t);
    t->n += 1;
    fw::launch_sup_check(L, t->g.N, t->u, t->thr, (int)t->n, t->flag);
  }
  int flag = fw::kNoBlowup;
  FW_CUDA(cudaMemcpyAsync(&flag, t->flag, sizeof(int), cudaMemcpyDeviceToHost, t->ctx->stream));
  FW_CUDA(cudaStreamSynchronize(t->ctx->stream));
  FW_CUDA(cudaGetLastError());
  if (flag != fw::kNoBlowup) {
    // as the reference's throw from step_tsfp2 (stepping.cpp:302-303): n is the offending step,
    // (u, v) the state right after it (later steps of this call were no-ops on the device)
    t->n = flag;
    const int none = fw::kNoBlowup;
    FW_CUDA(cudaMemcpyAsync(t->flag, &none, sizeof(int), cudaMemcpyHostToDevice, t->ctx->stream));
    FW_CUDA(cudaStreamSynchronize(t->ctx->stream));
    char b[128];
    snprintf(b, sizeof b, "sup|u| > %g at step %d", t->thr, flag);
    return set_err(FW_E_BLOWUP, b);
  }
  return FW_OK;
}

int fw_tsfp2_get(fw_tsfp2 t, double* u_host, double* v_host, long* n) {
  FW_SETDEV((t ? t->ctx : nullptr));
  if (!t) return set_err(FW_E_ARG, "null stepper");
  cudaStream_t st = t->ctx->stream;
  if (u_host) FW_CUDA(cudaMemcpyAsync(u_host, t->u, t->g.N * 8, cudaMemcpyDeviceToHost, st));
  if (v_host) FW_CUDA(cudaMemcpyAsync(v_host, t->v, t->g.N * 8, cudaMemcpyDeviceToHost, st));
  FW_CUDA(cudaStreamSynchronize(st));
  if (n) *n = t->n;
  return FW_OK;
}

}  // extern "C"

// ===========================================================================
// LFFP / CNFP two-level integrators (stepping.cpp:88-104, 119-138, 170-264): the
// reference's Stepper with the Laplacian seam served by the device apply; the state
// and every CG / Picard vector stay in HBM, only scalars cross to the host.

struct fw_wave_s {
  fw_ctx ctx = nullptr;
  fw::GridGeom g;
  fw_op A = nullptr;
  int method = 0, cubic = 0;
  double tau = 0, kappa = 1, thr = 0, picard_tol = 0, cg_tol = 0;
  int picard_max = 0, cg_max = 0;
  double* ub[3] = {nullptr, nullptr, nullptr};  // level L lives in ub[L % 3]
  long lvl = 1;                                 // level of cur (= n except after a blow-up)
  long n = 1, picard_total = 0;
  double *lu = nullptr, *rhs0 = nullptr, *rhs = nullptr, *wa = nullptr, *wb = nullptr;
  double *r = nullptr, *p = nullptr, *ap = nullptr, *part = nullptr, *scal = nullptr;
  double* hs = nullptr;  // pinned host scalars
  int* flag = nullptr;
};

namespace {

void wave_free(fw_wave t) {
  if (!t) return;
  fw_op_destroy(t->A);
  for (double* q : {t->ub[0], t->ub[1], t->ub[2], t->lu, t->rhs0, t->rhs, t->wa, t->wb, t->r, t->p, t->ap, t->part,
                    t->scal})
    if (q) cudaFree(q);
  if (t->hs) cudaFreeHost(t->hs);
  if (t->flag) cudaFree(t->flag);
  delete t;
}

// host values of k reductions queued into scal[0..k)
int wave_scalars(fw_wave t, int k) {
  FW_CUDA(cudaMemcpyAsync(t->hs, t->scal, k * sizeof(double), cudaMemcpyDeviceToHost, t->ctx->stream));
  FW_CUDA(cudaStreamSynchronize(t->ctx->stream));
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

// CG on (I + alpha L) x = rhs, warm start at rhs (stepping.cpp:183-221)
int wave_cg(fw_wave t, const double* rhs, double* x, double alpha) {
  auto L = t->ctx->L();
  const size_t N = t->g.N;
  cudaStream_t st = t->ctx->stream;
  FW_CUDA(cudaMemcpyAsync(x, rhs, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  FW_TRY(apply_device(t->A, x, t->lu, 0, nullptr, nullptr));
  fw::launch_cg_apply_a(L, N, alpha, x, t->lu, rhs, t->r);  // r = rhs - A x
  fw::launch_dot(L, N, 0, rhs, rhs, t->part, t->scal + 0);
  fw::launch_dot(L, N, 0, t->r, t->r, t->part, t->scal + 1);
  FW_TRY(wave_scalars(t, 2));
  const double rhs_norm = std::max(std::sqrt(t->hs[0]), 1e-300);
  double rr = t->hs[1];
  if (std::sqrt(rr) <= t->cg_tol * rhs_norm) return FW_OK;
  FW_CUDA(cudaMemcpyAsync(t->p, t->r, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  for (int it = 0; it < t->cg_max; ++it) {
    FW_TRY(apply_device(t->A, t->p, t->lu, 0, nullptr, nullptr));
    fw::launch_cg_apply_a(L, N, alpha, t->p, t->lu, nullptr, t->ap);  // ap = A p
    fw::launch_dot(L, N, 0, t->p, t->ap, t->part, t->scal);
    FW_TRY(wave_scalars(t, 1));
    const double pap = t->hs[0];
    if (pap == 0.0) return set_err(FW_E_CG_STAGNATED, "zero curvature in conjugate gradient");
    const double a = rr / pap;
    fw::launch_cg_step(L, N, a, t->p, t->ap, x, t->r);
    fw::launch_dot(L, N, 0, t->r, t->r, t->part, t->scal);
    FW_TRY(wave_scalars(t, 1));
    const double rr_new = t->hs[0];
    if (std::sqrt(rr_new) <= t->cg_tol * rhs_norm) return FW_OK;
    const double beta = rr_new / rr;
    rr = rr_new;
    fw::launch_cg_dir(L, N, beta, t->r, t->p);
  }
  return set_err(FW_E_CG_STAGNATED,
                 "conjugate gradient failed to converge in " + std::to_string(t->cg_max) + " iterations");
}

// one CNFP step into ub[(lvl + 1) % 3] (stepping.cpp:223-264); blow-up check left to the caller
int wave_cnfp(fw_wave t) {
  auto L = t->ctx->L();
  const size_t N = t->g.N;
  const double t2 = t->tau * t->tau;
  const double alpha = 0.5 * t->kappa * t2;
  const double* cur = t->ub[t->lvl % 3];
  const double* prev = t->ub[(t->lvl + 2) % 3];
  double* out = t->ub[(t->lvl + 1) % 3];
  FW_TRY(apply_device(t->A, prev, t->lu, 0, nullptr, nullptr));
  fw::launch_cnfp_rhs0(L, N, t2, alpha, t->cubic, cur, prev, t->lu, t->rhs0);
  if (!t->cubic) {
    FW_TRY(wave_cg(t, t->rhs0, out, alpha));
    ++t->picard_total;
    return FW_OK;
  }
  // Picard on w = u^{n+1}, starting from u^n; iterates alternate between two buffers
  double* w = t->wa;
  double* wn = t->wb;
  FW_CUDA(cudaMemcpyAsync(w, cur, N * sizeof(double), cudaMemcpyDeviceToDevice, t->ctx->stream));
  for (int it = 0; it < t->picard_max; ++it) {
    fw::launch_cnfp_rhs(L, N, t2, t->rhs0, w, t->rhs);
    FW_TRY(wave_cg(t, t->rhs, wn, alpha));
    fw::launch_dot(L, N, 1, wn, w, t->part, t->scal + 0);  // sum (w_next - w)^2
    fw::launch_dot(L, N, 0, wn, wn, t->part, t->scal + 1);  // |w_next|^2
    FW_TRY(wave_scalars(t, 2));
    ++t->picard_total;
    std::swap(w, wn);
    if (std::sqrt(t->hs[0]) <= t->picard_tol * std::max(1.0, std::sqrt(t->hs[1]))) {
      FW_CUDA(cudaMemcpyAsync(out, w, N * sizeof(double), cudaMemcpyDeviceToDevice, t->ctx->stream));
      return FW_OK;
    }
  }
  return set_err(FW_E_PICARD_DIVERGED, "fixed-point iteration cap hit at step " + std::to_string(t->n));
}

}  // namespace

extern "C" {

int fw_wave_create(fw_ctx ctx, int method, int dim, const int* J, const double* lo, const double* hi,
                   const double* order_values, int M, double kappa, int f_kind, const double* phi,
                   const double* psi, double tau, double picard_tol, int picard_max_iters, double inner_cg_tol,
                   int cg_max_iters, double blowup_factor, fw_wave* out) {
  if (!ctx || !out || !lo || !hi || !phi || !psi) return set_err(FW_E_ARG, "null argument");
  if (method != 0 && method != 1) return set_err(FW_E_ARG, "method must be 0 (LFFP) or 1 (CNFP)");
  if (f_kind != 0 && f_kind != 1) return set_err(FW_E_ARG, "f must be 0 (none) or 1 (cubic)");
  fw::GridGeom g;
  FW_TRY(check_grid(dim, J, lo, hi, &g));
  FW_CUDA(cudaSetDevice(ctx->device));
  fw_wave t = new fw_wave_s();
  t->ctx = ctx;
  t->g = g;
  t->method = method;
  t->cubic = f_kind;
  t->tau = tau;
  t->kappa = kappa;
  t->picard_tol = picard_tol;
  t->picard_max = picard_max_iters;
  t->cg_tol = inner_cg_tol;
  t->cg_max = cg_max_iters;
  int rc = op_create_internal(ctx, g, lo, hi, order_values, nullptr, M, &t->A);
  for (double** q : {&t->ub[0], &t->ub[1], &t->ub[2], &t->lu})
    if (rc == FW_OK) rc = dalloc(q, g.N);
  if (method == 1)
    for (double** q : {&t->rhs0, &t->rhs, &t->wa, &t->wb, &t->r, &t->p, &t->ap})
      if (rc == FW_OK) rc = dalloc(q, g.N);
  if (rc == FW_OK) rc = dalloc(&t->part, fw::wave_partials());
  if (rc == FW_OK) rc = dalloc(&t->scal, 4);
  if (rc == FW_OK) rc = dalloc(&t->flag, 1);
  if (rc == FW_OK && cudaMallocHost((void**)&t->hs, 4 * sizeof(double)) != cudaSuccess) rc = FW_E_OOM;
  if (rc != FW_OK) {
    wave_free(t);
    return rc == FW_E_OOM ? set_err(FW_E_OOM, "wave stepper allocation") : rc;
  }
  // blowup_threshold_ = factor * max(sup|phi|, 1e-300) (stepping.cpp:121), std::max semantics
  double sup = 0.0;
  for (size_t j = 0; j < g.N; ++j) sup = std::max(sup, std::fabs(phi[j]));
  t->thr = blowup_factor * std::max(sup, 1e-300);
  cudaStream_t st = ctx->stream;
  const int none = fw::kNoBlowup;
  cudaMemcpyAsync(t->flag, &none, sizeof(int), cudaMemcpyHostToDevice, st);
  // initial_levels (stepping.cpp:88-104): u^0 = phi, u^1 = Taylor start; psi staged in ub[2]
  cudaMemcpyAsync(t->ub[0], phi, g.N * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(t->ub[2], psi, g.N * 8, cudaMemcpyHostToDevice, st);
  rc = apply_device(t->A, t->ub[0], t->lu, 0, nullptr, nullptr);
  if (rc == FW_OK) {
    fw::launch_wave_start(ctx->L(), g.N, tau, kappa, t->cubic, t->ub[0], t->ub[2], t->lu, t->ub[1]);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) rc = set_err(FW_E_CUDA, std::string("wave setup: ") + cudaGetErrorString(e));
  }
  if (rc != FW_OK) {
    wave_free(t);
    return rc;
  }
  t->lvl = 1;
  t->n = 1;  // cur_ is u^1
  *out = t;
  return FW_OK;
}

void fw_wave_destroy(fw_wave t) {
  if (t && t->ctx) cudaSetDevice(t->ctx->device);
  if (t && t->ctx) cudaStreamSynchronize(t->ctx->stream);
  wave_free(t);
}

int fw_wave_step(fw_wave t, int nsteps) {
  FW_SETDEV((t ? t->ctx : nullptr));
  if (!t || nsteps < 0) return set_err(FW_E_ARG, "bad argument");
  auto L = t->ctx->L();
  const size_t N = t->g.N;
  cudaStream_t st = t->ctx->stream;
  const double t2 = t->tau * t->tau;
  const long lvl0 = t->lvl, n0 = t->n;
  if (t->method == 0) {
    // LFFP: the whole batch is enqueued; a blow-up freezes the later updates (stepping.cpp:170-181)
    for (int i = 0; i < nsteps; ++i) {
      const long l = lvl0 + i;
      FW_TRY(apply_device(t->A, t->ub[l % 3], t->lu, 0, nullptr, nullptr));
      fw::launch_lffp_update(L, N, t2, t->kappa, t->cubic, t->ub[l % 3], t->ub[(l + 2) % 3], t->lu,
                             t->ub[(l + 1) % 3], t->flag);
      fw::launch_sup_check(L, N, t->ub[(l + 1) % 3], t->thr, (int)(n0 + i + 1), t->flag);
    }
    t->lvl = lvl0 + nsteps;
    t->n = n0 + nsteps;
  } else {
    for (int i = 0; i < nsteps; ++i) {
      int rc = wave_cnfp(t);
      if (rc != FW_OK) return rc;  // state unchanged, n not incremented (the reference throws before ++n_)
      fw::launch_sup_check(L, N, t->ub[(t->lvl + 1) % 3], t->thr, (int)(t->n + 1), t->flag);
      int flag = fw::kNoBlowup;
      FW_CUDA(cudaMemcpyAsync(&flag, t->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
      FW_CUDA(cudaStreamSynchronize(st));
      t->n += 1;
      if (flag != fw::kNoBlowup) break;
      t->lvl += 1;
    }
  }
  int flag = fw::kNoBlowup;
  FW_CUDA(cudaMemcpyAsync(&flag, t->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  FW_CUDA(cudaStreamSynchronize(st));
  FW_CUDA(cudaGetLastError());
  if (flag != fw::kNoBlowup) {
    // the reference increments n_ and throws before rotating: state = the levels before step `flag`
    t->n = flag;
    t->lvl = lvl0 + (flag - n0) - 1;
    const int none = fw::kNoBlowup;
    FW_CUDA(cudaMemcpyAsync(t->flag, &none, sizeof(int), cudaMemcpyHostToDevice, st));
    FW_CUDA(cudaStreamSynchronize(st));
    char b[128];
    snprintf(b, sizeof b, "sup|u| > %g at step %d", t->thr, flag);
    return set_err(FW_E_BLOWUP, b);
  }
  return FW_OK;
}

int fw_wave_get(fw_wave t, double* cur_host, double* prev_host, long* n, long* picard_total) {
  FW_SETDEV((t ? t->ctx : nullptr));
  if (!t) return set_err(FW_E_ARG, "null stepper");
  cudaStream_t st = t->ctx->stream;
  if (cur_host) FW_CUDA(cudaMemcpyAsync(cur_host, t->ub[t->lvl % 3], t->g.N * 8, cudaMemcpyDeviceToHost, st));
  if (prev_host)
    FW_CUDA(cudaMemcpyAsync(prev_host, t->ub[(t->lvl + 2) % 3], t->g.N * 8, cudaMemcpyDeviceToHost, st));
  FW_CUDA(cudaStreamSynchronize(st));
  if (n) *n = t->n;
  if (picard_total) *picard_total = t->picard_total;
  return FW_OK;
}

}  // extern "C"

// ===========================================================================
// stage entry points: the pipeline's kernels on caller-provided device sub-arrays
// (used by the slab-decomposed multi-GPU apply, paper_2311_13049_b200/slab.py)

extern "C" {

int fw_stage_r2c(fw_ctx ctx, int dim, const int* J, const double* x_dev, double* H_dev, double scale) {
  FW_SETDEV(ctx);
  if (!ctx || !x_dev || !H_dev) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  FW_TRY(check_grid(dim, J, nullptr, nullptr, &g));
  fw::launch_stage_r2c(ctx->L(), g, x_dev, (double2*)H_dev, scale, scale != 1.0);
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

int fw_stage_c2c(fw_ctx ctx, int dim, const int* J, int axis, int dir, const double* src_dev, double* dst_dev,
                 const double* w_dev, long long src_ts, long long dst_ts, long long w_ts, int nterms, double scale) {
  FW_SETDEV(ctx);
  if (!ctx || !src_dev || !dst_dev || nterms < 1) return set_err(FW_E_ARG, "bad argument");
  fw::GridGeom g;
  FW_TRY(check_grid(dim, J, nullptr, nullptr, &g));
  if (axis < 0 || axis > dim - 2) return set_err(FW_E_ARG, "axis must be < dim-1 (the last axis is the halved one)");
  fw::launch_stage_c2c(ctx->L(), g, axis, dir < 0 ? -1 : +1, (const double2*)src_dev, (double2*)dst_dev, w_dev, src_ts,
                       dst_ts, w_ts, nterms, scale, scale != 1.0);
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

int fw_medium_coefficients(long long n, const double* gamma, const double* c0, double omega0, double* c_out,
                           double* eta_out, double* tau_coef_out) {
  if (n < 0 || !gamma || !c0 || !c_out || !eta_out || !tau_coef_out) return set_err(FW_E_ARG, "null argument");
  for (long long j = 0; j < n; ++j)  // seismic.cpp:14-19
    if (!(gamma[j] >= 0.0) || !(gamma[j] < 0.5)) {
      char b[128];
      snprintf(b, sizeof b, "gamma = %f outside [0, 0.5)", gamma[j]);
      return set_err(FW_E_GAMMA_RANGE, b);
    }
  for (long long j = 0; j < n; ++j) {  // seismic.cpp:30-39 (the same expressions as fw_seis_create)
    const double gj = gamma[j];
    const double cg = c0[j];
    const double scale = pow(cg, 2.0 * gj) * pow(omega0, -2.0 * gj);
    c_out[j] = cg * cos(0.5 * M_PI * gj);
    eta_out[j] = -scale * cos(M_PI * gj);
    tau_coef_out[j] = -(scale / cg) * sin(M_PI * gj);
  }
  return FW_OK;
}

int fw_ricker_initial(int dim, const int* J, const double* lo, const double* hi, double nu0, const double* xc,
                      double* out) {
  if (!J || !lo || !hi || !xc || !out) return set_err(FW_E_ARG, "null argument");
  fw::GridGeom g;
  FW_TRY(check_grid_ref(dim, J, lo, hi, &g));
  double h[3] = {0, 0, 0};
  for (int m = 0; m < dim; ++m) h[m] = (hi[m] - lo[m]) / J[m];  // grid.cpp:56
  const double a = M_PI * M_PI * nu0 * nu0;                        // seismic.cpp:72
  for (size_t j = 0; j < g.N; ++j) {
    size_t rem = j;
    double x[3] = {0, 0, 0};
    for (int m = dim - 1; m >= 0; --m) {  // Grid::point (grid.cpp:107-116)
      const size_t jm = rem % (size_t)J[m];
      rem /= (size_t)J[m];
      x[m] = lo[m] + jm * h[m];
    }
    double r2 = 0.0;
    for (int m = 0; m < dim; ++m) {
      const double d = x[m] - xc[m];
      r2 += d * d;
    }
    out[j] = (1.0 - 2.0 * a * r2) * exp(-a * r2);  // seismic.cpp:80
  }
  return FW_OK;
}

int fw_stage_seis_start(fw_ctx ctx, long long n, double tau, const double* phi, const double* psi, const double* c,
                        const double* eta, const double* tau_coef, const double* l1phi, const double* l2psi,
                        double* cur) {
  FW_SETDEV(ctx);
  if (!ctx || n < 0 || !phi || !psi || !c || !eta || !tau_coef || !l1phi || !l2psi || !cur)
    return set_err(FW_E_ARG, "null argument");
  fw::launch_seis_start(ctx->L(), (size_t)n, tau, phi, psi, c, eta, tau_coef, l1phi, l2psi, cur);
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

int fw_stage_seis_update(fw_ctx ctx, long long n, double tau, const double* cur, const double* prev,
                         const double* l2prev, const double* l1, const double* l2, const double* c, const double* eta,
                         const double* tau_coef, double* next, double thr, int step, int* flag_dev) {
  FW_SETDEV(ctx);
  if (!ctx || n < 0 || !cur || !prev || !l2prev || !l1 || !l2 || !c || !eta || !tau_coef || !next || !flag_dev)
    return set_err(FW_E_ARG, "null argument");
  fw::launch_seis_update(ctx->L(), (size_t)n, tau, cur, prev, l2prev, l1, l2, c, eta, tau_coef, next, thr, step,
                         flag_dev);
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

int fw_stage_seis_update_peers(fw_ctx ctx, long long n, double tau, const double* cur, const double* prev,
                               const double* l2prev, const double* l1, const double* l2, const double* c,
                               const double* eta, const double* tau_coef, double* next, double* l2out, double thr,
                               int step, int* flag_dev, int npeers, int* const* peer_flags_dev) {
  FW_SETDEV(ctx);
  if (!ctx || n < 0 || !cur || !prev || !l2prev || !l1 || !l2 || !c || !eta || !tau_coef || !next || !l2out || !flag_dev ||
      npeers < 0 || npeers > fw::kMaxPeers || (npeers > 0 && !peer_flags_dev))
    return set_err(FW_E_ARG, "bad argument");
  fw::PeerFlags pf;
  pf.n = npeers;
  for (int q = 0; q < npeers; ++q) pf.f[q] = peer_flags_dev[q];
  fw::launch_seis_update_peers(ctx->L(), (size_t)n, tau, cur, prev, l2prev, l1, l2, c, eta, tau_coef, next, l2out, thr,
                               step, flag_dev, pf);
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

// receive buffers for peer stores: plain cudaMalloc allocations, so that a peer's
// cudaIpcOpenMemHandle maps exactly this address (a handle maps the allocation BASE)
int fw_ipc_alloc(fw_ctx ctx, size_t bytes, void** dev_ptr_out) {
  FW_SETDEV(ctx);
  if (!ctx || !dev_ptr_out || bytes == 0) return set_err(FW_E_ARG, "bad argument");
  FW_CUDA(cudaMalloc(dev_ptr_out, bytes));
  return FW_OK;
}

int fw_ipc_free(fw_ctx ctx, void* dev_ptr) {
  FW_SETDEV(ctx);
  if (dev_ptr) FW_CUDA(cudaFree(dev_ptr));
  return FW_OK;
}

int fw_ipc_handle(const void* dev_ptr, unsigned char handle_out[64]) {
  if (!dev_ptr || !handle_out) return set_err(FW_E_ARG, "null argument");
  {  // a handle maps the allocation base: refuse interior pointers (e.g. a caching allocator's block)
    static PFN_cuMemGetAddressRange_v3020 range = nullptr;
    if (!range) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", (void**)&range, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        range = nullptr;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range && range(&base, &size, (CUdeviceptr)dev_ptr) == CUDA_SUCCESS && base != (CUdeviceptr)dev_ptr)
      return set_err(FW_E_ARG, "IPC export of an interior pointer (the peer would map the allocation base); "
                               "allocate the buffer with fw_ipc_alloc");
  }
  cudaIpcMemHandle_t h;
  FW_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  static_assert(sizeof(h) == 64, "CUDA IPC handle size");
  memcpy(handle_out, &h, 64);
  return FW_OK;
}

int fw_ipc_open(const unsigned char handle[64], void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return set_err(FW_E_ARG, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  FW_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return FW_OK;
}

int fw_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return set_err(FW_E_ARG, "null argument");
  FW_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return FW_OK;
}

int fw_stage_c2c_scatter(fw_ctx ctx, int dim, const int* J, int axis, int dir, const double* src_dev,
                         const double* w_dev, long long src_ts, long long w_ts, int nterms, double scale, int nq,
                         double* const* dst_q, long long blk, long long jstride, long long ostride,
                         long long tstride, long long base) {
  FW_SETDEV(ctx);
  if (!ctx || !src_dev || !dst_q || nterms < 1 || nq < 1 || nq > fw::kMaxScatter || blk < 1)
    return set_err(FW_E_ARG, "bad argument");
  fw::GridGeom g;
  FW_TRY(check_grid(dim, J, nullptr, nullptr, &g));
  if (axis < 0 || axis > dim - 2) return set_err(FW_E_ARG, "axis must be < dim-1 (the last axis is the halved one)");
  const int n = g.J[axis];
  if ((long long)nq * blk < n) return set_err(FW_E_ARG, "nq * blk must cover the axis");
  fw::Scatter sc{};
  for (int q = 0; q < nq; ++q) {
    if (!dst_q[q]) return set_err(FW_E_ARG, "null destination");
    sc.dst[q] = reinterpret_cast<double2*>(dst_q[q]);
  }
  sc.nq = nq;
  sc.blk = blk;
  sc.lgblk = -1;
  if (blk > 0 && (blk & (blk - 1)) == 0 && blk < (1ll << 30))
    for (sc.lgblk = 0; (1ll << sc.lgblk) < blk; ++sc.lgblk) {
    }
  sc.jstride = jstride;
  sc.ostride = ostride;
  sc.tstride = tstride;
  sc.base = base;
  long long S = g.hp1;
  for (int b = axis + 1; b <= g.d - 2; ++b) S *= g.J[b];
  long long outer = 1;
  for (int b = 0; b < axis; ++b) outer *= g.J[b];
  if (!fw::launch_lines(ctx->L(), n, dir < 0 ? -1 : +1, (const double2*)src_dev, nullptr, w_dev, S, outer, S, src_ts,
                        0, w_ts, nterms, 1, scale, scale != 1.0, nullptr, &sc))
    return set_err(FW_E_UNSUPPORTED, "fused transpose: axis length must be 256, 512 or 1024");
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

int fw_stage_c2r_accum(fw_ctx ctx, int dim, const int* J, const double* src_dev, long long src_ts, int m_first,
                       int m_last, const double* dev1_dev, double* out_dev, double* residue_dev) {
  FW_SETDEV(ctx);
  if (!ctx || !src_dev || !out_dev || m_last < m_first) return set_err(FW_E_ARG, "bad argument");
  fw::GridGeom g;
  FW_TRY(check_grid(dim, J, nullptr, nullptr, &g));
  fw::launch_stage_c2r(ctx->L(), g, (const double2*)src_dev, src_ts, m_first, m_last, dev1_dev, out_dev, residue_dev);
  FW_CUDA(cudaGetLastError());
  return FW_OK;
}

int fw_op_device_tables(fw_op op, const double** w_dev, const double** dev1_dev, int* m_last) {
  if (!op) return set_err(FW_E_ARG, "null op");
  if (w_dev) *w_dev = op->w;
  if (dev1_dev) *dev1_dev = op->dev1;
  if (m_last) *m_last = op->constant_order ? 0 : op->M;
  return FW_OK;
}

}  // extern "C"
