// flap_gpu.cpp — drop-in replacement of the reference's matrix-free operator entry
// points (proj/include/fracwave/flap.hpp:34-41, proj/src/flap.cpp:151-168) backed by
// the B200 C-ABI (include/fw_capi.h).  Built INTO the reference: flap.cpp is compiled
// with -Dapply_matrix_free=fwref_apply_matrix_free (etc.) so its CPU versions keep
// existing under other names, and every caller (SeismicStepper, MatrixFreeLaplacian,
// harness, tests) transparently reaches the GPU.  See INTEGRATION.md.
//
// Semantics follow the reference: GridMismatch when the field lives on another grid
// (flap.cpp:40-41), exact zeros for the perturbation of a constant order
// (flap.cpp:163-166), the imaginary residue through the optional pointer.  C-ABI
// status codes are re-thrown as the matching fwave exception type (errors.hpp).
// Every grid the reference accepts runs on the device (power-of-two axes on the real-transform
// pipeline, other lengths on the full-spectrum C2C form); lengths past the device transforms'
// reach raise fwave::Error: there is no silent CPU fallback.  The reference's own FFTW calls
// (Grid::dft, apply_toeplitz) are served by the device too (fftw_gpu.cpp).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "dropin_ctx.hpp"
#include "fracwave/errors.hpp"
#include "fracwave/flap.hpp"
#include "fw_capi.h"

namespace fwave {

namespace {

[[noreturn]] void rethrow(int rc) {
  const std::string msg = std::string("B200 backend: ") + fw_last_error();
  switch (rc) {
    case FW_E_GRID_MISMATCH: throw GridMismatch(msg);
    case FW_E_NEGATIVE_M: throw NegativeM(msg);
    case FW_E_ORDER_RANGE: throw OrderOutOfRange(msg);
    case FW_E_DEVIATION: throw DeviationTooLarge(msg);
    case FW_E_GAMMA_RANGE: throw GammaOutOfRange(msg);
    case FW_E_BLOWUP: throw BlowupDetected(msg);
    case FW_E_ODD_SIZE: throw OddSize(msg);
    case FW_E_EMPTY_INTERVAL: throw EmptyInterval(msg);
    case FW_E_DIM_RANGE: throw DimOutOfRange(msg);
    default: throw Error(msg);
  }
}

void check(int rc) {
  if (rc != FW_OK) rethrow(rc);
}

long g_calls = 0;

struct Entry {
  std::uint64_t hash;
  fw_op op;
};
std::unordered_map<const ExpansionOperator*, Entry> g_cache;

std::uint64_t mix(std::uint64_t h, const double* p, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i) {
    std::uint64_t x;
    std::memcpy(&x, p + i, 8);
    h ^= x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  }
  return h;
}

// fingerprint of everything uploaded (grid, M, s0, flags, tables)
std::uint64_t fingerprint(const ExpansionOperator& op) {
  const Grid& g = op.grid;
  std::uint64_t h = 1469598103934665603ull;
  double meta[12] = {double(g.dim()), double(op.M), op.order.s0(), op.constant_order ? 1.0 : 0.0};
  for (int m = 0; m < g.dim(); ++m) {
    meta[4 + 3 * m] = g.size(m);
    meta[5 + 3 * m] = g.lo(m);
    meta[6 + 3 * m] = g.hi(m);
  }
  h = mix(h, meta, 12);
  h = mix(h, op.base_symbol.data(), op.base_symbol.size());
  for (const auto& t : op.log_weights) h = mix(h, t.data(), t.size());
  if (!op.deviation_powers.empty()) h = mix(h, op.deviation_powers[0].data(), op.deviation_powers[0].size());
  return h;
}

fw_op device_op(const ExpansionOperator& op) {
  fw_ctx ctx = gpu_dropin::context();
  const std::uint64_t h = fingerprint(op);
  auto it = g_cache.find(&op);
  if (it != g_cache.end()) {
    if (it->second.hash == h) return it->second.op;
    fw_op_destroy(it->second.op);
    g_cache.erase(it);
  }
  const Grid& g = op.grid;
  int J[3] = {1, 1, 1};
  double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
  for (int m = 0; m < g.dim(); ++m) {
    J[m] = g.size(m);
    lo[m] = g.lo(m);
    hi[m] = g.hi(m);
  }
  std::vector<const double*> lw(op.M), dv(op.M);
  for (int m = 0; m < op.M; ++m) {
    lw[m] = op.log_weights[m].data();
    dv[m] = op.deviation_powers[m].data();
  }
  fw_op d = nullptr;
  check(fw_op_create_from_tables(ctx, g.dim(), J, lo, hi, op.M, op.order.s0(), op.constant_order ? 1 : 0,
                                 op.base_symbol.data(), op.M ? lw.data() : nullptr, op.M ? dv.data() : nullptr,
                                 &d));
  g_cache[&op] = Entry{h, d};
  return d;
}

Field apply_gpu(const ExpansionOperator& op, const Field& u, int m_first, double* imag_residue) {
  if (!u.grid().same_as(op.grid)) throw GridMismatch("field defined on a different grid than the operator");
  std::lock_guard<std::mutex> lock(gpu_dropin::mutex());
  fw_op d = device_op(op);
  Field out(op.grid, 0.0);
  check(fw_apply(d, u.values().data(), out.values().data(), m_first, imag_residue));
  ++g_calls;
  return out;
}

struct Report {
  ~Report() {
    if (std::getenv("FW_DROPIN_REPORT"))
      std::fprintf(stderr, "[fw-dropin] %ld operator applies ran on the B200 backend\n", g_calls);
  }
} g_report;

}  // namespace

namespace gpu_dropin {
std::mutex& mutex() {
  static std::mutex mu;
  return mu;
}
fw_ctx context() {
  static fw_ctx ctx = [] {
    fw_ctx c = nullptr;
    const char* dev = std::getenv("FW_DEVICE");
    check(fw_ctx_create(dev ? std::atoi(dev) : 0, &c));
    return c;
  }();
  return ctx;
}
}  // namespace gpu_dropin

Field apply_matrix_free(const ExpansionOperator& op, const Field& u, double* imag_residue) {
  return apply_gpu(op, u, 0, imag_residue);
}

// the device reduction order is fixed (ascending m), so "serial" is the same computation
Field apply_matrix_free_serial(const ExpansionOperator& op, const Field& u, double* imag_residue) {
  return apply_gpu(op, u, 0, imag_residue);
}

Field apply_perturbation(const ExpansionOperator& op, const Field& u, double* imag_residue) {
  if (op.constant_order) {  // flap.cpp:163-166
    if (!u.grid().same_as(op.grid)) throw GridMismatch("field defined on a different grid than the operator");
    if (imag_residue) *imag_residue = 0.0;
    return Field(op.grid, 0.0);
  }
  return apply_gpu(op, u, 1, imag_residue);
}

}  // namespace fwave
