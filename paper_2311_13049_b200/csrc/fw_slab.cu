// fw_slab.cu — the slab-decomposed SeismicStepper behind the C-ABI (one process per GPU),
// for C/C++ hosts (the reference's SeismicStepper, seismic.hpp:36-46, on C3/C4-sized grids).
//
// Rank r of P owns planes [r J0/P, (r+1) J0/P) of a 3D grid and only its slab of the two
// operators' tables (fw_op_create_slab).  One step (seismic.cpp:111-133):
//   R2C (axis 2) + C2C (axis 1) whose last pass stores straight into every rank's forward buffer
//   T [J0][J1/P][H] (fw_stage_c2c_scatter: peer memory, CUDA IPC)            | barrier
//   C2C (axis 0, x 1/N) of the own columns -> uhat (shared by both operators)
//   per operator: the all-terms axis-0 inverse (x w_m) scattered into every rank's Ts [nt][J0/P][J1][H]
//                                                                            | barrier
//   per operator: C2C (axis 1) + C2R with the ascending-m recombination -> L1, L2
//   the update into the next level; a blow-up mins the step into every rank's flag (peer memory)
// The communicator comes from an NCCL unique id (rank 0 makes it, the host distributes it):
// it exchanges the IPC handles once (all-gather) and is the device-side barrier between the
// phases (a one-word all-reduce on the context stream: stream-ordered, no host round trip).
// NCCL is loaded at run time (dlopen of libnccl.so.2): the library has no link-time dependency.
// The host reads the blow-up flag once per fw_slab_seis_step call and rewinds to the levels
// before the offending step, as the single-GPU stepper (seismic.cpp:124-129).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/fw_capi.h"
#include "fw_internal.h"

namespace {

// ---- NCCL, resolved at run time
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      x.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return x;
    }
    x.getUniqueId = (decltype(x.getUniqueId))dlsym(h, "ncclGetUniqueId");
    x.commInitRank = (decltype(x.commInitRank))dlsym(h, "ncclCommInitRank");
    x.commDestroy = (decltype(x.commDestroy))dlsym(h, "ncclCommDestroy");
    x.allReduce = (decltype(x.allReduce))dlsym(h, "ncclAllReduce");
    x.allGather = (decltype(x.allGather))dlsym(h, "ncclAllGather");
    x.errorString = (decltype(x.errorString))dlsym(h, "ncclGetErrorString");
    x.ok = x.getUniqueId && x.commInitRank && x.commDestroy && x.allReduce && x.allGather && x.errorString;
    if (!x.ok) x.why = "libnccl lacks an entry point";
    return x;
  }();
  return n;
}

}  // namespace

// errors: reuse the library's thread-local message through a tiny bridge (fw_capi.cu owns set_err)
extern "C" int fw_internal_set_error(int code, const char* msg);

#define SL_TRY(expr)             \
  do {                           \
    int rc_ = (expr);            \
    if (rc_ != FW_OK) return rc_; \
  } while (0)
#define SL_CUDA(call)                                                                                \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      return fw_internal_set_error(e_ == cudaErrorMemoryAllocation ? FW_E_OOM : FW_E_CUDA,           \
                                   (std::string(#call) + ": " + cudaGetErrorString(e_)).c_str());    \
  } while (0)
#define SL_NCCL(call)                                                                                \
  do {                                                                                               \
    ncclResult_t r_ = (call);                                                                        \
    if (r_ != ncclSuccess)                                                                           \
      return fw_internal_set_error(FW_E_NCCL, (std::string(#call) + ": " + nccl().errorString(r_)).c_str()); \
  } while (0)

struct fw_slab_seis_s {
  fw_ctx ctx = nullptr;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  int P = 1, rank = 0;
  int J[3] = {0, 0, 0}, J0l = 0, J1l = 0, H = 0;
  long long nloc = 0;
  double tau = 0, thr = 0;
  int M = 0, mlast = 0;
  fw_op op[2] = {nullptr, nullptr};
  const double* w[2] = {nullptr, nullptr};
  const double* dev1[2] = {nullptr, nullptr};
  // this rank's receive buffers (fw_ipc_alloc) and every rank's addresses of them
  void* own[4] = {nullptr, nullptr, nullptr, nullptr};  // T, Ts0, Ts1, flag
  std::vector<void*> ptr[4];
  std::vector<void*> opened;
  // scratch and state
  double *Y = nullptr, *uhat = nullptr, *Tsc = nullptr, *l1 = nullptr, *l2 = nullptr;
  double *ub[3] = {nullptr, nullptr, nullptr}, *ab[2] = {nullptr, nullptr};
  double *c = nullptr, *eta = nullptr, *tc = nullptr;
  int* bar = nullptr;  // barrier word
  long lvl = 1, n = 1;
  size_t table_bytes = 0;
  double* cur() { return ub[lvl % 3]; }
  double* prev() { return ub[(lvl + 2) % 3]; }
  double* ap() { return ab[(lvl + 1) % 2]; }
};

namespace {

int barrier(fw_slab_seis s) {
  if (s->P == 1) return FW_OK;
  SL_NCCL(nccl().allReduce(s->bar, s->bar, 1, ncclInt32, ncclSum, s->comm, s->stream));
  return FW_OK;
}

// one apply's forward phase: u (own planes) -> every rank's T (scatter)
int phase_forward(fw_slab_seis s, const double* u) {
  const int loc[3] = {s->J0l, s->J[1], s->J[2]};
  SL_TRY(fw_stage_r2c(s->ctx, 3, loc, u, s->Y, 1.0));
  std::vector<double*> dst(s->P);
  for (int q = 0; q < s->P; ++q) dst[q] = (double*)s->ptr[0][q];
  return fw_stage_c2c_scatter(s->ctx, 3, loc, 1, -1, s->Y, nullptr, 0, 0, 1, 1.0, s->P, dst.data(), s->J1l, s->H,
                              (long long)s->J1l * s->H, 0, (long long)s->rank * s->J0l * s->J1l * s->H);
}

int forward_spectrum(fw_slab_seis s) {
  const int tshape[3] = {s->J[0], s->J1l, s->J[2]};
  const double N = (double)s->J[0] * s->J[1] * s->J[2];
  return fw_stage_c2c(s->ctx, 3, tshape, 0, -1, (const double*)s->own[0], s->uhat, nullptr, 0,
                      (long long)s->J[0] * s->J1l * s->H, 0, 1, 1.0 / N);
}

int phase_inverse(fw_slab_seis s, int k, int m_first) {
  const int tshape[3] = {s->J[0], s->J1l, s->J[2]};
  const long long nh = (long long)s->J[0] * s->J1l * s->H;
  const int nt = s->mlast - m_first + 1;
  std::vector<double*> dst(s->P);
  for (int q = 0; q < s->P; ++q) dst[q] = (double*)s->ptr[1 + k][q];
  return fw_stage_c2c_scatter(s->ctx, 3, tshape, 0, +1, s->uhat, s->w[k] + (size_t)m_first * nh, 0, nh, nt, 1.0, s->P,
                              dst.data(), s->J0l, (long long)s->J[1] * s->H, 0, (long long)s->J0l * s->J[1] * s->H,
                              (long long)s->rank * s->J1l * s->H);
}

int phase_finish(fw_slab_seis s, int k, int m_first, double* out) {
  const int loc[3] = {s->J0l, s->J[1], s->J[2]};
  const long long nh = (long long)s->J0l * s->J[1] * s->H;
  const int nt = s->mlast - m_first + 1;
  SL_TRY(fw_stage_c2c(s->ctx, 3, loc, 1, +1, (const double*)s->own[1 + k], s->Tsc, nullptr, nh, nh, 0, nt, 1.0));
  return fw_stage_c2r_accum(s->ctx, 3, loc, s->Tsc, nt > 1 ? nh : 0, m_first, s->mlast, s->dev1[k], out, nullptr);
}

// out_k = A_k(u) for the listed operators (the constructor's applies)
int apply_ops(fw_slab_seis s, const double* u, int k0, int k1, double* out0, double* out1) {
  SL_TRY(phase_forward(s, u));
  SL_TRY(barrier(s));
  SL_TRY(forward_spectrum(s));
  for (int k = k0; k <= k1; ++k) SL_TRY(phase_inverse(s, k, 0));
  SL_TRY(barrier(s));
  if (k0 == 0) SL_TRY(phase_finish(s, 0, 0, out0));
  if (k1 == 1) SL_TRY(phase_finish(s, 1, 0, out1));
  return FW_OK;
}

void slab_free(fw_slab_seis s) {
  if (!s) return;
  if (s->ctx) {
    cudaSetDevice(fw_ctx_device(s->ctx));
    cudaStreamSynchronize(s->stream);
  }
  for (void* p : s->opened) fw_ipc_close(p);
  for (void* p : s->own)
    if (p) fw_ipc_free(s->ctx, p);
  for (double* p : {s->Y, s->uhat, s->Tsc, s->l1, s->l2, s->ub[0], s->ub[1], s->ub[2], s->ab[0], s->ab[1], s->c, s->eta,
                    s->tc})
    if (p) cudaFree(p);
  if (s->bar) cudaFree(s->bar);
  fw_op_destroy(s->op[0]);
  fw_op_destroy(s->op[1]);
  if (s->comm && nccl().ok) nccl().commDestroy(s->comm);
  delete s;
}

int slab_create(fw_slab_seis s, const unsigned char* nccl_id, const double* lo, const double* hi, const double* gamma,
                const double* c0, double omega0, const double* phi, const double* psi, double blowup_factor) {
  const size_t N = (size_t)s->J[0] * s->J[1] * s->J[2];
  // the medium of the own planes (derive_medium, seismic.cpp:14-39) and the two operators' slab tables
  std::vector<double> co(s->nloc), eta(s->nloc), tc(s->nloc), ord(N);
  SL_TRY(fw_medium_coefficients(s->nloc, gamma + (size_t)s->rank * s->nloc, c0 + (size_t)s->rank * s->nloc, omega0,
                                co.data(), eta.data(), tc.data()));
  for (size_t j = 0; j < N; ++j)  // derive_medium checks every point (seismic.cpp:14-19)
    if (!(gamma[j] >= 0.0) || !(gamma[j] < 0.5)) return fw_internal_set_error(FW_E_GAMMA_RANGE, "gamma outside [0, 0.5)");
  for (int k = 0; k < 2; ++k) {
    for (size_t j = 0; j < N; ++j) ord[j] = (k == 0 ? 1.0 : 0.5) + gamma[j];
    SL_TRY(fw_op_create_slab(s->ctx, s->J, lo, hi, ord.data(), nullptr, s->M, s->P, s->rank, &s->op[k]));
    int ml = 0;
    SL_TRY(fw_op_device_tables(s->op[k], &s->w[k], &s->dev1[k], &ml));
    s->mlast = ml;
    fw_op_info_t info;
    SL_TRY(fw_op_info(s->op[k], &info));
    s->table_bytes += info.device_bytes;
  }
  // buffers
  const size_t cplx = 2 * sizeof(double);
  const int nt = s->mlast + 1;
  const size_t bytes[4] = {(size_t)s->J[0] * s->J1l * s->H * cplx, (size_t)nt * s->J0l * s->J[1] * s->H * cplx,
                           (size_t)nt * s->J0l * s->J[1] * s->H * cplx, 256};
  for (int b = 0; b < 4; ++b) SL_TRY(fw_ipc_alloc(s->ctx, bytes[b], &s->own[b]));
  const int none = 0x7fffffff;
  SL_CUDA(cudaMemcpy(s->own[3], &none, sizeof(int), cudaMemcpyHostToDevice));
  const size_t nloc = (size_t)s->nloc, nhl = (size_t)s->J0l * s->J[1] * s->H;
  SL_CUDA(cudaMalloc(&s->Y, nhl * cplx));
  SL_CUDA(cudaMalloc(&s->uhat, bytes[0]));
  SL_CUDA(cudaMalloc(&s->Tsc, bytes[1]));
  for (double** p : {&s->l1, &s->l2, &s->ub[0], &s->ub[1], &s->ub[2], &s->ab[0], &s->ab[1], &s->c, &s->eta, &s->tc})
    SL_CUDA(cudaMalloc(p, nloc * sizeof(double)));
  SL_CUDA(cudaMalloc(&s->bar, sizeof(int)));
  SL_CUDA(cudaMemset(s->bar, 0, sizeof(int)));
  // the communicator and the peers' buffer addresses
  for (int b = 0; b < 4; ++b) s->ptr[b].assign(s->P, nullptr);
  if (s->P == 1) {
    for (int b = 0; b < 4; ++b) s->ptr[b][0] = s->own[b];
  } else {
    if (!nccl().ok) return fw_internal_set_error(FW_E_NCCL, nccl().why.c_str());
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    SL_NCCL(nccl().commInitRank(&s->comm, s->P, id, s->rank));
    unsigned char mine[4 * 64];
    for (int b = 0; b < 4; ++b) SL_TRY(fw_ipc_handle(s->own[b], mine + 64 * b));
    unsigned char *dh = nullptr, *dall = nullptr;
    SL_CUDA(cudaMalloc(&dh, sizeof(mine)));
    SL_CUDA(cudaMalloc(&dall, sizeof(mine) * s->P));
    std::vector<unsigned char> all(sizeof(mine) * s->P);
    SL_CUDA(cudaMemcpy(dh, mine, sizeof(mine), cudaMemcpyHostToDevice));
    SL_NCCL(nccl().allGather(dh, dall, sizeof(mine), ncclUint8, s->comm, s->stream));
    SL_CUDA(cudaMemcpyAsync(all.data(), dall, all.size(), cudaMemcpyDeviceToHost, s->stream));
    SL_CUDA(cudaStreamSynchronize(s->stream));
    cudaFree(dh);
    cudaFree(dall);
    for (int q = 0; q < s->P; ++q)
      for (int b = 0; b < 4; ++b) {
        if (q == s->rank) {
          s->ptr[b][q] = s->own[b];
          continue;
        }
        void* p = nullptr;
        SL_TRY(fw_ipc_open(all.data() + (size_t)q * sizeof(mine) + 64 * b, &p));
        s->opened.push_back(p);
        s->ptr[b][q] = p;
      }
  }
  // fields: phi, psi (own planes); the constructor (seismic.cpp:85-109): L1 phi, L2 psi, L2 phi, Taylor start
  SL_CUDA(cudaMemcpy(s->c, co.data(), nloc * 8, cudaMemcpyHostToDevice));
  SL_CUDA(cudaMemcpy(s->eta, eta.data(), nloc * 8, cudaMemcpyHostToDevice));
  SL_CUDA(cudaMemcpy(s->tc, tc.data(), nloc * 8, cudaMemcpyHostToDevice));
  double* d_phi = s->ub[0];  // prev at level 1
  double* d_psi = s->ub[2];  // scratch until the first step writes it
  SL_CUDA(cudaMemcpy(d_phi, phi + (size_t)s->rank * nloc, nloc * 8, cudaMemcpyHostToDevice));
  SL_CUDA(cudaMemcpy(d_psi, psi + (size_t)s->rank * nloc, nloc * 8, cudaMemcpyHostToDevice));
  double sup = 0.0;
  for (size_t j = 0; j < N; ++j) sup = sup > fabs(phi[j]) ? sup : fabs(phi[j]);
  s->thr = blowup_factor * (sup > 1e-300 ? sup : 1e-300);  // seismic.cpp:91-93
  s->lvl = 1;
  s->n = 1;
  SL_TRY(apply_ops(s, d_phi, 0, 1, s->l1, s->ab[0]));   // L1 phi, L2 phi (= L2prev at level 1)
  SL_TRY(apply_ops(s, d_psi, 1, 1, nullptr, s->l2));    // L2 psi
  SL_TRY(fw_stage_seis_start(s->ctx, s->nloc, s->tau, d_phi, d_psi, s->c, s->eta, s->tc, s->l1, s->l2, s->cur()));
  SL_TRY(barrier(s));
  SL_CUDA(cudaStreamSynchronize(s->stream));
  return FW_OK;
}

}  // namespace

extern "C" {

int fw_nccl_unique_id(unsigned char id_out[128]) {
  if (!id_out) return fw_internal_set_error(FW_E_ARG, "null argument");
  if (!nccl().ok) return fw_internal_set_error(FW_E_NCCL, nccl().why.c_str());
  ncclUniqueId id;
  SL_NCCL(nccl().getUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return FW_OK;
}

int fw_slab_seis_create(fw_ctx ctx, const unsigned char nccl_id[128], int P, int rank, const int* J, const double* lo,
                        const double* hi, const double* gamma, const double* c0, double omega0, int M,
                        const double* phi, const double* psi, double tau, double blowup_factor, fw_slab_seis* out) {
  if (!ctx || !J || !lo || !hi || !gamma || !c0 || !phi || !psi || !out || (P > 1 && !nccl_id))
    return fw_internal_set_error(FW_E_ARG, "null argument");
  if (P < 1 || P > fw::kMaxPeers || rank < 0 || rank >= P || J[0] % P || J[1] % P)
    return fw_internal_set_error(FW_E_ARG, "slab: 1 <= P <= 8, 0 <= rank < P, axes 0 and 1 divisible by P");
  SL_CUDA(cudaSetDevice(fw_ctx_device(ctx)));
  fw_slab_seis s = new fw_slab_seis_s();
  s->ctx = ctx;
  s->stream = (cudaStream_t)fw_ctx_stream(ctx);
  s->P = P;
  s->rank = rank;
  for (int m = 0; m < 3; ++m) s->J[m] = J[m];
  s->J0l = J[0] / P;
  s->J1l = J[1] / P;
  s->H = J[2] / 2 + 1;
  s->nloc = (long long)s->J0l * J[1] * J[2];
  s->tau = tau;
  s->M = M;
  const int rc = slab_create(s, nccl_id, lo, hi, gamma, c0, omega0, phi, psi, blowup_factor);
  if (rc != FW_OK) {
    slab_free(s);
    return rc;
  }
  *out = s;
  return FW_OK;
}

void fw_slab_seis_destroy(fw_slab_seis s) { slab_free(s); }

int fw_slab_seis_step(fw_slab_seis s, int nsteps) {
  if (!s || nsteps < 0) return fw_internal_set_error(FW_E_ARG, "bad argument");
  SL_CUDA(cudaSetDevice(fw_ctx_device(s->ctx)));
  int* flag = (int*)s->own[3];
  std::vector<int*> pf(s->P);
  for (int q = 0; q < s->P; ++q) pf[q] = (int*)s->ptr[3][q];
  for (int i = 0; i < nsteps; ++i) {
    SL_TRY(phase_forward(s, s->cur()));
    SL_TRY(barrier(s));
    SL_TRY(forward_spectrum(s));
    SL_TRY(phase_inverse(s, 0, 0));
    SL_TRY(phase_inverse(s, 1, 0));
    SL_TRY(barrier(s));
    SL_TRY(phase_finish(s, 0, 0, s->l1));
    SL_TRY(phase_finish(s, 1, 0, s->l2));
    SL_TRY(fw_stage_seis_update_peers(s->ctx, s->nloc, s->tau, s->cur(), s->prev(), s->ap(), s->l1, s->l2, s->c,
                                      s->eta, s->tc, s->ub[(s->lvl + 1) % 3], s->ab[s->lvl % 2], s->thr,
                                      (int)(s->n + 1), flag, s->P, pf.data()));
    s->lvl += 1;
    s->n += 1;
  }
  // once per call: after a barrier every rank's flag holds the earliest offending step of any rank
  SL_TRY(barrier(s));
  int v = 0x7fffffff;
  SL_CUDA(cudaMemcpyAsync(&v, flag, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  SL_CUDA(cudaStreamSynchronize(s->stream));
  if (v != 0x7fffffff) {
    s->lvl -= s->n - v + 1;  // the levels before the offending step (later updates were frozen)
    s->n = v;
    SL_TRY(barrier(s));  // every rank has read its flag before any resets it
    const int none = 0x7fffffff;
    SL_CUDA(cudaMemcpyAsync(flag, &none, sizeof(int), cudaMemcpyHostToDevice, s->stream));
    SL_CUDA(cudaStreamSynchronize(s->stream));
    char b[160];
    snprintf(b, sizeof b, "sup|u| > %g at step %d", s->thr, v);
    return fw_internal_set_error(FW_E_BLOWUP, b);
  }
  return FW_OK;
}

int fw_slab_seis_get(fw_slab_seis s, double* cur_host, double* prev_host, double* atten_prev_host, long* n) {
  if (!s) return fw_internal_set_error(FW_E_ARG, "null stepper");
  SL_CUDA(cudaSetDevice(fw_ctx_device(s->ctx)));
  const size_t b = (size_t)s->nloc * sizeof(double);
  if (cur_host) SL_CUDA(cudaMemcpyAsync(cur_host, s->cur(), b, cudaMemcpyDeviceToHost, s->stream));
  if (prev_host) SL_CUDA(cudaMemcpyAsync(prev_host, s->prev(), b, cudaMemcpyDeviceToHost, s->stream));
  if (atten_prev_host) SL_CUDA(cudaMemcpyAsync(atten_prev_host, s->ap(), b, cudaMemcpyDeviceToHost, s->stream));
  SL_CUDA(cudaStreamSynchronize(s->stream));
  if (n) *n = s->n;
  return FW_OK;
}

int fw_slab_seis_info(fw_slab_seis s, size_t* table_bytes, int* P, int* rank) {
  if (!s) return fw_internal_set_error(FW_E_ARG, "null stepper");
  if (table_bytes) *table_bytes = s->table_bytes;
  if (P) *P = s->P;
  if (rank) *rank = s->rank;
  return FW_OK;
}

}  // extern "C"
