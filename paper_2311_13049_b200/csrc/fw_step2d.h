// fw_step2d.h — parameters of the persistent 2D step kernel (fw_step2d.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace fw {

constexpr int kStep2dMaxTerms = 2 * 65;                 // nops <= 2, M <= 64
constexpr int kStep2dCStride = 1 + 2 * kStep2dMaxTerms;  // counters per set
constexpr int kTraceWords = 1024 * 16;                  // watchdog records: 2 x 8 words per CTA
// the mapped buffer also holds the warp-specialised kernel's phase timestamps of a
// -DFW_STEP2D_TRACE=1 build (2 x 32 x 136 x 8 + 2 x 160 x 2 x 136 words)
constexpr int kTraceAlloc = 2 * 32 * 136 * 8 + 2 * 160 * 2 * 136 > kTraceWords ? 2 * 32 * 136 * 8 + 2 * 160 * 2 * 136
                                                                                : kTraceWords;

struct Step2DParams {
  int J0, J1;
  int M, m_first, nops, nterms_total;
  const double* u;          // input field (cur)
  double2* Y;               // (J1/2+1) x J0 forward scratch, column-major Y[k][k0]
  double2* T;               // KRING x J0 x (J1/2+1) term ring
  const double* w[2];       // per op: [M+1][wcols][J0] weights (column-major per term)
  int wcols;                // columns per term in w (>= J1/2+1)
  const double* dev[2];     // per op: [M][J0][J1] deviation powers m = 1..M
  double* out[2];           // per op result (seismic: out[0] = L1, out[1] = new L2prev)
  double* residue;          // nullable, max-accumulated
  const double2* master;    // twiddle master table
  unsigned long long* counters;  // 2 sets x kStep2dCStride, zero-initialised
  unsigned long long* trace;     // optional watchdog records (mapped host memory), see fw_step2d.cu
  int cset, cstride;
  // seismic update
  int seismic;
  const double *prev, *ap, *c, *eta, *tc;
  double* next;
  double tau, thr;
  int step;   // step number of the launch's first step (blow-up flag value)
  int* flag;
  // multi-step seismic launches: nsteps steps, buffers rotating with the level L = lvl0 + s:
  // cur = ub[L % 3], prev = ub[(L + 2) % 3], next = ub[(L + 1) % 3], ap = ab[(L + 1) % 2],
  // new L2prev = ab[L % 2].  Applies and single steps use the plain pointers (nsteps = 1).
  int nsteps;
  double* ub[3];
  double* ab[2];
  long long lvl0;
  int dbg;  // timing experiments (FW_STEP2D_DBG), 0 in production
};

bool step2d_supported(int J0, int J1, int nsm);
int step2d_col_groups(int J1);
int step2d_wcols(int J1);
constexpr int kStep2dCG = 4;
#ifndef FW_S2D_RING
#define FW_S2D_RING 4  // measured: 4 -> 243.8, 3 -> 244.4, 5 -> 244.9, 6 -> 245.0, 7 -> 245.4 us/step; 2 deadlocks
#endif
constexpr int kStep2dRing = FW_S2D_RING;  // term slots of the global ring (8 / 12 measured slower)
static_assert(kStep2dRing >= 3, "the columns publish term t after pass 0 of t + 1: two slots deadlock");
cudaError_t launch_step2d(const Step2DParams& p, cudaStream_t st, int nsm);
// the time-multiplexed variant (fw_step2d_tm.cu): same parameters, tables and results
bool step2d_tm_supported(int J0, int J1, int nsm);
cudaError_t launch_step2d_tm(const Step2DParams& p, cudaStream_t st, int nsm);

// table relayouts for the persistent kernel
void launch_w_to_2d(cudaStream_t st, int J0, int J1, int M, const double* w, double* w2d);
void launch_dev_tables(cudaStream_t st, size_t N, int M, const double* dev1, double* dev);

}  // namespace fw
