// fw_kernels.cu — sm_100a kernels of the matrix-free variable-order apply.
//
// Generic multi-pass pipeline (all dimensions):
//   forward  : k_r2c_rows (last axis, real -> Hermitian half) then k_c2c_axis
//              for axes d-2..0 (1/N folded into the last pass; exact for 2^k N)
//   inverse  : k_c2c_axis on axis 0 for ALL terms at once (grid.y = term) with
//              the w_m multiply fused into its load, k_c2c_axis for axes
//              1..d-2, then k_c2r_accum: per row, every term's C2R in shared
//              memory with the (s-s0)^m recombination fused in registers in
//              ascending m, one write of the result.
// Compiled with --fmad=false: the only fused multiply-adds are the explicit
// fma() calls of the canonical FFT (fw_fft.cuh).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "fw_fft.cuh"
#include "fw_internal.h"

namespace fw {

namespace {

constexpr int kThreads = 256;
constexpr int kEmax = 16;  // accumulator elements per thread in k_c2r_accum

// line stride in shared memory so 8 consecutive lanes spanning `lpb` lines hit
// distinct 16-byte bank groups
__host__ __device__ inline int line_stride(int n, int lpb) {
  int pad = 0;
  switch (lpb) {
    case 8: pad = 1; break;
    case 4: pad = 2; break;
    case 2: pad = 4; break;
    default: pad = 1; break;
  }
  return n + pad;
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(__double_as_longlong(v)));
}

// ---------------------------------------------------------------------------
// forward, last axis: rows of nl reals -> nl/2+1 bins
__global__ void __launch_bounds__(kThreads) k_r2c_rows(const double* __restrict__ u, double2* __restrict__ Uh, int nl,
                                                      long long rows, int lpb, double sc, int do_scale,
                                                      const double2* __restrict__ master,
                                                      const BatchLine* __restrict__ bl) {
  if (bl) {  // batched: this field's pointers
    u = static_cast<const double*>(bl[blockIdx.z].src);
    Uh = static_cast<double2*>(bl[blockIdx.z].dst);
  }
  extern __shared__ double2 sm[];
  const int h = nl / 2;
  const int ls = line_stride(h + 1, lpb);
  double2* buf0 = sm;
  double2* buf1 = sm + lpb * ls;
  const long long row0 = (long long)blockIdx.x * lpb;
  const int nlines = (int)min((long long)lpb, rows - row0);
  for (int e = threadIdx.x; e < nlines * h; e += blockDim.x) {
    const int l = e / h, j = e - l * h;
    buf0[l * ls + j] = reinterpret_cast<const double2*>(u + (row0 + l) * nl)[j];
  }
  __syncthreads();
  const double2* Z = smem_c2c<-1>(buf0, buf1, h, nlines, ls, master);
  for (int e = threadIdx.x; e < nlines * (h + 1); e += blockDim.x) {
    const int l = e / (h + 1), k = e - l * (h + 1);
    double2 X = r2c_post(Z + l * ls, k, h, master);
    if (do_scale) {
      X.x *= sc;
      X.y *= sc;
    }
    Uh[(row0 + l) * (h + 1) + k] = X;
  }
}

// ---------------------------------------------------------------------------
// C2C along a strided axis of the half-spectrum array.  Line (o, in) holds
// elements o*n*S + in + j*S, j < n.  A block takes `lpb` consecutive `in`.
// blockIdx.y = term: src/dst/w advance by their term strides.
template <int DIR>
__global__ void __launch_bounds__(kThreads) k_c2c_axis(const double2* __restrict__ src, double2* __restrict__ dst,
                                                      const double* __restrict__ w, int n, long long S,
                                                      long long inner, long long src_ts, long long dst_ts,
                                                      long long w_ts, int lpb, double sc, int do_scale,
                                                      const double2* __restrict__ master,
                                                      const BatchLine* __restrict__ bl) {
  if (bl) {  // batched: this field's pointers
    src = static_cast<const double2*>(bl[blockIdx.z].src);
    dst = static_cast<double2*>(bl[blockIdx.z].dst);
    w = bl[blockIdx.z].w;
  }
  extern __shared__ double2 sm[];
  const int ls = line_stride(n, lpb);
  double2* buf0 = sm;
  double2* buf1 = sm + lpb * ls;
  const long long term = blockIdx.y;
  src += term * src_ts;
  dst += term * dst_ts;
  if (w) w += term * w_ts;
  const long long bpo = (inner + lpb - 1) / lpb;
  const long long o = blockIdx.x / bpo;
  const long long in0 = (blockIdx.x - o * bpo) * lpb;
  const int nlines = (int)min((long long)lpb, inner - in0);
  const long long base = o * (long long)n * S + in0;
  for (int e = threadIdx.x; e < n * nlines; e += blockDim.x) {
    const int j = e / nlines, l = e - j * nlines;
    const long long idx = base + (long long)j * S + l;
    double2 v = src[idx];
    if (w) {
      const double wk = __ldg(&w[idx]);
      v.x = wk * v.x;
      v.y = wk * v.y;
    }
    buf0[l * ls + j] = v;
  }
  __syncthreads();
  const double2* R = smem_c2c<DIR>(buf0, buf1, n, nlines, ls, master);
  for (int e = threadIdx.x; e < n * nlines; e += blockDim.x) {
    const int j = e / nlines, l = e - j * nlines;
    double2 v = R[l * ls + j];
    if (do_scale) {
      v.x *= sc;
      v.y *= sc;
    }
    dst[base + (long long)j * S + l] = v;
  }
}

// ---------------------------------------------------------------------------
// Per row: for m = m_first..m_last, C2R of (w_m .* src_m) and
// acc += (s-s0)^m .* x in ascending m (flap.cpp:21-36, 61-91).
// src_m = src + (m - m_first) * src_ts; weights applied here only when w != null (1D).
__global__ void __launch_bounds__(kThreads) k_c2r_accum(const double2* __restrict__ src, long long src_ts,
                                                       const double* __restrict__ w, long long w_ts, int m_first,
                                                       int m_last, const double* __restrict__ dev1,
                                                       double* __restrict__ out, int nl, long long rows, int lpb,
                                                       double* residue, const int* guard,
                                                       const double2* __restrict__ master,
                                                       const BatchLine* __restrict__ bl) {
  if (guard && *guard != kNoBlowup) return;
  if (bl) {  // batched: this field's pointers
    src = static_cast<const double2*>(bl[blockIdx.z].src);
    dev1 = bl[blockIdx.z].aux;
    out = bl[blockIdx.z].out;
  }
  extern __shared__ double2 sm[];
  const int h = nl / 2;
  const int ls = line_stride(h + 1, lpb);
  double2* bufX = sm;
  double2* bufZ = sm + lpb * ls;
  const long long row0 = (long long)blockIdx.x * lpb;
  const int nlines = (int)min((long long)lpb, rows - row0);
  const int nel = nlines * nl;
  double acc[kEmax], devm[kEmax], d1[kEmax];
#pragma unroll
  for (int i = 0; i < kEmax; ++i) {
    acc[i] = 0.0;
    devm[i] = 0.0;
    d1[i] = 0.0;
    const int e = threadIdx.x + i * blockDim.x;
    if (e < nel && dev1) d1[i] = dev1[row0 * nl + e];
  }
  double rmax = 0.0;
  for (int m = m_first; m <= m_last; ++m) {
    const double2* S = src + (long long)(m - m_first) * src_ts + row0 * (h + 1);
    const double* W = w ? w + (long long)m * w_ts + row0 * (h + 1) : nullptr;
    for (int e = threadIdx.x; e < nlines * (h + 1); e += blockDim.x) {
      const int l = e / (h + 1), k = e - l * (h + 1);
      double2 v = S[e];
      if (W) {
        const double wk = __ldg(&W[e]);
        v.x = wk * v.x;
        v.y = wk * v.y;
      }
      bufX[l * ls + k] = v;
    }
    __syncthreads();
    if (residue && threadIdx.x < nlines) {
      const double r = fabs(bufX[threadIdx.x * ls].y) + fabs(bufX[threadIdx.x * ls + h].y);
      rmax = fmax(rmax, r);
    }
    for (int e = threadIdx.x; e < nlines * h; e += blockDim.x) {
      const int l = e / h, k = e - l * h;
      const double2* X = bufX + l * ls;
      bufZ[l * ls + k] = c2r_pre(X[k], X[h - k], k, h, master);
    }
    __syncthreads();
    const double2* Z = smem_c2c<+1>(bufZ, bufX, h, nlines, ls, master);
#pragma unroll
    for (int i = 0; i < kEmax; ++i) {
      const int e = threadIdx.x + i * blockDim.x;
      if (e < nel) {
        const int l = e / nl, jj = e - l * nl;
        const double2 z = Z[l * ls + (jj >> 1)];
        const double x = (jj & 1) ? z.y : z.x;
        double v;
        if (m == 0) {
          v = x;
        } else {
          devm[i] = (m == 1) ? d1[i] : devm[i] * d1[i];
          v = devm[i] * x;
        }
        double p = 0.0;
        p += v;
        acc[i] += p;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kEmax; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    if (e < nel) out[row0 * nl + e] = acc[i];
  }
  if (residue && threadIdx.x < nlines) atomic_max_nonneg(residue, rmax);
}

// ---------------------------------------------------------------------------
__global__ void k_build_weights(long long Nh, int M, const double* __restrict__ mu2h,
                                const double* __restrict__ base, const double* __restrict__ logm,
                                double* __restrict__ w) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < Nh; k += (long long)gridDim.x * blockDim.x) {
    const double b = base[k];
    const double l = logm[k];
    const bool pos = mu2h[k] > 0.0;
    double lw = 0.0;
    w[k] = b;
    for (int m = 1; m <= M; ++m) {
      if (pos) lw = (m == 1) ? l : lw * l / m;
      w[(long long)m * Nh + k] = b * lw;
    }
  }
}

__global__ void k_weights_from_lw(long long Nh, int M, const double* __restrict__ base,
                                  const double* __restrict__ lw, double* __restrict__ w) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < Nh; k += (long long)gridDim.x * blockDim.x) {
    const double b = base[k];
    w[k] = b;
    for (int m = 1; m <= M; ++m) w[(long long)m * Nh + k] = b * lw[(long long)(m - 1) * Nh + k];
  }
}

__global__ void k_dev1(long long N, const double* __restrict__ s, double s0, double* __restrict__ dev1) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x)
    dev1[j] = s[j] - s0;
}

__global__ void k_seis_start(long long N, double tau, const double* __restrict__ phi, const double* __restrict__ psi,
                             const double* __restrict__ c, const double* __restrict__ eta,
                             const double* __restrict__ tc, const double* __restrict__ l1phi,
                             const double* __restrict__ l2psi, double* __restrict__ cur) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const double c2 = c[j] * c[j];
    cur[j] = phi[j] + tau * psi[j] + 0.5 * tau * tau * c2 * (eta[j] * l1phi[j] + tc[j] * l2psi[j]);
  }
}

__global__ void k_seis_update(long long N, double tau, const double* __restrict__ cur,
                              const double* __restrict__ prev, const double* __restrict__ ap,
                              const double* __restrict__ l1, const double* __restrict__ l2,
                              const double* __restrict__ c, const double* __restrict__ eta,
                              const double* __restrict__ tc, double* __restrict__ next, double thr, int step,
                              int* flag) {
  if (*flag != kNoBlowup) return;
  const double t2 = tau * tau;
  bool bad = false;
  // two points per thread and iteration (16-B accesses) when every array allows it; the arithmetic
  // per point is the scalar loop's
  const bool vec = (N % 2 == 0) &&
                   ((((uintptr_t)cur | (uintptr_t)prev | (uintptr_t)ap | (uintptr_t)l1 | (uintptr_t)l2 | (uintptr_t)c |
                      (uintptr_t)eta | (uintptr_t)tc | (uintptr_t)next) & 15) == 0);
  if (vec) {
    const long long N2 = N / 2;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N2; j += (long long)gridDim.x * blockDim.x) {
      const double2 cc = reinterpret_cast<const double2*>(c)[j], vc = reinterpret_cast<const double2*>(cur)[j];
      const double2 vp = reinterpret_cast<const double2*>(prev)[j], va = reinterpret_cast<const double2*>(ap)[j];
      const double2 v1 = reinterpret_cast<const double2*>(l1)[j], v2 = reinterpret_cast<const double2*>(l2)[j];
      const double2 ve = reinterpret_cast<const double2*>(eta)[j], vt = reinterpret_cast<const double2*>(tc)[j];
      const double c2x = cc.x * cc.x, c2y = cc.y * cc.y;
      const double vx = 2.0 * vc.x - vp.x + t2 * c2x * (ve.x * v1.x + vt.x * (v2.x - va.x) / tau);
      const double vy = 2.0 * vc.y - vp.y + t2 * c2y * (ve.y * v1.y + vt.y * (v2.y - va.y) / tau);
      reinterpret_cast<double2*>(next)[j] = make_double2(vx, vy);
      bad |= (fabs(vx) > thr) || (fabs(vy) > thr);
    }
  } else
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const double c2 = c[j] * c[j];
    const double v = 2.0 * cur[j] - prev[j] + t2 * c2 * (eta[j] * l1[j] + tc[j] * (l2[j] - ap[j]) / tau);
    next[j] = v;
    bad |= fabs(v) > thr;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicMin(flag, step);
}

// the slab stepper's update: as k_seis_update, plus the new L2prev copy (l2out) and the blow-up flag
// min-ed into every rank's flag (peer memory, system scope) so that after the next barrier every
// rank freezes its later updates (the state levels before the offending step stay intact)
__global__ void k_seis_update_peers(long long N, double tau, const double* __restrict__ cur,
                                    const double* __restrict__ prev, const double* __restrict__ ap,
                                    const double* __restrict__ l1, const double* __restrict__ l2,
                                    const double* __restrict__ c, const double* __restrict__ eta,
                                    const double* __restrict__ tc, double* __restrict__ next,
                                    double* __restrict__ l2out, double thr, int step, int* flag, PeerFlags peers) {
  if (*reinterpret_cast<volatile int*>(flag) != kNoBlowup) return;  // an earlier step blew up (on some rank)
  const double t2 = tau * tau;
  bool bad = false;
  // two points per thread and iteration (16-B accesses) when every array allows it; the arithmetic
  // per point is the scalar loop's
  const bool vec = (N % 2 == 0) &&
                   ((((uintptr_t)cur | (uintptr_t)prev | (uintptr_t)ap | (uintptr_t)l1 | (uintptr_t)l2 | (uintptr_t)c |
                      (uintptr_t)eta | (uintptr_t)tc | (uintptr_t)next | (uintptr_t)l2out) & 15) == 0);
  if (vec) {
    const long long N2 = N / 2;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N2; j += (long long)gridDim.x * blockDim.x) {
      const double2 cc = reinterpret_cast<const double2*>(c)[j], vc = reinterpret_cast<const double2*>(cur)[j];
      const double2 vp = reinterpret_cast<const double2*>(prev)[j], va = reinterpret_cast<const double2*>(ap)[j];
      const double2 v1 = reinterpret_cast<const double2*>(l1)[j], v2 = reinterpret_cast<const double2*>(l2)[j];
      const double2 ve = reinterpret_cast<const double2*>(eta)[j], vt = reinterpret_cast<const double2*>(tc)[j];
      const double c2x = cc.x * cc.x, c2y = cc.y * cc.y;
      const double vx = 2.0 * vc.x - vp.x + t2 * c2x * (ve.x * v1.x + vt.x * (v2.x - va.x) / tau);
      const double vy = 2.0 * vc.y - vp.y + t2 * c2y * (ve.y * v1.y + vt.y * (v2.y - va.y) / tau);
      reinterpret_cast<double2*>(next)[j] = make_double2(vx, vy);
      reinterpret_cast<double2*>(l2out)[j] = v2;
      bad |= (fabs(vx) > thr) || (fabs(vy) > thr);
    }
  } else
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const double c2 = c[j] * c[j];
    const double v = 2.0 * cur[j] - prev[j] + t2 * c2 * (eta[j] * l1[j] + tc[j] * (l2[j] - ap[j]) / tau);
    next[j] = v;
    l2out[j] = l2[j];
    bad |= fabs(v) > thr;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) {
    atomicMin(flag, step);
    for (int q = 0; q < peers.n; ++q) atomicMin_system(peers.f[q], step);
  }
}

__global__ void k_osc_rotate(long long Nh, const double* __restrict__ w, const double* __restrict__ cw,
                             const double* __restrict__ sw, double dt, double2* __restrict__ uh,
                             double2* __restrict__ vh) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < Nh; k += (long long)gridDim.x * blockDim.x) {
    double2 u = uh[k], v = vh[k];
    const double wk = w[k];
    if (wk == 0.0) {
      u.x += dt * v.x;
      u.y += dt * v.y;
    } else {
      const double c = cw[k], s = sw[k];
      const double2 u0 = u, v0 = v;
      u.x = u0.x * c + v0.x * (s / wk);
      u.y = u0.y * c + v0.y * (s / wk);
      v.x = -wk * u0.x * s + v0.x * c;
      v.y = -wk * u0.y * s + v0.y * c;
    }
    uh[k] = u;
    vh[k] = v;
  }
}

__global__ void k_tsfp2_kick(long long N, double tau, double kappa, int cubic, const double* __restrict__ u,
                             const double* __restrict__ pert, double* __restrict__ v, const int* guard) {
  if (guard && *guard != kNoBlowup) return;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const double fu = cubic ? u[j] * u[j] * u[j] : 0.0;
    v[j] += tau * (-kappa * pert[j] + fu);
  }
}

__global__ void k_sup_check(long long N, const double* __restrict__ u, double thr, int step, int* flag) {
  bool bad = false;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x)
    bad |= fabs(u[j]) > thr;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicMin(flag, step);
}

// ---------------------------------------------------------------------------

size_t smem_bytes(int n, int lpb) { return (size_t)2 * lpb * line_stride(n, lpb) * sizeof(double2); }

int elementwise_grid(size_t N) { return (int)std::min<size_t>((N + kThreads - 1) / kThreads, 148 * 16); }

template <class K>
void allow_smem(K, size_t) {}  // limits raised once per device in init_kernels()

void count(const LaunchCtx& L, int n = 1) {
  if (L.launches) *L.launches += n;
}

// (Sd: destination stride along the axis, 0 = the source's; only the register-resident line
// kernels take a different one, see term_row_stride)
void c2c_axis(const LaunchCtx& L, const GridGeom& g, int a, int dir, const double2* src, double2* dst,
              const double* w, long long src_ts, long long dst_ts, long long w_ts, int nterms, double sc,
              bool scale, long long Sd = 0) {
  const int n = g.J[a];
  long long S = g.hp1;
  for (int b = a + 1; b <= g.d - 2; ++b) S *= g.J[b];
  long long outer = 1;
  for (int b = 0; b < a; ++b) outer *= g.J[b];
  const long long inner = S;
  if (!L.generic_lines &&
      launch_lines(L, n, dir, src, dst, w, S, outer, inner, src_ts, dst_ts, w_ts, nterms, 1, sc, scale, nullptr,
                   nullptr, Sd))
    return;
  const int lpb = std::max(1, std::min(8, 4096 / n));
  const long long bpo = (inner + lpb - 1) / lpb;
  dim3 grid((unsigned)(outer * bpo), (unsigned)nterms);
  const size_t sm = smem_bytes(n, lpb);
  if (dir < 0) {
    allow_smem(k_c2c_axis<-1>, sm);
    k_c2c_axis<-1><<<grid, kThreads, sm, L.stream>>>(src, dst, w, n, S, inner, src_ts, dst_ts, w_ts, lpb, sc,
                                                      scale ? 1 : 0, L.master, nullptr);
  } else {
    allow_smem(k_c2c_axis<+1>, sm);
    k_c2c_axis<+1><<<grid, kThreads, sm, L.stream>>>(src, dst, w, n, S, inner, src_ts, dst_ts, w_ts, lpb, sc,
                                                      scale ? 1 : 0, L.master, nullptr);
  }
  count(L);
}

}  // namespace

// every line of length n (power of two <= 4096) along a strided axis of a complex array, in place:
// element j of line (o, in) at o n S + j S + in, in < S (canonical plan; x sc when scale)
void launch_c2c_lines(const LaunchCtx& L, int n, long long S, long long outer, int dir, double2* x, double sc,
                      bool scale) {
  if (!L.generic_lines && launch_lines(L, n, dir, x, x, nullptr, S, outer, S, 0, 0, 0, 1, 1, sc, scale, nullptr))
    return;
  const int lpb = std::max(1, std::min(8, 4096 / n));
  const long long bpo = (S + lpb - 1) / lpb;
  dim3 grid((unsigned)(outer * bpo), 1);
  const size_t sm = smem_bytes(n, lpb);
  if (dir < 0)
    k_c2c_axis<-1><<<grid, kThreads, sm, L.stream>>>(x, x, nullptr, n, S, S, 0, 0, 0, lpb, sc, scale ? 1 : 0, L.master,
                                                      nullptr);
  else
    k_c2c_axis<+1><<<grid, kThreads, sm, L.stream>>>(x, x, nullptr, n, S, S, 0, 0, 0, lpb, sc, scale ? 1 : 0, L.master,
                                                      nullptr);
  count(L);
}

void init_kernels() {
  const int lim = 227 * 1024;
  cudaFuncSetAttribute(k_r2c_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_c2c_axis<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_c2c_axis<+1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_c2r_accum, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
}

void launch_forward(const LaunchCtx& L, const GridGeom& g, const double* u, double2* Uh, bool scale) {
  const double inv = 1.0 / (double)g.N;
  const int h = g.nl / 2;
  if (L.generic_lines ||
      !launch_rows_r2c(L, g.nl, u, Uh, (long long)g.rows, 1, inv, scale && g.d == 1, nullptr)) {
    const int lpb = std::max(1, std::min(8, 2048 / h));
    const size_t sm = smem_bytes(h + 1, lpb);
    allow_smem(k_r2c_rows, sm);
    const unsigned nb = (unsigned)((g.rows + lpb - 1) / lpb);
    k_r2c_rows<<<nb, kThreads, sm, L.stream>>>(u, Uh, g.nl, (long long)g.rows, lpb, inv,
                                               (scale && g.d == 1) ? 1 : 0, L.master, nullptr);
    count(L);
  }
  for (int a = g.d - 2; a >= 0; --a)
    c2c_axis(L, g, a, -1, Uh, Uh, nullptr, 0, 0, 0, 1, inv, scale && a == 0);
}

static void c2r_accum(const LaunchCtx& L, const GridGeom& g, const double2* src, long long src_ts, const double* w,
                      long long w_ts, int m_first, int m_last, const double* dev1, double* out, double* residue,
                      const int* guard, long long xrs = 0) {
  if (!w && !L.generic_lines &&
      launch_rows_c2r(L, g.nl, src, src_ts, m_first, m_last, dev1, out, (long long)g.rows, 1, residue, guard,
                      nullptr, xrs))
    return;
  const int h = g.nl / 2;
  const int lpb = std::max(1, std::min(8, 4096 / g.nl));
  const size_t sm = smem_bytes(h + 1, lpb);
  allow_smem(k_c2r_accum, sm);
  const unsigned nb = (unsigned)((g.rows + lpb - 1) / lpb);
  k_c2r_accum<<<nb, kThreads, sm, L.stream>>>(src, src_ts, w, w_ts, m_first, m_last, dev1, out, g.nl,
                                              (long long)g.rows, lpb, residue, guard, L.master, nullptr);
  count(L);
}

void launch_inverse(const LaunchCtx& L, const GridGeom& g, const InverseArgs& a) {
  const int nterms = a.m_last - a.m_first + 1;
  if (g.d == 1) {
    c2r_accum(L, g, a.Uh, 0, a.w, (long long)g.Nh, a.m_first, a.m_last, a.dev1, a.out, a.residue, a.guard);
    return;
  }
  // axis 0 for all terms: T[t] = IFFT_0(w_{m_first+t} .* Uh); T's rows may be padded (term_row_stride)
  const long long xrs = term_row_stride(L, g, nterms);
  const long long tts = (long long)g.rows * xrs;
  c2c_axis(L, g, 0, +1, a.Uh, a.T, a.w + (long long)a.m_first * g.Nh, 0, tts, (long long)g.Nh, nterms, 1.0, false,
           xrs != g.hp1 ? xrs : 0);
  for (int ax = 1; ax <= g.d - 2; ++ax)
    c2c_axis(L, g, ax, +1, a.T, a.T, nullptr, tts, tts, 0, nterms, 1.0, false);
  c2r_accum(L, g, a.T, tts, nullptr, 0, a.m_first, a.m_last, a.dev1, a.out, a.residue, a.guard, xrs);
}

bool rows_resumable(const LaunchCtx& L, const GridGeom& g) {
  const int h = g.nl / 2;
  if (L.generic_lines || g.d < 2 || !(h == 128 || h == 256 || h == 512)) return false;
  for (int a = 0; a <= g.d - 2; ++a)
    if (!(g.J[a] == 256 || g.J[a] == 512 || g.J[a] == 1024)) return false;
  return true;
}

long long term_row_stride(const LaunchCtx& L, const GridGeom& g, int nterms) {
  const int h = g.nl / 2;
  const bool lines2d = FW_TERM_PAD && nterms > 1 && g.d == 2 && !L.generic_lines && (g.J[0] == 256 || g.J[0] == 512 || g.J[0] == 1024) &&
                       (h == 128 || h == 256 || h == 512);
  return lines2d ? (long long)((g.hp1 + 7) & ~7) : (long long)g.hp1;
}

void launch_irfft(const LaunchCtx& L, const GridGeom& g, double2* H, double* x, const int* guard) {
  for (int ax = 0; ax <= g.d - 2; ++ax) c2c_axis(L, g, ax, +1, H, H, nullptr, 0, 0, 0, 1, 1.0, false);
  c2r_accum(L, g, H, 0, nullptr, 0, 0, 0, nullptr, x, nullptr, guard);
}

void launch_build_weights(const LaunchCtx& L, size_t Nh, int M, const double* mu2h, const double* base,
                          const double* logm, double* w) {
  k_build_weights<<<elementwise_grid(Nh), kThreads, 0, L.stream>>>((long long)Nh, M, mu2h, base, logm, w);
  count(L);
}

void launch_weights_from_lw(const LaunchCtx& L, size_t Nh, int M, const double* base, const double* lw,
                            double* w) {
  k_weights_from_lw<<<elementwise_grid(Nh), kThreads, 0, L.stream>>>((long long)Nh, M, base, lw, w);
  count(L);
}

void launch_dev1(const LaunchCtx& L, size_t N, const double* s, double s0, double* dev1) {
  k_dev1<<<elementwise_grid(N), kThreads, 0, L.stream>>>((long long)N, s, s0, dev1);
  count(L);
}

void launch_seis_start(const LaunchCtx& L, size_t N, double tau, const double* phi, const double* psi,
                       const double* c, const double* eta, const double* tc, const double* l1phi,
                       const double* l2psi, double* cur) {
  k_seis_start<<<elementwise_grid(N), kThreads, 0, L.stream>>>((long long)N, tau, phi, psi, c, eta, tc, l1phi,
                                                              l2psi, cur);
  count(L);
}

void launch_seis_update(const LaunchCtx& L, size_t N, double tau, const double* cur, const double* prev,
                        const double* ap, const double* l1, const double* l2, const double* c, const double* eta,
                        const double* tc, double* next, double thr, int step, int* flag) {
  k_seis_update<<<elementwise_grid(N), kThreads, 0, L.stream>>>((long long)N, tau, cur, prev, ap, l1, l2, c, eta,
                                                               tc, next, thr, step, flag);
  count(L);
}

void launch_seis_update_peers(const LaunchCtx& L, size_t N, double tau, const double* cur, const double* prev,
                              const double* ap, const double* l1, const double* l2, const double* c, const double* eta,
                              const double* tc, double* next, double* l2out, double thr, int step, int* flag,
                              const PeerFlags& peers) {
  k_seis_update_peers<<<elementwise_grid(N), kThreads, 0, L.stream>>>((long long)N, tau, cur, prev, ap, l1, l2, c, eta,
                                                                     tc, next, l2out, thr, step, flag, peers);
  count(L);
}

void launch_osc_rotate(const LaunchCtx& L, size_t Nh, const double* w, const double* cw, const double* sw, double dt,
                       double2* uh, double2* vh) {
  k_osc_rotate<<<elementwise_grid(Nh), kThreads, 0, L.stream>>>((long long)Nh, w, cw, sw, dt, uh, vh);
  count(L);
}

void launch_tsfp2_kick(const LaunchCtx& L, size_t N, double tau, double kappa, int cubic, const double* u,
                       const double* pert, double* v, const int* guard) {
  k_tsfp2_kick<<<elementwise_grid(N), kThreads, 0, L.stream>>>((long long)N, tau, kappa, cubic, u, pert, v, guard);
  count(L);
}

void launch_sup_check(const LaunchCtx& L, size_t N, const double* u, double thr, int step, int* flag) {
  k_sup_check<<<elementwise_grid(N), kThreads, 0, L.stream>>>((long long)N, u, thr, step, flag);
  count(L);
}

}  // namespace fw

namespace fw {
// ---- stage entry points for distributed (slab) orchestration: the same kernels as the
// single-device pipeline, applied to a local sub-array
void launch_stage_r2c(const LaunchCtx& L, const GridGeom& g, const double* u, double2* H, double scale,
                      bool do_scale) {
  if (!L.generic_lines && launch_rows_r2c(L, g.nl, u, H, (long long)g.rows, 1, scale, do_scale, nullptr)) return;
  const int h = g.nl / 2;
  const int lpb = std::max(1, std::min(8, 2048 / h));
  const size_t sm = smem_bytes(h + 1, lpb);
  const unsigned nb = (unsigned)((g.rows + lpb - 1) / lpb);
  k_r2c_rows<<<nb, kThreads, sm, L.stream>>>(u, H, g.nl, (long long)g.rows, lpb, scale, do_scale ? 1 : 0,
                                             L.master, nullptr);
  count(L);
}
void launch_stage_c2c(const LaunchCtx& L, const GridGeom& g, int axis, int dir, const double2* src, double2* dst,
                      const double* w, long long src_ts, long long dst_ts, long long w_ts, int nterms, double scale,
                      bool do_scale) {
  c2c_axis(L, g, axis, dir, src, dst, w, src_ts, dst_ts, w_ts, nterms, scale, do_scale);
}
void launch_stage_c2r(const LaunchCtx& L, const GridGeom& g, const double2* src, long long src_ts, int m_first,
                      int m_last, const double* dev1, double* out, double* residue) {
  c2r_accum(L, g, src, src_ts, nullptr, 0, m_first, m_last, dev1, out, residue, nullptr);
}
// ---- batched multi-field pipeline (grid.z = field)
void launch_forward_batch(const LaunchCtx& L, const GridGeom& g, int F, const BatchLine* tab_r2c,
                          const BatchLine* tab_c2c, bool scale) {
  const double inv = 1.0 / (double)g.N;
  const int h = g.nl / 2;
  if (L.generic_lines ||
      !launch_rows_r2c(L, g.nl, nullptr, nullptr, (long long)g.rows, F, inv, scale && g.d == 1, tab_r2c)) {
    const int lpb = std::max(1, std::min(8, 2048 / h));
    const size_t sm = smem_bytes(h + 1, lpb);
    const unsigned nb = (unsigned)((g.rows + lpb - 1) / lpb);
    k_r2c_rows<<<dim3(nb, 1, F), kThreads, sm, L.stream>>>(nullptr, nullptr, g.nl, (long long)g.rows, lpb, inv,
                                                           (scale && g.d == 1) ? 1 : 0, L.master, tab_r2c);
    count(L);
  }
  for (int a = g.d - 2; a >= 0; --a) {
    const int n = g.J[a];
    long long S = g.hp1;
    for (int b = a + 1; b <= g.d - 2; ++b) S *= g.J[b];
    long long outer = 1;
    for (int b = 0; b < a; ++b) outer *= g.J[b];
    if (!L.generic_lines && launch_lines(L, n, -1, nullptr, nullptr, nullptr, S, outer, S, 0, 0, 0, 1, F, inv,
                                         scale && a == 0, tab_c2c))
      continue;
    const int lp = std::max(1, std::min(8, 4096 / n));
    const long long bpo = (S + lp - 1) / lp;
    k_c2c_axis<-1><<<dim3((unsigned)(outer * bpo), 1, F), kThreads, smem_bytes(n, lp), L.stream>>>(
        nullptr, nullptr, nullptr, n, S, S, 0, 0, 0, lp, inv, (scale && a == 0) ? 1 : 0, L.master, tab_c2c);
    count(L);
  }
}

void launch_inverse_batch(const LaunchCtx& L, const GridGeom& g, int F, int m_first, int m_last,
                          const BatchLine* tab0, const BatchLine* tab1, const BatchLine* tab2, const int* guard,
                          bool resume) {
  const int nterms = m_last - m_first + 1;
  for (int a = 0; a <= g.d - 2; ++a) {
    const int n = g.J[a];
    long long S = g.hp1;
    for (int b = a + 1; b <= g.d - 2; ++b) S *= g.J[b];
    long long outer = 1;
    for (int b = 0; b < a; ++b) outer *= g.J[b];
    const long long xrs = term_row_stride(L, g, nterms);
    const long long ts = (long long)g.rows * xrs;  // T's term stride (rows padded for 2D grids)
    if (!L.generic_lines && launch_lines(L, n, +1, nullptr, nullptr, nullptr, S, outer, S, a == 0 ? 0 : ts, ts,
                                         a == 0 ? (long long)g.Nh : 0, nterms, F, 1.0, false, a == 0 ? tab0 : tab1,
                                         nullptr, (a == 0 && xrs != g.hp1) ? xrs : 0))
      continue;
    const int lp = std::max(1, std::min(8, 4096 / n));
    const long long bpo = (S + lp - 1) / lp;
    k_c2c_axis<+1><<<dim3((unsigned)(outer * bpo), (unsigned)nterms, F), kThreads, smem_bytes(n, lp), L.stream>>>(
        nullptr, nullptr, nullptr, n, S, S, a == 0 ? 0 : ts, ts, a == 0 ? ts : 0, lp, 1.0, 0, L.master,
        a == 0 ? tab0 : tab1);
    count(L);
  }
  if (!L.generic_lines && launch_rows_c2r(L, g.nl, nullptr, (long long)g.rows * term_row_stride(L, g, nterms), m_first,
                                         m_last, nullptr, nullptr, (long long)g.rows, F, nullptr, guard, tab2,
                                         term_row_stride(L, g, nterms), resume ? 1 : 0))
    return;
  const int h = g.nl / 2;
  const int lpb = std::max(1, std::min(8, 4096 / g.nl));
  const unsigned nb = (unsigned)((g.rows + lpb - 1) / lpb);
  k_c2r_accum<<<dim3(nb, 1, F), kThreads, smem_bytes(h + 1, lpb), L.stream>>>(
      nullptr, (long long)g.Nh, nullptr, 0, m_first, m_last, nullptr, nullptr, g.nl, (long long)g.rows, lpb, nullptr,
      guard, L.master, tab2);
  count(L);
}

}  // namespace fw
