// fw_wave.cu — elementwise and reduction kernels of the two-level integrators
// behind the reference's Laplacian seam: leap-frog LFFP (stepping.cpp:170-181),
// Crank–Nicolson CNFP with Picard + conjugate gradients (stepping.cpp:183-264),
// and their Taylor start (stepping.cpp:88-104).  The operator applies are the
// hot-path kernels (fw_apply_device); what is here is O(N) glue.
//
// Every elementwise expression keeps the reference's evaluation order (the
// library is built with --fmad=false), so LFFP is bit-identical to the
// reference.  The CG dot products are deterministic (fixed two-level tree) but
// not the reference's serial sums, so CNFP agrees to the CG tolerance.
#include <cuda_runtime.h>

#include "fw_internal.h"

namespace fw {
namespace {

constexpr int kT = 256;
constexpr int kDotBlocks = 148 * 4;  // partial sums per reduction (fixed: deterministic order)

int grid_for(size_t N) { return (int)std::min<size_t>((N + kT - 1) / kT, 148 * 16); }

#define FW_GRID_STRIDE(j, N) \
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < (N); j += (long long)gridDim.x * blockDim.x)

// f(u) of Nonlinearity (stepping.cpp:60-80): none -> 0.0, cubic -> u*u*u
__device__ __forceinline__ double f_of(int cubic, double u) { return cubic ? u * u * u : 0.0; }

// u1 = phi + tau psi + (tau^2/2)(-kappa L phi + f(phi))   (stepping.cpp:97-100)
__global__ void k_wave_start(long long N, double tau, double kappa, int cubic, const double* __restrict__ phi,
                             const double* __restrict__ psi, const double* __restrict__ lphi, double* __restrict__ u1) {
  const double half_t2 = 0.5 * tau * tau;
  FW_GRID_STRIDE(i, N) {
    u1[i] = phi[i] + tau * psi[i] + half_t2 * (-kappa * lphi[i] + f_of(cubic, phi[i]));
  }
}

// next = 2 cur - prev + tau^2 (-kappa L cur + f(cur))   (stepping.cpp:175-176); no writes once
// the blow-up flag is set (a multi-step batch keeps the pre-blow-up levels for the host)
__global__ void k_lffp_update(long long N, double t2, double kappa, int cubic, const double* __restrict__ cur,
                              const double* __restrict__ prev, const double* __restrict__ lu, double* __restrict__ next,
                              const int* __restrict__ flag) {
  if (*flag != kNoBlowup) return;
  FW_GRID_STRIDE(i, N) {
    next[i] = 2.0 * cur[i] - prev[i] + t2 * (-kappa * lu[i] + f_of(cubic, cur[i]));
  }
}

// rhs0 = 2u^n - u^{n-1} - alpha L u^{n-1} + (t2/2) f(u^{n-1})   (stepping.cpp:225-227)
__global__ void k_cnfp_rhs0(long long N, double t2, double alpha, int cubic, const double* __restrict__ cur,
                            const double* __restrict__ prev, const double* __restrict__ lprev, double* __restrict__ rhs0) {
  FW_GRID_STRIDE(i, N) {
    rhs0[i] = 2.0 * cur[i] - prev[i] - alpha * lprev[i] + 0.5 * t2 * f_of(cubic, prev[i]);
  }
}

// rhs = rhs0 + (t2/2) f(w)   (stepping.cpp:238-239)
__global__ void k_cnfp_rhs(long long N, double t2, const double* __restrict__ rhs0, const double* __restrict__ w,
                           double* __restrict__ rhs) {
  FW_GRID_STRIDE(i, N) {
    double v = rhs0[i];
    v += 0.5 * t2 * (w[i] * w[i] * w[i]);
    rhs[i] = v;
  }
}

// apply_A(w) = w + alpha L w   (stepping.cpp:189-194); optionally r = rhs - apply_A(w) (stepping.cpp:197-199)
__global__ void k_cg_apply_a(long long N, double alpha, const double* __restrict__ w, const double* __restrict__ lw,
                             const double* __restrict__ rhs, double* __restrict__ out) {
  FW_GRID_STRIDE(i, N) {
    const double a = w[i] + alpha * lw[i];
    out[i] = rhs ? rhs[i] - a : a;
  }
}

// x += a p; r -= a ap   (stepping.cpp:209-212)
__global__ void k_cg_step(long long N, double a, const double* __restrict__ p, const double* __restrict__ ap,
                          double* __restrict__ x, double* __restrict__ r) {
  FW_GRID_STRIDE(i, N) {
    x[i] += a * p[i];
    r[i] -= a * ap[i];
  }
}

// p = r + beta p   (stepping.cpp:217)
__global__ void k_cg_dir(long long N, double beta, const double* __restrict__ r, double* __restrict__ p) {
  FW_GRID_STRIDE(i, N) { p[i] = r[i] + beta * p[i]; }
}

// deterministic reductions: per-thread strided sums -> block tree -> partial[block];
// then one block sums the kDotBlocks partials in a fixed tree.  MODE 0: sum a*b,
// MODE 1: sum (a-b)^2 (the Picard difference, stepping.cpp:241-245)
template <int MODE>
__global__ void __launch_bounds__(kT) k_dot_partial(long long N, const double* __restrict__ a,
                                                    const double* __restrict__ b, double* __restrict__ partial) {
  __shared__ double s[kT];
  double acc = 0.0;
  FW_GRID_STRIDE(i, N) {
    if (MODE == 0) {
      acc += a[i] * b[i];
    } else {
      const double d = a[i] - b[i];
      acc += d * d;
    }
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kT / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = s[0];
}

__global__ void __launch_bounds__(1024) k_dot_final(int n, const double* __restrict__ partial, double* __restrict__ out) {
  __shared__ double s[1024];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) acc += partial[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

}  // namespace

size_t wave_partials() { return kDotBlocks; }

void launch_wave_start(const LaunchCtx& L, size_t N, double tau, double kappa, int cubic, const double* phi,
                       const double* psi, const double* lphi, double* u1) {
  k_wave_start<<<grid_for(N), kT, 0, L.stream>>>((long long)N, tau, kappa, cubic, phi, psi, lphi, u1);
  if (L.launches) *L.launches += 1;
}

void launch_lffp_update(const LaunchCtx& L, size_t N, double t2, double kappa, int cubic, const double* cur,
                        const double* prev, const double* lu, double* next, const int* flag) {
  k_lffp_update<<<grid_for(N), kT, 0, L.stream>>>((long long)N, t2, kappa, cubic, cur, prev, lu, next, flag);
  if (L.launches) *L.launches += 1;
}

void launch_cnfp_rhs0(const LaunchCtx& L, size_t N, double t2, double alpha, int cubic, const double* cur,
                      const double* prev, const double* lprev, double* rhs0) {
  k_cnfp_rhs0<<<grid_for(N), kT, 0, L.stream>>>((long long)N, t2, alpha, cubic, cur, prev, lprev, rhs0);
  if (L.launches) *L.launches += 1;
}

void launch_cnfp_rhs(const LaunchCtx& L, size_t N, double t2, const double* rhs0, const double* w, double* rhs) {
  k_cnfp_rhs<<<grid_for(N), kT, 0, L.stream>>>((long long)N, t2, rhs0, w, rhs);
  if (L.launches) *L.launches += 1;
}

void launch_cg_apply_a(const LaunchCtx& L, size_t N, double alpha, const double* w, const double* lw,
                       const double* rhs, double* out) {
  k_cg_apply_a<<<grid_for(N), kT, 0, L.stream>>>((long long)N, alpha, w, lw, rhs, out);
  if (L.launches) *L.launches += 1;
}

void launch_cg_step(const LaunchCtx& L, size_t N, double a, const double* p, const double* ap, double* x, double* r) {
  k_cg_step<<<grid_for(N), kT, 0, L.stream>>>((long long)N, a, p, ap, x, r);
  if (L.launches) *L.launches += 1;
}

void launch_cg_dir(const LaunchCtx& L, size_t N, double beta, const double* r, double* p) {
  k_cg_dir<<<grid_for(N), kT, 0, L.stream>>>((long long)N, beta, r, p);
  if (L.launches) *L.launches += 1;
}

void launch_dot(const LaunchCtx& L, size_t N, int mode, const double* a, const double* b, double* partial,
                double* out) {
  if (mode == 0)
    k_dot_partial<0><<<kDotBlocks, kT, 0, L.stream>>>((long long)N, a, b, partial);
  else
    k_dot_partial<1><<<kDotBlocks, kT, 0, L.stream>>>((long long)N, a, b, partial);
  k_dot_final<<<1, 1024, 0, L.stream>>>(kDotBlocks, partial, out);
  if (L.launches) *L.launches += 2;
}

}  // namespace fw
