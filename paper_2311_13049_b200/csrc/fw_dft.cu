// fw_dft.cu — general-length complex DFTs on the device and the full-spectrum form of the apply.
//
// Grid::dft (grid.cpp:134-137) is an in-place, unnormalised d-dimensional C2C DFT of any even
// axis lengths (the reference Grid accepts every even J >= 4, grid.cpp:44-50).  On the device:
//   * power-of-two axes (<= 4096): the canonical Stockham plan of fw_fft.cuh (launch_c2c_lines);
//   * other lengths (<= 2048): Bluestein's chirp-z form, a cyclic convolution through the same
//     power-of-two FFT: with w_j = exp(sign i pi j^2 / n),  W^{jk} = w_j w_k / w_{k-j}, so
//     X_k = w_k sum_j (x_j w_j) conj(w_{k-j}) = w_k (a * b)_k  (length m = pow2 >= 2n-1);
//     the chirp (angle sign pi (j^2 mod 2n) / n in long double) and the transformed filter are
//     built once per (n, sign) and cached on the context.
// The full-spectrum apply is flap.cpp:38-92 in the reference's own C2C formulation (uhat =
// DFT(u)/N, per term IDFT(w_m .* uhat), acc += (s-s0)^m Re, max |Im|); it serves the grids the
// real-transform pipeline does not (non-power-of-two axes), with no CPU fallback.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <vector>

#include "fw_fft.cuh"
#include "fw_internal.h"

namespace fw {

namespace {

constexpr int kDftThreads = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// one line per block: x_j at line + j S, j < n
__global__ void __launch_bounds__(kDftThreads) k_bluestein(double2* __restrict__ x, int n, long long S, int m,
                                                           const double2* __restrict__ w,
                                                           const double2* __restrict__ bhat,
                                                           const double2* __restrict__ master) {
  extern __shared__ double2 sm[];
  double2* b0 = sm;
  double2* b1 = sm + m;
  const long long o = blockIdx.x / S, in = blockIdx.x - (blockIdx.x / S) * S;
  double2* line = x + o * (long long)n * S + in;
  for (int j = threadIdx.x; j < m; j += blockDim.x) b0[j] = j < n ? cmul(line[(long long)j * S], w[j]) : make_double2(0.0, 0.0);
  __syncthreads();
  double2* R = smem_c2c<-1>(b0, b1, m, 1, m, master);
  for (int j = threadIdx.x; j < m; j += blockDim.x) R[j] = cmul(R[j], bhat[j]);
  __syncthreads();
  double2* Q = smem_c2c<+1>(R, R == b0 ? b1 : b0, m, 1, m, master);
  for (int k = threadIdx.x; k < n; k += blockDim.x) line[(long long)k * S] = cmul(w[k], Q[k]);
}

// bhat = FFT_{-1}(B) / m, B[t] = conj(w_t) (t < n), B[m - t] = conj(w_t) (1 <= t < n), else 0
__global__ void __launch_bounds__(kDftThreads) k_chirp_filter(int n, int m, const double2* __restrict__ w,
                                                              double2* __restrict__ bhat,
                                                              const double2* __restrict__ master) {
  extern __shared__ double2 sm[];
  double2* b0 = sm;
  double2* b1 = sm + m;
  for (int t = threadIdx.x; t < m; t += blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (t < n)
      v = make_double2(w[t].x, -w[t].y);
    else if (m - t < n)
      v = make_double2(w[m - t].x, -w[m - t].y);
    b0[t] = v;
  }
  __syncthreads();
  const double2* R = smem_c2c<-1>(b0, b1, m, 1, m, master);
  const double inv = 1.0 / (double)m;
  for (int t = threadIdx.x; t < m; t += blockDim.x) bhat[t] = make_double2(R[t].x * inv, R[t].y * inv);
}

__global__ void k_real_to_complex(long long N, const double* __restrict__ u, double2* __restrict__ x) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x)
    x[j] = make_double2(u[j], 0.0);
}
__global__ void k_scale(long long N, double2* __restrict__ x, double s) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    x[j].x *= s;  // std::complex<double> *= double (grid.cpp:176-178, flap.cpp:49-50)
    x[j].y *= s;
  }
}
// buf = w .* uhat (flap.cpp:27; real weight times complex)
__global__ void k_weight(long long N, const double* __restrict__ w, const double2* __restrict__ uh,
                         double2* __restrict__ buf) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const double wk = w[j];
    buf[j] = make_double2(wk * uh[j].x, wk * uh[j].y);
  }
}
// term m of flap.cpp:21-36 + the ordered reduction (82-89): p = 0 + dev^m Re, out += p,
// dev^m by the reference recurrence (flap.cpp:124-133) in devm; residue = max |Im|
__global__ void k_accum_term(long long N, int m, int first, const double2* __restrict__ buf,
                             const double* __restrict__ dev1, double* __restrict__ devm, double* __restrict__ out,
                             double* residue, const int* guard) {
  if (guard && *guard != kNoBlowup) return;
  double rmax = 0.0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const double re = buf[j].x;
    double p = 0.0;
    if (m == 0) {
      p += re;
    } else {
      const double d = m == 1 ? dev1[j] : devm[j] * dev1[j];
      devm[j] = d;
      p += d * re;
    }
    out[j] = (first ? 0.0 : out[j]) + p;
    rmax = fmax(rmax, fabs(buf[j].y));
  }
  if (residue) {
#pragma unroll
    for (int off = 16; off; off >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
    if ((threadIdx.x & 31) == 0 && rmax > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(residue), (unsigned long long)__double_as_longlong(rmax));
  }
}
// out = Re(x), residue = max |Im|  (Grid::inverse, grid.cpp:181-197)
__global__ void k_real_part(long long N, const double2* __restrict__ x, double* __restrict__ out, double* residue) {
  double rmax = 0.0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    out[j] = x[j].x;
    rmax = fmax(rmax, fabs(x[j].y));
  }
  if (residue) {
#pragma unroll
    for (int off = 16; off; off >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
    if ((threadIdx.x & 31) == 0 && rmax > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(residue), (unsigned long long)__double_as_longlong(rmax));
  }
}
// spectrum *= |mu|^{2s} (flap.cpp:143-144), the multiplier computed on the host with glibc pow
__global__ void k_spectrum_mul(long long n, const double* __restrict__ f, double2* __restrict__ x) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const double fk = f[j];
    x[j].x *= fk;
    x[j].y *= fk;
  }
}

int egrid(long long N) { return (int)std::min<long long>((N + kDftThreads - 1) / kDftThreads, 148 * 16); }

bool is_pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }

}  // namespace

bool dft_length_supported(int n) { return is_pow2(n) ? n <= kTwMaster / 2 : (n >= 2 && n <= kMaxBluestein); }

void ChirpCache::release() {
  for (auto& e : entries) {
    if (e.w) cudaFree(e.w);
    if (e.bhat) cudaFree(e.bhat);
  }
  entries.clear();
}

cudaError_t ChirpCache::get(const LaunchCtx& L, int n, int sign, const Entry** out) {
  for (const auto& e : entries)
    if (e.n == n && e.sign == sign) {
      *out = &e;
      return cudaSuccess;
    }
  Entry e;
  e.n = n;
  e.sign = sign;
  e.m = 1;
  while (e.m < 2 * n - 1) e.m *= 2;
  std::vector<double2> w(n);
  for (long long j = 0; j < n; ++j) {  // angle sign pi (j^2 mod 2n) / n, exact argument reduction
    const long long q = (j * j) % (2LL * n);
    const long double ang = (long double)sign * 3.141592653589793238462643383279502884L * (long double)q / (long double)n;
    w[j] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  cudaError_t err;
  if ((err = cudaMalloc(&e.w, n * sizeof(double2))) != cudaSuccess) return err;
  if ((err = cudaMalloc(&e.bhat, e.m * sizeof(double2))) != cudaSuccess) {
    cudaFree(e.w);
    return err;
  }
  cudaMemcpyAsync(e.w, w.data(), n * sizeof(double2), cudaMemcpyHostToDevice, L.stream);
  const size_t sm = 2 * (size_t)e.m * sizeof(double2);
  cudaFuncSetAttribute(k_chirp_filter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_chirp_filter<<<1, kDftThreads, sm, L.stream>>>(n, e.m, e.w, e.bhat, L.master);
  if (L.launches) *L.launches += 1;
  if ((err = cudaStreamSynchronize(L.stream)) != cudaSuccess) return err;  // w (host vector) copied
  entries.push_back(e);
  *out = &entries.back();
  return cudaSuccess;
}

cudaError_t launch_dft(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, int sign, double2* x) {
  long long S = 1;
  for (int a = d - 1; a >= 0; --a) {
    const int n = J[a];
    long long outer = 1;
    for (int b = 0; b < a; ++b) outer *= J[b];
    if (is_pow2(n)) {
      launch_c2c_lines(L, n, S, outer, sign < 0 ? -1 : +1, x, 1.0, false);
    } else {
      const ChirpCache::Entry* e = nullptr;
      cudaError_t err = chirps.get(L, n, sign < 0 ? -1 : +1, &e);
      if (err != cudaSuccess) return err;
      const size_t sm = 2 * (size_t)e->m * sizeof(double2);
      cudaFuncSetAttribute(k_bluestein, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_bluestein<<<(unsigned)(outer * S), kDftThreads, sm, L.stream>>>(x, n, S, e->m, e->w, e->bhat, L.master);
      if (L.launches) *L.launches += 1;
    }
    S *= n;
  }
  return cudaGetLastError();
}

cudaError_t launch_full_forward(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, long long N,
                                const double* u, double2* uh, bool scale) {
  k_real_to_complex<<<egrid(N), kDftThreads, 0, L.stream>>>(N, u, uh);
  if (L.launches) *L.launches += 1;
  cudaError_t e = launch_dft(L, chirps, d, J, -1, uh);
  if (e != cudaSuccess) return e;
  if (scale) {
    k_scale<<<egrid(N), kDftThreads, 0, L.stream>>>(N, uh, 1.0 / (double)N);
    if (L.launches) *L.launches += 1;
  }
  return cudaGetLastError();
}

cudaError_t launch_full_apply(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, long long N,
                              const FullApplyArgs& a) {
  for (int m = a.m_first; m <= a.m_last; ++m) {
    k_weight<<<egrid(N), kDftThreads, 0, L.stream>>>(N, a.w + (size_t)m * N, a.uh, a.buf);
    if (L.launches) *L.launches += 1;
    cudaError_t e = launch_dft(L, chirps, d, J, +1, a.buf);
    if (e != cudaSuccess) return e;
    k_accum_term<<<egrid(N), kDftThreads, 0, L.stream>>>(N, m, m == a.m_first ? 1 : 0, a.buf, a.dev1, a.devm, a.out,
                                                        a.residue, a.guard);
    if (L.launches) *L.launches += 1;
  }
  return cudaGetLastError();
}

cudaError_t launch_real_part(const LaunchCtx& L, long long N, const double2* x, double* out, double* residue) {
  k_real_part<<<egrid(N), kDftThreads, 0, L.stream>>>(N, x, out, residue);
  if (L.launches) *L.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_spectrum_mul(const LaunchCtx& L, long long n, const double* f, double2* x) {
  k_spectrum_mul<<<egrid(n), kDftThreads, 0, L.stream>>>(n, f, x);
  if (L.launches) *L.launches += 1;
  return cudaGetLastError();
}

}  // namespace fw
