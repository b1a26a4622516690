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

// ---- dense operator (flap.cpp:170-243) and the Toeplitz fast path (flap.cpp:245-285)
// G[b][k] = |mu_k|^{2 s_j} (row j = j0 + b; 0 at k = 0)
__global__ void k_dense_symbol(long long N, int B, long long j0, const double* __restrict__ mu2,
                               const double* __restrict__ s, double2* __restrict__ G) {
  const long long tot = (long long)B * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / N, k = e - b * N;
    const double m2 = mu2[k];
    G[e] = make_double2(m2 > 0.0 ? pow(m2, s[j0 + b]) : 0.0, 0.0);
  }
}
// entries[j][l] = Re G_j[(j - l) mod J per axis] / N (flap.cpp:203-225)
__global__ void k_dense_gather(long long N, int B, long long j0, int d, int J0, int J1, int J2,
                               const double2* __restrict__ G, double* __restrict__ A) {
  const int J[3] = {J0, J1, J2};
  const long long tot = (long long)B * N;
  const double inv = 1.0 / (double)N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / N, l = e - b * N, j = j0 + b;
    int jm[3] = {0, 0, 0}, lm[3] = {0, 0, 0};
    long long rj = j, rl = l;
    for (int m = d - 1; m >= 0; --m) {
      jm[m] = (int)(rj % J[m]);
      rj /= J[m];
      lm[m] = (int)(rl % J[m]);
      rl /= J[m];
    }
    long long shift = 0;
    for (int m = 0; m < d; ++m) shift = shift * J[m] + (jm[m] - lm[m] + J[m]) % J[m];
    A[j * N + l] = G[b * N + shift].x * inv;
  }
}
// out[j] = sum_l A[j][l] u[l]: one warp per row (flap.cpp:233-241; tree-ordered sum)
__global__ void k_dense_matvec(long long N, const double* __restrict__ A, const double* __restrict__ u,
                               double* __restrict__ out) {
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  for (long long j = blockIdx.x * (long long)(blockDim.x / 32) + threadIdx.x / 32; j < N; j += warps) {
    const double* row = A + j * N;
    double acc = 0.0;
    for (long long l = threadIdx.x & 31; l < N; l += 32) acc += row[l] * u[l];
#pragma unroll
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) out[j] = acc;
  }
}
// circulant embedding at 2J of the symmetric Toeplitz column t/J; x = u zero-padded
__global__ void k_toeplitz_embed(int J, const double2* __restrict__ t, const double* __restrict__ u,
                                 double2* __restrict__ c, double2* __restrict__ x) {
  const int n = 2 * J;
  const double inv = 1.0 / (double)J;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double cv = 0.0;
    if (i < J)
      cv = t[i].x * inv;
    else if (i > J)
      cv = t[n - i].x * inv;
    c[i] = make_double2(cv, 0.0);
    x[i] = make_double2(i < J ? u[i] : 0.0, 0.0);
  }
}
__global__ void k_cmul_inplace(int n, double2* __restrict__ x, const double2* __restrict__ c) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double2 a = x[i], b = c[i];  // std::complex<double> *= (flap.cpp:275)
    x[i] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
}
__global__ void k_real_scale(int J, const double2* __restrict__ x, double* __restrict__ out, double scale) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < J; i += gridDim.x * blockDim.x) out[i] = x[i].x * scale;
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
  return launch_dft_batched(L, chirps, d, J, 1, sign, x);
}

cudaError_t launch_dft_batched(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, long long batch, int sign,
                               double2* x) {
  long long S = 1;
  for (int a = d - 1; a >= 0; --a) {
    const int n = J[a];
    long long outer = batch;
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

cudaError_t launch_dense_assemble(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, long long N,
                                  const double* mu2, const double* s, double2* G, long long rows_per_batch,
                                  double* A) {
  for (long long j0 = 0; j0 < N; j0 += rows_per_batch) {
    const int B = (int)std::min<long long>(rows_per_batch, N - j0);
    k_dense_symbol<<<egrid((long long)B * N), kDftThreads, 0, L.stream>>>(N, B, j0, mu2, s, G);
    cudaError_t e = launch_dft_batched(L, chirps, d, J, B, +1, G);
    if (e != cudaSuccess) return e;
    k_dense_gather<<<egrid((long long)B * N), kDftThreads, 0, L.stream>>>(N, B, j0, d, J[0], d > 1 ? J[1] : 1,
                                                                           d > 2 ? J[2] : 1, G, A);
    if (L.launches) *L.launches += 2;
  }
  return cudaGetLastError();
}

cudaError_t launch_dense_matvec(const LaunchCtx& L, long long N, const double* A, const double* u, double* out) {
  const int wpb = kDftThreads / 32;
  k_dense_matvec<<<(unsigned)std::min<long long>((N + wpb - 1) / wpb, 148 * 32), kDftThreads, 0, L.stream>>>(N, A, u,
                                                                                                            out);
  if (L.launches) *L.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_toeplitz(const LaunchCtx& L, ChirpCache& chirps, int J, double2* t, const double* u, double2* c,
                            double2* x, double* out) {
  const int n = 2 * J;
  cudaError_t e = launch_dft(L, chirps, 1, &J, +1, t);  // first column, flap.cpp:259-263
  if (e != cudaSuccess) return e;
  k_toeplitz_embed<<<egrid(n), kDftThreads, 0, L.stream>>>(J, t, u, c, x);
  if ((e = launch_dft(L, chirps, 1, &n, -1, c)) != cudaSuccess) return e;
  if ((e = launch_dft(L, chirps, 1, &n, -1, x)) != cudaSuccess) return e;
  k_cmul_inplace<<<egrid(n), kDftThreads, 0, L.stream>>>(n, x, c);
  if ((e = launch_dft(L, chirps, 1, &n, +1, x)) != cudaSuccess) return e;
  k_real_scale<<<egrid(J), kDftThreads, 0, L.stream>>>(J, x, out, 1.0 / n);
  if (L.launches) *L.launches += 4;
  return cudaGetLastError();
}

cudaError_t launch_spectrum_mul(const LaunchCtx& L, long long n, const double* f, double2* x) {
  k_spectrum_mul<<<egrid(n), kDftThreads, 0, L.stream>>>(n, f, x);
  if (L.launches) *L.launches += 1;
  return cudaGetLastError();
}

}  // namespace fw
