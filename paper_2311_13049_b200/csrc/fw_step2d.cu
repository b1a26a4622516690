// fw_step2d.cu — persistent single-launch 2D apply / seismic step for sm_100a.
//
// One cooperative launch of one CTA per SM does the whole seismic step (or one
// operator apply) on a J0 x J1 grid (half spectrum H = J1/2 + 1 columns):
//
//   F1  every CTA: R2C of its rows of u                        -> Y (global, L2)
//   --- grid counter ---
//   F2  column CTAs: C2C of their CG columns of Y, x 1/N       -> uhat (SHARED MEMORY, kept)
//   for t = (op, m), m = m_first..M of every operator, pipelined through a K-slot ring:
//     C(t) column CTAs: (w_m .* uhat) -> inverse C2C          -> T[t mod K] (global, L2)
//     R(t) every CTA : T rows -> C2R (pre-processing fused into the first pass)
//                      -> acc += (s-s0)^m .* x  (accumulators in registers,
//                      (s-s0)^m rows staged into shared memory by cp.async)
//   update (seismic.cpp:116-129) from the registers: next, new L2prev, blow-up flag
//
// The term intermediate T is the only global round trip per term (a 2D FFT is
// an all-to-all across SMs); the forward spectrum and the accumulators never
// leave the SM.  CTAs order themselves with monotone per-term counters
// (red.release / ld.acquire); the ring lets column work run K-1 terms ahead of
// row work.  Arithmetic is the canonical FFT of fw_fft.cuh (radix plan, twiddle
// values, fma placement), so results are bit-identical to the multi-pass path
// and to the CPU oracle.  Twiddles of every pass live in shared memory in a
// [k][r-1] layout (odd stride: conflict-free).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fw_fft.cuh"
#include "fw_internal.h"
#include "fw_step2d.h"

namespace fw {
namespace s2d {

constexpr int NT = 256;  // threads per CTA (8 warps, up to 255 registers each)
constexpr int KRING = 3;

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int npass(int n) { return (ilog2c(n) + 3) / 4; }
__host__ __device__ constexpr int radix(int n, int i) {
  return 1 << (ilog2c(n) / npass(n) + (i < ilog2c(n) % npass(n) ? 1 : 0));
}
__host__ __device__ constexpr int pprod(int n, int i) { return i == 0 ? 1 : pprod(n, i - 1) * radix(n, i - 1); }
__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
// per-pass twiddle table sizes / offsets of an N-point plan (pass 0 has none)
__host__ __device__ constexpr int twsize(int n, int pass) { return pass == 0 ? 0 : pprod(n, pass) * (radix(n, pass) - 1); }
__host__ __device__ constexpr int twoff(int n, int pass) { return pass <= 1 ? 0 : twoff(n, pass - 1) + twsize(n, pass - 1); }
__host__ __device__ constexpr int twtotal(int n) { return twoff(n, npass(n) - 1) + twsize(n, npass(n) - 1); }

// ---------------------------------------------------------------- sync helpers
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void wait_counter(const unsigned long long* cnt, unsigned long long target) {
  if (threadIdx.x == 0) {
    while (ld_acquire(cnt) < target) __nanosleep(20);
  }
  __syncthreads();
}
__device__ __forceinline__ void signal_counter(unsigned long long* cnt) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    red_release_add(cnt, 1ull);
  }
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int DIR>
__device__ __forceinline__ double2 dirw(double2 w) {
  return make_double2(w.x, DIR < 0 ? -w.y : w.y);
}

// Stockham butterfly of pass PASS (N-point plan) on register array a (butterfly i);
// tw = this N's per-pass table block.
template <int N, int PASS, int DIR>
__device__ __forceinline__ void butterfly(double2* a, int i, const double2* tw) {
  constexpr int R = radix(N, PASS);
  constexpr int p = pprod(N, PASS);
  if constexpr (p > 1) {
    const int k = i & (p - 1);
    const double2* t = tw + twoff(N, PASS) + k * (R - 1);
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const double2 w = dirw<DIR>(t[r - 1]);
      a[r] = cmulw(a[r], w.x, w.y);
    }
  }
  Dft<R, DIR>::run(a);
}

template <int N, int PASS>
__device__ __forceinline__ int out_index(int i, int r) {
  constexpr int R = radix(N, PASS);
  constexpr int p = pprod(N, PASS);
  const int k = i & (p - 1);
  return (i - k) * R + k + r * p;
}

template <int PADSH>
__device__ __forceinline__ int padq(int q) {
  return q + (q >> PADSH);
}

template <int T, bool LINE_FAST, int NLC>
__device__ __forceinline__ void bmap(int b, int& l, int& i) {
  if constexpr (LINE_FAST) {
    l = b % NLC;
    i = b / NLC;
  } else {
    l = b / T;
    i = b % T;
  }
}

// Middle pass PASS of an N-point C2C over nl lines, in place in shared memory.
template <int N, int PASS, int DIR, int PADSH, int LS, bool LINE_FAST, int NLMAX>
__device__ __forceinline__ void smem_pass(double2* buf, int nl, const double2* tw) {
  constexpr int R = radix(N, PASS);
  constexpr int T = N / R;
  constexpr int NB = cdiv(NLMAX * T, NT);
  const int tid = threadIdx.x;
  double2 a[NB][R];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    int l, i;
    bmap<T, LINE_FAST, NLMAX>(tid + j * NT, l, i);
    if (l < nl && i < T) {
#pragma unroll
      for (int r = 0; r < R; ++r) a[j][r] = buf[l * LS + padq<PADSH>(i + r * T)];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    int l, i;
    bmap<T, LINE_FAST, NLMAX>(tid + j * NT, l, i);
    if (l < nl && i < T) {
      butterfly<N, PASS, DIR>(a[j], i, tw);
#pragma unroll
      for (int r = 0; r < R; ++r) buf[l * LS + padq<PADSH>(out_index<N, PASS>(i, r))] = a[j][r];
    }
  }
  __syncthreads();
}

// --------------------------------------------------------------------------
template <int J0, int J1, int CG, int RMAX>
struct Geo {
  static constexpr int H = J1 / 2 + 1;               // half-spectrum columns
  static constexpr int h = J1 / 2;                   // row C2C length
  static constexpr int NG = (H + CG - 1) / CG;       // column groups
  static constexpr int PADC = ilog2c(radix(J0, 0));  // column pad shift
  static constexpr int PADR = ilog2c(radix(h, 0));   // row pad shift
  static constexpr int LSU = J0 + (CG == 4 ? 2 : CG == 2 ? 4 : 1);
  static constexpr int LSC0 = J0 + (J0 >> PADC);
  static constexpr int LSC = LSC0 + ((10 - LSC0 % 8) % 8);  // == 2 mod 8
  static constexpr int LSR = h + (h >> PADR) + 2;
  static constexpr int PC = npass(J0);
  static constexpr int PR = npass(h);
  static constexpr int RL = radix(h, PR - 1);  // last row pass
  static constexpr int TL = h / RL;
  static constexpr int NBL = cdiv(RMAX * TL, NT);  // last-pass butterflies per thread
  static constexpr int TWC = twtotal(J0);
  static constexpr int TWR = twtotal(h);
  static constexpr int TWP = h + 1;  // W_J1^k, k = 0..h
  static constexpr size_t SMEM_TW = sizeof(double2) * (TWC + TWR + TWP);
  static constexpr size_t SMEM_U = sizeof(double2) * CG * LSU;
  static constexpr size_t SMEM_W = sizeof(double2) * (CG * LSC > RMAX * LSR ? CG * LSC : RMAX * LSR);
  static constexpr size_t SMEM_D = sizeof(double) * RMAX * J1;  // (s-s0)^m staging
  static constexpr size_t SMEM = SMEM_TW + SMEM_U + SMEM_W + SMEM_D;
  static_assert(PC <= 3 && PR <= 3 && PR >= 2 && PC >= 2, "2 or 3 passes per FFT");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

// ---------------------------------------------------------------- column FFT
// J0-point C2C of the CTA's CG columns (lines interleaved fastest).  Pass 0 reads
// src(cc, q); the last pass writes sink(cc, q, value) in natural order q.
template <int J0, int CG, int DIR, int PADSH, int LSC, class Src, class Sink>
__device__ __forceinline__ void column_fft(double2* cbuf, const double2* tw, int ncols, Src src, Sink sink) {
  constexpr int P = npass(J0);
  const int tid = threadIdx.x;
  {
    constexpr int R = radix(J0, 0);
    constexpr int T = J0 / R;
    constexpr int NB = cdiv(CG * T, NT);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      int cc, i;
      bmap<T, true, CG>(tid + j * NT, cc, i);
      if (i < T && cc < ncols) {
        double2 a[R];
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = src(cc, i + r * T);
        Dft<R, DIR>::run(a);
#pragma unroll
        for (int r = 0; r < R; ++r) cbuf[cc * LSC + padq<PADSH>(i * R + r)] = a[r];
      }
    }
    __syncthreads();
  }
  if constexpr (P == 3) smem_pass<J0, 1, DIR, PADSH, LSC, true, CG>(cbuf, CG, tw);
  {
    constexpr int PL = P - 1;
    constexpr int R = radix(J0, PL);
    constexpr int T = J0 / R;
    constexpr int NB = cdiv(CG * T, NT);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      int cc, i;
      bmap<T, true, CG>(tid + j * NT, cc, i);
      if (i < T && cc < ncols) {
        double2 a[R];
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = cbuf[cc * LSC + padq<PADSH>(i + r * T)];
        butterfly<J0, PL, DIR>(a, i, tw);
#pragma unroll
        for (int r = 0; r < R; ++r) sink(cc, i + r * T, a[r]);
      }
    }
  }
}

// R2C post-processing X[k] from Z[k], Z[h-k] (fwcanon fwc_r2c), 1 <= k < h
__device__ __forceinline__ double2 post_r2c(double2 A, double2 Bz, double2 wk) {
  const double2 B = make_double2(Bz.x, -Bz.y);
  const double2 E = make_double2((A.x + B.x) * 0.5, (A.y + B.y) * 0.5);
  const double2 D = make_double2((A.x - B.x) * 0.5, (A.y - B.y) * 0.5);
  const double2 O = make_double2(D.y, -D.x);
  const double2 w = dirw<-1>(wk);
  const double2 t = cmulw(O, w.x, w.y);
  return make_double2(E.x + t.x, E.y + t.y);
}

// C2R pre-processing Z[k] from X[k], X[h-k] (fwcanon fwc_c2r)
__device__ __forceinline__ double2 pre_c2r(double2 A, double2 Xhk, bool k0, double2 wk) {
  double2 B = make_double2(Xhk.x, -Xhk.y);
  if (k0) {
    A.y = 0.0;
    B.y = 0.0;
  }
  const double2 E = make_double2(A.x + B.x, A.y + B.y);
  const double2 D = make_double2(A.x - B.x, A.y - B.y);
  const double2 O = cmulw(D, wk.x, wk.y);
  return make_double2(E.x - O.y, E.y + O.x);
}

// --------------------------------------------------------------------------
template <int J0, int J1, int CG, int RMAX>
__global__ void __launch_bounds__(NT, 1) k_step2d(const Step2DParams prm) {
  using G = Geo<J0, J1, CG, RMAX>;
  constexpr int H = G::H, h = G::h;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* twc = reinterpret_cast<double2*>(smem_raw);  // column plan tables
  double2* twr = twc + G::TWC;                          // row plan tables
  double2* twp = twr + G::TWR;                          // W_J1^k
  double2* uhat = reinterpret_cast<double2*>(smem_raw + G::SMEM_TW);
  double2* work = reinterpret_cast<double2*>(smem_raw + G::SMEM_TW + G::SMEM_U);
  double* devs = reinterpret_cast<double*>(smem_raw + G::SMEM_TW + G::SMEM_U + G::SMEM_W);
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  const int nblk = gridDim.x;

  // counters: this launch uses set `cset`, and clears the other set for the next launch
  unsigned long long* cnt = prm.counters + (size_t)prm.cset * prm.cstride;
  if (b == 0) {
    unsigned long long* other = prm.counters + (size_t)(prm.cset ^ 1) * prm.cstride;
    for (int e = tid; e < prm.cstride; e += NT) other[e] = 0ull;
  }
  if (prm.flag && *prm.flag != kNoBlowup) return;  // uniform across CTAs
  unsigned long long* cY = cnt;
  unsigned long long* cC = cnt + 1;
  unsigned long long* cR = cnt + 1 + prm.nterms_total;

  // twiddle tables (values = master entries, identical to fw_fft.cuh's twiddle())
  {
    auto fill = [&](double2* dst, int off, int p, int R) {
      const int n = p * (R - 1);
      for (int e = tid; e < n; e += NT) {
        const int k = e / (R - 1), r = e % (R - 1) + 1;
        dst[off + e] = prm.master[(r * k) * (kTwMaster / (p * R))];
      }
    };
    if constexpr (G::PC >= 2) fill(twc, twoff(J0, 1), pprod(J0, 1), radix(J0, 1));
    if constexpr (G::PC >= 3) fill(twc, twoff(J0, 2), pprod(J0, 2), radix(J0, 2));
    if constexpr (G::PR >= 2) fill(twr, twoff(h, 1), pprod(h, 1), radix(h, 1));
    if constexpr (G::PR >= 3) fill(twr, twoff(h, 2), pprod(h, 2), radix(h, 2));
    for (int e = tid; e <= h; e += NT) twp[e] = prm.master[e * (kTwMaster / J1)];
  }

  const int r0 = (int)(((long long)b * J0) / nblk);
  const int r1 = (int)(((long long)(b + 1) * J0) / nblk);
  const int nrows = r1 - r0;
  const bool has_cols = b < G::NG;
  const int c0 = b * CG;
  const int ncols = has_cols ? min(CG, H - c0) : 0;
  __syncthreads();

  // ------------------------------------------------ F1: forward rows -> Y
  {
    constexpr int R0 = radix(h, 0);
    constexpr int T0 = h / R0;
    constexpr int NB0 = cdiv(RMAX * T0, NT);
    const double2* u2 = reinterpret_cast<const double2*>(prm.u);
#pragma unroll
    for (int j = 0; j < NB0; ++j) {  // pass 0 straight from global: packed pairs z_q = x_2q + i x_2q+1
      const int bb = tid + j * NT, l = bb / T0, i = bb % T0;
      if (l < nrows) {
        double2 a[R0];
#pragma unroll
        for (int r = 0; r < R0; ++r) a[r] = u2[(size_t)(r0 + l) * h + i + r * T0];
        Dft<R0, -1>::run(a);
#pragma unroll
        for (int r = 0; r < R0; ++r) work[l * G::LSR + padq<G::PADR>(i * R0 + r)] = a[r];
      }
    }
    __syncthreads();
    if constexpr (G::PR == 3) smem_pass<h, 1, -1, G::PADR, G::LSR, false, RMAX>(work, nrows, twr);
#pragma unroll
    for (int j = 0; j < G::NBL; ++j) {  // last pass, written back to the slots it read
      const int bb = tid + j * NT, l = bb / G::TL, i = bb % G::TL;
      if (l < nrows) {
        double2 a[G::RL];
#pragma unroll
        for (int r = 0; r < G::RL; ++r) a[r] = work[l * G::LSR + padq<G::PADR>(i + r * G::TL)];
        butterfly<h, G::PR - 1, -1>(a, i, twr);
#pragma unroll
        for (int r = 0; r < G::RL; ++r) work[l * G::LSR + padq<G::PADR>(i + r * G::TL)] = a[r];
      }
    }
    __syncthreads();
    constexpr int NP = h / 2 + 1;
    for (int l = 0; l < nrows; ++l) {  // post-process pairs (k, h-k)
      const double2* Z = work + l * G::LSR;
      double2* Yr = prm.Y + (size_t)(r0 + l) * H;
      for (int jj = tid; jj < NP; jj += NT) {
        if (jj == 0) {
          const double2 z0 = Z[0];
          __stcg(&Yr[0], make_double2(z0.x + z0.y, 0.0));
          __stcg(&Yr[h], make_double2(z0.x - z0.y, 0.0));
        } else {
          const double2 A = Z[padq<G::PADR>(jj)];
          const double2 B = Z[padq<G::PADR>(h - jj)];
          __stcg(&Yr[jj], post_r2c(A, B, twp[jj]));
          if (jj != h - jj) __stcg(&Yr[h - jj], post_r2c(B, A, twp[h - jj]));
        }
      }
    }
    signal_counter(cY);
  }

  // ------------------------------------------------ F2: forward columns -> uhat (smem)
  if (has_cols) {
    wait_counter(cY, (unsigned long long)nblk);
    const double inv = 1.0 / ((double)J0 * (double)J1);
    const double2* Y = prm.Y;
    column_fft<J0, CG, -1, G::PADC, G::LSC>(
        work, twc, ncols, [&](int cc, int q) { return __ldcg(&Y[(size_t)q * H + c0 + cc]); },
        [&](int cc, int q, double2 v) { uhat[cc * G::LSU + q] = make_double2(v.x * inv, v.y * inv); });
    __syncthreads();
  }

  // ------------------------------------------------ terms
  const int M = prm.M;
  const int nterms = M + 1 - prm.m_first;
  const int ntot = prm.nops * nterms;

  auto column_term = [&](int t) {
    if (!has_cols) return;
    if (t >= KRING) wait_counter(&cR[t - KRING], (unsigned long long)nblk);
    const int op = t / nterms;
    const int m = prm.m_first + t % nterms;
    const double* w = prm.w[op] + ((size_t)m * G::NG + b) * (size_t)J0 * CG;  // [m][g][k0][CG]
    double2* T = prm.T + (size_t)(t % KRING) * J0 * H;
    column_fft<J0, CG, +1, G::PADC, G::LSC>(
        work, twc, ncols,
        [&](int cc, int q) {
          const double2 v = uhat[cc * G::LSU + q];
          const double wk = __ldg(&w[(size_t)q * CG + cc]);
          return make_double2(wk * v.x, wk * v.y);
        },
        [&](int cc, int q, double2 v) { __stcg(&T[(size_t)q * H + c0 + cc], v); });
    signal_counter(&cC[t]);
  };

  double acc[G::NBL][G::RL][2];
#pragma unroll
  for (int j = 0; j < G::NBL; ++j)
#pragma unroll
    for (int r = 0; r < G::RL; ++r) acc[j][r][0] = acc[j][r][1] = 0.0;

  double rmax = 0.0;
  auto row_term = [&](int t) {
    wait_counter(&cC[t], (unsigned long long)G::NG);
    const int op = t / nterms;
    const int m = prm.m_first + t % nterms;
    const double2* T = prm.T + (size_t)(t % KRING) * J0 * H;
    if (m >= 1) {  // stage (s-s0)^m rows asynchronously
      const double* dv = prm.dev[op] + (size_t)(m - 1) * J0 * J1 + (size_t)r0 * J1;
      const int nchunk = nrows * J1 / 2;
      for (int e = tid; e < nchunk; e += NT) cp_async16(devs + 2 * e, dv + 2 * e);
      cp_async_commit();
    }
    {  // pass 0 with the C2R pre-processing fused: unit i pairs butterflies i and T0-i
      constexpr int R0 = radix(h, 0);
      constexpr int T0 = h / R0;
      constexpr int NU = T0 / 2 + 1;  // units per row
      constexpr int NBU = cdiv(RMAX * NU, NT);
#pragma unroll
      for (int j = 0; j < NBU; ++j) {
        const int bb = tid + j * NT, l = bb / NU, i = bb % NU;
        if (l < nrows) {
          const double2* X = T + (size_t)(r0 + l) * H;
          const int i2 = T0 - i;  // mirror butterfly; for i == 0 this walks X[T0 (r+1)], ending at X[h]
          double2 XA[R0], XB[R0];
#pragma unroll
          for (int r = 0; r < R0; ++r) XA[r] = __ldcg(&X[i + r * T0]);
#pragma unroll
          for (int r = 0; r < R0; ++r) XB[r] = __ldcg(&X[i2 + r * T0]);
          double2 a[R0];
          if (i == 0) {
            if (prm.residue) rmax = fmax(rmax, fabs(XA[0].y) + fabs(XB[R0 - 1].y));
#pragma unroll
            for (int r = 0; r < R0; ++r)  // k = r*T0, h-k = (R0-r)*T0 = XB[R0-1-r]
              a[r] = pre_c2r(XA[r], XB[R0 - 1 - r], r == 0, twp[r * T0]);
            Dft<R0, +1>::run(a);
#pragma unroll
            for (int r = 0; r < R0; ++r) work[l * G::LSR + padq<G::PADR>(r)] = a[r];
          } else {
            // butterfly i: k = i + r*T0, h-k = (T0-i) + (R0-1-r)*T0 -> XB[R0-1-r]
#pragma unroll
            for (int r = 0; r < R0; ++r) a[r] = pre_c2r(XA[r], XB[R0 - 1 - r], false, twp[i + r * T0]);
            Dft<R0, +1>::run(a);
#pragma unroll
            for (int r = 0; r < R0; ++r) work[l * G::LSR + padq<G::PADR>(i * R0 + r)] = a[r];
            if (i2 != i) {  // butterfly T0-i: k = i2 + r*T0, h-k = i + (R0-1-r)*T0 -> XA[R0-1-r]
#pragma unroll
              for (int r = 0; r < R0; ++r) a[r] = pre_c2r(XB[r], XA[R0 - 1 - r], false, twp[i2 + r * T0]);
              Dft<R0, +1>::run(a);
#pragma unroll
              for (int r = 0; r < R0; ++r) work[l * G::LSR + padq<G::PADR>(i2 * R0 + r)] = a[r];
            }
          }
        }
      }
      __syncthreads();
    }
    if constexpr (G::PR == 3) smem_pass<h, 1, +1, G::PADR, G::LSR, false, RMAX>(work, nrows, twr);
    if (m >= 1) {
      cp_async_wait_all();
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < G::NBL; ++j) {  // last pass + recombination in registers
      const int bb = tid + j * NT, l = bb / G::TL, i = bb % G::TL;
      if (l < nrows) {
        double2 a[G::RL];
#pragma unroll
        for (int r = 0; r < G::RL; ++r) a[r] = work[l * G::LSR + padq<G::PADR>(i + r * G::TL)];
        butterfly<h, G::PR - 1, +1>(a, i, twr);
        const double2* dv2 = reinterpret_cast<const double2*>(devs + l * J1);
#pragma unroll
        for (int r = 0; r < G::RL; ++r) {
          const int q = i + r * G::TL;  // x[2q], x[2q+1]
          double v0 = a[r].x, v1 = a[r].y;
          if (m >= 1) {
            const double2 d = dv2[q];
            v0 = d.x * v0;
            v1 = d.y * v1;
          }
          double p0 = 0.0, p1 = 0.0;
          p0 += v0;
          p1 += v1;
          acc[j][r][0] += p0;
          acc[j][r][1] += p1;
        }
      }
    }
    signal_counter(&cR[t]);
    if (m == M && !(prm.seismic && op == prm.nops - 1)) {  // operator complete: hand over
#pragma unroll
      for (int j = 0; j < G::NBL; ++j) {
        const int bb = tid + j * NT, l = bb / G::TL, i = bb % G::TL;
        if (l < nrows) {
          double2* o = reinterpret_cast<double2*>(prm.out[op] + (size_t)(r0 + l) * J1);
#pragma unroll
          for (int r = 0; r < G::RL; ++r) {
            o[i + r * G::TL] = make_double2(acc[j][r][0], acc[j][r][1]);
            acc[j][r][0] = acc[j][r][1] = 0.0;
          }
        }
      }
    }
  };

  // pipeline: C(0..K-2) ; for t: R(t), C(t+K-1)
  for (int t = 0; t < KRING - 1 && t < ntot; ++t) column_term(t);
  for (int t = 0; t < ntot; ++t) {
    row_term(t);
    if (t + KRING - 1 < ntot) column_term(t + KRING - 1);
  }
  if (prm.residue && rmax > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(prm.residue), (unsigned long long)__double_as_longlong(rmax));

  // ------------------------------------------------ seismic update (seismic.cpp:116-129)
  if (prm.seismic) {
    bool bad = false;
    const double tau = prm.tau;
    const double t2 = tau * tau;
#pragma unroll
    for (int j = 0; j < G::NBL; ++j) {
      const int bb = tid + j * NT, l = bb / G::TL, i = bb % G::TL;
      if (l < nrows) {
        const size_t rowoff = (size_t)(r0 + l) * J1;
        const double2* cur = reinterpret_cast<const double2*>(prm.u + rowoff);
        const double2* prev = reinterpret_cast<const double2*>(prm.prev + rowoff);
        const double2* ap = reinterpret_cast<const double2*>(prm.ap + rowoff);
        const double2* l1 = reinterpret_cast<const double2*>(prm.out[0] + rowoff);
        const double2* c = reinterpret_cast<const double2*>(prm.c + rowoff);
        const double2* eta = reinterpret_cast<const double2*>(prm.eta + rowoff);
        const double2* tc = reinterpret_cast<const double2*>(prm.tc + rowoff);
        double2* nx = reinterpret_cast<double2*>(prm.next + rowoff);
        double2* l2o = reinterpret_cast<double2*>(prm.out[1] + rowoff);
#pragma unroll
        for (int r = 0; r < G::RL; ++r) {
          const int q = i + r * G::TL;
          const double2 vc = cur[q], vp = prev[q], va = ap[q], v1 = l1[q], cc = c[q], ve = eta[q], vt = tc[q];
          const double l2x = acc[j][r][0], l2y = acc[j][r][1];
          const double c2x = cc.x * cc.x, c2y = cc.y * cc.y;
          const double nx0 = 2.0 * vc.x - vp.x + t2 * c2x * (ve.x * v1.x + vt.x * (l2x - va.x) / tau);
          const double nx1 = 2.0 * vc.y - vp.y + t2 * c2y * (ve.y * v1.y + vt.y * (l2y - va.y) / tau);
          nx[q] = make_double2(nx0, nx1);
          l2o[q] = make_double2(l2x, l2y);
          bad |= (fabs(nx0) > prm.thr) || (fabs(nx1) > prm.thr);
        }
      }
    }
    if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicMin(prm.flag, prm.step);
  }
}

template <int J0, int J1, int CG, int RMAX>
cudaError_t launch_t(const Step2DParams& p, cudaStream_t st, int nblk) {
  using G = Geo<J0, J1, CG, RMAX>;
  if ((J0 + nblk - 1) / nblk > RMAX || G::NG > nblk) return cudaErrorInvalidConfiguration;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_step2d<J0, J1, CG, RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    attr = true;
  }
  void* args[] = {(void*)&p};
  return cudaLaunchCooperativeKernel((void*)k_step2d<J0, J1, CG, RMAX>, dim3(nblk), dim3(NT), args, G::SMEM, st);
}

}  // namespace s2d

bool step2d_supported(int J0, int J1, int nsm) {
  if (!((J0 == 1024 && J1 == 1024) || (J0 == 512 && J1 == 512) || (J0 == 256 && J1 == 256) ||
        (J0 == 512 && J1 == 1024) || (J0 == 1024 && J1 == 512)))
    return false;
  const int H = J1 / 2 + 1;
  const int ng = (H + kStep2dCG - 1) / kStep2dCG;
  return nsm >= 148 && ng <= nsm;
}

int step2d_col_groups(int J1) { return (J1 / 2 + 1 + kStep2dCG - 1) / kStep2dCG; }

cudaError_t launch_step2d(const Step2DParams& p, cudaStream_t st, int nsm) {
  const int J0 = p.J0, J1 = p.J1;
  if (J0 == 1024 && J1 == 1024) return s2d::launch_t<1024, 1024, 4, 7>(p, st, nsm);
  if (J0 == 512 && J1 == 512) return s2d::launch_t<512, 512, 4, 4>(p, st, nsm);
  if (J0 == 256 && J1 == 256) return s2d::launch_t<256, 256, 4, 2>(p, st, nsm);
  if (J0 == 512 && J1 == 1024) return s2d::launch_t<512, 1024, 4, 4>(p, st, nsm);
  if (J0 == 1024 && J1 == 512) return s2d::launch_t<1024, 512, 4, 7>(p, st, nsm);
  return cudaErrorInvalidValue;
}

}  // namespace fw

namespace fw {
namespace {
// w[m][k0][c] (c < H) -> w2d[m][g][k0][CG] (zero padded past H)
__global__ void k_w_to_2d(int J0, int H, int NG, int M, const double* __restrict__ w, double* __restrict__ w2d) {
  const long long total = (long long)(M + 1) * NG * J0 * kStep2dCG;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int cc = (int)(e % kStep2dCG);
    long long r = e / kStep2dCG;
    const int k0 = (int)(r % J0);
    r /= J0;
    const int g = (int)(r % NG);
    const int m = (int)(r / NG);
    const int c = g * kStep2dCG + cc;
    w2d[e] = c < H ? w[((long long)m * J0 + k0) * H + c] : 0.0;
  }
}
// dev[m-1][j] = (s - s0)^m by the reference recurrence dev_m = dev_{m-1} * dev_1 (flap.cpp:131)
__global__ void k_dev_tables(long long N, int M, const double* __restrict__ dev1, double* __restrict__ dev) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const double d1 = dev1[j];
    double d = d1;
    for (int m = 1; m <= M; ++m) {
      if (m > 1) d = d * d1;
      dev[(long long)(m - 1) * N + j] = d;
    }
  }
}
}  // namespace

void launch_w_to_2d(cudaStream_t st, int J0, int J1, int M, const double* w, double* w2d) {
  const int H = J1 / 2 + 1;
  const int NG = (H + kStep2dCG - 1) / kStep2dCG;
  k_w_to_2d<<<148 * 8, 256, 0, st>>>(J0, H, NG, M, w, w2d);
}

void launch_dev_tables(cudaStream_t st, size_t N, int M, const double* dev1, double* dev) {
  if (M < 1) return;
  k_dev_tables<<<148 * 8, 256, 0, st>>>((long long)N, M, dev1, dev);
}

}  // namespace fw
