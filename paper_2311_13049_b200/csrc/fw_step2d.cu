// fw_step2d.cu — persistent, warp-specialised single-launch 2D apply / seismic step (sm_100a).
//
// One cooperative launch of one CTA per SM does the whole seismic step (or one
// operator apply) on a J0 x J1 grid (half spectrum H = J1/2 + 1 columns).  CTA b
// owns 4 half-spectrum columns (group b) and RMAX rows.  Its warps are
// specialised and progress independently (no CTA-wide barrier after setup):
//
//   column warps (4, one column each)            row warps (RMAX, one row each)
//   F2: wait all rows -> C2C of its column of     F1: R2C of its row of u -> Y row
//       Y (x 1/N) -> uhat column (SHARED MEM,     R(t), t = (op, m) in order:
//       kept for the whole step)                     wait all columns of T[t%3];
//   C(t), t = (op, m) in order:                      C2R with the pre-processing
//       wait T slot free (rows of t-3 done);         fused into its loads; acc +=
//       IFFT(w_m .* uhat) ; the 4 warps                (s-s0)^m .* x in registers
//       transpose through smem and store           update (seismic.cpp:116-129)
//       64-byte row chunks of T[t%3]                  from the registers
//
// Producer/consumer ordering between warps of all CTAs uses monotone counters
// counted in rows / columns (red.release.gpu / ld.acquire.gpu), two counter sets
// alternating between launches.  Only the term intermediate T round-trips
// through global memory (a 2D FFT is an all-to-all across SMs).
// Arithmetic is the canonical FFT of fw_fft.cuh (radix plan, twiddle values,
// fma placement): results are bit-identical to the multi-pass path and to the
// CPU oracle.  Per-pass twiddle tables live in shared memory in a [k][r-1]
// layout (odd stride, conflict-free).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fw_fft.cuh"
#include "fw_internal.h"
#include "fw_step2d.h"

namespace fw {
namespace s2d {

constexpr int KRING = 3;
constexpr int NWC = 4;  // column warps per CTA (= columns per CTA)

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int npass(int n) { return (ilog2c(n) + 3) / 4; }
__host__ __device__ constexpr int radix(int n, int i) {
  return 1 << (ilog2c(n) / npass(n) + (i < ilog2c(n) % npass(n) ? 1 : 0));
}
__host__ __device__ constexpr int pprod(int n, int i) { return i == 0 ? 1 : pprod(n, i - 1) * radix(n, i - 1); }
__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
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
// whole warp waits until *cnt >= target
__device__ __forceinline__ void warp_wait(const unsigned long long* cnt, unsigned long long target) {
  if ((threadIdx.x & 31) == 0) {
    while (ld_acquire(cnt) < target) __nanosleep(20);
  }
  __syncwarp();
}
// the warp's global writes are done -> publish v
__device__ __forceinline__ void warp_signal(unsigned long long* cnt, unsigned long long v) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    red_release_add(cnt, v);
  }
}
// named barriers: 1..4 = the warp pair of column p, 5 = all 8 column warps
__device__ __forceinline__ void colbar() { asm volatile("bar.sync 5, 256;" ::: "memory"); }
__device__ __forceinline__ void pairbar(int p) { asm volatile("bar.sync %0, 64;" ::"r"(1 + p) : "memory"); }
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// optional instrumentation: trace[(sel*16 + warp)*136 + t][4] = globaltimer at phase marks
#define FW_TRACE(t, slot)                                                                              \
  do {                                                                                                 \
    if (prm.trace && (threadIdx.x & 31) == 0 && (blockIdx.x == 0 || blockIdx.x == 100))               \
      prm.trace[(((size_t)(blockIdx.x == 0 ? 0 : 1) * 16 + (threadIdx.x >> 5)) * 136 + (t)) * 4 + (slot)] = \
          gtimer();                                                                                    \
  } while (0)

template <int DIR>
__device__ __forceinline__ double2 dirw(double2 w) {
  return make_double2(w.x, DIR < 0 ? -w.y : w.y);
}

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

// Middle pass PASS of an N-point C2C held by ONE warp in buf (padded), in place.
template <int N, int PASS, int DIR, int PADSH>
__device__ __forceinline__ void warp_pass(double2* buf, const double2* tw) {
  constexpr int R = radix(N, PASS);
  constexpr int T = N / R;
  constexpr int NB = T / 32;
  static_assert(T % 32 == 0, "warp pass needs >= 32 butterflies");
  const int lane = threadIdx.x & 31;
  double2 a[NB][R];
#pragma unroll
  for (int j = 0; j < NB; ++j)
#pragma unroll
    for (int r = 0; r < R; ++r) a[j][r] = buf[padq<PADSH>(lane + 32 * j + r * T)];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int i = lane + 32 * j;
    butterfly<N, PASS, DIR>(a[j], i, tw);
#pragma unroll
    for (int r = 0; r < R; ++r) buf[padq<PADSH>(out_index<N, PASS>(i, r))] = a[j][r];
  }
  __syncwarp();
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

// joint column-transpose area: element (k0, cc) of the CTA's 4 columns, XOR swizzled
__device__ __forceinline__ int jidx(int k0, int cc) { return k0 * 4 + (cc ^ ((k0 >> 1) & 3)); }

// --------------------------------------------------------------------------
template <int J0, int J1, int RMAX>
struct Geo {
  static constexpr int H = J1 / 2 + 1;
  static constexpr int h = J1 / 2;
  static constexpr int NG = (H + NWC - 1) / NWC;
  static constexpr int NT = 512;  // 8 column warps (2 per column) + 8 row warps
  static constexpr int PADC = ilog2c(radix(J0, 0));
  static constexpr int PADR = 4;
  static constexpr int LCOL = J0 + (J0 >> PADC) + 2;  // per column-warp work buffer
  static constexpr int LROW = h + (h >> PADR) + 2;    // per row-warp work buffer
  static constexpr int PC = npass(J0);
  static constexpr int PR = npass(h);
  static constexpr int TWC = twtotal(J0);
  static constexpr int TWR = twtotal(h);
  static constexpr int TWP = h + 1;
  static constexpr size_t OFF_TWR = TWC;
  static constexpr size_t OFF_TWP = TWC + TWR;
  static constexpr size_t OFF_U = TWC + TWR + TWP;         // uhat [4][J0]
  static constexpr size_t OFF_CW = OFF_U + (size_t)NWC * J0;  // column work [4][LCOL]
  static constexpr size_t OFF_RW = OFF_CW + (size_t)NWC * LCOL;  // row work [RMAX][LROW]
  static constexpr size_t NELEM = OFF_RW + (size_t)RMAX * LROW;
  static constexpr size_t SMEM = NELEM * sizeof(double2);
  static_assert(PC >= 2 && PC <= 3 && PR >= 2 && PR <= 3, "2 or 3 passes per FFT");
  static_assert(NWC * LCOL >= 4 * J0 && NWC * J0 >= 4 * J0, "joint transpose area");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(RMAX <= 8, "at most 8 row warps");
};

// ---------------------------------------------------------------- column pair: J0-point C2C
// Two warps (64 threads, ct2 = 0..63, pair barrier `pbar`) transform one column.
// Pass 0 reads src(q) (q = i + r*T0); the last pass writes each butterfly's
// outputs back to the slots it read, so `work` ends holding the column in
// natural order (padded).  `sync0` separates pass 0 from the rest (the caller's
// barrier when the pass-0 source is shared with other warps).
template <int J0, int DIR, int PADSH, class Src, class Sync0, class PBar>
__device__ __forceinline__ void column_c2c(double2* work, const double2* tw, int ct2, Src src, Sync0 sync0,
                                           PBar pbar) {
  constexpr int P = npass(J0);
  {
    constexpr int R = radix(J0, 0);
    constexpr int T = J0 / R;
    static_assert(T == 64, "column pass 0: one butterfly per pair thread");
    const int i = ct2;
    double2 a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = src(i + r * T);
    Dft<R, DIR>::run(a);
#pragma unroll
    for (int r = 0; r < R; ++r) work[padq<PADSH>(i * R + r)] = a[r];
    sync0();
  }
  if constexpr (P == 3) {  // middle pass, in place across the pair
    constexpr int R = radix(J0, 1);
    constexpr int T = J0 / R;
    constexpr int NB = T / 64;
    static_assert(T % 64 == 0, "column middle pass");
    double2 a[NB][R];
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) a[j][r] = work[padq<PADSH>(ct2 + 64 * j + r * T)];
    pbar();
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int i = ct2 + 64 * j;
      butterfly<J0, 1, DIR>(a[j], i, tw);
#pragma unroll
      for (int r = 0; r < R; ++r) work[padq<PADSH>(out_index<J0, 1>(i, r))] = a[j][r];
    }
    pbar();
  }
  {
    constexpr int PL = P - 1;
    constexpr int R = radix(J0, PL);
    constexpr int T = J0 / R;
    static_assert(T % 64 == 0, "column last pass");
#pragma unroll
    for (int j = 0; j < T / 64; ++j) {
      const int i = ct2 + 64 * j;
      double2 a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = work[padq<PADSH>(i + r * T)];
      butterfly<J0, PL, DIR>(a, i, tw);
#pragma unroll
      for (int r = 0; r < R; ++r) work[padq<PADSH>(i + r * T)] = a[r];
    }
  }
}

// --------------------------------------------------------------------------
template <int J0, int J1, int RMAX>
__global__ void __launch_bounds__(Geo<J0, J1, RMAX>::NT, 1) k_step2d(const Step2DParams prm) {
  using G = Geo<J0, J1, RMAX>;
  constexpr int H = G::H, h = G::h, NT = G::NT;
  extern __shared__ __align__(16) double2 sm[];
  double2* twc = sm;
  double2* twr = sm + G::OFF_TWR;
  double2* twp = sm + G::OFF_TWP;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.x;
  const int nblk = gridDim.x;

  unsigned long long* cnt = prm.counters + (size_t)prm.cset * prm.cstride;
  if (b == 0) {
    unsigned long long* other = prm.counters + (size_t)(prm.cset ^ 1) * prm.cstride;
    for (int e = tid; e < prm.cstride; e += NT) other[e] = 0ull;
  }
  if (prm.flag && *prm.flag != kNoBlowup) return;  // uniform across CTAs
  unsigned long long* cY = cnt;                          // rows forward-transformed
  unsigned long long* cC = cnt + 1;                      // columns of T[t] stored
  unsigned long long* cR = cnt + 1 + prm.nterms_total;  // rows of T[t] consumed

  {  // twiddle tables (values = master entries, identical to fw_fft.cuh's twiddle())
    auto fill = [&](double2* dst, int off, int p, int R) {
      const int n = p * (R - 1);
      for (int e = tid; e < n; e += NT) {
        const int k = e / (R - 1), r = e % (R - 1) + 1;
        dst[off + e] = prm.master[(r * k) * (kTwMaster / (p * R))];
      }
    };
    fill(twc, twoff(J0, 1), pprod(J0, 1), radix(J0, 1));
    if constexpr (G::PC >= 3) fill(twc, twoff(J0, 2), pprod(J0, 2), radix(J0, 2));
    fill(twr, twoff(h, 1), pprod(h, 1), radix(h, 1));
    if constexpr (G::PR >= 3) fill(twr, twoff(h, 2), pprod(h, 2), radix(h, 2));
    for (int e = tid; e <= h; e += NT) twp[e] = prm.master[e * (kTwMaster / J1)];
  }
  __syncthreads();

  const int M = prm.M;
  const int nterms = M + 1 - prm.m_first;
  const int ntot = prm.nops * nterms;

  if (warp < 2 * NWC) {
    // ============================================ column warps (pairs)
    setmaxnreg_dec<96>();
    if (b >= G::NG) return;
    const int cw = warp >> 1;              // column of the pair
    const int ct2 = ((warp & 1) << 5) | lane;  // 0..63 within the pair
    const int c0 = b * NWC;
    const int c = c0 + cw;
    const int ncols = min(NWC, H - c0);
    const bool valid = c < H;
    double2* uhat = sm + G::OFF_U + (size_t)cw * J0;
    double2* work = sm + G::OFF_CW + (size_t)cw * G::LCOL;
    double2* works = sm + G::OFF_CW;   // the 4 column work buffers (line stride LCOL)
    double2* joint_u = sm + G::OFF_U;  // F2 staging (uhat not yet valid)
    const int ct = tid;                // 0..255 within the column warps
    auto pb = [cw] { pairbar(cw); };

    // ---- F2: forward columns -> uhat
    warp_wait(cY, (unsigned long long)J0);
    colbar();  // all column warps have seen every row
    for (int e = ct; e < J0 * 4; e += 2 * NWC * 32) {
      const int k0 = e >> 2, cc = e & 3;
      joint_u[jidx(k0, cc)] = (c0 + cc < H) ? __ldcg(&prm.Y[(size_t)k0 * H + c0 + cc]) : make_double2(0.0, 0.0);
    }
    colbar();
    // pass 0 reads joint_u (shared by all column warps): barrier before uhat is overwritten
    column_c2c<J0, -1, G::PADC>(work, twc, ct2, [&](int q) { return joint_u[jidx(q, cw)]; }, [] { colbar(); }, pb);
    pb();
    {
      const double inv = 1.0 / ((double)J0 * (double)J1);
      for (int q = ct2; q < J0; q += 64) {
        const double2 v = work[padq<G::PADC>(q)];
        uhat[q] = make_double2(v.x * inv, v.y * inv);
      }
      pb();
    }

    // ---- C(t): inverse columns -> T[t % KRING]
    for (int t = 0; t < ntot; ++t) {
      const int op = t / nterms;
      const int m = prm.m_first + t % nterms;
      FW_TRACE(t, 0);
      if (t >= KRING) warp_wait(&cR[t - KRING], (unsigned long long)J0);
      FW_TRACE(t, 1);
      const double* w = prm.w[op] + ((size_t)m * (G::NG * NWC) + c) * J0;  // [m][c][k0]
      column_c2c<J0, +1, G::PADC>(
          work, twc, ct2,
          [&](int q) {
            const double2 v = uhat[q];
            const double wk = valid ? __ldg(&w[q]) : 0.0;
            return make_double2(wk * v.x, wk * v.y);
          },
          pb, pb);
      colbar();  // the 4 columns are complete in the 4 work buffers
      FW_TRACE(t, 2);
      double2* T = prm.T + (size_t)(t % KRING) * J0 * H;
      for (int e = ct; e < J0 * 4; e += 2 * NWC * 32) {  // 64-byte row chunks of the 4 columns
        const int k0 = e >> 2, cc = e & 3;
        if (cc < ncols) __stcg(&T[(size_t)k0 * H + c0 + cc], works[cc * G::LCOL + padq<G::PADC>(k0)]);
      }
      colbar();  // stores issued by all column threads; work buffers free again
      if (ct == 0) {
        __threadfence();
        red_release_add(&cC[t], (unsigned long long)ncols);
      }
      FW_TRACE(t, 3);
    }
    return;
  }

  // ============================================ row warps
  setmaxnreg_inc<160>();
  const int rw = warp - 2 * NWC;
  const int r0 = (int)(((long long)b * J0) / nblk);
  const int r1 = (int)(((long long)(b + 1) * J0) / nblk);
  if (rw >= r1 - r0) return;
  const int row = r0 + rw;
  double2* work = sm + G::OFF_RW + (size_t)rw * G::LROW;
  constexpr int R0 = radix(h, 0);
  constexpr int T0 = h / R0;
  constexpr int RL = radix(h, G::PR - 1);
  constexpr int TL = h / RL;
  constexpr int NBL = TL / 32;
  static_assert(TL % 32 == 0, "row last pass");

  // ---- F1: R2C of the row -> Y
  {
    const double2* u2 = reinterpret_cast<const double2*>(prm.u) + (size_t)row * h;
#pragma unroll
    for (int j = 0; j < T0 / 32; ++j) {
      const int i = lane + 32 * j;
      double2 a[R0];
#pragma unroll
      for (int r = 0; r < R0; ++r) a[r] = u2[i + r * T0];
      Dft<R0, -1>::run(a);
#pragma unroll
      for (int r = 0; r < R0; ++r) work[padq<G::PADR>(i * R0 + r)] = a[r];
    }
    __syncwarp();
    if constexpr (G::PR == 3) warp_pass<h, 1, -1, G::PADR>(work, twr);
#pragma unroll
    for (int j = 0; j < NBL; ++j) {
      const int i = lane + 32 * j;
      double2 a[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) a[r] = work[padq<G::PADR>(i + r * TL)];
      butterfly<h, G::PR - 1, -1>(a, i, twr);
#pragma unroll
      for (int r = 0; r < RL; ++r) work[padq<G::PADR>(i + r * TL)] = a[r];
    }
    __syncwarp();
    double2* Yr = prm.Y + (size_t)row * H;
    for (int jj = lane; jj <= h / 2; jj += 32) {
      if (jj == 0) {
        const double2 z0 = work[0];
        __stcg(&Yr[0], make_double2(z0.x + z0.y, 0.0));
        __stcg(&Yr[h], make_double2(z0.x - z0.y, 0.0));
      } else {
        const double2 A = work[padq<G::PADR>(jj)];
        const double2 B = work[padq<G::PADR>(h - jj)];
        __stcg(&Yr[jj], post_r2c(A, B, twp[jj]));
        if (jj != h - jj) __stcg(&Yr[h - jj], post_r2c(B, A, twp[h - jj]));
      }
    }
    warp_signal(cY, 1ull);
  }

  // ---- R(t): C2R + recombination
  double acc[NBL][RL][2];
#pragma unroll
  for (int j = 0; j < NBL; ++j)
#pragma unroll
    for (int r = 0; r < RL; ++r) acc[j][r][0] = acc[j][r][1] = 0.0;
  double rmax = 0.0;

  for (int t = 0; t < ntot; ++t) {
    const int op = t / nterms;
    const int m = prm.m_first + t % nterms;
    FW_TRACE(t, 0);
    warp_wait(&cC[t], (unsigned long long)H);
    FW_TRACE(t, 1);
    const double2* X = prm.T + (size_t)(t % KRING) * J0 * H + (size_t)row * H;
    // pass 0 with the pre-processing fused.  Butterfly i needs X[i + r T0] and
    // X[h - i - r T0] = X[(T0 - i) + (R0-1-r) T0]: lane L takes butterflies L and
    // T0-L (lane 0: butterflies 0 and T0/2, both self-contained) -- every X once.
    static_assert(T0 == 64, "pass-0 pairing assumes 64 butterflies");
    {
      const int i1 = lane;                        // 0..31
      const int i2 = (lane == 0) ? T0 / 2 : T0 - lane;
      double2 XA[R0], XB[R0];
#pragma unroll
      for (int r = 0; r < R0; ++r) XA[r] = __ldcg(&X[i1 + r * T0]);
#pragma unroll
      for (int r = 0; r < R0; ++r) XB[r] = __ldcg(&X[i2 + r * T0]);
      double2 xh = make_double2(0.0, 0.0);
      if (lane == 0) xh = __ldcg(&X[h]);
      double2 a[R0];
      if (lane == 0) {
        if (prm.residue) rmax = fmax(rmax, fabs(XA[0].y) + fabs(xh.y));
        // butterfly 0: k = r T0, h-k = (R0-r) T0 -> XA[R0-r] (r >= 1), X[h] (r = 0)
#pragma unroll
        for (int r = 0; r < R0; ++r) a[r] = pre_c2r(XA[r], r == 0 ? xh : XA[R0 - r], r == 0, twp[r * T0]);
        Dft<R0, +1>::run(a);
#pragma unroll
        for (int r = 0; r < R0; ++r) work[padq<G::PADR>(r)] = a[r];
        // butterfly T0/2 (self-mirror): h-k = T0/2 + (R0-1-r) T0 -> XB[R0-1-r]
#pragma unroll
        for (int r = 0; r < R0; ++r) a[r] = pre_c2r(XB[r], XB[R0 - 1 - r], false, twp[T0 / 2 + r * T0]);
        Dft<R0, +1>::run(a);
#pragma unroll
        for (int r = 0; r < R0; ++r) work[padq<G::PADR>((T0 / 2) * R0 + r)] = a[r];
      } else {
#pragma unroll
        for (int r = 0; r < R0; ++r) a[r] = pre_c2r(XA[r], XB[R0 - 1 - r], false, twp[i1 + r * T0]);
        Dft<R0, +1>::run(a);
#pragma unroll
        for (int r = 0; r < R0; ++r) work[padq<G::PADR>(i1 * R0 + r)] = a[r];
#pragma unroll
        for (int r = 0; r < R0; ++r) a[r] = pre_c2r(XB[r], XA[R0 - 1 - r], false, twp[i2 + r * T0]);
        Dft<R0, +1>::run(a);
#pragma unroll
        for (int r = 0; r < R0; ++r) work[padq<G::PADR>(i2 * R0 + r)] = a[r];
      }
      warp_signal(&cR[t], 1ull);  // this row of T[t] has been consumed: the slot may be reused
      FW_TRACE(t, 2);
    }
    if constexpr (G::PR == 3) warp_pass<h, 1, +1, G::PADR>(work, twr);
    const double* dv = (m >= 1) ? prm.dev[op] + (size_t)(m - 1) * J0 * J1 + (size_t)row * J1 : nullptr;
#pragma unroll
    for (int j = 0; j < NBL; ++j) {
      const int i = lane + 32 * j;
      double2 a[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) a[r] = work[padq<G::PADR>(i + r * TL)];
      double2 d[RL];
      if (dv) {
#pragma unroll
        for (int r = 0; r < RL; ++r) d[r] = __ldg(reinterpret_cast<const double2*>(dv) + i + r * TL);
      }
      butterfly<h, G::PR - 1, +1>(a, i, twr);
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        double v0 = a[r].x, v1 = a[r].y;
        if (dv) {
          v0 = d[r].x * v0;
          v1 = d[r].y * v1;
        }
        double p0 = 0.0, p1 = 0.0;
        p0 += v0;
        p1 += v1;
        acc[j][r][0] += p0;
        acc[j][r][1] += p1;
      }
    }
    __syncwarp();  // work buffer reads done before the next term's pass 0 writes
    FW_TRACE(t, 3);
    if (m == M && !(prm.seismic && op == prm.nops - 1)) {  // operator complete: hand over
      double2* o = reinterpret_cast<double2*>(prm.out[op] + (size_t)row * J1);
#pragma unroll
      for (int j = 0; j < NBL; ++j)
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          o[lane + 32 * j + r * TL] = make_double2(acc[j][r][0], acc[j][r][1]);
          acc[j][r][0] = acc[j][r][1] = 0.0;
        }
    }
  }
  if (prm.residue && rmax > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(prm.residue), (unsigned long long)__double_as_longlong(rmax));

  // ---- seismic update (seismic.cpp:116-129)
  if (prm.seismic) {
    bool bad = false;
    const double tau = prm.tau;
    const double t2 = tau * tau;
    const size_t rowoff = (size_t)row * J1;
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
    for (int j = 0; j < NBL; ++j)
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int q = lane + 32 * j + r * TL;
        const double2 vc = cur[q], vp = prev[q], va = ap[q], v1 = l1[q], cc = c[q], ve = eta[q], vt = tc[q];
        const double l2x = acc[j][r][0], l2y = acc[j][r][1];
        const double c2x = cc.x * cc.x, c2y = cc.y * cc.y;
        const double nx0 = 2.0 * vc.x - vp.x + t2 * c2x * (ve.x * v1.x + vt.x * (l2x - va.x) / tau);
        const double nx1 = 2.0 * vc.y - vp.y + t2 * c2y * (ve.y * v1.y + vt.y * (l2y - va.y) / tau);
        nx[q] = make_double2(nx0, nx1);
        l2o[q] = make_double2(l2x, l2y);
        bad |= (fabs(nx0) > prm.thr) || (fabs(nx1) > prm.thr);
      }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(prm.flag, prm.step);
  }
}

template <int J0, int J1, int RMAX>
cudaError_t launch_t(const Step2DParams& p, cudaStream_t st, int nblk) {
  using G = Geo<J0, J1, RMAX>;
  if ((J0 + nblk - 1) / nblk > RMAX || G::NG > nblk) return cudaErrorInvalidConfiguration;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_step2d<J0, J1, RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    attr = true;
  }
  void* args[] = {(void*)&p};
  return cudaLaunchCooperativeKernel((void*)k_step2d<J0, J1, RMAX>, dim3(nblk), dim3(G::NT), args, G::SMEM, st);
}

}  // namespace s2d

bool step2d_supported(int J0, int J1, int nsm) {
  if (!((J0 == 1024 && J1 == 1024) || (J0 == 512 && J1 == 1024)))
    return false;
  const int H = J1 / 2 + 1;
  const int ng = (H + kStep2dCG - 1) / kStep2dCG;
  return nsm >= 148 && ng <= nsm;
}

int step2d_col_groups(int J1) { return (J1 / 2 + 1 + kStep2dCG - 1) / kStep2dCG; }

cudaError_t launch_step2d(const Step2DParams& p, cudaStream_t st, int nsm) {
  const int J0 = p.J0, J1 = p.J1;
  if (J0 == 1024 && J1 == 1024) return s2d::launch_t<1024, 1024, 7>(p, st, nsm);
  if (J0 == 512 && J1 == 1024) return s2d::launch_t<512, 1024, 4>(p, st, nsm);
  return cudaErrorInvalidValue;
}

}  // namespace fw

namespace fw {
namespace {
// w[m][k0][c] (c < H) -> w2d[m][c][k0] (column-major per term; columns past H zero)
__global__ void k_w_to_2d(int J0, int H, int NC, int M, const double* __restrict__ w, double* __restrict__ w2d) {
  const long long total = (long long)(M + 1) * NC * J0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int k0 = (int)(e % J0);
    const long long r = e / J0;
    const int c = (int)(r % NC);
    const int m = (int)(r / NC);
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
  const int NC = ((H + kStep2dCG - 1) / kStep2dCG) * kStep2dCG;
  k_w_to_2d<<<148 * 8, 256, 0, st>>>(J0, H, NC, M, w, w2d);
}

void launch_dev_tables(cudaStream_t st, size_t N, int M, const double* dev1, double* dev) {
  if (M < 1) return;
  k_dev_tables<<<148 * 8, 256, 0, st>>>((long long)N, M, dev1, dev);
}

}  // namespace fw
