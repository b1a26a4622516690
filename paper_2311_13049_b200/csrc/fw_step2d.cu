// fw_step2d.cu — persistent, warp-specialised single-launch 2D apply / seismic step (sm_100a).
//
// One cooperative launch of one CTA per SM does the whole seismic step (or one
// operator apply) on a J0 x J1 grid (half spectrum H = J1/2 + 1 columns,
// h = J1/2).  CTA b owns two mirror column pairs {k, h-k} of the half spectrum
// (4 columns) and up to RMAX rows.  Its 16 warps are specialised and progress
// independently (no CTA-wide barrier after setup):
//
//   column warps (8: a warp pair per column)       row warps (up to 8: one per row)
//   F2: wait all rows -> C2C of its column of      F1: R2C of its row of u -> Y row
//       Y, x 1/N -> uhat column (SHARED MEMORY,     R(t), t = (op, m) in order:
//       kept for the whole step)                      wait all of Z[t%3]; h-point
//   C(t), t = (op, m) in order:                       C2C of its row of Z; acc +=
//       wait slot free (rows of t-3 done);            (s-s0)^m .* x in registers
//       IFFT(w_m .* uhat) of the 4 columns; the    update (seismic.cpp:116-129) from
//       C2R pre-processing of each mirror pair        the registers
//       (k, h-k) -> Z[t%3] (global)
//
// Because a CTA owns both columns k and h-k, the C2R pre-processing
// Z_k = f(X_k, X_{h-k}) happens in the column phase, so rows only run a plain
// h-point C2C.  Producer/consumer ordering between warps of all CTAs uses
// monotone counters counted in rows / Z columns (red.release.gpu /
// ld.acquire.gpu), two counter sets alternating between launches.  Only the
// term intermediate Z round-trips through global memory (a 2D FFT is an
// all-to-all across SMs).  Registers are split with setmaxnreg (column warps
// 96, row warps 160).  Arithmetic is the canonical FFT of fw_fft.cuh (radix
// plan, twiddle values, fma placement, pre-processing formula): results are
// bit-identical to the multi-pass path and to the CPU oracle.  Per-pass twiddle
// tables live in shared memory in a [k][r-1] layout (odd stride, conflict-free).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fw_fft.cuh"
#include "fw_internal.h"
#include "fw_step2d.h"

namespace fw {
namespace s2d {

constexpr int KRING = kStep2dRing;
constexpr int NWC = 4;  // columns per CTA (two mirror pairs)

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int npass(int n) { return (ilog2c(n) + 3) / 4; }
__host__ __device__ constexpr int radix(int n, int i) {
  return 1 << (ilog2c(n) / npass(n) + (i < ilog2c(n) % npass(n) ? 1 : 0));
}
__host__ __device__ constexpr int pprod(int n, int i) { return i == 0 ? 1 : pprod(n, i - 1) * radix(n, i - 1); }
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
    while (ld_acquire(cnt) < target) {
    }
  }
  __syncwarp();
}
// the warp's prior memory accesses are done -> publish v (release is cumulative
// over the lanes ordered before it by __syncwarp)
__device__ __forceinline__ void warp_signal(unsigned long long* cnt, unsigned long long v) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) red_release_add(cnt, v);
}
// named barriers: 1, 2 = column group g (4 warps), 5 = all 8 column warps
__device__ __forceinline__ void colbar() { asm volatile("bar.sync 5, 256;" ::: "memory"); }
__device__ __forceinline__ void groupbar(int g) { asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory"); }
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
// bulk prefetch of [p, p + bytes) into L2 (bytes multiple of 16)
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
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

// ---------------------------------------------------------------- TMEM as accumulator storage
// Row accumulators live in tensor memory (tcgen05.ld/st, 32 lanes x 32 columns of 32 bit
// per call): they would otherwise pin 64 registers per row thread across the whole step.
__device__ __forceinline__ void tmem_ld32(unsigned taddr, unsigned (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st32(unsigned taddr, const unsigned (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
               :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
               : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

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

// F2 staging: element (k0, cc) of the CTA's 4 columns, XOR swizzled
__device__ __forceinline__ int jidx(int k0, int cc) { return k0 * 4 + (cc ^ ((k0 >> 1) & 3)); }

// --------------------------------------------------------------------------
// Column slots: slot 0 = {0, h}, slot s in [1, h/2) = {s, h-s}, slot h/2 = {h/2}.
// CTA b owns slots 2b and 2b+1; column warp pair cw: slot 2b + (cw >> 1), member cw & 1.
template <int J0, int J1, int RMAX>
struct Geo {
  static constexpr int H = J1 / 2 + 1;
  static constexpr int h = J1 / 2;
  static constexpr int NSLOT = h / 2 + 1;
  static constexpr int NG = (NSLOT + 1) / 2;  // CTAs with columns
  static constexpr int NT = 512;               // 8 column warps (2 groups of 4) + 8 row warps
  static constexpr int PADC = ilog2c(radix(J0, 0));
  static constexpr int PADR = 4;
  static constexpr int LCOL = J0 + (J0 >> PADC) + 2;  // per column work buffer
  static constexpr int LROW = h + (h >> PADR) + 2;    // per row-warp work buffer
  static constexpr int PC = npass(J0);
  static constexpr int PR = npass(h);
  static constexpr int TWC = twtotal(J0);
  static constexpr int TWR = twtotal(h);
  static constexpr int TWP = h + 1;
  static constexpr size_t OFF_TWR = TWC;
  static constexpr size_t OFF_TWP = TWC + TWR;
  static constexpr size_t OFF_U = TWC + TWR + TWP;              // uhat [4][J0]
  static constexpr size_t OFF_CW = OFF_U + (size_t)NWC * J0;      // column work [2][LCOL] (one per group)
  static constexpr size_t OFF_RW = OFF_CW + (size_t)2 * LCOL;    // row work [RMAX][LROW]
  static constexpr size_t NELEM = OFF_RW + (size_t)RMAX * LROW;
  static constexpr size_t SMEM = NELEM * sizeof(double2);
  static_assert(PC >= 2 && PC <= 3 && PR >= 2 && PR <= 3, "2 or 3 passes per FFT");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(RMAX <= 8, "at most 8 row warps");
  static_assert(h / radix(h, 0) % 32 == 0, "row pass 0 lane mapping");
};

// ---------------------------------------------------------------- column group: J0-point C2C
// Four warps (128 threads, cg = 0..127, group barrier `gbar`) transform one column.
// Pass 0 reads src(q) (q = i + r*T0); the last pass writes each butterfly's
// outputs back to the slots it read, so `work` ends holding the column in
// natural order (padded).
template <int J0, int DIR, int PADSH, class Src, class GBar>
__device__ __forceinline__ void column_c2c(double2* work, const double2* tw, int cg, Src src, GBar gbar) {
  constexpr int P = npass(J0);
  {
    constexpr int R = radix(J0, 0);
    constexpr int T = J0 / R;
    static_assert(T <= 128, "column pass 0");
    if (cg < T) {
      const int i = cg;
      double2 a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = src(i + r * T);
      Dft<R, DIR>::run(a);
#pragma unroll
      for (int r = 0; r < R; ++r) work[padq<PADSH>(i * R + r)] = a[r];
    }
    gbar();
  }
  if constexpr (P == 3) {  // middle pass, in place across the group
    constexpr int R = radix(J0, 1);
    constexpr int T = J0 / R;
    static_assert(T <= 128, "column middle pass: at most one butterfly per thread");
    double2 a[R];
    if (cg < T) {
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = work[padq<PADSH>(cg + r * T)];
    }
    gbar();
    if (cg < T) {
      butterfly<J0, 1, DIR>(a, cg, tw);
#pragma unroll
      for (int r = 0; r < R; ++r) work[padq<PADSH>(out_index<J0, 1>(cg, r))] = a[r];
    }
    gbar();
  }
  {
    constexpr int PL = P - 1;
    constexpr int R = radix(J0, PL);
    constexpr int T = J0 / R;
#pragma unroll 1
    for (int i = cg; i < T; i += 128) {
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
  unsigned long long* cC = cnt + 1;                      // Z columns of term t stored
  unsigned long long* cR = cnt + 1 + prm.nterms_total;  // rows of Z[t] consumed

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
  __shared__ unsigned tmem_base_sh;
  if (warp == 0) {  // 128 TMEM columns: row accumulators (2 row warps per lane quadrant x 64 columns)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem_base = tmem_base_sh;

  const int M = prm.M;
  const int nterms = M + 1 - prm.m_first;
  const int ntot = prm.nops * nterms;

  if (warp < 2 * NWC) {
    // ============================================ column warps (2 groups of 4)
    if (b >= G::NG) return;
    const int g = warp >> 2;       // group: member g of each mirror slot (0: k = s, 1: k = h - s)
    const int cg = tid & 127;      // thread within the group
    const int ct = tid;            // 0..255 within the column warps
    // column q = 2*sl + member of this CTA: slot s -> {s, h-s}; slot 0 -> {0, h}; slot h/2 -> {h/2, -}
    auto colno = [&](int q) {
      const int s = 2 * b + (q >> 1);
      if (s >= G::NSLOT) return -1;
      if (s == 0) return (q & 1) ? h : 0;
      if (s == h / 2) return (q & 1) ? -1 : h / 2;
      return (q & 1) ? h - s : s;
    };
    double2* works = sm + G::OFF_CW;  // the 2 group work buffers (line stride LCOL)
    double2* work = works + (size_t)g * G::LCOL;
    auto gb = [g] { groupbar(g); };
    int nz = 0;
    for (int q = 0; q < 4; ++q) {
      const int col = colno(q);
      if (col >= 0 && col < h) ++nz;  // column h feeds Z_0 and produces no Z of its own
    }

    // ---- F2: forward columns -> uhat (pass 0 straight from Y)
    warp_wait(cY, (unsigned long long)J0);
    colbar();  // every column thread has seen all rows
    const double inv = 1.0 / ((double)J0 * (double)J1);
    for (int sl = 0; sl < 2; ++sl) {
      const int q = 2 * sl + g;
      const int col = colno(q);
      double2* uh = sm + G::OFF_U + (size_t)q * J0;
      column_c2c<J0, -1, G::PADC>(
          work, twc, cg,
          [&](int k0) { return col >= 0 ? __ldcg(&prm.Y[(size_t)k0 * H + col]) : make_double2(0.0, 0.0); }, gb);
      gb();
      for (int k0 = cg; k0 < J0; k0 += 128) {
        const double2 v = work[padq<G::PADC>(k0)];
        uh[k0] = make_double2(v.x * inv, v.y * inv);
      }
      gb();
    }

    double rmax = 0.0;
    // ---- C(t): inverse columns -> pre-processed Z[t % KRING]
    for (int t = 0; t < ntot; ++t) {
      const int op = t / nterms;
      const int m = prm.m_first + t % nterms;
      FW_TRACE(t, 0);
      if (t >= KRING) warp_wait(&cR[t - KRING], (unsigned long long)J0);
      FW_TRACE(t, 1);
      double2* Z = prm.T + (size_t)(t % KRING) * J0 * h;
      for (int sl = 0; sl < 2; ++sl) {
        const int q = 2 * sl + g;
        const int col = colno(q);
        const bool valid = col >= 0;
        const double2* uh = sm + G::OFF_U + (size_t)q * J0;
        const double* w = prm.w[op] + ((size_t)m * prm.wcols + (valid ? col : 0)) * J0;  // [m][c][k0]
        if (cg == 0 && valid) {  // the next use of this column's weights -> L2
          const int t1 = sl == 0 ? t : t + 1;
          if (t1 < ntot) {
            const int op1 = t1 / nterms, m1 = prm.m_first + t1 % nterms;
            const int q1 = sl == 0 ? q + 2 : q - 2;
            const int col1 = colno(q1);
            if (col1 >= 0) prefetch_l2(prm.w[op1] + ((size_t)m1 * prm.wcols + col1) * J0, J0 * sizeof(double));
          }
        }
        column_c2c<J0, +1, G::PADC>(
            work, twc, cg,
            [&](int k0) {
              const double2 v = uh[k0];
              const double wk = valid ? __ldg(&w[k0]) : 0.0;
              return make_double2(wk * v.x, wk * v.y);
            },
            gb);
        colbar();  // both members of slot 2b + sl are complete in the 2 work buffers
        FW_TRACE(t, 2);
        // C2R pre-processing of the mirror pair -> Z rows (k = s and k = h - s)
        const int kA = colno(2 * sl), kB = colno(2 * sl + 1);
        for (int e = ct; e < J0 * 2; e += 256) {
          const int k0 = e >> 1, mbr = e & 1;
          const int k = mbr ? kB : kA;
          if (k < 0 || k == h) continue;
          const double2 X = works[mbr * G::LCOL + padq<G::PADC>(k0)];
          double2 z;
          if (k == 0) {  // Z_0 from X_0 and X_h
            const double2 B = works[G::LCOL + padq<G::PADC>(k0)];
            if (prm.residue) rmax = fmax(rmax, fabs(X.y) + fabs(B.y));
            z = pre_c2r(X, B, true, twp[0]);
          } else if (k == h / 2) {
            z = pre_c2r(X, X, false, twp[k]);
          } else {
            z = pre_c2r(X, works[(mbr ^ 1) * G::LCOL + padq<G::PADC>(k0)], false, twp[k]);
          }
          __stcg(&Z[(size_t)k0 * h + k], z);
        }
        colbar();  // work buffers free again
      }
      if (ct == 0) red_release_add(&cC[t], (unsigned long long)nz);
      FW_TRACE(t, 3);
    }
    if (prm.residue && rmax > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(prm.residue), (unsigned long long)__double_as_longlong(rmax));
    return;
  }

  // ============================================ row warps
  const int rw = warp - 2 * NWC;
  const int r0 = (int)(((long long)b * J0) / nblk);
  const int r1 = (int)(((long long)(b + 1) * J0) / nblk);
  if (rw < r1 - r0) {
  const int row = r0 + rw;
  // this warp's 64 TMEM columns in its lane quadrant: butterfly j uses columns [32 j, 32 j + 32)
  const unsigned tacc = tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + 64u * (unsigned)((warp - 2 * NWC) >> 2);
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

  // ---- R(t): h-point C2C of the pre-processed row + recombination
  static_assert(NBL * RL * 2 * 2 == 64, "row accumulator = 64 TMEM columns per lane");
  {
    unsigned z[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) z[e] = 0u;
#pragma unroll
    for (int j = 0; j < NBL; ++j) tmem_st32(tacc + 32u * j, z);
  }

  for (int t = 0; t < ntot; ++t) {
    const int op = t / nterms;
    const int m = prm.m_first + t % nterms;
    if (lane == 0 && t + 1 < ntot) {  // next term's (s-s0)^m row -> L2
      const int op1 = (t + 1) / nterms, m1 = prm.m_first + (t + 1) % nterms;
      if (m1 >= 1) prefetch_l2(prm.dev[op1] + (size_t)(m1 - 1) * J0 * J1 + (size_t)row * J1, J1 * sizeof(double));
    }
    FW_TRACE(t, 0);
    warp_wait(&cC[t], (unsigned long long)h);
    FW_TRACE(t, 1);
    const double2* Zr = prm.T + (size_t)(t % KRING) * J0 * h + (size_t)row * h;
#pragma unroll
    for (int j = 0; j < T0 / 32; ++j) {  // pass 0 (p = 1) straight from global
      const int i = lane + 32 * j;
      double2 a[R0];
#pragma unroll
      for (int r = 0; r < R0; ++r) a[r] = __ldcg(&Zr[i + r * T0]);
      Dft<R0, +1>::run(a);
#pragma unroll
      for (int r = 0; r < R0; ++r) work[padq<G::PADR>(i * R0 + r)] = a[r];
    }
    warp_signal(&cR[t], 1ull);  // this row of Z[t] has been consumed: the slot may be reused
    FW_TRACE(t, 2);
    if constexpr (G::PR == 3) warp_pass<h, 1, +1, G::PADR>(work, twr);
    const double* dv = (m >= 1) ? prm.dev[op] + (size_t)(m - 1) * J0 * J1 + (size_t)row * J1 : nullptr;
#pragma unroll
    for (int j = 0; j < NBL; ++j) {
      const int i = lane + 32 * j;
      asm volatile("" ::: "memory");  // keep the butterflies sequential (register pressure)
      double2 a[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) a[r] = work[padq<G::PADR>(i + r * TL)];
      double2 d[RL];
      if (dv) {
#pragma unroll
        for (int r = 0; r < RL; ++r) d[r] = __ldg(reinterpret_cast<const double2*>(dv) + i + r * TL);
      }
      butterfly<h, G::PR - 1, +1>(a, i, twr);
      unsigned v[32];
      tmem_ld32(tacc + 32u * j, v);
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
        double a0 = __hiloint2double((int)v[4 * r + 1], (int)v[4 * r]);
        double a1 = __hiloint2double((int)v[4 * r + 3], (int)v[4 * r + 2]);
        a0 += p0;
        a1 += p1;
        v[4 * r] = (unsigned)__double2loint(a0);
        v[4 * r + 1] = (unsigned)__double2hiint(a0);
        v[4 * r + 2] = (unsigned)__double2loint(a1);
        v[4 * r + 3] = (unsigned)__double2hiint(a1);
      }
      tmem_st32(tacc + 32u * j, v);
    }
    __syncwarp();  // work buffer reads done before the next term's pass 0 writes
    FW_TRACE(t, 3);
    if (m == M && !(prm.seismic && op == prm.nops - 1)) {  // operator complete: hand over
      double2* o = reinterpret_cast<double2*>(prm.out[op] + (size_t)row * J1);
#pragma unroll
      for (int j = 0; j < NBL; ++j) {
        unsigned v[32];
        tmem_ld32(tacc + 32u * j, v);
#pragma unroll
        for (int r = 0; r < RL; ++r)
          o[lane + 32 * j + r * TL] = make_double2(__hiloint2double((int)v[4 * r + 1], (int)v[4 * r]),
                                                   __hiloint2double((int)v[4 * r + 3], (int)v[4 * r + 2]));
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0u;
        tmem_st32(tacc + 32u * j, v);
      }
    }
  }

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
    for (int j = 0; j < NBL; ++j) {
      unsigned v[32];
      tmem_ld32(tacc + 32u * j, v);
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int q = lane + 32 * j + r * TL;
        const double2 vc = cur[q], vp = prev[q], va = ap[q], v1 = l1[q], cc = c[q], ve = eta[q], vt = tc[q];
        const double l2x = __hiloint2double((int)v[4 * r + 1], (int)v[4 * r]);
        const double l2y = __hiloint2double((int)v[4 * r + 3], (int)v[4 * r + 2]);
        const double c2x = cc.x * cc.x, c2y = cc.y * cc.y;
        const double nx0 = 2.0 * vc.x - vp.x + t2 * c2x * (ve.x * v1.x + vt.x * (l2x - va.x) / tau);
        const double nx1 = 2.0 * vc.y - vp.y + t2 * c2y * (ve.y * v1.y + vt.y * (l2y - va.y) / tau);
        nx[q] = make_double2(nx0, nx1);
        l2o[q] = make_double2(l2x, l2y);
        bad |= (fabs(nx0) > prm.thr) || (fabs(nx1) > prm.thr);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(prm.flag, prm.step);
  }
  }  // active row warp
  // all row warps are done with tensor memory: release it
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("bar.sync 7, 256;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 2 * NWC)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem_base) : "memory");
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
  if (!((J0 == 1024 && J1 == 1024) || (J0 == 512 && J1 == 1024))) return false;
  const int nslot = J1 / 4 + 1;
  return nsm >= 148 && (nslot + 1) / 2 <= nsm;
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

int step2d_wcols(int J1) { return step2d_col_groups(J1) * kStep2dCG; }

void launch_w_to_2d(cudaStream_t st, int J0, int J1, int M, const double* w, double* w2d) {
  const int H = J1 / 2 + 1;
  k_w_to_2d<<<148 * 8, 256, 0, st>>>(J0, H, step2d_wcols(J1), M, w, w2d);
}

void launch_dev_tables(cudaStream_t st, size_t N, int M, const double* dev1, double* dev) {
  if (M < 1) return;
  k_dev_tables<<<148 * 8, 256, 0, st>>>((long long)N, M, dev1, dev);
}

}  // namespace fw
