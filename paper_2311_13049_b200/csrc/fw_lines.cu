// fw_lines.cu — register-resident line FFTs along a strided axis (generic multi-pass path).
//
// One kernel family for the C2C passes of the multi-pass pipeline (3D grids, 2D
// grids the persistent kernel does not serve, the slab stages): a block owns L
// consecutive lines of one axis (line-fastest thread mapping, so every global
// access of a warp is a contiguous run over L lines), thread (l, i) owns
// butterfly i of line l in every pass.  Pass 0 reads its inputs straight from
// global memory (optionally x w_m), the last pass writes straight to global
// memory (optionally x scale); in between the line lives once in shared memory
// in an in-place-per-butterfly layout (the canonical Stockham plan of
// fw_fft.cuh, only the storage order differs), one barrier per pass boundary.
// Bit-identical to k_c2c_axis / the CPU oracle (same radix plan, twiddles,
// fma placement).
//
// Kernels: k_lines<n, dir> (one term per blockIdx.y), k_lines_terms<n> (every term of the
// first inverse axis per block, uhat parked in tensor memory), k_rows_r2c<h> / k_rows_c2r<h>
// (per row of the last axis; the C2R keeps (s-s0) and (s-s0)^{m-1} in tensor memory and
// recombines the terms in registers).  Shared-memory layouts are bank-conflict-free for each
// kernel's thread mapping (tools/layouts/).  Build switches (-D..., A/B only; defaults are the
// measured best): FW_LINES_TERMS, FW_LT_PREFETCH, FW_LT_TARGET, FW_LT_DBUF,
// FW_LT_MINB{256,512,512W}, FW_LINES_SWZ, FW_LINES_WIDE, FW_WIDE_STRIDE, FW_LINES_NTH256,
// FW_LINES_MINB{256,512,1024}, FW_C2R_PAD, FW_C2R_XB2, FW_C2R_RPB{128,256}, FW_C2R_MINB{,128,256},
// FW_C2R_WSYNC, FW_C2R_BULK, FW_C2R_TM8, FW_ZERO_PLUS (and FW_TERM_PAD in fw_internal.h).
// Block shapes are chosen spill-free: every kernel here compiles with a zero stack frame except
// the 256-point all-terms inverse (24 B).
#include <cuda_runtime.h>

#include <algorithm>

#include "fw_fft.cuh"
#include "fw_internal.h"

namespace fw {
namespace lines {

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int npass(int n) { return (ilog2c(n) + 3) / 4; }
__host__ __device__ constexpr int radix(int n, int i) {
  return 1 << (ilog2c(n) / npass(n) + (i < ilog2c(n) % npass(n) ? 1 : 0));
}
__host__ __device__ constexpr int pprod(int n, int i) { return i == 0 ? 1 : pprod(n, i - 1) * radix(n, i - 1); }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

#ifndef FW_LINES_SWZ
#define FW_LINES_SWZ 1
#endif
#ifndef FW_LINES_WIDE
#define FW_LINES_WIDE 1
#endif
#ifndef FW_WIDE_STRIDE
#define FW_WIDE_STRIDE (512 << 10)  // bytes
#endif
template <int N, int NTH = 256>
struct Plan {
  static constexpr int P = npass(N);
  static constexpr int R0 = radix(N, 0), R1 = radix(N, 1), R2 = P > 2 ? radix(N, 2) : 1;
  static constexpr int T0 = N / R0, T1 = N / R1, T2 = N / R2;
  static constexpr int TMAX = cmax(T0, cmax(T1, P > 2 ? T2 : 0));
  // threads per block of the line kernels (launch_n picks 512 for long strides: 8 / 4 lines of
  // n = 512 / 1024 give 128 / 64 B contiguous per global access)
  static constexpr int NTHR = NTH;
  static constexpr int L = NTHR / TMAX;  // lines per block
  static constexpr int S1 = ilog2c(R1), ST = ilog2c(T1);
  // padded position; the line stride is odd so the L lines of a quarter warp hit distinct banks
  __device__ static __forceinline__ int pad(int p) { return p + (p >> S1) + (p >> ST); }
  static constexpr int LS = ((N - 1) + ((N - 1) >> S1) + ((N - 1) >> ST) + 1) | 1;
  // pass-0 output logical e -> position of pass-1 input (e % T1, e / T1) = (e % T1) R1 + e / T1
  __device__ static __forceinline__ int p0out(int e) { return pad((e % T1) * R1 + e / T1); }
  __device__ static __forceinline__ int p1(int i, int r) { return pad(i * R1 + r); }
  // pass-2 input logical e: the pass-1 slot (i1, r1) that produced it
  __device__ static __forceinline__ int p2in(int e) {
    const int i1 = (e / (R0 * R1)) * R0 + e % R0, r1 = (e / R0) % R1;
    return pad(i1 * R1 + r1);
  }
  // line kernels (line-fastest thread mapping, L lines per block): logical in-place slot p of
  // line l at lpos(l, p).  n = 512 / 1024: unpadded lines with an XOR swizzle of the 16-B slot
  // within its 128-B group (every pass bank-conflict-free, checked by enumerating the
  // quarter-warp bank groups of each access; the padding above gives 2-way conflicts there);
  // n = 256: the padding above (already conflict-free)
  // (the XOR term reads only bits >= 3 of p, so it permutes slots within their 8-slot group)
  // (searched per (n, L): tools/layouts/search_line_swizzle.py)
  static constexpr int SWA = N == 512 || N == 1024 ? 3 : 0;
  static constexpr int SWB = N == 512 ? (L == 8 ? 0 : 6) : N == 1024 ? 7 : 0;  // 0: single term
  static constexpr int SWL = N == 512 ? (L == 8 ? 1 : 2) : (L == 4 ? 2 : 4);
  static constexpr int LLS = (FW_LINES_SWZ && SWA) ? N : LS;
  __device__ static __forceinline__ int lpos(int l, int p) {
    if constexpr (FW_LINES_SWZ && SWA != 0)
      return l * N + (p ^ ((((p >> SWA) ^ (SWB ? (p >> SWB) : 0)) + SWL * l) & 7));
    else
      return l * LS + pad(p);
  }
  __device__ static __forceinline__ int q0out(int e) { return (e % T1) * R1 + e / T1; }
  __device__ static __forceinline__ int q1(int i, int r) { return i * R1 + r; }
  __device__ static __forceinline__ int q2in(int e) {
    const int i1 = (e / (R0 * R1)) * R0 + e % R0, r1 = (e / R0) % R1;
    return i1 * R1 + r1;
  }
  static_assert(P == 2 || P == 3, "2- or 3-pass plans");
  static_assert(L >= 1 && L * TMAX == NTHR, "whole lines per block");
};

// twiddled radix-R butterfly of pass PASS (p = pprod > 1): twiddles = master entries
template <int N, int PASS, int DIR>
__device__ __forceinline__ void bfly(double2* a, int i, const double2* __restrict__ master) {
  constexpr int R = radix(N, PASS);
  constexpr int p = pprod(N, PASS);
  if constexpr (p > 1) {
    const int k = i & (p - 1);
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const double2 w = __ldg(&master[(r * k) * (kTwMaster / (p * R))]);
      a[r] = cmulw(a[r], w.x, DIR < 0 ? -w.y : w.y);
    }
  }
  Dft<R, DIR>::run(a);
}

// blocks per SM the register allocation of k_lines<N> is bounded for (shared memory allows 3
// at N = 256, 6 at N = 512 / 1024)
#ifndef FW_LINES_NTH256
#define FW_LINES_NTH256 128  // threads per block of the 256-point line passes: 8 lines per block (256: 16 lines; A/B)
#endif
#ifndef FW_LINES_MINB256
#define FW_LINES_MINB256 3  // (of FW_LINES_NTH256 threads)
#endif
#ifndef FW_LINES_MINB512
#define FW_LINES_MINB512 4
#endif
#ifndef FW_LINES_MINB1024
#define FW_LINES_MINB1024 2
#endif
// (the 512 / 1024 bounds are for 256-thread blocks; 512-thread blocks get half)
template <int N, int NTH>
__host__ __device__ constexpr int lines_minb() {
  return N == 256 ? FW_LINES_MINB256 : (N == 512 ? FW_LINES_MINB512 : FW_LINES_MINB1024) * 256 / NTH;
}

// C2C of lines of length N along an axis of stride S (line (o, in): o*N*S + in + j*S).
// blockIdx.y = term (src/dst/w advance by their term strides), blockIdx.z = field (bl).
template <int N, int DIR, bool SCAT, int NTH>
__global__ void __launch_bounds__(NTH, (lines_minb<N, NTH>())) k_lines(const double2* __restrict__ src, double2* __restrict__ dst,
                                               const double* __restrict__ w, long long S, long long inner,
                                               long long src_ts, long long dst_ts, long long w_ts, double sc,
                                               int do_scale, const double2* __restrict__ master,
                                               const BatchLine* __restrict__ bl, const __grid_constant__ Scatter scat) {
  using PL = Plan<N, NTH>;
  constexpr int L = PL::L;
  extern __shared__ double2 sm[];  // L lines x LS
  if (bl) {
    src = static_cast<const double2*>(bl[blockIdx.z].src);
    dst = static_cast<double2*>(bl[blockIdx.z].dst);
    w = bl[blockIdx.z].w;
  }
  const long long term = blockIdx.y;
  src += term * src_ts;
  dst += term * dst_ts;
  if (w) w += term * w_ts;
  const long long bpo = (inner + L - 1) / L;
  const long long o = blockIdx.x / bpo;
  const long long in0 = (blockIdx.x - o * bpo) * L;
  const int l = threadIdx.x % L, i = threadIdx.x / L;
  const bool live = in0 + l < inner;
  const long long base = o * (long long)N * S + in0 + l;
  double2* line = sm;  // slot p of this thread's line at PL::lpos(l, p)

  {  // pass 0 (no twiddles): global -> registers -> shared
    constexpr int R = PL::R0, T = PL::T0;
    if (i < T) {
      double2 a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long idx = base + (long long)(i + r * T) * S;
        double2 v = live ? src[idx] : make_double2(0.0, 0.0);
        if (w && live) {
          const double wk = __ldg(&w[idx]);
          v.x = wk * v.x;
          v.y = wk * v.y;
        }
        a[r] = v;
      }
      Dft<R, DIR>::run(a);
#pragma unroll
      for (int r = 0; r < R; ++r) line[PL::lpos(l, PL::q0out(i * R + r))] = a[r];
    }
  }
  __syncthreads();
  if constexpr (PL::P == 3) {  // middle pass, in place
    constexpr int R = PL::R1, T = PL::T1;
    if (i < T) {
      double2 a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = line[PL::lpos(l, PL::q1(i, r))];
      bfly<N, 1, DIR>(a, i, master);
#pragma unroll
      for (int r = 0; r < R; ++r) line[PL::lpos(l, PL::q1(i, r))] = a[r];
    }
    __syncthreads();
  }
  {  // last pass: shared -> registers -> global (natural order q = i + r T)
    constexpr int LAST = PL::P - 1;
    constexpr int R = radix(N, LAST), T = N / R;
    if (i < T) {
      double2 a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = line[PL::lpos(l, LAST == 1 ? PL::q1(i, r) : PL::q2in(i + r * T))];
      bfly<N, LAST, DIR>(a, i, master);
      if (live) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double2 v = a[r];
          if (do_scale) {
            v.x *= sc;
            v.y *= sc;
          }
          const int j = i + r * T;
          if constexpr (SCAT) {  // fused transpose: straight into the destination rank's buffer
            int q, jr;
            if (scat.lgblk >= 0) {  // power-of-two block: 32-bit shift and mask
              q = j >> scat.lgblk;
              jr = j & ((1 << scat.lgblk) - 1);
            } else {
              q = (int)(j / scat.blk);
              jr = (int)(j - q * scat.blk);
            }
            scat.dst[q][term * scat.tstride + (long long)jr * scat.jstride + o * scat.ostride + in0 + l + scat.base] =
                v;
          } else {
            dst[base + (long long)j * S] = v;
          }
        }
      }
    }
  }
}


// ---------------------------------------------------------------- tensor memory (per-thread state)
// A warp reaches the 32 TMEM lanes of its quadrant (warp % 4); thread = lane, 32-bit columns.
__host__ __device__ constexpr int pow2ceil(int n) { return n <= 1 ? 1 : 2 * pow2ceil((n + 1) / 2); }
__device__ __forceinline__ void tm_ld16(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tm_st16(unsigned taddr, const unsigned* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
               ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
               : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double tm_get(const unsigned* v, int k) {
  return __hiloint2double((int)v[2 * k + 1], (int)v[2 * k]);
}
__device__ __forceinline__ void tm_set(unsigned* v, int k, double x) {
  v[2 * k] = (unsigned)__double2loint(x);
  v[2 * k + 1] = (unsigned)__double2hiint(x);
}

// the reference's per-term partial 0.0 + v (flap.cpp:83-89: partials start from a zeroed
// vector; differs from v only for v = -0.0).  An integer form that keeps the fp64 pipe free
// measured no faster.
// FW_ZERO_PLUS=0 drops the addition: the sum the partial is added to is never -0 (it starts at
// +0, and x + y = -0 needs x = y = -0), and s + (-0) = s + (+0) for every s other than -0, so the
// accumulated bits are the same (A/B).
#ifndef FW_ZERO_PLUS
#define FW_ZERO_PLUS 0
#endif
__device__ __forceinline__ double zero_plus(double v) {
#if FW_ZERO_PLUS
  double p = 0.0;
  p += v;
  return p;
#else
  return v;
#endif
}

// twiddled butterfly of pass PASS with the twiddles from a shared-memory table [k][r-1]
// (values = master entries: bit-identical to bfly())
template <int N, int PASS, int DIR>
__device__ __forceinline__ void bfly_s(double2* a, int i, const double2* tw) {
  constexpr int R = radix(N, PASS);
  constexpr int p = pprod(N, PASS);
  if constexpr (p > 1) {
    const double2* t = tw + (i & (p - 1)) * (R - 1);
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const double2 w = t[r - 1];
      a[r] = cmulw(a[r], w.x, DIR < 0 ? -w.y : w.y);
    }
  }
  Dft<R, DIR>::run(a);
}

// R2C post-processing (r2c_post) with the master entry of W_{2h}^k given (conjugated here as twiddle<-1> does)
__device__ __forceinline__ double2 r2c_post_w(const double2* Z, int k, int h, double2 wm) {
  if (k == 0) return make_double2(Z[0].x + Z[0].y, 0.0);
  if (k == h) return make_double2(Z[0].x - Z[0].y, 0.0);
  const double2 A = Z[k];
  const double2 Bz = Z[h - k];
  const double2 B = make_double2(Bz.x, -Bz.y);
  const double2 E = make_double2((A.x + B.x) * 0.5, (A.y + B.y) * 0.5);
  const double2 D = make_double2((A.x - B.x) * 0.5, (A.y - B.y) * 0.5);
  const double2 O = make_double2(D.y, -D.x);
  const double2 t = cmulw(O, wm.x, -wm.y);
  return make_double2(E.x + t.x, E.y + t.y);
}

// C2R pre-processing (c2r_pre) with W_{2h}^k given
__device__ __forceinline__ double2 c2r_pre_w(double2 A, double2 Xhk, bool k0, double2 w) {
  double2 B = make_double2(Xhk.x, -Xhk.y);
  if (k0) {
    A.y = 0.0;
    B.y = 0.0;
  }
  const double2 E = make_double2(A.x + B.x, A.y + B.y);
  const double2 D = make_double2(A.x - B.x, A.y - B.y);
  const double2 O = cmulw(D, w.x, w.y);
  return make_double2(E.x - O.y, E.y + O.x);
}

// bulk copies (TMA engine) with mbarrier completion: the X rows of the row C2R
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n FW_LMBW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra FW_LMBW_%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}

// Per row of the last axis (NL reals, h = NL/2 complex, rows contiguous): for every
// term m = m_first..m_last in ascending order, C2R of the half-spectrum row src_m
// (flap.cpp:21-36: pre-processing Z_q = f(X_q, X_{h-q}), h-point C2C, real parts
// interleaved) and acc += 0 + (s-s0)^m .* x with (s-s0)^m = (s-s0)^{m-1} (s-s0) carried
// per element (flap.cpp:61-91, 124-133).  Thread (row, i) owns butterfly i of every
// pass; its outputs q = i + r T_last and their accumulators stay in registers across
// the terms.  Everything a term needs besides its spectrum row is on chip: (s-s0) and
// the running power (s-s0)^{m-1} of the thread's outputs live in TENSOR MEMORY (loaded
// once per launch), the twiddles in one shared-memory table per block; the next term's
// row lands by cp.async while the current term's passes run.
#ifndef FW_C2R_PAD
#define FW_C2R_PAD 1  // 0: Plan<H>'s line padding in the row C2R (A/B)
#endif
#ifndef FW_C2R_RPB128
#define FW_C2R_RPB128 8  // rows per block of the h = 128 row C2R
#endif
#ifndef FW_C2R_XB2
#define FW_C2R_XB2 0  // h = 256 / 512 (h = 128 always double-buffers; at 16 rows per block it gained nothing)
#endif
#ifndef FW_C2R_MINB
#define FW_C2R_MINB 2  // blocks per SM the register allocation is bounded for
#endif
#ifndef FW_C2R_RPB256
#define FW_C2R_RPB256 8  // rows per block of the h = 256 row C2R (0: as many as fit two blocks per SM, 12)
#endif
#ifndef FW_C2R_MINB256
#define FW_C2R_MINB256 FW_C2R_MINB
#endif
#ifndef FW_C2R_MINB128
#define FW_C2R_MINB128 3  // the same for the h = 128 row C2R (8-row blocks of 128 threads)
#endif
#ifndef FW_C2R_TM8
#define FW_C2R_TM8 1  // h = 128 row C2R with 8 threads per row (0: 16; A/B)
#endif
#ifndef FW_C2R_BULK
#define FW_C2R_BULK 1  // X rows by one bulk copy per row (TMA engine, mbarrier per warp) when a row's threads share a warp (0: 16-B cp.async per thread; A/B)
#endif
#ifndef FW_C2R_WSYNC
#define FW_C2R_WSYNC 1  // warp barriers between the passes when a row's threads share a warp (0: block barriers, A/B)
#endif
template <int H>
struct C2RPlan {
  using P = Plan<H>;
  static constexpr int RL = radix(H, P::P - 1);      // last-pass radix
  static constexpr int TL = H / RL;
  // threads per row.  h = 128 (radix 16 then 8: 8 butterflies in pass 0, 16 in the last pass):
  // 8 threads per row, each with BOTH last-pass butterflies i and i + 8 -- with 16 threads the
  // pre-processing and pass 0 (two thirds of the row's fp64 work) ran on half the lanes
  static constexpr int TM = (H == 128 && FW_C2R_TM8) ? 8 : P::TMAX;
  static constexpr int NB = TL / TM;                 // last-pass butterflies per thread
  // X row stride (natural order, odd; 128-B aligned rows measured 1-3 % slower)
  static constexpr int XS = (H + 1) | 1;
  // twiddles: pre-processing W_{2H}^k (k <= H), pass 1 [k < R0][R1 - 1], pass 2 [k < R0 R1][R2 - 1]
  static constexpr int TW1 = P::R0 * (P::R1 - 1);
  static constexpr int TW2 = P::P > 2 ? P::R0 * P::R1 * (P::R2 - 1) : 0;
  static constexpr int TWN = (H + 1) + TW1 + TW2;
  // work layout: the in-place-per-butterfly positions of Plan<H> with a padding chosen for this
  // kernel's row-major thread mapping (Plan's padding suits the line-fastest mapping of k_lines
  // and gives 2-way conflicts in the last pass here): one pad term p >> PADA makes every pass
  // bank-conflict-free at h = 128 / 256 (checked by enumerating the quarter-warp bank groups of
  // each access); h = 512 keeps Plan's padding (already conflict-free)
  static constexpr int PADA = !FW_C2R_PAD ? 0 : H == 128 ? 3 : H == 256 ? 4 : 0;
  __device__ static __forceinline__ int pad(int p) { return PADA ? p + (p >> PADA) : P::pad(p); }
  static constexpr int LS = PADA ? (((H - 1) + ((H - 1) >> PADA) + 1) | 1) : P::LS;
  __device__ static __forceinline__ int p0out(int e) { return pad((e % P::T1) * P::R1 + e / P::T1); }
  __device__ static __forceinline__ int p1(int i, int r) { return pad(i * P::R1 + r); }
  __device__ static __forceinline__ int p2in(int e) {
    const int i1 = (e / (P::R0 * P::R1)) * P::R0 + e % P::R0, r1 = (e / P::R0) % P::R1;
    return pad(i1 * P::R1 + r1);
  }
  static constexpr size_t ROWB = (size_t)(XS + LS) * sizeof(double2);
  static constexpr size_t CAP = 112640;  // two blocks per SM
  static constexpr int RPB0 = (size_t)(256 / TM) * ROWB + TWN * sizeof(double2) <= CAP
                                  ? 256 / TM
                                  : (int)((CAP - TWN * sizeof(double2)) / ROWB);
  // h = 128: half-size blocks (8 rows, 4 warps), four per SM, X double-buffered (measured at C3:
  // 6.34 -> ~6.0 ms per step against 16-row blocks, two per SM)
  static constexpr int RPB = H == 128 ? FW_C2R_RPB128 : (H == 256 && FW_C2R_RPB256 > 0) ? FW_C2R_RPB256 : RPB0;
  static constexpr int MINB = H == 128 ? FW_C2R_MINB128 : H == 256 ? FW_C2R_MINB256 : FW_C2R_MINB;
  static constexpr int NT = RPB * TM;
  // X rows double-buffered (next term and the one after in flight) when that keeps RPB
  static constexpr int NXB = (FW_C2R_XB2 || H == 128) && (size_t)TWN * sizeof(double2) + (size_t)RPB * (ROWB + XS * sizeof(double2)) <= CAP ? 2 : 1;
  static constexpr size_t SMEM = (size_t)TWN * sizeof(double2) + (size_t)RPB * (ROWB + (NXB - 1) * XS * sizeof(double2));
  // tensor memory per warp and last-pass butterfly: (s-s0) at [0, 4 RL), (s-s0)^{m-1} at [4 RL, 8 RL)
  // (two columns per double)
  static constexpr int TMC = 8 * RL * NB;
  static constexpr int NSLOT = (NT / 32 + 3) / 4;
  static constexpr int TMALLOC = pow2ceil(NSLOT * TMC < 32 ? 32 : NSLOT * TMC);
  static_assert(RPB >= 1 && NT % 32 == 0, "whole warps");
  static_assert(TL == TM * NB && (NB == 1 || P::P == 2), "every thread owns NB RL outputs");
  static_assert(RL % 4 == 0, "16-column chunks");
  static_assert(TMALLOC <= 256, "two blocks per SM in tensor memory");
};

template <int H>
__global__ void __launch_bounds__(C2RPlan<H>::NT, C2RPlan<H>::MINB) k_rows_c2r(const double2* __restrict__ src, long long src_ts,
                                                            int m_first, int m_last, const double* __restrict__ dev1,
                                                            double* __restrict__ out, long long rows, double* residue,
                                                            const int* guard, const double2* __restrict__ master,
                                                            const BatchLine* __restrict__ bl, long long xrs, int resume) {
  using RP = C2RPlan<H>;
  using PL = Plan<H>;
  constexpr int TM = RP::TM, RPB = RP::RPB, RL = RP::RL, TL = RP::TL, NL = 2 * H, NT = RP::NT, NB = RP::NB;
  if (guard && *guard != kNoBlowup) return;
  if (bl) {
    src = static_cast<const double2*>(bl[blockIdx.z].src);
    dev1 = bl[blockIdx.z].aux;
    out = bl[blockIdx.z].out;
  }
  // [X rows: NXB x RPB x XS][twiddles: TWN][work: RPB x LS]
  extern __shared__ __align__(128) double2 sm[];
  __shared__ unsigned tbase_sh;
  const int tid = threadIdx.x;
  const int rl = tid / TM, i = tid % TM;
  const long long row = (long long)blockIdx.x * RPB + rl;
  const bool live = row < rows;
  constexpr int NXB = RP::NXB;
  double2* Xb = sm + rl * RP::XS;  // natural-order X of this row (NXB buffers)
  double2* twpre = sm + NXB * RPB * RP::XS;
  double2* tw1 = twpre + (H + 1);
  double2* tw2 = tw1 + RP::TW1;
  double2* Wk = twpre + RP::TWN + rl * RP::LS;  // FFT work (in-place layout)

  const double* d1row = dev1 ? dev1 + (live ? row : 0) * NL : nullptr;
  // X rows arrive NXB terms ahead: a buffer is refilled as soon as pass 0 of its term has read it,
  // and lands during the following terms' passes.  When a row's threads share a warp, lane 0 of the
  // warp issues ONE bulk copy per row of the warp (the TMA engine writes the row into shared
  // memory; 16-B cp.async per thread cost three times the shared-memory wavefronts of the row)
  // and the warp waits on its own mbarrier; otherwise 16-B cp.async, one commit group per term.
  // (h = 128: the 2-KB rows measured 2 % slower by bulk copy at C3, 1.7 % faster at h = 256, C5)
  constexpr bool BULK = FW_C2R_BULK && FW_C2R_WSYNC && 32 % TM == 0 && H >= 256;
  __shared__ __align__(8) unsigned long long xbar[BULK ? NT / 32 : 1][2];
  auto fetch = [&](int m) {
    if constexpr (BULK) {
      if ((tid & 31) == 0) {
        constexpr int RPW = 32 / TM;  // rows per warp
        const long long row0 = (long long)blockIdx.x * RPB + (tid / 32) * RPW;
        const int b = (m - m_first) % NXB;
        int nlive = 0;
        for (int r = 0; r < RPW; ++r) nlive += (row0 + r < rows && m <= m_last) ? 1 : 0;
        mbar_expect_tx(&xbar[tid / 32][b], (unsigned)(nlive * (H + 1) * sizeof(double2)));
        for (int r = 0; r < nlive; ++r)
          bulk_g2s(sm + ((tid / 32) * RPW + r) * RP::XS + b * RPB * RP::XS,
                   src + (long long)(m - m_first) * src_ts + (row0 + r) * xrs, (unsigned)((H + 1) * sizeof(double2)),
                   &xbar[tid / 32][b]);
      }
      return;
    }
    if (live && m <= m_last) {
      const double2* S = src + (long long)(m - m_first) * src_ts + row * xrs;
      double2* X = Xb + ((m - m_first) % NXB) * RPB * RP::XS;
      for (int k = i; k <= H; k += TM)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(&X[k])),
                     "l"(S + k)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if constexpr (BULK) {
    if ((tid & 31) == 0) {
      mbar_init(&xbar[tid / 32][0], 1);
      mbar_init(&xbar[tid / 32][1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
  }
  fetch(m_first);
  if (NXB > 1) fetch(m_first + 1);

  // twiddle tables (values = master entries, as twiddle() / bfly() read them)
  for (int e = tid; e <= H; e += NT) twpre[e] = master[e * (kTwMaster / (2 * H))];
  for (int e = tid; e < RP::TW1; e += NT) {
    constexpr int R = PL::R1, p = PL::R0;
    const int k = e / (R - 1), r = e % (R - 1) + 1;
    tw1[e] = master[(r * k) * (kTwMaster / (p * R))];
  }
  if constexpr (PL::P > 2) {
    for (int e = tid; e < RP::TW2; e += NT) {
      constexpr int R = PL::R2, p = PL::R0 * PL::R1;
      const int k = e / (R - 1), r = e % (R - 1) + 1;
      tw2[e] = master[(r * k) * (kTwMaster / (p * R))];
    }
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tbase_sh)),
                 "n"(RP::TMALLOC)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = tid >> 5;
  // butterfly bb of the last pass (index i + bb TM): (s-s0) at tdev + bb 8 RL, the running power 4 RL further
  const unsigned tdev = tbase_sh + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * RP::TMC);
  const unsigned tpow = tdev + 4 * RL;
  if (d1row) {  // (s-s0) of this thread's outputs -> tensor memory, once
#pragma unroll
    for (int bb = 0; bb < NB; ++bb) {
#pragma unroll
      for (int c4 = 0; c4 < RL / 4; ++c4) {
        unsigned v[16];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const int q = i + bb * TM + (4 * c4 + rr) * TL;
          const double2 d = live ? __ldg(reinterpret_cast<const double2*>(d1row) + q) : make_double2(0.0, 0.0);
          tm_set(v, 2 * rr, d.x);
          tm_set(v, 2 * rr + 1, d.y);
        }
        tm_st16(tdev + bb * 8 * RL + 16 * c4, v);
        if (resume && m_first > 1) {
          // a later chunk of the operator's terms: the running power (s-s0)^{m_first-1} by the same
          // recurrence the earlier chunks ran, (s-s0)^m = (s-s0)^{m-1} (s-s0) (flap.cpp:131)
          unsigned pw[16];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const double d1 = tm_get(v, e);
            double d = d1;
            for (int m = 2; m < m_first; ++m) d = d * d1;
            tm_set(pw, e, d);
          }
          tm_st16(tpow + bb * 8 * RL + 16 * c4, pw);
        }
      }
    }
    tm_wait_st();
  }

  // a row's TM threads exchange data only among themselves (its X row, its work buffer): when
  // they share a warp (h = 128 / 256: 16 threads per row) the pass boundaries need a warp barrier
  // only, and the block's warps run through the terms independently of each other
  auto rowsync = [] {
    if constexpr (FW_C2R_WSYNC && 32 % TM == 0)
      __syncwarp();
    else
      __syncthreads();
  };
  double acc[NB][2 * RL];
#pragma unroll
  for (int bb = 0; bb < NB; ++bb)
#pragma unroll
    for (int e = 0; e < 2 * RL; ++e) acc[bb][e] = 0.0;
  if (resume && live) {  // partial sums of the operator's earlier terms (written by the previous chunk's launch)
#pragma unroll
    for (int bb = 0; bb < NB; ++bb)
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const double2 o = reinterpret_cast<const double2*>(out + row * NL)[i + bb * TM + r * TL];
        acc[bb][2 * r] = o.x;
        acc[bb][2 * r + 1] = o.y;
      }
  }
  double rmax = 0.0;
  for (int m = m_first; m <= m_last; ++m) {
    if constexpr (BULK)
      mbar_wait(&xbar[tid / 32][(m - m_first) % NXB], (unsigned)((m - m_first) / NXB) & 1u);
    else if (NXB > 1)
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // term m landed (m + 1 may be in flight)
    else
      asm volatile("cp.async.wait_all;" ::: "memory");
    rowsync();  // X of term m complete; every thread is done with the previous term's work buffer
    const double2* X = Xb + ((m - m_first) % NXB) * RPB * RP::XS;
    if (residue && live && i == 0) rmax = fmax(rmax, fabs(X[0].y) + fabs(X[H].y));
    {  // C2R pre-processing + pass 0 (no twiddles) -> work
      constexpr int R = PL::R0, T = PL::T0;
      if (i < T) {
        double2 a[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int q = i + r * T;
          a[r] = c2r_pre_w(X[q], X[H - q], q == 0, twpre[q]);
        }
        Dft<R, +1>::run(a);
#pragma unroll
        for (int r = 0; r < R; ++r) Wk[RP::p0out(i * R + r)] = a[r];
      }
    }
    rowsync();
    fetch(m + NXB);  // X is free again
    if constexpr (PL::P == 3) {
      constexpr int R = PL::R1, T = PL::T1;
      if (i < T) {
        double2 a[R];
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = Wk[RP::p1(i, r)];
        bfly_s<H, 1, +1>(a, i, tw1);
#pragma unroll
        for (int r = 0; r < R; ++r) Wk[RP::p1(i, r)] = a[r];
      }
      rowsync();
    }
#pragma unroll
    for (int bb = 0; bb < NB; ++bb) {  // last pass -> outputs z_q, q = ib + r TL: reals x[2q], x[2q+1]
      constexpr int LAST = PL::P - 1;
      const int ib = i + bb * TM;
      double2 a[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) a[r] = Wk[LAST == 1 ? RP::p1(ib, r) : RP::p2in(ib + r * TL)];
      bfly_s<H, LAST, +1>(a, ib, LAST == 1 ? tw1 : tw2);
      if (m == 0 || !d1row) {
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          acc[bb][2 * r] += zero_plus(a[r].x);
          acc[bb][2 * r + 1] += zero_plus(a[r].y);
        }
      } else {
#pragma unroll
        for (int c4 = 0; c4 < RL / 4; ++c4) {
          unsigned dv[16], pv[16];
          tm_ld16(tdev + bb * 8 * RL + 16 * c4, dv);
          if (m > 1) tm_ld16(tpow + bb * 8 * RL + 16 * c4, pv);
          tm_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) {  // element e of the chunk: output r = 4 c4 + e / 2, real part e % 2
            const int r = 4 * c4 + e / 2;
            const double x = (e & 1) ? a[r].y : a[r].x;
            double d = tm_get(dv, e);
            if (m > 1) d = tm_get(pv, e) * d;  // (s-s0)^m = (s-s0)^{m-1} (s-s0)
            tm_set(pv, e, d);
            acc[bb][2 * r + (e & 1)] += zero_plus(d * x);
          }
          tm_st16(tpow + bb * 8 * RL + 16 * c4, pv);
        }
        tm_wait_st();
      }
    }
  }
  if (live) {
#pragma unroll
    for (int bb = 0; bb < NB; ++bb)
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int q = i + bb * TM + r * TL;
        reinterpret_cast<double2*>(out + row * NL)[q] = make_double2(acc[bb][2 * r], acc[bb][2 * r + 1]);
      }
  }
  if (residue && live && i == 0 && rmax > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(residue), (unsigned long long)__double_as_longlong(rmax));
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase_sh), "n"(RP::TMALLOC)
                 : "memory");
}

// All terms of an inverse along a strided axis in one pass over the spectrum: out_m =
// C2C(w_m .* uhat) for m in the launch's term range (flap.cpp:64-71 weights fused into
// pass 0).  Same thread mapping and arithmetic as k_lines<N, +1> with grid.y = terms, but a
// block loops over the terms itself: its lines of uhat are read from HBM ONCE and parked in
// tensor memory (pass-0 inputs of each thread), so a launch streams uhat once, w_m once and
// writes the M+1 outputs (instead of re-reading uhat per term).  The next term's weights
// are loaded while the current term's passes run.
#ifndef FW_LT_MINB512
#define FW_LT_MINB512 2  // blocks per SM of the 256-thread 512-point all-terms inverse
#endif
#ifndef FW_LT_DBUF
#define FW_LT_DBUF 0  // 1: double-buffered lines in the 512-point all-terms inverse (measured 1 % slower at C5; A/B)
#endif
#ifndef FW_LT_LD2
#define FW_LT_LD2 1
#endif
#ifndef FW_LT_LD1
#define FW_LT_LD1 1
#endif
#ifndef FW_LT_MINB512W
#define FW_LT_MINB512W 1  // blocks per SM of the 512-thread 512-point all-terms inverse
#endif
#ifndef FW_LT_MINB256
#define FW_LT_MINB256 0  // blocks per SM of the 256-point all-terms inverse (0: 512 / threads)
#endif
#ifndef FW_LT_PREFETCH
#define FW_LT_PREFETCH 1  // next term's weights loaded during the current term's passes
#endif
template <int N, int NTH>
struct TermPlan {
  using P = Plan<N, NTH>;
  static constexpr int TW1 = P::P > 2 ? P::R0 * (P::R1 - 1) : 0;  // pass-1 twiddles of a 3-pass plan
  static constexpr int TWL = pprod(N, P::P - 1) * (radix(N, P::P - 1) - 1);  // last pass
  static constexpr int TWN = TW1 + TWL;
  // line buffers: two at N = 512 (term t + 1's pass 0 fills the other one while slower warps
  // still read term t's last pass: one block barrier per term fewer), one otherwise (shared memory)
  static constexpr int NBUF = (FW_LT_DBUF && N == 512) ? 2 : 1;
  static constexpr size_t SMEM = (size_t)(TWN + NBUF * P::L * P::LLS) * sizeof(double2);
  static constexpr int TMC = 4 * P::R0;  // columns per warp: R0 complex pass-0 inputs
  static constexpr int NSLOT = P::NTHR / 128;  // warps per TMEM lane quadrant
  static constexpr int TMALLOC = pow2ceil(NSLOT * TMC < 32 ? 32 : NSLOT * TMC);
};

template <int N, bool SCAT, int NTH>
__global__ void __launch_bounds__(NTH, (N == 512 && NTH == 256) ? FW_LT_MINB512 : (N == 512 && NTH == 512) ? FW_LT_MINB512W : (N == 256 && FW_LT_MINB256 > 0) ? FW_LT_MINB256 : 512 / NTH) k_lines_terms(const double2* __restrict__ src, double2* __restrict__ dst,
                                                        const double* __restrict__ w, long long S, long long inner,
                                                        long long dst_ts, long long w_ts, int nterms, int tchunk,
                                                        double sc, int do_scale, const double2* __restrict__ master,
                                                        const BatchLine* __restrict__ bl, const __grid_constant__ Scatter scat,
                                                        long long Sd) {
  using PL = Plan<N, NTH>;
  using TP = TermPlan<N, NTH>;
  constexpr int L = PL::L, R0 = PL::R0, T0 = PL::T0, LAST = PL::P - 1;
  constexpr int RLST = radix(N, LAST), TLST = N / RLST;
  extern __shared__ double2 sm[];
  __shared__ unsigned tbase_sh;
  if (bl) {
    src = static_cast<const double2*>(bl[blockIdx.z].src);
    if constexpr (!SCAT) dst = static_cast<double2*>(bl[blockIdx.z].dst);
    w = bl[blockIdx.z].w;
  }
  // this block's terms [t0, t1) (blockIdx.y = chunk: small grids split the term range)
  const int t0 = blockIdx.y * tchunk, t1 = min(nterms, t0 + tchunk);
  w += (long long)t0 * w_ts;
  double2* tw1 = sm;
  double2* twl = sm + TP::TW1;
  double2* lines_sm = sm + TP::TWN;
  const int tid = threadIdx.x;
  const long long bpo = (inner + L - 1) / L;
  const long long o = blockIdx.x / bpo;
  const long long in0 = (blockIdx.x - o * bpo) * L;
  const int l = tid % L, i = tid / L;
  const bool live = in0 + l < inner;
  const long long base = o * (long long)N * S + in0 + l;
  const long long dbase = o * (long long)N * Sd + in0 + l;  // destination (Sd != S: padded rows, inner < S)
  double2* line = lines_sm;  // slot p of this thread's line at PL::lpos(l, p)  (buffer term % NBUF)

  if constexpr (PL::P > 2) {
    for (int e = tid; e < TP::TW1; e += PL::NTHR) {
      constexpr int R = PL::R1, p = PL::R0;
      const int k = e / (R - 1), r = e % (R - 1) + 1;
      tw1[e] = master[(r * k) * (kTwMaster / (p * R))];
    }
  }
  for (int e = tid; e < TP::TWL; e += PL::NTHR) {
    constexpr int R = RLST, p = pprod(N, LAST);
    const int k = e / (R - 1), r = e % (R - 1) + 1;
    twl[e] = master[(r * k) * (kTwMaster / (p * R))];
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tbase_sh)),
                 "n"(TP::TMALLOC)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = tid >> 5;
  const unsigned tu = tbase_sh + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * TP::TMC);
  // pass-0 holders: i < T0 (warp-uniform: i = tid / L and T0 L is a multiple of 32)
  static_assert((T0 * L) % 32 == 0, "warp-uniform pass-0 threads");
  const bool p0 = i < T0;
  double wk[R0];  // this term's weights (loaded one term ahead)
  if (p0) {
#pragma unroll
    for (int c = 0; c < R0 / 4; ++c) {  // uhat -> tensor memory, 4 complex (16 columns) per store
      unsigned v[16];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const long long idx = base + (long long)(i + (4 * c + rr) * T0) * S;
        const double2 x = live ? src[idx] : make_double2(0.0, 0.0);
        tm_set(v, 2 * rr, x.x);
        tm_set(v, 2 * rr + 1, x.y);
      }
      tm_st16(tu + 16 * c, v);
    }
    tm_wait_st();
#pragma unroll
    for (int r = 0; r < R0; ++r) wk[r] = live ? __ldg(&w[base + (long long)(i + r * T0) * S]) : 0.0;
  }
  for (int term = t0; term < t1; ++term) {
    if constexpr (TP::NBUF > 1) line = lines_sm + ((term - t0) & 1) * (L * PL::LLS);
    if (p0) {  // pass 0: w_m .* uhat (no twiddles)
      if (!FW_LT_PREFETCH && term > t0) {
        const double* wn = w + (long long)(term - t0) * w_ts;
#pragma unroll
        for (int r = 0; r < R0; ++r) wk[r] = live ? __ldg(&wn[base + (long long)(i + r * T0) * S]) : 0.0;
      }
      double2 a[R0];
      if constexpr (FW_LT_LD1 && R0 == 8) {  // both tensor-memory loads in flight, one wait
        unsigned v[32];
        tm_ld16(tu, v);
        tm_ld16(tu + 16, v + 16);
        tm_wait_ld();
#pragma unroll
        for (int r = 0; r < R0; ++r)
          a[r] = live ? make_double2(wk[r] * tm_get(v, 2 * r), wk[r] * tm_get(v, 2 * r + 1)) : make_double2(0.0, 0.0);
      } else if constexpr (FW_LT_LD2 && R0 == 16) {  // two loads in flight per wait
#pragma unroll
        for (int c = 0; c < R0 / 8; ++c) {
          unsigned v[32];
          tm_ld16(tu + 32 * c, v);
          tm_ld16(tu + 32 * c + 16, v + 16);
          tm_wait_ld();
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int r = 8 * c + rr;
            a[r] = live ? make_double2(wk[r] * tm_get(v, 2 * rr), wk[r] * tm_get(v, 2 * rr + 1)) : make_double2(0.0, 0.0);
          }
        }
      } else {
#pragma unroll
      for (int c = 0; c < R0 / 4; ++c) {
        unsigned v[16];
        tm_ld16(tu + 16 * c, v);
        tm_wait_ld();
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const int r = 4 * c + rr;
          a[r] = live ? make_double2(wk[r] * tm_get(v, 2 * rr), wk[r] * tm_get(v, 2 * rr + 1)) : make_double2(0.0, 0.0);
        }
      }
      }
      if (FW_LT_PREFETCH && term + 1 < t1) {
        const double* wn = w + (long long)(term + 1 - t0) * w_ts;
#pragma unroll
        for (int r = 0; r < R0; ++r) wk[r] = live ? __ldg(&wn[base + (long long)(i + r * T0) * S]) : 0.0;
      }
      Dft<R0, +1>::run(a);
#pragma unroll
      for (int r = 0; r < R0; ++r) line[PL::lpos(l, PL::q0out(i * R0 + r))] = a[r];
    }
    __syncthreads();
    if constexpr (PL::P == 3) {
      constexpr int R = PL::R1, T = PL::T1;
      if (i < T) {
        double2 a[R];
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = line[PL::lpos(l, PL::q1(i, r))];
        bfly_s<N, 1, +1>(a, i, tw1);
#pragma unroll
        for (int r = 0; r < R; ++r) line[PL::lpos(l, PL::q1(i, r))] = a[r];
      }
      __syncthreads();
    }
    if (i < TLST) {  // last pass: shared -> registers -> global (natural order q = i + r T)
      double2 a[RLST];
#pragma unroll
      for (int r = 0; r < RLST; ++r) a[r] = line[PL::lpos(l, LAST == 1 ? PL::q1(i, r) : PL::q2in(i + r * TLST))];
      bfly_s<N, LAST, +1>(a, i, twl);
      if (live) {
#pragma unroll
        for (int r = 0; r < RLST; ++r) {
          double2 v = a[r];
          if (do_scale) {
            v.x *= sc;
            v.y *= sc;
          }
          const int j = i + r * TLST;
          if constexpr (SCAT) {
            int q, jr;
            if (scat.lgblk >= 0) {  // power-of-two block: 32-bit shift and mask
              q = j >> scat.lgblk;
              jr = j & ((1 << scat.lgblk) - 1);
            } else {
              q = (int)(j / scat.blk);
              jr = (int)(j - q * scat.blk);
            }
            scat.dst[q][term * scat.tstride + (long long)jr * scat.jstride + o * scat.ostride + in0 + l + scat.base] =
                v;
          } else {
            dst[(long long)term * dst_ts + dbase + (long long)j * Sd] = v;
          }
        }
      }
    }
    // the line buffer takes the next term's pass 0 (with two buffers the barriers of the next
    // term order its reuse the term after)
    if constexpr (TP::NBUF == 1) __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase_sh), "n"(TP::TMALLOC)
                 : "memory");
}

// row plan of the R2C kernel (the block shape of the earlier shared-memory C2R)
template <int H>
struct RowPlan {
  using P = Plan<H>;
  static constexpr int TM = P::TMAX;
  static constexpr int RL = radix(H, P::P - 1);
  static constexpr int TL = H / RL;
  static constexpr size_t ROWB = (size_t)(((H + 1) | 1) + P::LS) * sizeof(double2) + (size_t)2 * H * sizeof(double);
  static constexpr int RPB = (256 / TM) * ROWB <= 112640 ? 256 / TM : (int)(112640 / ROWB);
  static constexpr int NT = RPB * TM;
};

// Per row of the last axis: R2C of NL = 2H reals (z_j = x_2j + i x_2j+1, H-point C2C,
// split X_k = f(Z_k, Z_{H-k})) into H+1 bins, x scale when do_scale.  Same plan/threads as
// k_rows_c2r; pass 0 reads the row straight from global memory.
template <int H>
__global__ void __launch_bounds__(256) k_rows_r2c(const double* __restrict__ u, double2* __restrict__ Uh,
                                                  long long rows, double sc, int do_scale,
                                                  const double2* __restrict__ master,
                                                  const BatchLine* __restrict__ bl) {
  using RP = RowPlan<H>;
  using PL = Plan<H>;
  using XP = C2RPlan<H>;  // work layout of the row-major mapping (conflict-free padding)
  constexpr int TM = RP::TM, RPB = RP::RPB, RL = RP::RL, TL = RP::TL;
  if (bl) {
    u = static_cast<const double*>(bl[blockIdx.z].src);
    Uh = static_cast<double2*>(bl[blockIdx.z].dst);
  }
  extern __shared__ double2 sm[];
  const int rl = threadIdx.x / TM, i = threadIdx.x % TM;
  const long long row = (long long)blockIdx.x * RPB + rl;
  const bool live = row < rows;
  // [twiddles: post-processing W_{2H}^k (k <= H), pass 1, pass 2 -- the row C2R's table][work: RPB x LS]
  // (values = the master entries; one table per block instead of scattered master reads per thread)
  double2* twpre = sm;
  double2* tw1 = twpre + (H + 1);
  double2* tw2 = tw1 + XP::TW1;
  for (int e = threadIdx.x; e <= H; e += RP::NT) twpre[e] = master[e * (kTwMaster / (2 * H))];
  for (int e = threadIdx.x; e < XP::TW1; e += RP::NT) {
    constexpr int R = PL::R1, p = PL::R0;
    const int k = e / (R - 1), r = e % (R - 1) + 1;
    tw1[e] = master[(r * k) * (kTwMaster / (p * R))];
  }
  if constexpr (PL::P > 2) {
    for (int e = threadIdx.x; e < XP::TW2; e += RP::NT) {
      constexpr int R = PL::R2, p = PL::R0 * PL::R1;
      const int k = e / (R - 1), r = e % (R - 1) + 1;
      tw2[e] = master[(r * k) * (kTwMaster / (p * R))];
    }
  }
  __syncthreads();
  double2* Wk = sm + XP::TWN + rl * XP::LS;  // FFT work, then the natural-order result
  // a row's threads exchange data only among themselves: a warp barrier when they share a warp
  auto rowsync = [] {
    if constexpr (FW_C2R_WSYNC && 32 % TM == 0)
      __syncwarp();
    else
      __syncthreads();
  };
  const double2* z = reinterpret_cast<const double2*>(u) + row * H;
  {  // pass 0 straight from global
    constexpr int R = PL::R0, T = PL::T0;
    if (i < T) {
      double2 a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = live ? z[i + r * T] : make_double2(0.0, 0.0);
      Dft<R, -1>::run(a);
#pragma unroll
      for (int r = 0; r < R; ++r) Wk[XP::p0out(i * R + r)] = a[r];
    }
  }
  rowsync();
  if constexpr (PL::P == 3) {
    constexpr int R = PL::R1, T = PL::T1;
    if (i < T) {
      double2 a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = Wk[XP::p1(i, r)];
      bfly_s<H, 1, -1>(a, i, tw1);
#pragma unroll
      for (int r = 0; r < R; ++r) Wk[XP::p1(i, r)] = a[r];
    }
    rowsync();
  }
  {
    constexpr int LAST = PL::P - 1;
    double2 a[RL];
    if (i < TL) {
#pragma unroll
      for (int r = 0; r < RL; ++r) a[r] = Wk[LAST == 1 ? XP::p1(i, r) : XP::p2in(i + r * TL)];
      bfly_s<H, LAST, -1>(a, i, LAST == 1 ? tw1 : tw2);
    }
    rowsync();  // every read of the work layout is done: store the natural-order result
    if (i < TL) {
#pragma unroll
      for (int r = 0; r < RL; ++r) Wk[i + r * TL] = a[r];
    }
  }
  rowsync();
  if (live) {
    double2* X = Uh + row * (H + 1);
    for (int k = i; k <= H; k += TM) {
      double2 v = r2c_post_w(Wk, k, H, twpre[k]);
      if (do_scale) {
        v.x *= sc;
        v.y *= sc;
      }
      X[k] = v;
    }
  }
}

#ifndef FW_LT_TARGET
#define FW_LT_TARGET 1184  // blocks the all-terms inverse aims for (4 waves x 2 blocks x 148 SMs)
#endif
#ifndef FW_LINES_TERMS
#define FW_LINES_TERMS 1  // 0: one block per (lines, term), uhat re-read per term
#endif
static_assert(FW_LINES_TERMS || !FW_TERM_PAD, "padded term scratch rows need the all-terms inverse (FW_LINES_TERMS=0: build with -DFW_TERM_PAD=0)");
template <int N, int NTH>
bool launch_nt(const LaunchCtx& L, int dir, const double2* src, double2* dst, const double* w, long long S,
              long long outer, long long inner, long long src_ts, long long dst_ts, long long w_ts, int nterms,
              int nfields, double sc, bool scale, const BatchLine* bl, const Scatter* scatter, long long Sd) {
  constexpr int LPB = Plan<N, NTH>::L;
  constexpr size_t SMEM = (size_t)LPB * Plan<N, NTH>::LLS * sizeof(double2);
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_lines<N, -1, false, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    cudaFuncSetAttribute(k_lines<N, +1, false, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    cudaFuncSetAttribute(k_lines<N, -1, true, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    cudaFuncSetAttribute(k_lines<N, +1, true, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  });
  const long long bpo = (inner + LPB - 1) / LPB;
  const Scatter none{};
  const Scatter& sc_ = scatter ? *scatter : none;
  const int f = scale ? 1 : 0;
  if (FW_LINES_TERMS && dir > 0 && src_ts == 0 && nterms > 1 && (w || (bl && w_ts != 0))) {  // (launch_n's `terms`)
    // every term of an inverse from one uhat: one pass over the spectrum (k_lines_terms)
    constexpr size_t TSM = TermPlan<N, NTH>::SMEM;
    static std::atomic<unsigned long long> tattr{0};
    once_per_device(tattr, [] {
      cudaFuncSetAttribute(k_lines_terms<N, false, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TSM);
      cudaFuncSetAttribute(k_lines_terms<N, true, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TSM);
    });
    // enough blocks to fill the GPU: split the term range when the lines alone give fewer than
    // ~4 waves of two blocks per SM (uhat is then read once per chunk)
    const long long nb = outer * bpo * nfields;
    const int nchunk = (int)std::min<long long>(nterms, std::max<long long>(1, (FW_LT_TARGET + nb - 1) / nb));
    const int tchunk = (nterms + nchunk - 1) / nchunk;
    const dim3 tgrid((unsigned)(outer * bpo), (unsigned)((nterms + tchunk - 1) / tchunk), (unsigned)nfields);
    if (scatter)
      k_lines_terms<N, true, NTH><<<tgrid, Plan<N, NTH>::NTHR, TSM, L.stream>>>(src, dst, w, S, inner, dst_ts, w_ts, nterms, tchunk, sc,
                                                             f, L.master, bl, sc_, Sd);
    else
      k_lines_terms<N, false, NTH><<<tgrid, Plan<N, NTH>::NTHR, TSM, L.stream>>>(src, dst, w, S, inner, dst_ts, w_ts, nterms, tchunk,
                                                              sc, f, L.master, bl, sc_, Sd);
    if (L.launches) *L.launches += 1;
    return true;
  }
  if (Sd != S) return false;  // only the all-terms inverse writes a differently strided destination
  const dim3 grid((unsigned)(outer * bpo), (unsigned)nterms, (unsigned)nfields);
  if (dir < 0) {
    if (scatter)
      k_lines<N, -1, true, NTH><<<grid, Plan<N, NTH>::NTHR, SMEM, L.stream>>>(src, dst, w, S, inner, src_ts, dst_ts, w_ts, sc, f, L.master,
                                                           bl, sc_);
    else
      k_lines<N, -1, false, NTH><<<grid, Plan<N, NTH>::NTHR, SMEM, L.stream>>>(src, dst, w, S, inner, src_ts, dst_ts, w_ts, sc, f,
                                                            L.master, bl, sc_);
  } else {
    if (scatter)
      k_lines<N, +1, true, NTH><<<grid, Plan<N, NTH>::NTHR, SMEM, L.stream>>>(src, dst, w, S, inner, src_ts, dst_ts, w_ts, sc, f, L.master,
                                                           bl, sc_);
    else
      k_lines<N, +1, false, NTH><<<grid, Plan<N, NTH>::NTHR, SMEM, L.stream>>>(src, dst, w, S, inner, src_ts, dst_ts, w_ts, sc, f,
                                                            L.master, bl, sc_);
  }
  if (L.launches) *L.launches += 1;
  return true;
}

// 512-thread blocks (8 / 4 lines per block: 128 / 64 B contiguous per global access) for every
// 512 / 1024-point line pass, except the all-terms inverse on short strides, which keeps
// 256-thread blocks (measured: C4 step 97.6 -> 83 ms, C5 unchanged; tools/lt_stride.py)
template <int N>
bool launch_n(const LaunchCtx& L, int dir, const double2* src, double2* dst, const double* w, long long S,
              long long outer, long long inner, long long src_ts, long long dst_ts, long long w_ts, int nterms,
              int nfields, double sc, bool scale, const BatchLine* bl, const Scatter* scatter, long long Sd) {
  const bool terms = dir > 0 && src_ts == 0 && nterms > 1 && (w || (bl && w_ts != 0));
  const bool wide = FW_LINES_WIDE && (N == 1024 || !terms || S * (long long)sizeof(double2) >= FW_WIDE_STRIDE);
  if constexpr (N == 256)
    return launch_nt<N, FW_LINES_NTH256>(L, dir, src, dst, w, S, outer, inner, src_ts, dst_ts, w_ts, nterms, nfields, sc, scale, bl, scatter, Sd);
  else
    return wide ? launch_nt<N, 512>(L, dir, src, dst, w, S, outer, inner, src_ts, dst_ts, w_ts, nterms, nfields, sc, scale, bl, scatter, Sd) : launch_nt<N, 256>(L, dir, src, dst, w, S, outer, inner, src_ts, dst_ts, w_ts, nterms, nfields, sc, scale, bl, scatter, Sd);
}

template <int H>
bool launch_rows_r2c_t(const LaunchCtx& L, const double* u, double2* Uh, long long rows, int nfields, double sc,
                       bool scale, const BatchLine* bl) {
  using RP = RowPlan<H>;
  constexpr size_t SMEM = (size_t)(C2RPlan<H>::TWN + RP::RPB * C2RPlan<H>::LS) * sizeof(double2);
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_rows_r2c<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  });
  const dim3 grid((unsigned)((rows + RP::RPB - 1) / RP::RPB), 1, (unsigned)nfields);
  k_rows_r2c<H><<<grid, RP::NT, SMEM, L.stream>>>(u, Uh, rows, sc, scale ? 1 : 0, L.master, bl);
  if (L.launches) *L.launches += 1;
  return true;
}

template <int H>
bool launch_rows(const LaunchCtx& L, const double2* src, long long src_ts, int m_first, int m_last,
                 const double* dev1, double* out, long long rows, int nfields, double* residue, const int* guard,
                 const BatchLine* bl, long long xrs, int resume) {
  using RP = C2RPlan<H>;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_rows_c2r<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RP::SMEM);
  });
  const dim3 grid((unsigned)((rows + RP::RPB - 1) / RP::RPB), 1, (unsigned)nfields);
  k_rows_c2r<H><<<grid, RP::NT, RP::SMEM, L.stream>>>(src, src_ts, m_first, m_last, dev1, out, rows, residue, guard,
                                                    L.master, bl, xrs > 0 ? xrs : (long long)(H + 1), resume);
  if (L.launches) *L.launches += 1;
  return true;
}

}  // namespace lines

bool launch_lines(const LaunchCtx& L, int n, int dir, const double2* src, double2* dst, const double* w,
                  long long S, long long outer, long long inner, long long src_ts, long long dst_ts, long long w_ts,
                  int nterms, int nfields, double sc, bool scale, const BatchLine* bl, const Scatter* scatter,
                  long long Sd) {
  if (Sd <= 0) Sd = S;
  switch (n) {
    case 256:
      return lines::launch_n<256>(L, dir, src, dst, w, S, outer, inner, src_ts, dst_ts, w_ts, nterms, nfields, sc,
                                  scale, bl, scatter, Sd);
    case 512:
      return lines::launch_n<512>(L, dir, src, dst, w, S, outer, inner, src_ts, dst_ts, w_ts, nterms, nfields, sc,
                                  scale, bl, scatter, Sd);
    case 1024:
      return lines::launch_n<1024>(L, dir, src, dst, w, S, outer, inner, src_ts, dst_ts, w_ts, nterms, nfields, sc,
                                   scale, bl, scatter, Sd);
    default:
      return false;
  }
}

bool launch_rows_r2c(const LaunchCtx& L, int nl, const double* u, double2* Uh, long long rows, int nfields,
                     double sc, bool scale, const BatchLine* bl) {
  switch (nl / 2) {
    case 128:
      return lines::launch_rows_r2c_t<128>(L, u, Uh, rows, nfields, sc, scale, bl);
    case 256:
      return lines::launch_rows_r2c_t<256>(L, u, Uh, rows, nfields, sc, scale, bl);
    case 512:
      return lines::launch_rows_r2c_t<512>(L, u, Uh, rows, nfields, sc, scale, bl);
    default:
      return false;
  }
}

bool launch_rows_c2r(const LaunchCtx& L, int nl, const double2* src, long long src_ts, int m_first, int m_last,
                     const double* dev1, double* out, long long rows, int nfields, double* residue, const int* guard,
                     const BatchLine* bl, long long xrs, int resume) {
  switch (nl / 2) {
    case 128:
      return lines::launch_rows<128>(L, src, src_ts, m_first, m_last, dev1, out, rows, nfields, residue, guard, bl, xrs, resume);
    case 256:
      return lines::launch_rows<256>(L, src, src_ts, m_first, m_last, dev1, out, rows, nfields, residue, guard, bl, xrs, resume);
    case 512:
      return lines::launch_rows<512>(L, src, src_ts, m_first, m_last, dev1, out, rows, nfields, residue, guard, bl, xrs, resume);
    default:
      return false;
  }
}

}  // namespace fw
