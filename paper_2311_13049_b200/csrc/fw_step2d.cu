// fw_step2d.cu — persistent, warp-specialised single-launch 2D apply / seismic step (sm_100a).
//
// One cooperative launch (one CTA per SM, 768 threads) does a whole seismic step
// (seismic.cpp:111-133: two M-term applies sharing one forward transform, plus
// the update) or one operator apply (flap.cpp:38-92) on a J0 x J1 grid
// (half spectrum H = J1/2 + 1 columns, h = J1/2).  Warp roles:
//
//   column warps 0-7 (2 groups of 4)            row warps 8-23 (8 pairs; RMAX active)
//   group g owns mirror slot b + g*gridDim:      pair p owns row r0 + p
//   columns {s, h-s} of the half spectrum        F1: R2C of its row of u -> Y (global)
//   F2: wait all rows, C2C of its 2 columns      R(t), t = (op, m) in ascending order:
//       of Y, x 1/N -> uhat in TENSOR MEMORY         wait for the TMA tile of Z[t] (mbarrier),
//   C(t), t = (op, m):                               pass 0 tile -> work, release the tile,
//       a = w_m .* uhat (TMEM), IFFT of both         passes 1-2 in place, x (s-s0)^m, accumulate
//       columns, C2R pre-processing of the pair      in TENSOR MEMORY (ascending m); operator
//       in registers -> Z[t % 6] (column-major,      done: write L1 / fused seismic update
//       global), publish (red.release)           pair RMAX: tile producer (one lane): wait for
//                                                    the columns of term t, TMA the CTA's 8 rows
//                                                    of Z[t] into the 128-B-swizzled tile
//
// Producer/consumer ordering between CTAs uses monotone counters (rows
// transformed, Z columns stored per term, rows consumed per term;
// red.release.gpu / red.relaxed.gpu / ld.acquire.gpu), two counter sets
// alternating between launches; inside a CTA named barriers (column groups,
// row pairs) and the full/empty mbarriers of the tile.  Every FFT pass is in
// place per butterfly with padded, bank-conflict-free positions.  Registers are
// split with setmaxnreg (column warps 112, row warps 64).  Arithmetic is the
// canonical FFT of fw_fft.cuh (radix plan, twiddle values, fma placement,
// pre-processing formula): results are bit-identical to the multi-pass path
// and to the CPU oracle (tests/test_gpu_parity.py).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "fw_fft.cuh"
#include "fw_internal.h"
#include "fw_step2d.h"

namespace fw {
namespace s2d {

constexpr int KRING = kStep2dRing;

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
__device__ __forceinline__ void st_release_cta_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_cta_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void red_relaxed_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Spin with acquire loads.  (Measured: relaxed polling + one acquire, with or without
// __nanosleep backoff, is 3-5 % slower for the whole step although the acquire load
// invalidates L1 (CCTL.IVALL) every iteration.)
__device__ __forceinline__ void spin_until(const unsigned long long* cnt, unsigned long long target) {
  while (ld_acquire(cnt) < target) {
  }
}
// whole warp waits until *cnt >= target
__device__ __forceinline__ void warp_wait(const unsigned long long* cnt, unsigned long long target) {
  if ((threadIdx.x & 31) == 0) spin_until(cnt, target);
  __syncwarp();
}
// the warp's prior memory accesses are done -> publish v (release is cumulative
// over the lanes ordered before it by __syncwarp)
__device__ __forceinline__ void warp_signal(unsigned long long* cnt, unsigned long long v) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) red_release_add(cnt, v);
}
// named barriers: 1, 2 = column group g (4 warps), 5 = all 8 column warps
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
// L2 residency: the streamed tables (weights, deviation powers) are read once per step and
// marked evict-first, the term ring Z (re-read a term later, rewritten 6 terms later)
// evict-last, so that most of the ring is overwritten in L2 instead of written back.
#ifndef FW_S2D_STREAM_EF
#define FW_S2D_STREAM_EF 1  // streamed tables evict-first (0: evict-normal, A/B)
#endif
__device__ __forceinline__ unsigned long long pol_evict_first() {
  unsigned long long p;
#if FW_S2D_STREAM_EF
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#else
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ unsigned long long pol_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_stream(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_stream2(const double2* p, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
#ifndef FW_S2D_ZKEEP
#define FW_S2D_ZKEEP 1  // term-ring stores with the evict-last hint (0: plain stores, A/B)
#endif
__device__ __forceinline__ void st_keep(double2* p, double2 v, unsigned long long pol) {
#if FW_S2D_ZKEEP
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
#else
  (void)pol;
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
#endif
}
__device__ __forceinline__ void prefetch_l2_hint(const void* p, unsigned bytes, unsigned long long pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned vtid() {
  unsigned x;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(x));
  return x;
}
__device__ __forceinline__ unsigned vctaid() {
  unsigned x;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(x));
  return x;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// optional instrumentation (build with -DFW_STEP2D_TRACE=1, then FW_TRACE=1 at run time):
// trace[(sel*32 + warp)*136 + t][8] = globaltimer at phase marks.  Compiled out by default:
// the address arithmetic would cost registers in the hot loops.
#ifndef FW_STEP2D_TRACE
#define FW_STEP2D_TRACE 0
#endif
// timing experiments (build with -DFW_STEP2D_EXPERIMENTS=1, select with FW_STEP2D_DBG=bits; the
// results are wrong by design): compiled out of the product kernel
#ifndef FW_STEP2D_EXPERIMENTS
#define FW_STEP2D_EXPERIMENTS 0
#endif
#define FW_DBG(bits) (FW_STEP2D_EXPERIMENTS && (prm.dbg & (bits)))
// per-thread FFT twiddles (column passes 1-2, row pass 2) held in tensor memory instead of
// being re-read from shared memory every term
#ifndef FW_S2D_TWTM
#define FW_S2D_TWTM 1
#endif
// warp roles: the SM's schedulers issue from the highest eligible warp id first, so the column
// warps (the per-term critical path) take warps 16-23 and the row warps 0-15 (0: the round-1
// layout, column warps 0-7, row warps 8-23; A/B)
#ifndef FW_S2D_COLHI
#define FW_S2D_COLHI 1
#endif
// publication of a term's Z columns (red.release.gpu on the term counter): by a publisher lane
// in an otherwise idle row warp, told through a monotone shared-memory counter per column group,
// so that the release fence's drain of the Z stores is off the column warps' critical path
// (0: the column group's first thread publishes term t-1 after pass 0 of term t; A/B)
#ifndef FW_S2D_PUBLISHER
#define FW_S2D_PUBLISHER 1
#endif
// ring-slot wait (Z[gt % KRING] consumed everywhere) by the group's first thread only, its
// acquire load overlapping the weight loads (the group barrier after pass 0 orders the other
// threads' Z stores after it); 0: every column warp waits after the weights (A/B)
#ifndef FW_S2D_RING1
#define FW_S2D_RING1 1
#endif
// the column warps take half of the step's fused update (idle otherwise at the step's tail; 0: the
// row warps do all of it; A/B)
#ifndef FW_S2D_TAILHELP
#define FW_S2D_TAILHELP 1
#endif
constexpr int kColW0 = FW_S2D_COLHI ? 16 : 0;  // first column warp
constexpr int kRowW0 = FW_S2D_COLHI ? 0 : 8;   // first row warp
// L2 promotion of the tile TMA loads (A/B)
#ifndef FW_S2D_L2PROMO
#define FW_S2D_L2PROMO CU_TENSOR_MAP_L2_PROMOTION_NONE  // measured 0.2 % faster than L2_256B
#endif
// seismic update inputs prefetched into L2 this many terms before the step's last term (0 = off)
#ifndef FW_S2D_UPF
#define FW_S2D_UPF 0
#endif
#if FW_STEP2D_TRACE
#define FW_TRACE(t, slot)                                                                            \
  do {                                                                                                 \
    if (prm.trace && (threadIdx.x & 31) == 0 && (blockIdx.x == 0 || blockIdx.x == 100))               \
      prm.trace[(((size_t)(blockIdx.x == 0 ? 0 : 1) * 32 + (threadIdx.x >> 5)) * 136 + (t)) * 8 + (slot)] = \
          gtimer();                                                                                    \
  } while (0)
#else
#define FW_TRACE(t, slot) \
  do {                    \
  } while (0)
#endif

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

// ---------------------------------------------------------------- async copies (bulk + mbarrier)
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
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* b,
                                              unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n FW_MBW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra FW_MBW_%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}

// --------------------------------------------------------------------------
// Geometry.  Column slots: slot 0 = {0, h}, slot s in [1, h/2) = {s, h-s},
// slot h/2 = {h/2}.  Column group g (warps 4g..4g+3) of CTA b owns slot
// b + g * gridDim.x and transforms both members of the pair at once.  Row pair
// p (warps 8+2p, 9+2p: 64 lanes, one radix-8 butterfly per lane and pass) owns
// row r0 + p of the CTA's rows [r0, r1).
//
// Shared-memory layouts are chosen so that every FFT pass is IN PLACE PER
// BUTTERFLY (a butterfly writes its outputs to the slots its inputs came from):
// a thread then holds one butterfly at a time, and the padding below makes every
// pass conflict-free.  Only where data lives changes; the arithmetic is the
// canonical Stockham plan of fw_fft.cuh.
template <int J0, int J1, int RMAX>
struct Geo {
  static constexpr int H = J1 / 2 + 1;
  static constexpr int h = J1 / 2;
  static constexpr int NSLOT = h / 2 + 1;
  static constexpr int NT = 768;  // 8 column warps (2 groups of 4) + 16 row warps (8 pairs)
  // column plan (J0 points, 3 passes)
  static constexpr int CR0 = radix(J0, 0), CR1 = radix(J0, 1), CR2 = radix(J0, 2);
  static constexpr int CT0 = J0 / CR0, CT1 = J0 / CR1, CT2 = J0 / CR2;
  static constexpr int CP1 = CR0;  // pprod(J0, 1)
  static constexpr int CL1 = ilog2c(CR1), CLT = ilog2c(CT1);
  // row plan (h points, 3 radix-8 passes of 64 butterflies)
  static constexpr int RR0 = radix(h, 0), RR1 = radix(h, 1), RR2 = radix(h, 2);
  static constexpr int RT = h / RR0;
  static constexpr int RP1 = RR0;
  static constexpr int RLT = ilog2c(RT);
  static constexpr int LCOL = J0 + (J0 >> CL1) + (J0 >> CLT) + 1;  // per column work buffer
  static constexpr int LROW = (h + (h >> RLT)) | 1;                // per row work buffer (odd)
  // the current term's weights of the CTA's columns, landed by bulk copy: [2 groups][2 members][J0]
  // doubles; then the C2R pre-processing twiddles of each group's pair (W_J1^kA, W_J1^kB)
  static constexpr size_t OFF_W = 0;
  static constexpr size_t OFF_TWQ = OFF_W + (size_t)2 * J0;
  static constexpr size_t OFF_CW = OFF_TWQ + 8;                    // column work [2 groups][2 members][LCOL]
  static constexpr size_t OFF_RW = OFF_CW + (size_t)4 * LCOL;      // row work [RMAX][LROW]
  // next term's 8 rows of Z: two TMA boxes [256 k][8 rows] (128-B swizzled), 1 KB aligned at run time
  static constexpr size_t OFF_TILE = OFF_RW + (size_t)RMAX * LROW;
  static constexpr size_t TILE_ELEMS = (size_t)h * 8;
  static constexpr size_t NELEM = OFF_TILE + 64 + TILE_ELEMS;
  static constexpr size_t SMEM = NELEM * sizeof(double2);
  // tensor memory: [0,128) row accumulators (16 warps x 32 columns), [128, 128 + 8 CR0) uhat
  static constexpr int TM_U = 128;
  // (FW_S2D_TWTM) [256, 368) column twiddles (2 groups x 2 passes x 28), [368, 480) row pass-2
  // twiddles (4 warps x 28), per lane quadrant
  static constexpr int TM_TWC = 256;
  static constexpr int TM_TWR = 368;
  // [480, 508) row pass-1 twiddles: lane (32 q + j) holds the set of butterfly index j & 7 (all
  // row warps of quadrant q read it)
  static constexpr int TM_TWR1 = 480;
  static constexpr int TM_COLS = 512;
  static_assert(FW_S2D_TWTM && FW_S2D_PUBLISHER, "twiddles in tensor memory; the publisher lane loads the weights");
  static_assert(TM_U + 2 * 4 * CR0 <= 256 && TM_TWR + 4 * 28 <= TM_TWR1 && TM_TWR1 + 28 <= 512, "tensor memory budget");
  static_assert(CR1 == 8 && CR2 == 8, "radix-8 column passes 1-2");
  static_assert(2 * CT0 == 128, "column pass 0: one butterfly per group thread");
  static_assert(npass(J0) == 3 && npass(h) == 3, "3-pass plans");
  static_assert(RR0 == 8 && RR1 == 8 && RR2 == 8 && RT == 64, "row pair: one radix-8 butterfly per lane");
  static_assert(SMEM + 128 <= 227 * 1024, "shared memory budget (with the static barriers)");
  static_assert(RMAX < 8, "one row pair is the tile producer and the publisher");
  static_assert(h % 256 == 0, "whole TMA boxes");

  // column layouts: pass-1 input (i, r) = logical i + CT1 r lives at i CR1 + r
  __device__ static __forceinline__ int cpad(int pos) { return pos + (pos >> CL1) + (pos >> CLT); }
  __device__ static __forceinline__ int c_p0out(int e) { return cpad((e % CT1) * CR1 + e / CT1); }
  __device__ static __forceinline__ int c_p1(int i, int r) { return cpad(i * CR1 + r); }
  __device__ static __forceinline__ int c_p2in(int e) {
    const int i = (e / (CP1 * CR1)) * CP1 + e % CP1, r = (e / CP1) % CR1;
    return cpad(i * CR1 + r);
  }
  // the padded positions of a butterfly's R elements are base + r * stride (checked exhaustively
  // for the instantiated sizes): pass-0 outputs, pass-1 and pass-2 inputs / rows
  static constexpr int CS0 = CR1 + 1, CS2 = CT2 + CT2 / CR1 + 1;
  static constexpr int RS0 = RT + 1, RS1 = 8, RS2 = 1;
  // row layouts: pass-0 input natural; passes 0 and 1 in place
  __device__ static __forceinline__ int rpad(int pos) { return pos + (pos >> RLT); }
  __device__ static __forceinline__ int r_p1raw(int e) { return e / RR0 + RT * (e % RR0); }
  __device__ static __forceinline__ int r_p1in(int e) { return rpad(r_p1raw(e)); }
  __device__ static __forceinline__ int r_p2in(int e) {
    const int i1 = (e / (RP1 * RR1)) * RP1 + e % RP1, r1 = (e / RP1) % RR1;
    return rpad(r_p1raw(i1 + RT * r1));
  }
};

__device__ __forceinline__ void tmem_ld32_nw(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16_nw(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16_nw(unsigned taddr, const unsigned* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
               :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
               : "memory");
}
__device__ __forceinline__ void tmem_ld4(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld4_nw(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st4_nw(unsigned taddr, const unsigned* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void tmem_ld8_nw(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8_nw(unsigned taddr, const unsigned* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double tm_d(const unsigned* v, int k) { return __hiloint2double((int)v[2 * k + 1], (int)v[2 * k]); }
__device__ __forceinline__ void tm_put(unsigned* v, int k, double x) {
  v[2 * k] = (unsigned)__double2loint(x);
  v[2 * k + 1] = (unsigned)__double2hiint(x);
}
// this thread's 7 twiddles of one radix-8 pass (butterfly index fixed across terms): 28 TMEM
// columns = 7 x (re, im) as pairs of 32-bit halves.  Values = the table entries, so the
// butterflies below are bit-identical to butterfly() reading shared memory.
__device__ __forceinline__ void tw_park(unsigned taddr, const double2* t) {
  unsigned v[28];
#pragma unroll
  for (int r = 0; r < 7; ++r) {
    tm_put(v, 2 * r, t[r].x);
    tm_put(v, 2 * r + 1, t[r].y);
  }
  tmem_st16_nw(taddr, v);
  tmem_st8_nw(taddr + 16, v + 16);
  tmem_st4_nw(taddr + 24, v + 24);
  tmem_wait_st();
}
// the same from the master table: the 7 twiddles of butterfly index k of a radix-8 pass with
// p = pprod (entries r k (kTwMaster / (8 p)), r = 1..7 = the per-pass table of butterfly())
__device__ __forceinline__ void tw_park_master(unsigned taddr, const double2* master, int k, int p) {
  double2 t[7];
#pragma unroll
  for (int r = 0; r < 7; ++r) t[r] = __ldg(&master[((r + 1) * k) * (kTwMaster / (8 * p))]);
  tw_park(taddr, t);
}
template <int DIR>
__device__ __forceinline__ void tw_load(unsigned taddr, double2 (&w)[7]) {
  unsigned v[28];
  tmem_ld16_nw(taddr, v);
  tmem_ld8_nw(taddr + 16, v + 16);
  tmem_ld4_nw(taddr + 24, v + 24);
  tmem_wait_ld();
#pragma unroll
  for (int r = 0; r < 7; ++r) w[r] = dirw<DIR>(make_double2(tm_d(v, 2 * r), tm_d(v, 2 * r + 1)));
}
// the same, twiddles applied in two halves (row warps run at 64 registers)
template <int DIR>
__device__ __forceinline__ void butterfly_tm8_lean(double2* a, unsigned taddr) {
  {
    unsigned v[16];
    tmem_ld16_nw(taddr, v);
    tmem_wait_ld();
#pragma unroll
    for (int r = 1; r <= 4; ++r) {
      const double2 w = dirw<DIR>(make_double2(tm_d(v, 2 * (r - 1)), tm_d(v, 2 * (r - 1) + 1)));
      a[r] = cmulw(a[r], w.x, w.y);
    }
  }
  {
    unsigned v[12];
    tmem_ld8_nw(taddr + 16, v);
    tmem_ld4_nw(taddr + 24, v + 8);
    tmem_wait_ld();
#pragma unroll
    for (int r = 5; r <= 7; ++r) {
      const double2 w = dirw<DIR>(make_double2(tm_d(v, 2 * (r - 5)), tm_d(v, 2 * (r - 5) + 1)));
      a[r] = cmulw(a[r], w.x, w.y);
    }
  }
  Dft<8, DIR>::run(a);
}
template <int DIR>
__device__ __forceinline__ void butterfly_w8(double2* a, const double2 (&w)[7]) {
#pragma unroll
  for (int r = 1; r < 8; ++r) a[r] = cmulw(a[r], w[r - 1].x, w[r - 1].y);
  Dft<8, DIR>::run(a);
}
__device__ __forceinline__ void pairbar(int p) { asm volatile("bar.sync %0, 64;" ::"r"(4 + p) : "memory"); }

// ---------------------------------------------------------------- column group: 2 x J0-point C2C
// 128 threads (cg), both members of a mirror pair.  Pass 0 takes each thread's CR0
// inputs in registers (member cg / CT0, butterfly cg % CT0, element q = cg % CT0 + r CT0);
// passes 1 and 2 run one butterfly at a time in place; pass 2 hands the natural-order
// outputs q = i + r CT2 of both members to epilogue(i, X0[], X1[]).
template <class G, int DIR, class GBar, class Hook, class Epi, class Mark>
__device__ __forceinline__ void column_pair(double2* work, const double2* tw, unsigned ttw, int cg,
                                            double2 (&a)[G::CR0], GBar gbar, Hook after_pass0, Epi epilogue,
                                            Mark mark) {
  constexpr int J0 = G::CT0 * G::CR0;
  {
    const int mbr = cg / G::CT0, I = cg % G::CT0;
    Dft<G::CR0, DIR>::run(a);
    double2* wb = work + mbr * G::LCOL;
#pragma unroll
    for (int r = 0; r < G::CR0; ++r) wb[G::c_p0out(I * G::CR0) + r * G::CS0] = a[r];
  }
  gbar();
  mark(3);
  after_pass0();
  static_assert(!FW_S2D_TWTM || (G::CT1 <= 128 && G::CT2 <= 128), "one butterfly per thread and pass");
#pragma unroll 1
  for (int i = cg; i < G::CT1; i += 128) {  // butterfly i of both members (same twiddles)
    double2 c0[G::CR1], c1[G::CR1];
#pragma unroll
    for (int r = 0; r < G::CR1; ++r) {
      c0[r] = work[G::c_p1(i, 0) + r];
      c1[r] = work[G::LCOL + G::c_p1(i, 0) + r];
    }
    if (FW_S2D_TWTM) {  // i == cg: the thread's parked pass-1 twiddles
      double2 w[7];
      tw_load<DIR>(ttw, w);
      butterfly_w8<DIR>(c0, w);
      butterfly_w8<DIR>(c1, w);
    } else {
      butterfly<J0, 1, DIR>(c0, i, tw);
      butterfly<J0, 1, DIR>(c1, i, tw);
    }
#pragma unroll
    for (int r = 0; r < G::CR1; ++r) {
      work[G::c_p1(i, 0) + r] = c0[r];
      work[G::LCOL + G::c_p1(i, 0) + r] = c1[r];
    }
  }
  gbar();
  mark(4);
#pragma unroll 1
  for (int i = cg; i < G::CT2; i += 128) {
    double2 c0[G::CR2], c1[G::CR2];
#pragma unroll
    for (int r = 0; r < G::CR2; ++r) {
      const int p = G::c_p2in(i) + r * G::CS2;
      c0[r] = work[p];
      c1[r] = work[G::LCOL + p];
    }
    if (FW_S2D_TWTM) {
      double2 w[7];
      tw_load<DIR>(ttw + 28, w);
      butterfly_w8<DIR>(c0, w);
      butterfly_w8<DIR>(c1, w);
    } else {
      butterfly<J0, 2, DIR>(c0, i, tw);
      butterfly<J0, 2, DIR>(c1, i, tw);
    }
    epilogue(i, c0, c1);
  }
}

// ---------------------------------------------------------------- row pair: h-point C2C
// passes 0 and 1 in place (pass-0 input in natural order, padded); returns after the
// pair barrier that follows pass 1.  Lane l (0..63) owns butterfly l of every pass.
template <class G, int DIR>
__device__ __forceinline__ void row_passes01(double2* work, unsigned ttw1, int l, int pair) {
  {
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = work[G::rpad(l) + r * G::RS0];
    Dft<8, DIR>::run(a);
#pragma unroll
    for (int r = 0; r < 8; ++r) work[G::rpad(l) + r * G::RS0] = a[r];
  }
  pairbar(pair);
  {
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = work[G::r_p1in(l) + r * G::RS1];
    butterfly_tm8_lean<DIR>(a, ttw1);
#pragma unroll
    for (int r = 0; r < 8; ++r) work[G::r_p1in(l) + r * G::RS1] = a[r];
  }
  pairbar(pair);
}

// ---------------------------------------------------------------- fused seismic update
// (seismic.cpp:116-129) of outputs q = l + 64 r, r in [rb, re), of NW row warps at once (their
// loads in flight together); the L2 sums come from each row warp's tensor-memory accumulators
// (lane quadrant of the calling warp).  Returns this lane's blow-up test.
template <class G, int NW>
__device__ __forceinline__ bool seis_update_part(const Step2DParams& prm, int s, const int (&row)[NW],
                                                 const int (&l)[NW], const unsigned (&tacc)[NW],
                                                 const bool (&on)[NW], int rb, int re, bool frozen) {
  constexpr int J1 = 2 * G::h;
  const double tau = prm.tau;
  const double t2 = tau * tau;
  const bool ms = prm.nsteps > 1;
  const double* ucur = ms ? prm.ub[(int)((prm.lvl0 + s) % 3)] : prm.u;
  const double* uprev = ms ? prm.ub[(int)((prm.lvl0 + s + 2) % 3)] : prm.prev;
  const double* aprev = ms ? prm.ab[(int)((prm.lvl0 + s + 1) % 2)] : prm.ap;
  double* unext = ms ? prm.ub[(int)((prm.lvl0 + s + 1) % 3)] : prm.next;
  double* aout = ms ? prm.ab[(int)((prm.lvl0 + s) % 2)] : prm.out[1];
  bool bad = false;
#pragma unroll 1
  for (int r = rb; r < re; ++r) {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      if (!on[w]) continue;  // warp-uniform
      unsigned v[4];
      tmem_ld4(tacc[w] + 4u * r, v);
      const size_t rowoff = (size_t)row[w] * J1;
      const int q = l[w] + r * G::RT;
      const double2 vc = reinterpret_cast<const double2*>(ucur + rowoff)[q];
      const double2 vp = reinterpret_cast<const double2*>(uprev + rowoff)[q];
      const double2 va = reinterpret_cast<const double2*>(aprev + rowoff)[q];
      const double2 v1 = reinterpret_cast<const double2*>(prm.out[0] + rowoff)[q];
      const double2 cc = reinterpret_cast<const double2*>(prm.c + rowoff)[q];
      const double2 ve = reinterpret_cast<const double2*>(prm.eta + rowoff)[q];
      const double2 vt = reinterpret_cast<const double2*>(prm.tc + rowoff)[q];
      const double l2x = tm_d(v, 0), l2y = tm_d(v, 1);
      const double c2x = cc.x * cc.x, c2y = cc.y * cc.y;
      const double nx0 = 2.0 * vc.x - vp.x + t2 * c2x * (ve.x * v1.x + vt.x * (l2x - va.x) / tau);
      const double nx1 = 2.0 * vc.y - vp.y + t2 * c2y * (ve.y * v1.y + vt.y * (l2y - va.y) / tau);
      if (!frozen) {
        reinterpret_cast<double2*>(unext + rowoff)[q] = make_double2(nx0, nx1);
        reinterpret_cast<double2*>(aout + rowoff)[q] = make_double2(l2x, l2y);
      }
      bad |= (fabs(nx0) > prm.thr) || (fabs(nx1) > prm.thr);
    }
  }
  return bad;
}
// the step's tail: the active row warps and the active column groups' warps meet on named
// barrier 12 before and after the fused update (the column warps take outputs r = 4..7 of the
// row warps of their lane quadrant, see k_step2d)
__device__ __forceinline__ void tailbar(int nthreads) { asm volatile("bar.sync 12, %0;" ::"r"(nthreads) : "memory"); }

// --------------------------------------------------------------------------
template <int J0, int J1, int RMAX>
__global__ void __launch_bounds__(768, 1) k_step2d(const Step2DParams prm, const __grid_constant__ CUtensorMap zmap) {
  using G = Geo<J0, J1, RMAX>;
  constexpr int H = G::H, h = G::h, NT = G::NT;
  constexpr int CR0 = G::CR0, CT0 = G::CT0;
  extern __shared__ __align__(16) double2 sm[];
  __shared__ unsigned tmem_base_sh;
  __shared__ __align__(8) unsigned long long tile_full, tile_empty;  // row tile pipeline (TMA producer)
  __shared__ unsigned zdone[2];  // terms of the launch whose Z stores group g has issued (-> publisher)
  __shared__ unsigned ringok;    // terms of the launch whose ring slot is free (<- loader)
  __shared__ __align__(8) unsigned long long wfull[2], wempty[2];  // weights of group g (bulk copy)
  double2* twq = sm + G::OFF_TWQ;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.x;
  const int nblk = gridDim.x;

  // launch marks (tracing only): warp slot 31 of the trace, [step % 64][entry, exit]
  auto launch_mark = [&](int which) {
    if (FW_STEP2D_TRACE && prm.trace && tid == 0 && (b == 0 || b == 100))
      prm.trace[((size_t)(b == 0 ? 0 : 1) * 32 + 31) * 136 * 8 + (size_t)(prm.step & 63) * 2 + which] = gtimer();
  };
  launch_mark(0);
  unsigned long long* cnt = prm.counters + (size_t)prm.cset * prm.cstride;
  if (b == 0) {
    unsigned long long* other = prm.counters + (size_t)(prm.cset ^ 1) * prm.cstride;
    for (int e = tid; e < prm.cstride; e += NT) other[e] = 0ull;
  }
  if (prm.flag && *prm.flag != kNoBlowup) return;  // uniform across CTAs
  unsigned long long* cY = cnt;                          // rows forward-transformed
  unsigned long long* cC = cnt + 1;                      // Z columns of term t stored
  unsigned long long* cR = cnt + 1 + prm.nterms_total;  // rows of Z[t] consumed

  // FFT twiddles live in tensor memory (parked below, values = the master entries, identical to
  // fw_fft.cuh's twiddle()); shared memory keeps only the pre-processing twiddles of the pairs
  if (tid < 2) {
    const int sl = b + tid * nblk;
    const int kA = sl == 0 ? 0 : sl;
    const int kB = sl == 0 ? h : h - sl;
    twq[2 * tid] = sl < G::NSLOT ? prm.master[kA * (kTwMaster / J1)] : make_double2(0.0, 0.0);
    twq[2 * tid + 1] = sl < G::NSLOT ? prm.master[kB * (kTwMaster / J1)] : make_double2(0.0, 0.0);
    zdone[tid] = 0u;
  }
  if (tid == 0) {
    ringok = (unsigned)KRING;
    for (int g = 0; g < 2; ++g) {
      mbar_init(&wfull[g], 1);
      mbar_init(&wempty[g], 4);  // one arrive per column warp of the group
    }
    const int nr0 = (int)(((long long)(b + 1) * J0) / nblk) - (int)(((long long)b * J0) / nblk);
    mbar_init(&tile_full, 1);
    mbar_init(&tile_empty, 2 * nr0);  // one arrive per consumer warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tmem_base_sh)),
                 "n"(G::TM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem_base = tmem_base_sh;
  if (warp >= kRowW0 && warp < kRowW0 + 4)  // one row warp per lane quadrant: row pass-1 twiddles
    tw_park_master(tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)G::TM_TWR1, prm.master,
                   lane & (pprod(h, 1) - 1), pprod(h, 1));
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  const int M = prm.M;
  const int nterms = M + 1 - prm.m_first;
  const int ntot = prm.nops * nterms;

  if (warp >= kColW0 && warp < kColW0 + 8) {
    // ============================================ column warps (2 groups of 4)
    setmaxnreg_inc<112>();
    const int g = (warp - kColW0) >> 2;  // group
    const int cg = tid & 127;  // thread within the group
    const int slot = b + g * nblk;
    const int mbr = cg / CT0, i0 = cg % CT0;
    auto colno = [&](int m_) {
      if (slot >= G::NSLOT) return -1;
      if (slot == 0) return m_ ? h : 0;
      if (slot == h / 2) return m_ ? -1 : h / 2;
      return m_ ? h - slot : slot;
    };
    if (slot < G::NSLOT) {
      double2* work = sm + G::OFF_CW + (size_t)g * 2 * G::LCOL;  // members at +0, +LCOL
      auto gb = [g] { groupbar(g); };
      const int mycol = colno(mbr);
      const int kA = colno(0), kB = colno(1);
      int nz = 0;
      if (kA >= 0 && kA < h) ++nz;
      if (kB >= 0 && kB < h) ++nz;  // column h feeds Z_0 and produces no Z of its own
      // this thread's uhat values: TMEM lane (32 (warp & 3) + lane), columns TM_U + g 4 CR0 + [0, 4 CR0)
      const unsigned tu = tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)(G::TM_U + g * 4 * CR0);
      // this thread's pass-1 / pass-2 twiddles (butterfly index cg in both passes) -> TMEM
      const unsigned ttw = tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)(G::TM_TWC + g * 56);
      tw_park_master(ttw, prm.master, cg & (pprod(J0, 1) - 1), pprod(J0, 1));
      tw_park_master(ttw + 28, prm.master, cg & (pprod(J0, 2) - 1), pprod(J0, 2));

      double rmax = 0.0;
#pragma unroll 1
      for (int s = 0; s < prm.nsteps; ++s) {  // launch steps (counters are cumulative over them)
      // ---- F2: forward columns -> uhat (pass 0 straight from Y) -> tensor memory
      FW_TRACE(135, 0);
      warp_wait(cY, (unsigned long long)(s + 1) * J0);
      FW_TRACE(135, 1);
      gb();  // every thread of the group has seen all rows
      {
        double2 a[CR0];
#pragma unroll
        for (int r = 0; r < CR0; ++r)
          a[r] = mycol >= 0 ? __ldcg(&prm.Y[(size_t)mycol * J0 + i0 + r * CT0]) : make_double2(0.0, 0.0);
        double2 x0[G::CR2], x1[G::CR2];
        int ix = 0;
        column_pair<G, -1>(
            work, nullptr, ttw, cg, a, gb, [] {},
            [&](int i, const double2* c0, const double2* c1) {
              ix = i;
#pragma unroll
              for (int r = 0; r < G::CR2; ++r) {
                x0[r] = c0[r];
                x1[r] = c1[r];
              }
            },
            [](int) {});
        FW_TRACE(135, 3);
        gb();  // pass-2 reads done: the buffers may take the natural-order result
        if (cg < G::CT2) {
#pragma unroll
          for (int r = 0; r < G::CR2; ++r) {
            work[ix + r * G::CT2] = x0[r];
            work[G::LCOL + ix + r * G::CT2] = x1[r];
          }
        }
        gb();
        const double inv = 1.0 / ((double)J0 * (double)J1);
#pragma unroll
        for (int c = 0; c < 4 * CR0; c += 32) {
          unsigned v[32];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const double2 x = work[mbr * G::LCOL + i0 + (c / 4 + k) * CT0];
            tm_put(v, 2 * k, x.x * inv);
            tm_put(v, 2 * k + 1, x.y * inv);
          }
          tmem_st32(tu + c, v);
        }
        gb();
      }
      FW_TRACE(135, 2);

      // ---- C(t): inverse columns -> pre-processed Z[gt % KRING] (gt = s ntot + t), column-major Z[k][k0]
      for (int t = 0; t < ntot; ++t) {
        // per-thread constants re-derived from the special registers each term (volatile reads
        // are not hoisted): fewer live registers across the FFT passes
        const int tidc = (int)vtid();
        const int g_ = (tidc >> 7) - kColW0 / 4, cg_ = tidc & 127;
        const int slot_ = (int)vctaid() + g_ * nblk;
        const int i0_ = cg_ % CT0;
        const int kA_ = slot_ == 0 ? 0 : slot_;
        const int kB_ = slot_ == 0 ? h : (slot_ == h / 2 ? -1 : h - slot_);
        const int mycol_ = (cg_ / CT0) ? kB_ : kA_;
        const int nz_ = (kA_ < h) + (kB_ >= 0 && kB_ < h);
        double2* work_ = sm + G::OFF_CW + (size_t)g_ * 2 * G::LCOL;
        const unsigned tu_ = tmem_base + ((unsigned)(32 * ((tidc >> 5) & 3)) << 16) + (unsigned)(G::TM_U + g_ * 4 * CR0);
        auto gb_ = [g_] { groupbar(g_); };
        FW_TRACE(t, 0);
        const int op = t / nterms, m = prm.m_first + t % nterms;
        (void)op;
        (void)m;
        double2 a[CR0];
        const int gt = s * ntot + t;  // term index over the launch
        {
          // this term's weights of the group's columns, landed in shared memory by the loader lane
          mbar_wait(&wfull[g_], (unsigned)gt & 1u);
          const double* ws = reinterpret_cast<const double*>(sm + G::OFF_W) + (size_t)(2 * g_ + cg_ / CT0) * J0 + i0_;
          double wk[CR0];
#pragma unroll
          for (int r = 0; r < CR0; ++r) wk[r] = (mycol_ >= 0 && !FW_DBG(2)) ? ws[r * CT0] : 0.5;
          __syncwarp();
          if ((tidc & 31) == 0) mbar_arrive(&wempty[g_]);  // the buffer may take the next term's weights
#pragma unroll
          for (int c = 0; c < 4 * CR0; c += 32) {
            unsigned v[32];
            tmem_ld32_nw(tu_ + c, v);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 8; ++k)
              a[c / 4 + k] = make_double2(wk[c / 4 + k] * tm_d(v, 2 * k), wk[c / 4 + k] * tm_d(v, 2 * k + 1));
          }
        }
        FW_TRACE(t, 1);
        // ring slot gt % KRING free (rows of term gt - KRING consumed everywhere; the loader lane
        // polls the global counter): the group's first thread, ordered before every Z store of the
        // term by the group barrier after pass 0  (128: timing experiment without the ring wait)
        if (cg_ == 0 && !FW_DBG(128))
          while (ld_acquire_cta_u32(&ringok) <= (unsigned)gt) {
          }
        // the warp reconverges here: the group barriers below are bar.sync (.aligned), which a
        // diverged warp must not reach (measured with the DBG 32 timing build: lanes 1-31 arriving
        // while lane 0 still spun let the group pass without it)
        __syncwarp();
        FW_TRACE(t, 2);
#if FW_STEP2D_TRACE
        if (prm.trace && cg_ == 0 && vctaid() < 160)
          prm.trace[2 * 32 * 136 * 8 + 160 * 2 * 136 + ((size_t)vctaid() * 2 + g_) * 136 + t] = gtimer();
#endif
        double2* Z = prm.T + (size_t)(gt % KRING) * J0 * h;
        // the previous term's Z columns are published once this term's pass 0 is done:
        // by then its stores have drained and the release fence is cheap
        if (FW_DBG(8)) Z = prm.T + (size_t)(KRING - 1) * J0 * h;  // all terms into one slot
        if (FW_DBG(32)) {  // timing experiment: columns skip the FFT
          gb_();
          if (FW_S2D_PUBLISHER) {
            if (cg_ == 0) st_release_cta_u32(&zdone[g_], (unsigned)gt + 1u);
          } else if (cg_ == 0 && t > 0) {
            red_release_add(&cC[t - 1], (unsigned long long)nz_);
          }
          continue;
        }
        const unsigned ttw_ = tmem_base + ((unsigned)(32 * ((tidc >> 5) & 3)) << 16) + (unsigned)(G::TM_TWC + g_ * 56);
        column_pair<G, +1>(work_, nullptr, ttw_, cg_, a, gb_, [&] {
          if (!FW_S2D_PUBLISHER && cg_ == 0 && t > 0) {
            if (FW_DBG(64))
              red_relaxed_add(&cC[t - 1], (unsigned long long)nz_);  // timing: publication without the fence
            else
              red_release_add(&cC[t - 1], (unsigned long long)nz_);
          }
        }, [&](int i, const double2* xa, const double2* xb) {
#pragma unroll
          for (int r = 0; r < G::CR2; ++r) {
            const int k0 = i + r * G::CT2;
            if (kA_ == 0) {  // Z_0 from X_0 and X_h (member 1 = column h has no Z of its own)
              if (prm.residue) rmax = fmax(rmax, fabs(xa[r].y) + fabs(xb[r].y));
              st_keep(&Z[k0], pre_c2r(xa[r], xb[r], true, twq[2 * g_]), pol_evict_last());
            } else if (kA_ == h / 2) {
              st_keep(&Z[(size_t)kA_ * J0 + k0], pre_c2r(xa[r], xa[r], false, twq[2 * g_]), pol_evict_last());
            } else {
              st_keep(&Z[(size_t)kA_ * J0 + k0], pre_c2r(xa[r], xb[r], false, twq[2 * g_]), pol_evict_last());
              st_keep(&Z[(size_t)kB_ * J0 + k0], pre_c2r(xb[r], xa[r], false, twq[2 * g_ + 1]), pol_evict_last());
            }
          }
        }, [&](int sl) { FW_TRACE(t, sl); });
        FW_TRACE(t, 5);
        gb_();  // work_ buffers free again; all Z stores of the group issued
        if (FW_S2D_PUBLISHER && cg_ == 0) st_release_cta_u32(&zdone[g_], (unsigned)gt + 1u);  // -> publisher
        FW_TRACE(t, 6);
#if FW_STEP2D_TRACE
        if (prm.trace && cg_ == 0 && vctaid() < 160)
          prm.trace[2 * 32 * 136 * 8 + ((size_t)vctaid() * 2 + g_) * 136 + t] = gtimer();
#endif
      }
      if (!FW_S2D_PUBLISHER && cg == 0 && ntot > 0) red_release_add(&cC[ntot - 1], (unsigned long long)nz);
      if (FW_S2D_TAILHELP && prm.seismic) {
        // help with the step's update: outputs r = 4..7 of row warps q + 8g and q + 8g + 4 (lane
        // quadrant q = this warp's), whose accumulators this warp can read from tensor memory
        const int nrow = (int)(((long long)(b + 1) * J0) / nblk) - (int)(((long long)b * J0) / nblk);
        const int ngrp = 1 + (b + nblk < G::NSLOT);
        const int q = warp & 3;
        int rowv[2], lv[2];
        unsigned tav[2];
        bool onv[2];
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const int rw = q + 8 * g + 4 * w;
          onv[w] = rw < 2 * nrow;
          rowv[w] = (int)(((long long)b * J0) / nblk) + (rw >> 1);
          lv[w] = (rw & 1) * 32 + lane;
          tav[w] = tmem_base + ((unsigned)(32 * q) << 16) + 32u * (unsigned)(rw >> 2);
        }
        tailbar((2 * nrow + 4 * ngrp) * 32);
        const bool frozen = s > 0 && *reinterpret_cast<volatile int*>(prm.flag) < prm.step + s;
        const bool bad = seis_update_part<G, 2>(prm, s, rowv, lv, tav, onv, 4, 8, frozen);
        if (__any_sync(0xffffffffu, bad) && lane == 0 && !FW_DBG(-1)) atomicMin(prm.flag, prm.step + s);
        tailbar((2 * nrow + 4 * ngrp) * 32);
      }
      }  // steps
      if (prm.residue && rmax > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(prm.residue),
                  (unsigned long long)__double_as_longlong(rmax));
    }
  } else {
    // ============================================ row warps (8 pairs)
    setmaxnreg_dec<64>();
    const int rw = warp - kRowW0;
    const int pair = rw >> 1;
    const int l = (rw & 1) * 32 + lane;  // lane within the pair = butterfly index
    const int r0 = (int)(((long long)b * J0) / nblk);
    const int r1 = (int)(((long long)(b + 1) * J0) / nblk);
    const int nr = r1 - r0;
    const bool active = pair < nr;
    const int row = r0 + (active ? pair : 0);
    // this warp's 32 TMEM columns in its lane quadrant: (s-s0)^m-weighted sums of outputs l + 64 r
    const unsigned tacc = tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + 32u * (unsigned)(rw >> 2);
    // this lane's pass-2 twiddles (butterfly index l) -> TMEM, once per launch; pass-1 twiddles
    // were parked per lane quadrant before the role split
    const unsigned ttw2 = tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)(G::TM_TWR + 28 * (rw >> 2));
    const unsigned ttw1 = tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)G::TM_TWR1;
    tw_park_master(ttw2, prm.master, l & (pprod(h, 2) - 1), pprod(h, 2));
    double2* work = sm + G::OFF_RW + (size_t)(active ? pair : 0) * G::LROW;
    // the tile: rows r0..r0+7 of Z[t] as two [256 k][8 rows] TMA boxes, 128-B swizzled
    double2* tile;
    {
      const unsigned base = smem_u32(sm + G::OFF_TILE);
      tile = sm + G::OFF_TILE + (((base + 1023u) & ~1023u) - base) / 16u;
    }
    // element k = l + 64 r of row slot rs: chunk (rs ^ (k & 7)) of the 128-B line of k
    auto tile_at = [&](int l_, int rs, int r) -> const double2& {
      return tile[l_ * 8 + (rs ^ (l_ & 7)) + r * 64 * 8];
    };
    // (s-s0)^m row of term t: global (streamed once), L2-prefetched one term ahead
    auto dev_row = [&](int t, int row) -> const double2* {
      const int op1 = t / nterms, m1 = prm.m_first + t % nterms;
      return m1 < 1 ? nullptr
                    : reinterpret_cast<const double2*>(prm.dev[op1] + (size_t)(m1 - 1) * J0 * J1 + (size_t)row * J1);
    };

    if (rw == 2 * RMAX) {
      // ---- tile producer (one lane of an otherwise idle warp): Z[t] -> tile by TMA as soon as
      // the columns of term t are published and the consumers are done with tile t-1
      if (lane == 0) {
        const int gtot = prm.nsteps * ntot;
        for (int gt = 0; gt < gtot; ++gt) {  // term index over the launch's steps
          const int t = gt % ntot;
          // term t's columns first (its latency overlaps the consumers' pass 0 of the previous term)
          FW_TRACE(t, 0);
          spin_until(&cC[t], (unsigned long long)(gt / ntot + 1) * h);
          FW_TRACE(t, 1);
          if (gt > 0) {
            mbar_wait(&tile_empty, (unsigned)(gt - 1) & 1u);
            FW_TRACE(t, 2);
            // the CTA's rows of the previous term are consumed (in shared memory / registers):
            // the ring slot may be reused.  No release fence needed.
            red_relaxed_add(&cR[(gt - 1) % ntot], (unsigned long long)nr);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy Z stores -> TMA reads
          if (!FW_DBG(4)) {
            mbar_expect_tx(&tile_full, (unsigned)(G::TILE_ELEMS * sizeof(double2)));
            for (int bx = 0; bx < h / 256; ++bx)
              tma_load_3d(tile + (size_t)bx * 256 * 8, &zmap, 2 * r0, bx * 256, gt % KRING, &tile_full);
            FW_TRACE(t, 3);
          } else {
            mbar_arrive(&tile_full);
          }
        }
        if (gtot > 0) {
          mbar_wait(&tile_empty, (unsigned)(gtot - 1) & 1u);
          red_relaxed_add(&cR[ntot - 1], (unsigned long long)nr);
        }
      }
      __syncwarp();  // reconverge before the kernel's final (aligned) barrier
    }

    if (rw == 2 * RMAX + 1 && lane == 0) {
      // ---- loader + publisher (one lane of the other idle warp), one event loop over the
      // launch's terms gt:
      //  * weights: as soon as group g's column warps have read term gt-1's weights (wempty), the
      //    bulk copies of term gt's weights of its two columns land in shared memory (wfull);
      //  * ring: once the columns have started term gt-1, poll the global "rows of term gt-KRING
      //    consumed" counter and post ring slot gt as free (ringok, st.release.cta);
      //  * publication: term gt's Z columns of this CTA are stored once every active group has
      //    counted it in zdone (st.release.cta after the group barrier that follows its Z stores);
      //    one red.release.gpu makes them visible to every tile producer (cumulative over the
      //    groups' stores: they precede the release in causality order).  The release fence's
      //    drain is off the column warps' critical path.
      int ng = 0;
      unsigned long long nzs = 0;
      int colA[2] = {-1, -1}, colB[2] = {-1, -1};
      unsigned bytes[2] = {0u, 0u};
      for (int g = 0; g < 2; ++g) {
        const int sl = b + g * nblk;
        if (sl >= G::NSLOT) continue;
        ++ng;
        colA[g] = sl == 0 ? 0 : sl;
        colB[g] = sl == 0 ? h : (sl == h / 2 ? -1 : h - sl);
        nzs += (unsigned long long)((colA[g] < h) + (colB[g] >= 0 && colB[g] < h));
        bytes[g] = (unsigned)((colA[g] >= 0) + (colB[g] >= 0)) * (unsigned)(J0 * sizeof(double));
      }
      const unsigned long long pol = pol_evict_first();
      auto issue = [&](int g, int gt) {
        const int t = gt % ntot;
        const int op = t / nterms, m = prm.m_first + t % nterms;
        double* dst = reinterpret_cast<double*>(sm + G::OFF_W) + (size_t)(2 * g) * J0;
        const double* src = prm.w[op] + (size_t)m * prm.wcols * J0;
        mbar_expect_tx(&wfull[g], bytes[g]);
        if (colA[g] >= 0) bulk_g2s_hint(dst, src + (size_t)colA[g] * J0, J0 * sizeof(double), &wfull[g], pol);
        if (colB[g] >= 0) bulk_g2s_hint(dst + J0, src + (size_t)colB[g] * J0, J0 * sizeof(double), &wfull[g], pol);
      };
      const int gtot = prm.nsteps * ntot;
      int nl[2] = {1, 1};
      if (gtot > 0)
        for (int g = 0; g < ng; ++g) issue(g, 0);
      int np = 0, nr = KRING;
      while (np < gtot) {
        int nlmin = gtot;
        for (int g = 0; g < ng; ++g) {
          if (nl[g] < gtot && mbar_test(&wempty[g], (unsigned)(nl[g] - 1) & 1u)) {
            issue(g, nl[g]);
            ++nl[g];
          }
          nlmin = min(nlmin, nl[g]);
        }
        if (nr < gtot && nr <= nlmin &&
            ld_acquire(&cR[(nr - KRING) % ntot]) >= (unsigned long long)((nr - KRING) / ntot + 1) * J0) {
          st_release_cta_u32(&ringok, (unsigned)nr + 1u);
          ++nr;
        }
        bool done = true;
        for (int g = 0; g < ng; ++g) done = done && ld_acquire_cta_u32(&zdone[g]) > (unsigned)np;
        if (done) {
          red_release_add(&cC[np % ntot], nzs);
          ++np;
        }
      }
    }
    if (rw == 2 * RMAX + 1) __syncwarp();  // the loader's warp reconverges before the final barrier

    // this step's state buffers (multi-step launches rotate them with the level)
    auto lvl_u = [&](int s, int d) -> double* { return prm.ub[(int)((prm.lvl0 + s + d) % 3)]; };
    auto lvl_a = [&](int s, int d) -> double* { return prm.ab[(int)((prm.lvl0 + s + d) % 2)]; };
#pragma unroll 1
    for (int s = 0; active && s < prm.nsteps; ++s) {
    {
      FW_TRACE(135, 0);
      // ---- F1: R2C of the row -> Y
      const double2* u2 = reinterpret_cast<const double2*>(prm.nsteps > 1 ? lvl_u(s, 0) : prm.u) + (size_t)row * h;
#pragma unroll
      for (int r = 0; r < 8; ++r) work[G::rpad(l) + r * G::RS0] = u2[l + r * G::RT];
      pairbar(pair);
      row_passes01<G, -1>(work, ttw1, l, pair);
      double2 a[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) a[r] = work[G::r_p2in(l) + r * G::RS2];
      butterfly_tm8_lean<-1>(a, ttw2);
      pairbar(pair);
#pragma unroll
      for (int r = 0; r < 8; ++r) work[G::rpad(l) + r * G::RS0] = a[r];
      pairbar(pair);
      // Y is stored column-major, Y[k][k0] (the forward column pass reads each column contiguously)
      double2* Yc = prm.Y + row;
#pragma unroll
      for (int it = 0; it < h / 128 + 1; ++it) {
        const int jj = l + 64 * it;
        if (jj > h / 2) break;
        if (jj == 0) {
          const double2 z0 = work[0];
          __stcg(&Yc[0], make_double2(z0.x + z0.y, 0.0));
          __stcg(&Yc[(size_t)h * J0], make_double2(z0.x - z0.y, 0.0));
        } else {
          const double2 wa = __ldg(&prm.master[jj * (kTwMaster / J1)]);
          const double2 wb = __ldg(&prm.master[(h - jj) * (kTwMaster / J1)]);
          const double2 A = work[G::rpad(jj)];
          const double2 B = work[G::rpad(h - jj)];
          __stcg(&Yc[(size_t)jj * J0], post_r2c(A, B, wa));
          if (jj != h - jj) __stcg(&Yc[(size_t)(h - jj) * J0], post_r2c(B, A, wb));
        }
      }
      pairbar(pair);  // both warps' Y stores precede the signal
      if (!(rw & 1)) warp_signal(cY, 1ull);
      FW_TRACE(135, 1);
      unsigned z[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) z[e] = 0u;
      tmem_st32(tacc, z);
    }

    // ---- R(t): h-point C2C of the pre-processed row + recombination
    for (int t = 0; t < ntot; ++t) {
      // per-thread constants re-derived from the special registers each term (volatile reads
      // are not hoisted): cheaper than keeping them live, the row warps run at 64 registers
      const int tidr = (int)vtid();
      const int rw_ = (tidr >> 5) - kRowW0, pair_ = rw_ >> 1, l_ = (rw_ & 1) * 32 + (tidr & 31);
      const int row_ = (int)(((long long)vctaid() * J0) / nblk) + pair_;
      double2* work_ = sm + G::OFF_RW + (size_t)pair_ * G::LROW;
      const unsigned tacc_ = tmem_base + ((unsigned)(32 * ((tidr >> 5) & 3)) << 16) + 32u * (unsigned)(rw_ >> 2);
      const int op = t / nterms;
      const int m = prm.m_first + t % nterms;
      FW_TRACE(t, 0);
      if (l_ == 0 && t + 1 < ntot) {  // the next term's (s-s0)^m row_ -> L2
        const double2* d = dev_row(t + 1, row_);
        if (d) prefetch_l2_hint(d, J1 * sizeof(double), pol_evict_first());
      }
      if (FW_S2D_UPF > 0 && prm.seismic && t == ntot - FW_S2D_UPF && l_ >= 1 && l_ <= 7) {
        // the update's seven input rows (seismic.cpp:116-129) -> L2 while the last terms run:
        // the update sits on the step's critical path and is otherwise HBM-latency bound
        const bool ms = prm.nsteps > 1;
        const double* src[7] = {ms ? lvl_u(s, 0) : prm.u, ms ? lvl_u(s, 2) : prm.prev, ms ? lvl_a(s, 1) : prm.ap,
                                prm.out[0], prm.c, prm.eta, prm.tc};
        prefetch_l2(src[l_ - 1] + (size_t)row_ * J1, J1 * sizeof(double));
      }
      mbar_wait(&tile_full, (unsigned)(s * ntot + t) & 1u);
      FW_TRACE(t, 2);
      {  // pass 0 (p = 1): tile -> work_ (natural positions)
        double2 a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = tile_at(l_, pair_, r);
        Dft<8, +1>::run(a);
#pragma unroll
        for (int r = 0; r < 8; ++r) work_[G::rpad(l_) + r * G::RS0] = a[r];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_empty);  // this warp is done with tile t
      FW_TRACE(t, 4);
      if (FW_DBG(16)) continue;  // timing experiment: rows do pass 0 only
      pairbar(pair_);
      {
        double2 a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = work_[G::r_p1in(l_) + r * G::RS1];
        butterfly_tm8_lean<+1>(a, tmem_base + ((unsigned)(32 * ((tidr >> 5) & 3)) << 16) + (unsigned)G::TM_TWR1);
#pragma unroll
        for (int r = 0; r < 8; ++r) work_[G::r_p1in(l_) + r * G::RS1] = a[r];
      }
      pairbar(pair_);
      FW_TRACE(t, 5);
      const double2* dv = FW_DBG(1) ? nullptr : dev_row(t, row_);
      {
        double2 a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = work_[G::r_p2in(l_) + r * G::RS2];
        butterfly_tm8_lean<+1>(a, tmem_base + ((unsigned)(32 * ((tidr >> 5) & 3)) << 16) +
                                      (unsigned)(G::TM_TWR + 28 * (rw_ >> 2)));
#pragma unroll
        for (int qt = 0; qt < 4; ++qt) {
          double2 d[2];
          if (dv) {
#pragma unroll
            for (int r = 0; r < 2; ++r) d[r] = ld_stream2(&dv[l_ + (2 * qt + r) * G::RT], pol_evict_first());
          }
          unsigned v[8];
          tmem_ld8_nw(tacc_ + 8u * qt, v);
          tmem_wait_ld();
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            double v0 = a[2 * qt + r].x, v1 = a[2 * qt + r].y;
            if (dv) {
              v0 = d[r].x * v0;
              v1 = d[r].y * v1;
            }
            double p0 = 0.0, p1 = 0.0;  // the reference's per-term partial: 0 + dev * x
            p0 += v0;
            p1 += v1;
            tm_put(v, 2 * r, tm_d(v, 2 * r) + p0);
            tm_put(v, 2 * r + 1, tm_d(v, 2 * r + 1) + p1);
          }
          tmem_st8_nw(tacc_ + 8u * qt, v);
        }
        tmem_wait_st();
      }
      FW_TRACE(t, 6);
      pairbar(pair_);  // pass-2 reads of the work_ buffer are done
      FW_TRACE(t, 7);
      if (m == M && !(prm.seismic && op == prm.nops - 1)) {  // operator complete: hand over
        double2* o = reinterpret_cast<double2*>(prm.out[op] + (size_t)row_ * J1);
        unsigned v[32];
        tmem_ld32(tacc_, v);
#pragma unroll
        for (int r = 0; r < 8; ++r) o[l_ + r * G::RT] = make_double2(tm_d(v, 2 * r), tm_d(v, 2 * r + 1));
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0u;
        tmem_st32(tacc_, v);
      }
    }

    // ---- seismic update (seismic.cpp:116-129)
    FW_TRACE(135, 6);
    if (prm.seismic) {
      // a blow-up in an EARLIER step of this launch: keep the state the host restores
      // (this step would overwrite the offending step's prev / L2prev)
      const bool frozen = s > 0 && *reinterpret_cast<volatile int*>(prm.flag) < prm.step + s;
      bool bad;
      if (FW_S2D_TAILHELP) {
        // outputs r = 0..3 here, r = 4..7 by the column warp of this lane quadrant when its group
        // is active (otherwise all eight)
        const int ngrp = 1 + (b + nblk < G::NSLOT);
        const bool helped = ((rw >> 3) < ngrp);
        tailbar((2 * nr + 4 * ngrp) * 32);
        const int rowv[1] = {row}, lv[1] = {l};
        const unsigned tav[1] = {tacc};
        const bool onv[1] = {true};
        bad = seis_update_part<G, 1>(prm, s, rowv, lv, tav, onv, 0, helped ? 4 : 8, frozen);
        if (__any_sync(0xffffffffu, bad) && lane == 0 && !FW_DBG(-1)) atomicMin(prm.flag, prm.step + s);
        tailbar((2 * nr + 4 * ngrp) * 32);
      } else {
        const int rowv[1] = {row}, lv[1] = {l};
        const unsigned tav[1] = {tacc};
        const bool onv[1] = {true};
        bad = seis_update_part<G, 1>(prm, s, rowv, lv, tav, onv, 0, 8, frozen);
        if (__any_sync(0xffffffffu, bad) && lane == 0 && !FW_DBG(-1)) atomicMin(prm.flag, prm.step + s);
      }
      FW_TRACE(135, 2);
    }
    }  // steps
  }
  // everyone is done with tensor memory: release it
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(G::TM_COLS) : "memory");
  launch_mark(1);
}

template <int J0, int J1, int RMAX>
cudaError_t launch_t(const Step2DParams& p, cudaStream_t st, int nblk) {
  using G = Geo<J0, J1, RMAX>;
  if ((J0 + nblk - 1) / nblk > RMAX || 2 * nblk < G::NSLOT) return cudaErrorInvalidConfiguration;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_step2d<J0, J1, RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
  });
  // the term ring as a 3D tensor of doubles [KRING][h][2 J0]; box = 8 rows (128 B) x 256 k
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode)
      return cudaErrorNotSupported;
  }
  constexpr int h = J1 / 2;
  CUtensorMap zmap;
  const cuuint64_t dims[3] = {(cuuint64_t)2 * J0, (cuuint64_t)h, (cuuint64_t)KRING};
  const cuuint64_t strides[2] = {(cuuint64_t)2 * J0 * sizeof(double), (cuuint64_t)2 * J0 * h * sizeof(double)};
  const cuuint32_t box[3] = {16, 256, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (encode(&zmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)p.T, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, FW_S2D_L2PROMO,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  void* args[] = {(void*)&p, (void*)&zmap};
  return cudaLaunchCooperativeKernel((void*)k_step2d<J0, J1, RMAX>, dim3(nblk), dim3(G::NT), args, G::SMEM, st);
}

}  // namespace s2d

bool step2d_supported(int J0, int J1, int nsm) {
  if (!((J0 == 1024 && J1 == 1024) || (J0 == 512 && J1 == 1024))) return false;
  const int nslot = J1 / 4 + 1;
  return nsm >= 148 && nslot <= 2 * nsm;
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
