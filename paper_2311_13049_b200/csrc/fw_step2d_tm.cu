// fw_step2d_tm.cu — persistent single-launch 2D apply / seismic step (sm_100a), time-multiplexed.
//
// One cooperative launch (one CTA per SM) does every step of a seismic advance
// (seismic.cpp:111-133: two M-term applies sharing one forward transform, plus the
// update) or one operator apply (flap.cpp:38-92) on a J0 x J1 grid (half spectrum
// H = J1/2 + 1 columns, h = J1/2).  CTA b owns the column mirror slots b and b + gridDim
// (columns {s, h-s}) and the rows [r0, r1) (<= 8).
//
// All 16 compute warps run the same phase at a time (the CTA's columns, then its rows),
// so every FFT pass has a butterfly per thread and the SM's fp64 pipes and shared
// memory serve one phase at full width; one producer warp streams the operands:
//
//   step s:   F1   R2C of the CTA's rows of u -> Yt (column-major half spectrum, global)
//             F2   (all rows published) forward C2C of the CTA's columns x 1/N -> uhat in TENSOR MEMORY
//             COL(0), COL(1), then for t: COL(t+2), ROW(t)          t = (op, m), ascending
//             update (seismic.cpp:116-129) after the last ROW
//   COL(t)    w_m (bulk-copied to shared memory by the producer) .* uhat, inverse C2C of the
//             4 columns (radix 16/8/8, one butterfly per thread), C2R pre-processing of each
//             mirror pair (partner lane by shuffle) -> Z[t % K] (global ring, column-major [k][k0])
//   ROW(t)    the CTA's rows of Z[t] (TMA, 128-B swizzled tile, issued by the producer once every
//             CTA has published its columns), h-point C2C, x (s-s0)^m, accumulated in ascending m
//             in TENSOR MEMORY (flap.cpp:82-90)
//
// Cross-CTA ordering: monotone counters (rows forward-transformed, Z columns stored per term,
// CTAs done reading term t), red.release / ld.acquire, two counter sets alternating between
// launches.  Inside the CTA: one named barrier for the compute warps, mbarriers for the
// producer's weight and tile copies.  Every pass is in place per butterfly in padded,
// bank-conflict-free shared-memory layouts (tools/layouts/check_step2d.py).  The arithmetic is
// the canonical FFT of fw_fft.cuh (radix plan, twiddle values, fma placement, pre-processing
// formula): bit-identical to the multi-pass path and to the CPU oracle (tests/test_gpu_parity.py,
// tests/test_gpu_configs.py).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "fw_fft.cuh"
#include "fw_internal.h"
#include "fw_step2d.h"

namespace fw {
namespace s2dtm {

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
__device__ __forceinline__ void red_relaxed_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Watchdog: a wait that has not been satisfied after kWatchdogNs is a protocol bug; the kernel
// records where (when a diagnostics buffer is attached: FW_TRACE=1 maps it in host memory, so it
// survives the trap) and traps, so that the host sees an error instead of a hung GPU.
constexpr unsigned long long kWatchdogNs = 4000000000ull;
__device__ __noinline__ void wd_fail(unsigned long long* diag, int site, long long seen, long long want, int gt) {
  if (diag) {
    unsigned long long* r = diag + (size_t)blockIdx.x * 16 + (site >= 5 ? 8 : 0);  // producer | compute
    r[0] = (unsigned long long)site;
    r[1] = threadIdx.x;
    r[2] = (unsigned long long)seen;
    r[3] = (unsigned long long)want;
    r[4] = (unsigned long long)gt;
    r[5] = gtimer();
    __threadfence_system();
  }
  asm volatile("trap;");
}
__device__ __forceinline__ void spin_until(const unsigned long long* cnt, unsigned long long target,
                                           unsigned long long* diag, int site, int gt) {
  if (ld_acquire(cnt) >= target) return;
  const unsigned long long t0 = gtimer();
  unsigned long long v;
  while ((v = ld_acquire(cnt)) < target) {
    if (gtimer() - t0 > kWatchdogNs) wd_fail(diag, site, (long long)v, (long long)target, gt);
  }
}
// named barrier 1: the 16 compute warps
constexpr int NCOMP = 512;
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, 512;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

__device__ __forceinline__ unsigned long long pol_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_stream2(const double2* p, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
// term-ring stores: evict-last (re-read a term later, overwritten K terms later)
__device__ __forceinline__ void st_keep(double2* p, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void prefetch_l2_hint(const void* p, unsigned bytes, unsigned long long pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
               : "memory");
}

// ---------------------------------------------------------------- tensor memory
__device__ __forceinline__ void tmem_ld32_nw(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32_nw(unsigned taddr, const unsigned* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
               :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
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
__device__ __forceinline__ void tmem_ld4_nw(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double tm_d(const unsigned* v, int k) { return __hiloint2double((int)v[2 * k + 1], (int)v[2 * k]); }
__device__ __forceinline__ void tm_put(unsigned* v, int k, double x) {
  v[2 * k] = (unsigned)__double2loint(x);
  v[2 * k + 1] = (unsigned)__double2hiint(x);
}

// ---------------------------------------------------------------- canonical butterflies
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
__device__ __forceinline__ double2 shfl_x1(double2 v) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 1), __shfl_xor_sync(0xffffffffu, v.y, 1));
}

// ---------------------------------------------------------------- async copies (bulk / TMA + mbarrier)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity, unsigned long long* diag, int site,
                                          int gt) {
  if (mbar_try(b, parity)) return;
  const unsigned long long t0 = gtimer();
  while (!mbar_try(b, parity)) {
    if (gtimer() - t0 > kWatchdogNs) wd_fail(diag, site, -1, (long long)parity, gt);
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b,
                                         unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(b))
      : "memory");
}

// --------------------------------------------------------------------------
// Geometry.  Column slots: slot 0 = {0, h}, slot s in [1, h/2) = {s, h-s}, slot h/2 = {h/2};
// CTA b owns slots b (g = 0) and b + gridDim (g = 1), i.e. columns c = 2 g + member.
//   column pass 0: thread u < 4 CT0 -> column c = u / CT0, butterfly u % CT0
//   column passes 1-2: thread u < 4 CT1 -> member u & 1, butterfly (u >> 1) % CT1, slot (u >> 1) / CT1
//     (the two members of a mirror pair on adjacent lanes: pre-processing partner by shuffle)
//   rows: lane -> row slot lane & 7, butterfly 4 warp + (lane >> 3)
//     (a quarter warp = the 8 rows at one butterfly: 128-B tile lines, odd row stride)
// Shared-memory layouts are in place per butterfly (a butterfly writes its outputs where its
// inputs were); the padding makes every pass conflict-free for these mappings.
template <int J0, int J1>
struct Geo {
  static constexpr int H = J1 / 2 + 1;
  static constexpr int h = J1 / 2;
  static constexpr int NSLOT = h / 2 + 1;
  // 16 compute warps + one producer warpgroup (warp 16 streams; 17-19 only balance the register
  // file: one producer warp per SM sub-partition, so setmaxnreg can give the compute warps 120)
  static constexpr int NT = NCOMP + 128;
  // column plan (J0 points, 3 passes)
  static constexpr int CR0 = radix(J0, 0), CR1 = radix(J0, 1), CR2 = radix(J0, 2);
  static constexpr int CT0 = J0 / CR0, CT1 = J0 / CR1, CT2 = J0 / CR2;
  static constexpr int CP1 = CR0;
  static constexpr int CL1 = ilog2c(CR1), CLT = ilog2c(CT1);
  // row plan (h points, 3 radix-8 passes of 64 butterflies)
  static constexpr int RR0 = radix(h, 0), RR1 = radix(h, 1), RR2 = radix(h, 2);
  static constexpr int RT = h / RR0;
  static constexpr int RP1 = RR0;
  static constexpr int RLT = ilog2c(RT);
  // per-column stride = 4 (mod 8): the two members of a pair hit disjoint bank quads
  static constexpr int LCOLM = ((J0 + (J0 >> CL1) + (J0 >> CLT) + 1 + 3) / 8) * 8 + 4;
  static constexpr int LROW = (h + (h >> RLT)) | 1;  // per row (odd stride)
  static constexpr int TWC = twtotal(J0);
  static constexpr int TWR = twtotal(h);
  static constexpr int TWP = h + 1;
  static constexpr size_t OFF_TWR = TWC;
  static constexpr size_t OFF_TWP = TWC + TWR;
  static constexpr size_t OFF_W = (OFF_TWP + TWP + 1) & ~(size_t)1;  // work: columns [4][LCOLM] | rows [8][LROW]
  static constexpr size_t WORK = (4 * LCOLM > 8 * LROW) ? 4 * LCOLM : 8 * LROW;
  static constexpr size_t OFF_WB = OFF_W + WORK;  // weights of the next COL: [4][J0] doubles
  static constexpr size_t OFF_TILE = OFF_WB + (size_t)4 * J0 / 2;
  static constexpr size_t TILE_ELEMS = (size_t)h * 8;  // [h k][8 rows], two 128-B-swizzled TMA boxes
  static constexpr size_t NELEM = OFF_TILE + 64 + TILE_ELEMS;
  static constexpr size_t SMEM = NELEM * sizeof(double2);
  // tensor memory, per warp w (lane quadrant w & 3, slot w >> 2): [0, 128) uhat (8 complex per pass-0
  // thread: 32 columns), [128, 256) row accumulators (32 columns), [256, 480) the thread's column
  // twiddles of passes 1 and 2 (2 x 28 columns)
  static constexpr int TM_U = 0, TM_ACC = 128, TM_TW = 256, TM_COLS = 512;
  // column pass 0: CR0 = 16 -> every compute thread holds half a radix-16 butterfly; CR0 = 8 -> the
  // first 4 CT0 threads hold a whole one.  Either way 8 elements per thread.
  static constexpr bool P0SPLIT = CR0 == 16;
  static_assert(P0SPLIT ? 8 * CT0 == NCOMP : (CR0 == 8 && 4 * CT0 <= NCOMP), "pass-0 mapping");
  static_assert(CR1 == 8 && CR2 == 8 && npass(J0) == 3, "column passes 1-2 radix 8");
  static_assert(4 * CT0 <= NCOMP && 4 * CT1 <= NCOMP, "one butterfly per thread and column pass");
  static_assert(npass(h) == 3 && RR0 == 8 && RR1 == 8 && RR2 == 8 && RT == 64, "row: 3 radix-8 passes");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(h % 256 == 0, "whole TMA boxes");

  __device__ static __forceinline__ int cpad(int pos) { return pos + (pos >> CL1) + (pos >> CLT); }
  __device__ static __forceinline__ int c_p0out(int e) { return cpad((e % CT1) * CR1 + e / CT1); }
  __device__ static __forceinline__ int c_p1(int i, int r) { return cpad(i * CR1 + r); }
  __device__ static __forceinline__ int c_p2in(int e) {
    const int i = (e / (CP1 * CR1)) * CP1 + e % CP1, r = (e / CP1) % CR1;
    return cpad(i * CR1 + r);
  }
  static constexpr int CS0 = CR1 + 1, CS2 = CT2 + CT2 / CR1 + 1;
  static constexpr int RS0 = RT + 1, RS1 = 8, RS2 = 1;
  __device__ static __forceinline__ int rpad(int pos) { return pos + (pos >> RLT); }
  __device__ static __forceinline__ int r_p1in(int e) { return rpad(e / RR0 + RT * (e % RR0)); }
  __device__ static __forceinline__ int r_p2in(int e) {
    const int i1 = (e / (RP1 * RR1)) * RP1 + e % RP1, r1 = (e / RP1) % RR1;
    return rpad((i1 + RT * r1) / RR0 + RT * ((i1 + RT * r1) % RR0));
  }
};

// the column of member mbr of slot `slot` (-1: none)
template <int h, int NSLOT>
__device__ __forceinline__ int colno(int slot, int mbr) {
  if (slot >= NSLOT) return -1;
  if (slot == 0) return mbr ? h : 0;
  if (slot == h / 2) return mbr ? -1 : h / 2;
  return mbr ? h - slot : slot;
}

// ---------------------------------------------------------------- column twiddles in tensor memory
// A column thread's 7 twiddles of pass 1 and of pass 2 (its butterfly index is fixed across terms)
// are parked once per launch: 28 TMEM columns each = 7 x (re, im) as 32-bit halves.  The values are
// the shared-memory table entries, so the butterflies are bit-identical to butterfly().
__device__ __forceinline__ void tmem_st16_nw(unsigned taddr, const unsigned* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
               :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
               : "memory");
}
__device__ __forceinline__ void tmem_ld16_nw(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st4_nw(unsigned taddr, const unsigned* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
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
template <int DIR>
__device__ __forceinline__ void butterfly_tm8(double2 (&a)[8], unsigned taddr) {
  unsigned v[28];
  tmem_ld16_nw(taddr, v);
  tmem_ld8_nw(taddr + 16, v + 16);
  tmem_ld4_nw(taddr + 24, v + 24);
  tmem_wait_ld();
#pragma unroll
  for (int r = 1; r < 8; ++r) {
    const double2 w = dirw<DIR>(make_double2(tm_d(v, 2 * (r - 1)), tm_d(v, 2 * (r - 1) + 1)));
    a[r] = cmulw(a[r], w.x, w.y);
  }
  Dft<8, DIR>::run(a);
}

// ---------------------------------------------------------------- column passes 1 and 2
// pass 1 in place; pass 2 returns the natural-order outputs k0 = i + CT2 r in x[]
// (twiddles from the thread's tensor-memory slots ttw, ttw + 28)
template <class G, int DIR>
__device__ __forceinline__ void col_passes12(double2* work, unsigned ttw, int tid, double2 (&x)[8]) {
  const int mbr = tid & 1, i = (tid >> 1) % G::CT1, g = (tid >> 1) / G::CT1;
  double2* wb = work + (2 * g + mbr) * G::LCOLM;
  if (g < 2) {
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = wb[G::c_p1(i, 0) + r];
    butterfly_tm8<DIR>(a, ttw);
#pragma unroll
    for (int r = 0; r < 8; ++r) wb[G::c_p1(i, 0) + r] = a[r];
  }
  cbar();
  if (g < 2) {
#pragma unroll
    for (int r = 0; r < 8; ++r) x[r] = wb[G::c_p2in(i) + r * G::CS2];
    butterfly_tm8<DIR>(x, ttw + 28);
  }
}

// ---------------------------------------------------------------- column pass 0
// CR0 = 16: every compute thread holds half a radix-16 butterfly: column c = tid >> 7, butterfly
// I = 8 ((tid >> 4) & 7) + (tid & 7), half hh = (tid >> 3) & 1 (partner lane ^ 8; a quarter warp is
// 8 butterflies of one half: conflict-free stores).  DFT_16 as fw_fft.cuh (4 DFT_4, W16, 4 DFT_4):
// the thread's first-stage DFT_4s are j2 = 2 hh + {0, 1}, its second-stage ones k1 = 2 hh + {0, 1},
// after swapping four values with the partner half.  Element e < 8 is the input / output slot
// r = 2 hh + (e & 1) + 4 (e >> 1).  CR0 = 8: thread tid < 4 CT0 holds butterfly tid % CT0 of column
// tid / CT0 whole, r = e.
template <class G>
struct P0 {
  int c, I, hh;
  bool act;
  __device__ __forceinline__ explicit P0(int tid) {
    if constexpr (G::P0SPLIT) {
      c = tid >> 7;
      I = 8 * ((tid >> 4) & 7) + (tid & 7);
      hh = (tid >> 3) & 1;
      act = true;
    } else {
      c = tid / G::CT0;
      I = tid % G::CT0;
      hh = 0;
      act = tid < 4 * G::CT0;
    }
  }
  __device__ __forceinline__ int r(int e) const {
    if constexpr (G::P0SPLIT)
      return 2 * hh + (e & 1) + 4 * (e >> 1);
    else
      return e;
  }
};
template <class G, int DIR>
__device__ __forceinline__ void col_pass0(double2 (&a)[8], const P0<G>& p, double2* wb) {
  if constexpr (G::P0SPLIT) {
    double2 F[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) dft4v<DIR>(a[j], a[2 + j], a[4 + j], a[6 + j], F[j][0], F[j][1], F[j][2], F[j][3]);
    if (p.hh == 0) {  // j2 = 0 (no twiddles), j2 = 1
      F[1][1] = w16<DIR>(F[1][1], 1);
      F[1][2] = w16<DIR>(F[1][2], 2);
      F[1][3] = w16<DIR>(F[1][3], 3);
    } else {  // j2 = 2, 3
      F[0][1] = w16<DIR>(F[0][1], 2);
      F[0][2] = w16<DIR>(F[0][2], 4);
      F[0][3] = w16<DIR>(F[0][3], 6);
      F[1][1] = w16<DIR>(F[1][1], 3);
      F[1][2] = w16<DIR>(F[1][2], 6);
      F[1][3] = w16<DIR>(F[1][3], 9);
    }
    // R[jj][j]: the partner's first-stage output (its j2 = 2 (1 - hh) + jj) at this thread's k1 = 2 hh + j
    double2 R[2][2];
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const double2 snd = p.hh ? F[jj][j] : F[jj][2 + j];
        R[jj][j] = make_double2(__shfl_xor_sync(0xffffffffu, snd.x, 8), __shfl_xor_sync(0xffffffffu, snd.y, 8));
      }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double2 o0 = p.hh ? F[0][2 + j] : F[0][j], o1 = p.hh ? F[1][2 + j] : F[1][j];
      const double2 x0 = p.hh ? R[0][j] : o0, x1 = p.hh ? R[1][j] : o1;
      const double2 x2 = p.hh ? o0 : R[0][j], x3 = p.hh ? o1 : R[1][j];
      dft4v<DIR>(x0, x1, x2, x3, a[j], a[2 + j], a[4 + j], a[6 + j]);
    }
  } else {
    Dft<8, DIR>::run(a);
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) wb[G::c_p0out(p.I * G::CR0) + p.r(e) * G::CS0] = a[e];
}

// row pass 1 of one row (butterfly l) in place
template <class G, int DIR>
__device__ __forceinline__ void row_pass1(double2* wr, const double2* twr, int l) {
  double2 a[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) a[r] = wr[G::r_p1in(l) + r * G::RS1];
  butterfly<G::h, 1, DIR>(a, l, twr);
#pragma unroll
  for (int r = 0; r < 8; ++r) wr[G::r_p1in(l) + r * G::RS1] = a[r];
}

// --------------------------------------------------------------------------
template <int J0, int J1>
__global__ void __launch_bounds__(Geo<J0, J1>::NT, 1) k_step2d(const Step2DParams prm, const __grid_constant__ CUtensorMap zmap) {
  using G = Geo<J0, J1>;
  constexpr int h = G::h, NSLOT = G::NSLOT;
  constexpr int CR0 = G::CR0, CT0 = G::CT0, CT2 = G::CT2;
  extern __shared__ __align__(16) double2 sm[];
  __shared__ unsigned tmem_base_sh;
  __shared__ __align__(8) unsigned long long wfull, wempty, tfull, tempty;
  double2* twc = sm;
  double2* twr = sm + G::OFF_TWR;
  double2* twp = sm + G::OFF_TWP;
  double2* work = sm + G::OFF_W;
  double* wbuf = reinterpret_cast<double*>(sm + G::OFF_WB);
  double2* tile;
  {
    const unsigned base = smem_u32(sm + G::OFF_TILE);
    tile = sm + G::OFF_TILE + (((base + 1023u) & ~1023u) - base) / 16u;
  }
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.x;
  const int nblk = gridDim.x;

  unsigned long long* cnt = prm.counters + (size_t)prm.cset * prm.cstride;
  if (b == 0) {
    unsigned long long* other = prm.counters + (size_t)(prm.cset ^ 1) * prm.cstride;
    for (int e = tid; e < prm.cstride; e += G::NT) other[e] = 0ull;
  }
  if (prm.flag && *prm.flag != kNoBlowup) return;  // uniform across CTAs
  unsigned long long* cY = cnt;                          // rows forward-transformed
  unsigned long long* cC = cnt + 1;                      // Z columns of term t stored
  unsigned long long* cR = cnt + 1 + prm.nterms_total;  // CTAs done reading Z[t]

  {  // twiddle tables (values = master entries, identical to fw_fft.cuh's twiddle())
    auto fill = [&](double2* dst, int off, int p, int R) {
      const int n = p * (R - 1);
      for (int e = tid; e < n; e += G::NT) {
        const int k = e / (R - 1), r = e % (R - 1) + 1;
        dst[off + e] = prm.master[(r * k) * (kTwMaster / (p * R))];
      }
    };
    fill(twc, twoff(J0, 1), pprod(J0, 1), radix(J0, 1));
    fill(twc, twoff(J0, 2), pprod(J0, 2), radix(J0, 2));
    fill(twr, twoff(h, 1), pprod(h, 1), radix(h, 1));
    fill(twr, twoff(h, 2), pprod(h, 2), radix(h, 2));
    for (int e = tid; e <= h; e += G::NT) twp[e] = prm.master[e * (kTwMaster / J1)];
  }
  if (tid == 0) {
    mbar_init(&wfull, 1);
    mbar_init(&wempty, 1);
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 1);
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

  const int M = prm.M;
  const int nterms = M + 1 - prm.m_first;
  const int ntot = prm.nops * nterms;
  const int gtot = prm.nsteps * ntot;
  const int r0 = (int)(((long long)b * J0) / nblk);
  const int nr = (int)(((long long)(b + 1) * J0) / nblk) - r0;

  if (warp >= NCOMP / 32) {
    // ============================================ producer warpgroup (one lane of warp 16)
    setmaxnreg_dec<32>();
    if (warp == NCOMP / 32 && lane == 0) {
      const unsigned long long pf = pol_evict_first();
      auto wissue = [&](int gt) {  // weights of COL(gt) -> wbuf
        const int t = gt % ntot;
        const int op = t / nterms, m = prm.m_first + t % nterms;
        unsigned bytes = 0;
        for (int c = 0; c < 4; ++c) bytes += colno<h, NSLOT>(b + (c >> 1) * nblk, c & 1) >= 0 ? J0 * 8u : 0u;
        mbar_expect_tx(&wfull, bytes);
        for (int c = 0; c < 4; ++c) {
          const int col = colno<h, NSLOT>(b + (c >> 1) * nblk, c & 1);
          if (col >= 0)
            bulk_g2s(wbuf + (size_t)c * J0, prm.w[op] + ((size_t)m * prm.wcols + col) * J0, J0 * 8u, &wfull, pf);
        }
      };
      auto zissue = [&](int gt) {  // Z[gt] rows of this CTA -> tile, once every column is stored
        const int t = gt % ntot;
        const int op = t / nterms, m = prm.m_first + t % nterms;
        if (m >= 1)  // this term's (s-s0)^m rows -> L2 (read by ROW(gt) a phase later)
          for (int rho = 0; rho < nr; ++rho)
            prefetch_l2_hint(prm.dev[op] + (size_t)(m - 1) * J0 * J1 + (size_t)(r0 + rho) * J1, J1 * 8u, pf);
        spin_until(&cC[t], (unsigned long long)(gt / ntot + 1) * h, prm.trace, 1, gt);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy Z stores -> TMA reads
        mbar_expect_tx(&tfull, (unsigned)(G::TILE_ELEMS * sizeof(double2)));
        for (int bx = 0; bx < h / 256; ++bx)
          tma_load_3d(tile + (size_t)bx * 256 * 8, &zmap, 2 * r0, bx * 256, gt % KRING, &tfull);
      };
      if (gtot > 0) wissue(0);
      for (int gt = 0; gt < gtot; ++gt) {
        const int t = gt % ntot;
        mbar_wait(&wempty, (unsigned)gt & 1u, prm.trace, 2, gt);  // COL(gt) has read its weights
        if (gt + 1 < gtot) wissue(gt + 1);
        if (t >= 1) {  // Z[gt-1]: the tile is free once ROW(gt-2) has read it
          if (gt - 2 >= 0) mbar_wait(&tempty, (unsigned)(gt - 2) & 1u, prm.trace, 3, gt);
          zissue(gt - 1);
        }
        if (t == ntot - 1) {
          if (gt - 1 >= 0) mbar_wait(&tempty, (unsigned)(gt - 1) & 1u, prm.trace, 4, gt);
          zissue(gt);
        }
      }
    }
  } else {
    // ============================================ compute warps
    setmaxnreg_inc<112>();  // per sub-partition: 4 x 32 x 112 + 32 x 32 < 16 K registers
    // row mapping
    const int rho = lane & 7;
    const int l = 4 * warp + (lane >> 3);
    const bool ract = rho < nr;
    const int row = r0 + (ract ? rho : 0);
    double2* wrow = work + (size_t)rho * G::LROW;
    const unsigned tacc = tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)(G::TM_ACC + 32 * (warp >> 2));
    // column pass-0 mapping
    const P0<G> p0m(tid);
    const bool p0 = p0m.act;
    const int col0 = p0 ? colno<h, NSLOT>(b + (p0m.c >> 1) * nblk, p0m.c & 1) : -1;
    const unsigned tq = tmem_base + ((unsigned)(32 * (warp & 3)) << 16);  // this warp's lane quadrant
    const unsigned tu = tq + (unsigned)(G::TM_U + 32 * (warp >> 2));
    const unsigned ttw = tq + (unsigned)(G::TM_TW + 56 * (warp >> 2));
    // column pass-1/2 mapping
    const int cm = tid & 1, cg = (tid >> 1) / G::CT1, ci = (tid >> 1) % G::CT1;
    const int slot = b + cg * nblk;
    const int kA = slot == 0 ? 0 : slot;
    const int kB = slot == 0 ? h : (slot == h / 2 ? -1 : h - slot);
    int nz = 0;  // Z columns this CTA stores per term
    for (int gg = 0; gg < 2; ++gg) {
      const int sl = b + gg * nblk;
      nz += sl >= NSLOT ? 0 : (sl == 0 || sl == h / 2 ? 1 : 2);
    }
    double rmax = 0.0;
    int pend = -1;  // term whose Z columns are stored but not yet published (cC)

    auto lvl_u = [&](int s, int d) -> double* { return prm.ub[(int)((prm.lvl0 + s + d) % 3)]; };
    auto lvl_a = [&](int s, int d) -> double* { return prm.ab[(int)((prm.lvl0 + s + d) % 2)]; };

    // ---- COL(gt): inverse column transform of term gt -> Z ring
    auto col_phase = [&](int s, int t) {
      const int gt = s * ntot + t;
      if (tid == 0 && gt >= KRING)  // ring slot free: every CTA has read term gt - K
        spin_until(&cR[(gt - KRING) % ntot], (unsigned long long)((gt - KRING) / ntot + 1) * nblk, prm.trace, 5, gt);
      if (p0) {
        mbar_wait(&wfull, (unsigned)gt & 1u, prm.trace, 6, gt);
        double wk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) wk[e] = col0 >= 0 ? wbuf[p0m.c * J0 + p0m.I + p0m.r(e) * CT0] : 0.0;
        double2 a[8];
        {
          unsigned v[32];
          tmem_ld32_nw(tu, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) a[e] = make_double2(wk[e] * tm_d(v, 2 * e), wk[e] * tm_d(v, 2 * e + 1));
        }
        col_pass0<G, +1>(a, p0m, work + p0m.c * G::LCOLM);
      }
      cbar();
      if (tid == 0) {
        mbar_arrive(&wempty);
        if (pend >= 0) red_release_add(&cC[pend], (unsigned long long)nz);  // deferred: the stores have drained
      }
      pend = -1;
      double2 x[8];
      col_passes12<G, +1>(work, ttw, tid, x);
      if (cg < 2) {
        double2 y[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) y[r] = shfl_x1(x[r]);
        if (slot < NSLOT) {
          const unsigned long long pkeep = pol_evict_last();
          double2* Z = prm.T + (size_t)(gt % KRING) * J0 * h;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int k0 = ci + r * CT2;
            const double2 xa = cm ? y[r] : x[r], xb = cm ? x[r] : y[r];
            if (kA == 0) {  // Z_0 from X_0 and X_h (column h has no Z of its own)
              if (!cm) {
                if (prm.residue) rmax = fmax(rmax, fabs(xa.y) + fabs(xb.y));
                st_keep(&Z[k0], pre_c2r(xa, xb, true, twp[0]), pkeep);
              }
            } else if (kA == h / 2) {
              if (!cm) st_keep(&Z[(size_t)kA * J0 + k0], pre_c2r(xa, xa, false, twp[kA]), pkeep);
            } else if (!cm) {
              st_keep(&Z[(size_t)kA * J0 + k0], pre_c2r(xa, xb, false, twp[kA]), pkeep);
            } else {
              st_keep(&Z[(size_t)kB * J0 + k0], pre_c2r(xb, xa, false, twp[kB]), pkeep);
            }
          }
        }
      }
      cbar();  // every Z store of the CTA issued (and the column buffers free)
      // publish term t after the next phase's first barrier (its release then finds the stores
      // drained); with a single term ROW(t) itself comes next and waits for it: publish now
      if (ntot == 1) {
        if (tid == 0) red_release_add(&cC[t], (unsigned long long)nz);
      } else {
        pend = t;
      }
    };

    // ---- ROW(gt): the CTA's rows of Z[gt], C2R + (s-s0)^m, accumulate
    auto row_phase = [&](int s, int t) {
      const int gt = s * ntot + t;
      const int op = t / nterms, m = prm.m_first + t % nterms;
      mbar_wait(&tfull, (unsigned)gt & 1u, prm.trace, 7, gt);
      {
        double2 a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = tile[l * 8 + (rho ^ (l & 7)) + r * 64 * 8];
        Dft<8, +1>::run(a);
        if (ract) {
#pragma unroll
          for (int r = 0; r < 8; ++r) wrow[G::rpad(l) + r * G::RS0] = a[r];
        }
      }
      cbar();
      if (tid == 0) {
        mbar_arrive(&tempty);  // tile read: the producer may load the next term
        red_relaxed_add(&cR[t], 1ull);  // the ring slot's bytes are in shared memory
        if (pend >= 0) red_release_add(&cC[pend], (unsigned long long)nz);
      }
      pend = -1;
      // tcgen05.ld/st are warp-collective: every lane runs the row code (lanes of a row slot past
      // the CTA's rows work on scratch in their own buffer); only global accesses are guarded
      double2 d[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) d[r] = make_double2(0.0, 0.0);
      if (m >= 1 && ract) {
        const double2* dv = reinterpret_cast<const double2*>(prm.dev[op] + (size_t)(m - 1) * J0 * J1 + (size_t)row * J1);
        const unsigned long long pf = pol_evict_first();
#pragma unroll
        for (int r = 0; r < 8; ++r) d[r] = ld_stream2(&dv[l + r * G::RT], pf);
      }
      row_pass1<G, +1>(wrow, twr, l);
      cbar();
      {
        double2 a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = wrow[G::r_p2in(l) + r * G::RS2];
        butterfly<h, 2, +1>(a, l, twr);
#pragma unroll
        for (int qt = 0; qt < 4; ++qt) {
          unsigned v[8];
          tmem_ld8_nw(tacc + 8u * qt, v);
          tmem_wait_ld();
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            double v0 = a[2 * qt + r].x, v1 = a[2 * qt + r].y;
            if (m >= 1) {
              v0 = d[2 * qt + r].x * v0;
              v1 = d[2 * qt + r].y * v1;
            }
            double q0 = 0.0, q1 = 0.0;  // the reference's per-term partial: 0 + dev * x
            q0 += v0;
            q1 += v1;
            tm_put(v, 2 * r, tm_d(v, 2 * r) + q0);
            tm_put(v, 2 * r + 1, tm_d(v, 2 * r + 1) + q1);
          }
          tmem_st8_nw(tacc + 8u * qt, v);
        }
        tmem_wait_st();
      }
      cbar();  // pass-2 reads done: the work buffer may take the next column pass 0
      if (m == M && !(prm.seismic && op == prm.nops - 1)) {  // operator complete: hand over
        double2* o = reinterpret_cast<double2*>(prm.out[op] + (size_t)row * J1);
        unsigned v[32];
        tmem_ld32_nw(tacc, v);
        tmem_wait_ld();
        if (ract) {
#pragma unroll
          for (int r = 0; r < 8; ++r) o[l + r * G::RT] = make_double2(tm_d(v, 2 * r), tm_d(v, 2 * r + 1));
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0u;
        tmem_st32_nw(tacc, v);
        tmem_wait_st();
      }
    };

    {  // zero the accumulators; park this thread's column twiddles of passes 1 and 2
      unsigned z[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) z[e] = 0u;
      tmem_st32_nw(tacc, z);
      tmem_wait_st();
      tw_park(ttw, twc + twoff(J0, 1) + (ci & (pprod(J0, 1) - 1)) * 7);
      tw_park(ttw + 28, twc + twoff(J0, 2) + (ci & (pprod(J0, 2) - 1)) * 7);
    }

#pragma unroll 1
    for (int s = 0; s < prm.nsteps; ++s) {
      // ---- F1: R2C of the CTA's rows -> Yt[k][k0]
      {
        const double2* u2 = reinterpret_cast<const double2*>(prm.nsteps > 1 ? lvl_u(s, 0) : prm.u) + (size_t)row * h;
        double2 a[8];
        if (ract) {
#pragma unroll
          for (int r = 0; r < 8; ++r) a[r] = u2[l + r * G::RT];
          Dft<8, -1>::run(a);
#pragma unroll
          for (int r = 0; r < 8; ++r) wrow[G::rpad(l) + r * G::RS0] = a[r];
        }
        cbar();
        if (ract) row_pass1<G, -1>(wrow, twr, l);
        cbar();
        if (ract) {  // pass 2 in place: output q = l + RT r where its butterfly read its inputs
#pragma unroll
          for (int r = 0; r < 8; ++r) a[r] = wrow[G::r_p2in(l) + r * G::RS2];
          butterfly<h, 2, -1>(a, l, twr);
#pragma unroll
          for (int r = 0; r < 8; ++r) wrow[G::r_p2in(l) + r * G::RS2] = a[r];
        }
        cbar();
        if (ract) {
          auto zq = [&](int q) -> double2 { return wrow[G::r_p2in(q % G::RT) + (q / G::RT) * G::RS2]; };
          for (int jj = l; jj <= h / 2; jj += G::RT) {
            if (jj == 0) {
              const double2 z0 = zq(0);
              __stcg(&prm.Y[row], make_double2(z0.x + z0.y, 0.0));
              __stcg(&prm.Y[(size_t)h * J0 + row], make_double2(z0.x - z0.y, 0.0));
            } else {
              const double2 A = zq(jj);
              const double2 B = zq(h - jj);
              __stcg(&prm.Y[(size_t)jj * J0 + row], post_r2c(A, B, twp[jj]));
              if (jj != h - jj) __stcg(&prm.Y[(size_t)(h - jj) * J0 + row], post_r2c(B, A, twp[h - jj]));
            }
          }
        }
        cbar();
        if (tid == 0) red_release_add(cY, (unsigned long long)nr);
      }
      // ---- F2: forward columns (all rows published) -> uhat in tensor memory
      {
        if (tid == 0) spin_until(cY, (unsigned long long)(s + 1) * J0, prm.trace, 8, s);
        cbar();
        if (p0) {
          double2 a[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            a[e] = col0 >= 0 ? __ldcg(&prm.Y[(size_t)col0 * J0 + p0m.I + p0m.r(e) * CT0]) : make_double2(0.0, 0.0);
          col_pass0<G, -1>(a, p0m, work + p0m.c * G::LCOLM);
        }
        cbar();
        {
          double2 x[8];
          col_passes12<G, -1>(work, ttw, tid, x);
          if (cg < 2) {  // in place: output k0 = ci + CT2 r where its butterfly read its inputs
            double2* wb = work + (2 * cg + cm) * G::LCOLM;
#pragma unroll
            for (int r = 0; r < 8; ++r) wb[G::c_p2in(ci) + r * G::CS2] = x[r];
          }
        }
        cbar();
        if (p0) {
          const double inv = 1.0 / ((double)J0 * (double)J1);
          const double2* wb = work + p0m.c * G::LCOLM;
          unsigned v[32];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int k0 = p0m.I + p0m.r(e) * CT0;
            const double2 xx = wb[G::c_p2in(k0 % CT2) + (k0 / CT2) * G::CS2];
            tm_put(v, 2 * e, xx.x * inv);
            tm_put(v, 2 * e + 1, xx.y * inv);
          }
          tmem_st32_nw(tu, v);
          tmem_wait_st();
        }
        cbar();
      }

      // ---- the terms: COL runs two terms ahead of ROW
      col_phase(s, 0);
      if (ntot > 1) col_phase(s, 1);
#pragma unroll 1
      for (int t = 0; t < ntot; ++t) {
        if (t + 2 < ntot) col_phase(s, t + 2);
        row_phase(s, t);
      }

      // ---- seismic update (seismic.cpp:116-129)
      if (prm.seismic) {
        bool bad = false;
        {
          const double tau = prm.tau;
          const double t2 = tau * tau;
          const size_t rowoff = (size_t)row * J1;
          const bool ms = prm.nsteps > 1;
          const double2* cur = reinterpret_cast<const double2*>((ms ? lvl_u(s, 0) : prm.u) + rowoff);
          const double2* prev = reinterpret_cast<const double2*>((ms ? lvl_u(s, 2) : prm.prev) + rowoff);
          const double2* ap = reinterpret_cast<const double2*>((ms ? lvl_a(s, 1) : prm.ap) + rowoff);
          // a blow-up in an EARLIER step of this launch: keep the state the host restores
          const bool frozen = s > 0 && *reinterpret_cast<volatile int*>(prm.flag) < prm.step + s;
          const double2* l1 = reinterpret_cast<const double2*>(prm.out[0] + rowoff);
          const double2* c = reinterpret_cast<const double2*>(prm.c + rowoff);
          const double2* eta = reinterpret_cast<const double2*>(prm.eta + rowoff);
          const double2* tc = reinterpret_cast<const double2*>(prm.tc + rowoff);
          double2* nx = reinterpret_cast<double2*>((ms ? lvl_u(s, 1) : prm.next) + rowoff);
          double2* l2o = reinterpret_cast<double2*>((ms ? lvl_a(s, 0) : prm.out[1]) + rowoff);
#pragma unroll 1
          for (int r = 0; r < 8; ++r) {
            unsigned v[4];
            tmem_ld4_nw(tacc + 4u * r, v);
            tmem_wait_ld();
            if (ract) {
              const int q = l + r * G::RT;
              const double2 vc = cur[q], vp = prev[q], va = ap[q], v1 = l1[q], cc = c[q], ve = eta[q], vt = tc[q];
              const double l2x = tm_d(v, 0), l2y = tm_d(v, 1);
              const double c2x = cc.x * cc.x, c2y = cc.y * cc.y;
              const double nx0 = 2.0 * vc.x - vp.x + t2 * c2x * (ve.x * v1.x + vt.x * (l2x - va.x) / tau);
              const double nx1 = 2.0 * vc.y - vp.y + t2 * c2y * (ve.y * v1.y + vt.y * (l2y - va.y) / tau);
              if (!frozen) {
                nx[q] = make_double2(nx0, nx1);
                l2o[q] = make_double2(l2x, l2y);
              }
              bad |= (fabs(nx0) > prm.thr) || (fabs(nx1) > prm.thr);
            }
          }
          unsigned z[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) z[e] = 0u;
          tmem_st32_nw(tacc, z);
          tmem_wait_st();
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(prm.flag, prm.step + s);
        cbar();  // the next step's F1 reads this step's `next` rows
      }
    }  // steps
    if (prm.residue && rmax > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(prm.residue), (unsigned long long)__double_as_longlong(rmax));
  }
  // everyone is done with tensor memory: release it
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(G::TM_COLS) : "memory");
}

template <int J0, int J1>
cudaError_t launch_t(const Step2DParams& p, cudaStream_t st, int nblk) {
  using G = Geo<J0, J1>;
  if ((J0 + nblk - 1) / nblk > 8 || 2 * nblk < G::NSLOT) return cudaErrorInvalidConfiguration;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_step2d<J0, J1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
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
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  void* args[] = {(void*)&p, (void*)&zmap};
  return cudaLaunchCooperativeKernel((void*)k_step2d<J0, J1>, dim3(nblk), dim3(G::NT), args, G::SMEM, st);
}

}  // namespace s2dtm

bool step2d_tm_supported(int J0, int J1, int nsm) {
  if (!((J0 == 1024 && J1 == 1024) || (J0 == 512 && J1 == 1024))) return false;
  return nsm >= 148 && J1 / 4 + 1 <= 2 * nsm && (J0 + nsm - 1) / nsm <= 8;
}

cudaError_t launch_step2d_tm(const Step2DParams& p, cudaStream_t st, int nsm) {
  const int J0 = p.J0, J1 = p.J1;
  if (J0 == 1024 && J1 == 1024) return s2dtm::launch_t<1024, 1024>(p, st, nsm);
  if (J0 == 512 && J1 == 1024) return s2dtm::launch_t<512, 1024>(p, st, nsm);
  return cudaErrorInvalidValue;
}

}  // namespace fw
