// fw_fft.cuh — device side of the canonical fp64 FFT.
//
// Power-of-two Stockham passes (radix 16/8/4/2, radix sequence from
// fw_radices()), fixed in-register DFT kernels, twiddles from one host-computed
// master table, explicit fma() in complex products and no other contraction
// (the TU is compiled with --fmad=false).  Real transforms use the half-length
// packing formulation.  The same definition is implemented independently for
// the CPU oracle (oracle/fwshim/fwcanon.c); identical inputs give identical bits.
#pragma once

#include <cuda_runtime.h>

namespace fw {

constexpr int kTwMaster = 8192;  // master twiddle table length (max transform length)

__host__ __device__ inline int fw_radices(int n, int* radix) {
  int L = 0;
  while ((1 << L) < n) ++L;
  if (L == 0) return 0;
  const int P = (L + 3) / 4;
  const int base = L / P, extra = L % P;
  for (int i = 0; i < P; ++i) radix[i] = 1 << (base + (i < extra ? 1 : 0));
  return P;
}

#define FW_SQRT1_2 0.70710678118654752440084436210484904
#define FW_COS_PI_8 0.92387953251128675612818318939678829
#define FW_SIN_PI_8 0.38268343236508977172845998403039887

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// a * (wr, wi)
__device__ __forceinline__ double2 cmulw(double2 a, double wr, double wi) {
  return make_double2(fma(a.x, wr, -(a.y * wi)), fma(a.x, wi, a.y * wr));
}
template <int DIR>
__device__ __forceinline__ double2 rot(double2 a) {  // * (DIR i)
  return DIR < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}
template <int DIR>
__device__ __forceinline__ double2 w8_1(double2 x) {
  return DIR < 0 ? make_double2((x.x + x.y) * FW_SQRT1_2, (x.y - x.x) * FW_SQRT1_2)
                 : make_double2((x.x - x.y) * FW_SQRT1_2, (x.y + x.x) * FW_SQRT1_2);
}
template <int DIR>
__device__ __forceinline__ double2 w8_3(double2 x) {
  return DIR < 0 ? make_double2((x.y - x.x) * FW_SQRT1_2, -((x.x + x.y) * FW_SQRT1_2))
                 : make_double2(-((x.x + x.y) * FW_SQRT1_2), (x.x - x.y) * FW_SQRT1_2);
}

template <int DIR>
__device__ __forceinline__ void dft4v(double2 x0, double2 x1, double2 x2, double2 x3, double2& o0,
                                      double2& o1, double2& o2, double2& o3) {
  const double2 t0 = cadd(x0, x2), t1 = csub(x0, x2);
  const double2 t2 = cadd(x1, x3), t3 = rot<DIR>(csub(x1, x3));
  o0 = cadd(t0, t2);
  o1 = cadd(t1, t3);
  o2 = csub(t0, t2);
  o3 = csub(t1, t3);
}

template <int R, int DIR>
struct Dft;

template <int DIR>
struct Dft<2, DIR> {
  __device__ __forceinline__ static void run(double2* a) {
    const double2 t = a[0];
    a[0] = cadd(t, a[1]);
    a[1] = csub(t, a[1]);
  }
};

template <int DIR>
struct Dft<4, DIR> {
  __device__ __forceinline__ static void run(double2* a) { dft4v<DIR>(a[0], a[1], a[2], a[3], a[0], a[1], a[2], a[3]); }
};

template <int DIR>
struct Dft<8, DIR> {
  __device__ __forceinline__ static void run(double2* a) {
    double2 E0, E1, E2, E3, O0, O1, O2, O3;
    dft4v<DIR>(a[0], a[2], a[4], a[6], E0, E1, E2, E3);
    dft4v<DIR>(a[1], a[3], a[5], a[7], O0, O1, O2, O3);
    O1 = w8_1<DIR>(O1);
    O2 = rot<DIR>(O2);
    O3 = w8_3<DIR>(O3);
    a[0] = cadd(E0, O0); a[4] = csub(E0, O0);
    a[1] = cadd(E1, O1); a[5] = csub(E1, O1);
    a[2] = cadd(E2, O2); a[6] = csub(E2, O2);
    a[3] = cadd(E3, O3); a[7] = csub(E3, O3);
  }
};

template <int DIR>
__device__ __forceinline__ double2 w16(double2 x, int e) {
  constexpr double sd = DIR < 0 ? -1.0 : 1.0;
  switch (e) {
    case 1: return cmulw(x, FW_COS_PI_8, sd * FW_SIN_PI_8);
    case 2: return w8_1<DIR>(x);
    case 3: return cmulw(x, FW_SIN_PI_8, sd * FW_COS_PI_8);
    case 4: return rot<DIR>(x);
    case 6: return w8_3<DIR>(x);
    case 9: return cmulw(x, -FW_COS_PI_8, -(sd * FW_SIN_PI_8));
    default: return x;
  }
}

template <int DIR>
struct Dft<16, DIR> {
  __device__ __forceinline__ static void run(double2* a) {
    double2 F[4][4];
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2)
      dft4v<DIR>(a[j2], a[j2 + 4], a[j2 + 8], a[j2 + 12], F[j2][0], F[j2][1], F[j2][2], F[j2][3]);
#pragma unroll
    for (int j2 = 1; j2 < 4; ++j2)
#pragma unroll
      for (int k1 = 1; k1 < 4; ++k1) F[j2][k1] = w16<DIR>(F[j2][k1], j2 * k1);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
      dft4v<DIR>(F[0][k1], F[1][k1], F[2][k1], F[3][k1], a[k1], a[k1 + 4], a[k1 + 8], a[k1 + 12]);
  }
};

// twiddle W_n^t for direction DIR from the master table (cos, sin)(2 pi t / 8192)
template <int DIR>
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ master, int t, int n) {
  const double2 w = __ldg(&master[t * (kTwMaster / n)]);
  return make_double2(w.x, DIR < 0 ? -w.y : w.y);
}

// One Stockham pass of radix R over `lines` lines of length n held in shared
// memory (line l at src + l*ls), all threads of the block cooperating.
template <int R, int DIR>
__device__ __forceinline__ void stockham_pass(const double2* src, double2* dst, int n, int p, int lines,
                                              int ls, const double2* __restrict__ master) {
  const int T = n / R;
  const int tstep_n = n;  // twiddle index r*k*(n/(p*R)) in a length-n table
  const int total = lines * T;
  for (int b = threadIdx.x; b < total; b += blockDim.x) {
    const int line = b / T;
    const int i = b - line * T;
    const int k = i & (p - 1);
    const double2* s = src + line * ls;
    double2 a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = s[i + r * T];
    if (p > 1) {
      const int ts = n / (p * R);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const double2 w = twiddle<DIR>(master, r * k * ts, tstep_n);
        a[r] = cmulw(a[r], w.x, w.y);
      }
    }
    Dft<R, DIR>::run(a);
    const int j = (i - k) * R + k;
    double2* d = dst + line * ls;
#pragma unroll
    for (int r = 0; r < R; ++r) d[j + r * p] = a[r];
  }
}

// Full C2C of `lines` lines of length n in shared memory.  Data starts in
// buf0; returns the buffer (buf0 or buf1) holding the result.
template <int DIR>
__device__ inline double2* smem_c2c(double2* buf0, double2* buf1, int n, int lines, int ls,
                                    const double2* __restrict__ master) {
  int radix[8];
  const int np = fw_radices(n, radix);
  double2* src = buf0;
  double2* dst = buf1;
  int p = 1;
  for (int pass = 0; pass < np; ++pass) {
    const int R = radix[pass];
    switch (R) {
      case 16: stockham_pass<16, DIR>(src, dst, n, p, lines, ls, master); break;
      case 8: stockham_pass<8, DIR>(src, dst, n, p, lines, ls, master); break;
      case 4: stockham_pass<4, DIR>(src, dst, n, p, lines, ls, master); break;
      default: stockham_pass<2, DIR>(src, dst, n, p, lines, ls, master); break;
    }
    __syncthreads();
    double2* t = src;
    src = dst;
    dst = t;
    p *= R;
  }
  return src;
}

// R2C post-processing for bin k of a length-n real transform (h = n/2) from
// the half-length C2C result Z (fwcanon.c fwc_r2c).
__device__ __forceinline__ double2 r2c_post(const double2* Z, int k, int h, const double2* __restrict__ master) {
  if (k == 0) return make_double2(Z[0].x + Z[0].y, 0.0);
  if (k == h) return make_double2(Z[0].x - Z[0].y, 0.0);
  const double2 A = Z[k];
  const double2 Bz = Z[h - k];
  const double2 B = make_double2(Bz.x, -Bz.y);
  const double2 E = make_double2((A.x + B.x) * 0.5, (A.y + B.y) * 0.5);
  const double2 D = make_double2((A.x - B.x) * 0.5, (A.y - B.y) * 0.5);
  const double2 O = make_double2(D.y, -D.x);
  const double2 w = twiddle<-1>(master, k, 2 * h);
  const double2 t = cmulw(O, w.x, w.y);
  return make_double2(E.x + t.x, E.y + t.y);
}

// C2R pre-processing: Z[k] from bins X[k], X[h-k] (fwcanon.c fwc_c2r)
__device__ __forceinline__ double2 c2r_pre(double2 A, double2 Xhk, int k, int h, const double2* __restrict__ master) {
  double2 B = make_double2(Xhk.x, -Xhk.y);
  if (k == 0) {
    A.y = 0.0;
    B.y = 0.0;
  }
  const double2 E = make_double2(A.x + B.x, A.y + B.y);
  const double2 D = make_double2(A.x - B.x, A.y - B.y);
  const double2 w = twiddle<+1>(master, k, 2 * h);
  const double2 O = cmulw(D, w.x, w.y);
  return make_double2(E.x - O.y, E.y + O.x);
}

}  // namespace fw
