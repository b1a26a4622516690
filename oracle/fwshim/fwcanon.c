/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.  Canonical fp64 FFT (see fwcanon.h and
 * DESIGN.md §3).  Compile with -ffp-contract=off: the only fused operations
 * are the explicit fma() calls below.
 */
#include "fwcanon.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define C_SQRT1_2 0.70710678118654752440084436210484904
#define C_COS_PI_8 0.92387953251128675612818318939678829
#define C_SIN_PI_8 0.38268343236508977172845998403039887

int fwc_is_pow2(long n) { return n >= 1 && (n & (n - 1)) == 0; }

void fwc_twiddle(long t, long n, double* c, double* s) {
  t %= n;
  if (t < 0) t += n;
  if (t == 0) {
    *c = 1.0;
    *s = 0.0;
    return;
  }
  if (n % 4 != 0) {
    if (2 * t == n) {
      *c = -1.0;
      *s = 0.0;
      return;
    }
    const double ang = (2.0 * M_PI) * ((double)t / (double)n);
    *c = cos(ang);
    *s = sin(ang);
    return;
  }
  const long quarter = n / 4;
  const long q = t / quarter;
  const long tq = t - q * quarter; /* [0, n/4) */
  double cc, ss;
  if (tq == 0) {
    cc = 1.0;
    ss = 0.0;
  } else if (8 * tq <= n) {
    const double ang = (2.0 * M_PI) * ((double)tq / (double)n);
    cc = cos(ang);
    ss = sin(ang);
  } else {
    const long tr = quarter - tq;
    const double ang = (2.0 * M_PI) * ((double)tr / (double)n);
    cc = sin(ang);
    ss = cos(ang);
  }
  switch (q) {
    case 0: *c = cc; *s = ss; break;
    case 1: *c = -ss; *s = cc; break;
    case 2: *c = -cc; *s = -ss; break;
    default: *c = ss; *s = -cc; break;
  }
}

int fwc_radices(int n, int* radix) {
  int L = 0;
  while ((1 << L) < n) ++L;
  if (L == 0) return 0;
  const int P = (L + 3) / 4;
  const int base = L / P, extra = L % P;
  for (int i = 0; i < P; ++i) radix[i] = 1 << (base + (i < extra ? 1 : 0));
  return P;
}

void fwc_plan1d_init(fwc_plan1d* p, int n) {
  memset(p, 0, sizeof(*p));
  p->n = n;
  p->npass = fwc_radices(n, p->radix);
  p->tw = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)(n > 0 ? n : 1));
  for (int t = 0; t < n; ++t) fwc_twiddle(t, n, &p->tw[t].re, &p->tw[t].im);
}

void fwc_plan1d_free(fwc_plan1d* p) {
  free(p->tw);
  p->tw = NULL;
}

/* ---- complex helpers (exact expression forms are part of the definition) ---- */
static inline fwc_cd cadd(fwc_cd a, fwc_cd b) { fwc_cd r = {a.re + b.re, a.im + b.im}; return r; }
static inline fwc_cd csub(fwc_cd a, fwc_cd b) { fwc_cd r = {a.re - b.re, a.im - b.im}; return r; }
/* a * w with w = (wr, wi) */
static inline fwc_cd cmulw(fwc_cd a, double wr, double wi) {
  fwc_cd r = {fma(a.re, wr, -(a.im * wi)), fma(a.re, wi, a.im * wr)};
  return r;
}
/* multiply by dir*i */
static inline fwc_cd rot(fwc_cd a, int dir) {
  fwc_cd r;
  if (dir < 0) { r.re = a.im; r.im = -a.re; }
  else { r.re = -a.im; r.im = a.re; }
  return r;
}
/* multiply by W8^1 = (c, dir c) */
static inline fwc_cd w8_1(fwc_cd x, int dir) {
  fwc_cd r;
  if (dir < 0) { r.re = (x.re + x.im) * C_SQRT1_2; r.im = (x.im - x.re) * C_SQRT1_2; }
  else { r.re = (x.re - x.im) * C_SQRT1_2; r.im = (x.im + x.re) * C_SQRT1_2; }
  return r;
}
/* multiply by W8^3 = (-c, dir c) */
static inline fwc_cd w8_3(fwc_cd x, int dir) {
  fwc_cd r;
  if (dir < 0) { r.re = (x.im - x.re) * C_SQRT1_2; r.im = -((x.re + x.im) * C_SQRT1_2); }
  else { r.re = -((x.re + x.im) * C_SQRT1_2); r.im = (x.re - x.im) * C_SQRT1_2; }
  return r;
}

static inline void dft2(fwc_cd* a) {
  fwc_cd t = a[0];
  a[0] = cadd(t, a[1]);
  a[1] = csub(t, a[1]);
}

/* in: x0..x3 (may alias out) */
static inline void dft4v(fwc_cd x0, fwc_cd x1, fwc_cd x2, fwc_cd x3, int dir, fwc_cd* out) {
  const fwc_cd t0 = cadd(x0, x2), t1 = csub(x0, x2);
  const fwc_cd t2 = cadd(x1, x3), t3 = rot(csub(x1, x3), dir);
  out[0] = cadd(t0, t2);
  out[1] = cadd(t1, t3);
  out[2] = csub(t0, t2);
  out[3] = csub(t1, t3);
}

static inline void dft4(fwc_cd* a, int dir) { dft4v(a[0], a[1], a[2], a[3], dir, a); }

static inline void dft8(fwc_cd* a, int dir) {
  fwc_cd E[4], O[4];
  dft4v(a[0], a[2], a[4], a[6], dir, E);
  dft4v(a[1], a[3], a[5], a[7], dir, O);
  O[1] = w8_1(O[1], dir);
  O[2] = rot(O[2], dir);
  O[3] = w8_3(O[3], dir);
  for (int k = 0; k < 4; ++k) {
    a[k] = cadd(E[k], O[k]);
    a[k + 4] = csub(E[k], O[k]);
  }
}

static inline fwc_cd w16(fwc_cd x, int e, int dir) {
  const double sd = dir < 0 ? -1.0 : 1.0;
  switch (e) {
    case 0: return x;
    case 1: return cmulw(x, C_COS_PI_8, sd * C_SIN_PI_8);
    case 2: return w8_1(x, dir);
    case 3: return cmulw(x, C_SIN_PI_8, sd * C_COS_PI_8);
    case 4: return rot(x, dir);
    case 6: return w8_3(x, dir);
    default: /* 9 */ return cmulw(x, -C_COS_PI_8, -(sd * C_SIN_PI_8));
  }
}

static inline void dft16(fwc_cd* a, int dir) {
  fwc_cd F[4][4];
  for (int j2 = 0; j2 < 4; ++j2) dft4v(a[j2], a[j2 + 4], a[j2 + 8], a[j2 + 12], dir, F[j2]);
  for (int j2 = 1; j2 < 4; ++j2)
    for (int k1 = 1; k1 < 4; ++k1) F[j2][k1] = w16(F[j2][k1], j2 * k1, dir);
  for (int k1 = 0; k1 < 4; ++k1) {
    fwc_cd X[4];
    dft4v(F[0][k1], F[1][k1], F[2][k1], F[3][k1], dir, X);
    for (int k2 = 0; k2 < 4; ++k2) a[k1 + 4 * k2] = X[k2];
  }
}

static inline void dftR(fwc_cd* a, int R, int dir) {
  switch (R) {
    case 2: dft2(a); break;
    case 4: dft4(a, dir); break;
    case 8: dft8(a, dir); break;
    default: dft16(a, dir); break;
  }
}

void fwc_c2c(const fwc_plan1d* P, fwc_cd* x, fwc_cd* scratch, int dir) {
  const int n = P->n;
  if (n <= 1) return;
  fwc_cd* src = x;
  fwc_cd* dst = scratch;
  int p = 1;
  const double sd = dir < 0 ? -1.0 : 1.0;
  for (int pass = 0; pass < P->npass; ++pass) {
    const int R = P->radix[pass];
    const int T = n / R;
    const int tstep = n / (p * R);
    for (int i = 0; i < T; ++i) {
      const int k = i & (p - 1);
      fwc_cd a[16];
      for (int r = 0; r < R; ++r) a[r] = src[i + r * T];
      if (p > 1) {
        for (int r = 1; r < R; ++r) {
          const fwc_cd w = P->tw[(long)r * k * tstep];
          a[r] = cmulw(a[r], w.re, sd * w.im);
        }
      }
      dftR(a, R, dir);
      const int j = (i - k) * R + k;
      for (int r = 0; r < R; ++r) dst[j + r * p] = a[r];
    }
    fwc_cd* t = src;
    src = dst;
    dst = t;
    p *= R;
  }
  if (src != x) memcpy(x, src, sizeof(fwc_cd) * (size_t)n);
}

void fwc_r2c(const fwc_plan1d* half, const fwc_cd* twn, const double* x, fwc_cd* X,
             fwc_cd* scratch) {
  const int h = half->n;
  for (int j = 0; j < h; ++j) {
    X[j].re = x[2 * j];
    X[j].im = x[2 * j + 1];
  }
  fwc_c2c(half, X, scratch, -1);
  /* post-process in a copy of Z (X holds Z[0..h-1]) */
  fwc_cd* Z = scratch;
  memcpy(Z, X, sizeof(fwc_cd) * (size_t)h);
  X[0].re = Z[0].re + Z[0].im;
  X[0].im = 0.0;
  X[h].re = Z[0].re - Z[0].im;
  X[h].im = 0.0;
  for (int k = 1; k < h; ++k) {
    const fwc_cd A = Z[k];
    const fwc_cd B = {Z[h - k].re, -Z[h - k].im};
    const fwc_cd E = {(A.re + B.re) * 0.5, (A.im + B.im) * 0.5};
    const fwc_cd D = {(A.re - B.re) * 0.5, (A.im - B.im) * 0.5};
    const fwc_cd O = {D.im, -D.re};
    const fwc_cd t = cmulw(O, twn[k].re, -twn[k].im);
    X[k].re = E.re + t.re;
    X[k].im = E.im + t.im;
  }
}

void fwc_c2r(const fwc_plan1d* half, const fwc_cd* twn, const fwc_cd* X, double* x,
             fwc_cd* scratch) {
  const int h = half->n;
  fwc_cd* Z = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)h);
  for (int k = 0; k < h; ++k) {
    fwc_cd A = X[k];
    fwc_cd B = {X[h - k].re, -X[h - k].im};
    if (k == 0) {
      A.im = 0.0;
      B.im = 0.0;
    }
    const fwc_cd E = {A.re + B.re, A.im + B.im};
    const fwc_cd D = {A.re - B.re, A.im - B.im};
    const fwc_cd O = cmulw(D, twn[k].re, twn[k].im);
    Z[k].re = E.re - O.im;
    Z[k].im = E.im + O.re;
  }
  fwc_c2c(half, Z, scratch, +1);
  for (int j = 0; j < h; ++j) {
    x[2 * j] = Z[j].re;
    x[2 * j + 1] = Z[j].im;
  }
  free(Z);
}

/* ---------------------------- multi-dimensional ---------------------------- */

int fwc_realnd_init(fwc_realnd* p, int d, const int* n) {
  memset(p, 0, sizeof(*p));
  if (d < 1 || d > 3) return -1;
  p->d = d;
  for (int a = 0; a < d; ++a) {
    if (!fwc_is_pow2(n[a]) || n[a] < 2) return -1;
    p->n[a] = n[a];
  }
  if (n[d - 1] < 4) return -1;
  for (int a = 0; a < d; ++a) fwc_plan1d_init(&p->ax[a], n[a]);
  fwc_plan1d_init(&p->half, n[d - 1] / 2);
  return 0;
}

void fwc_realnd_free(fwc_realnd* p) {
  for (int a = 0; a < p->d; ++a) fwc_plan1d_free(&p->ax[a]);
  fwc_plan1d_free(&p->half);
}

size_t fwc_realnd_nhalf(const fwc_realnd* p) {
  size_t rows = 1;
  for (int a = 0; a + 1 < p->d; ++a) rows *= (size_t)p->n[a];
  return rows * (size_t)(p->n[p->d - 1] / 2 + 1);
}

/* C2C along axis a (< d-1) of the half-spectrum array H */
static void half_axis_pass(const fwc_realnd* p, fwc_cd* H, int a, int dir) {
  const int d = p->d;
  const size_t hp1 = (size_t)(p->n[d - 1] / 2 + 1);
  size_t inner = hp1; /* stride of axis a */
  for (int b = a + 1; b < d - 1; ++b) inner *= (size_t)p->n[b];
  size_t outer = 1;
  for (int b = 0; b < a; ++b) outer *= (size_t)p->n[b];
  const int na = p->n[a];
  const long total = (long)(outer * inner);
#pragma omp parallel
  {
    fwc_cd* line = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)na);
    fwc_cd* scr = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)na);
#pragma omp for schedule(static)
    for (long li = 0; li < total; ++li) {
      const size_t o = (size_t)li / inner, in = (size_t)li % inner;
      fwc_cd* base = H + o * inner * (size_t)na + in;
      for (int j = 0; j < na; ++j) line[j] = base[(size_t)j * inner];
      fwc_c2c(&p->ax[a], line, scr, dir);
      for (int j = 0; j < na; ++j) base[(size_t)j * inner] = line[j];
    }
    free(line);
    free(scr);
  }
}

void fwc_realnd_forward(const fwc_realnd* p, const double* x, fwc_cd* H) {
  const int d = p->d;
  const int nl = p->n[d - 1];
  const int h = nl / 2;
  size_t rows = 1;
  for (int a = 0; a + 1 < d; ++a) rows *= (size_t)p->n[a];
#pragma omp parallel
  {
    fwc_cd* scr = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)h);
#pragma omp for schedule(static)
    for (long r = 0; r < (long)rows; ++r)
      fwc_r2c(&p->half, p->ax[d - 1].tw, x + (size_t)r * nl, H + (size_t)r * (h + 1), scr);
    free(scr);
  }
  for (int a = d - 2; a >= 0; --a) half_axis_pass(p, H, a, -1);
}

void fwc_realnd_backward(const fwc_realnd* p, fwc_cd* H, double* x, double* imag0,
                         double* imagh) {
  const int d = p->d;
  const int nl = p->n[d - 1];
  const int h = nl / 2;
  size_t rows = 1;
  for (int a = 0; a + 1 < d; ++a) rows *= (size_t)p->n[a];
  for (int a = 0; a <= d - 2; ++a) half_axis_pass(p, H, a, +1);
#pragma omp parallel
  {
    fwc_cd* scr = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)h);
#pragma omp for schedule(static)
    for (long r = 0; r < (long)rows; ++r) {
      const fwc_cd* Hr = H + (size_t)r * (h + 1);
      if (imag0) imag0[r] = Hr[0].im;
      if (imagh) imagh[r] = Hr[h].im;
      fwc_c2r(&p->half, p->ax[d - 1].tw, Hr, x + (size_t)r * nl, scr);
    }
    free(scr);
  }
}
