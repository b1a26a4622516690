/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product path.
 *
 * FFTW3 API shim for building the reference (/root/reference/proj) unmodified.
 * FFTW3 (third-party, version unpinned in proj/CMakeLists.txt:13-14, absent
 * from this image) is replaced by a restatement of the transform it computes:
 * the unnormalized rank-d DFT  X[k] = sum_j x[j] exp(sign * 2 pi i <j,k/n>),
 * row-major, in place or out of place, thread-safe new-array execute
 * (grid.hpp:49-51 relies on that).
 *
 * Execution paths (all compute the same DFT up to fp64 rounding):
 *  - real forward: sign = -1, every imaginary part exactly 0, all dims powers of
 *    two -> canonical R2C (fwcanon.c) on the half spectrum, the other half
 *    filled by exact conjugate mirroring.
 *  - Hermitian backward: sign = +1, X[k', n-p] == conj(X[-k', p]) exactly for
 *    0 < p < n/2 -> canonical C2C over axes 0..d-2 then C2R over the last axis.
 *    The imaginary part of the result is the exact remainder
 *    Im Y0[j'] + (-1)^j Im Yh[j'] from the p = 0 and p = n/2 planes.
 *  - general: canonical C2C (powers of two) or mixed-radix Cooley-Tukey along
 *    every axis.
 */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "fwcanon.h"

struct fwshim_plan_s {
  int rank;
  int n[3];
  int sign;
  fftw_complex* in;
  fftw_complex* out;
  int pow2;
  fwc_realnd real; /* valid when pow2 && last >= 4 */
  int real_ok;
  fwc_plan1d ax[3]; /* per-axis C2C plans when pow2 */
};

static long g_real_fwd = 0, g_herm_bwd = 0, g_general = 0;

void fwshim_stats(long* real_fwd, long* herm_bwd, long* general) {
  if (real_fwd) *real_fwd = __atomic_load_n(&g_real_fwd, __ATOMIC_RELAXED);
  if (herm_bwd) *herm_bwd = __atomic_load_n(&g_herm_bwd, __ATOMIC_RELAXED);
  if (general) *general = __atomic_load_n(&g_general, __ATOMIC_RELAXED);
}

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out,
                        int sign, unsigned flags) {
  (void)flags;
  if (rank < 1 || rank > 3) return NULL;
  struct fwshim_plan_s* p = (struct fwshim_plan_s*)calloc(1, sizeof(*p));
  p->rank = rank;
  p->sign = sign;
  p->in = in;
  p->out = out;
  p->pow2 = 1;
  for (int a = 0; a < rank; ++a) {
    p->n[a] = n[a];
    if (!fwc_is_pow2(n[a])) p->pow2 = 0;
  }
  if (p->pow2) {
    for (int a = 0; a < rank; ++a) fwc_plan1d_init(&p->ax[a], n[a]);
    p->real_ok = (n[rank - 1] >= 4) && fwc_realnd_init(&p->real, rank, n) == 0;
  }
  return p;
}

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
  return fftw_plan_dft(1, &n, in, out, sign, flags);
}

void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  if (p->pow2) {
    for (int a = 0; a < p->rank; ++a) fwc_plan1d_free(&p->ax[a]);
    if (p->real_ok) fwc_realnd_free(&p->real);
  }
  free(p);
}

/* ----------------------- general mixed-radix C2C -------------------------- */

static int smallest_factor(int n) {
  if (n % 4 == 0) return 4;
  if (n % 2 == 0) return 2;
  for (int f = 3; f * f <= n; f += 2)
    if (n % f == 0) return f;
  return n;
}

/* out[k] = sum_j x[j*stride] e^{sign 2 pi i jk/n}, recursive DIT */
static void mixed_fft(const fwc_cd* x, int n, long stride, fwc_cd* out, int sign) {
  if (n == 1) {
    out[0] = x[0];
    return;
  }
  const int r = smallest_factor(n);
  const int m = n / r;
  for (int q = 0; q < r; ++q) mixed_fft(x + q * stride, m, stride * r, out + q * m, sign);
  fwc_cd* t = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)r);
  fwc_cd* y = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)n);
  for (int k = 0; k < m; ++k) {
    for (int q = 0; q < r; ++q) {
      double c, s;
      fwc_twiddle((long)q * k, n, &c, &s);
      s *= sign;
      const fwc_cd a = out[q * m + k];
      t[q].re = a.re * c - a.im * s;
      t[q].im = a.re * s + a.im * c;
    }
    for (int sidx = 0; sidx < r; ++sidx) {
      double re = 0.0, im = 0.0;
      for (int q = 0; q < r; ++q) {
        double c, s;
        fwc_twiddle((long)q * sidx, r, &c, &s);
        s *= sign;
        re += t[q].re * c - t[q].im * s;
        im += t[q].re * s + t[q].im * c;
      }
      y[k + sidx * m].re = re;
      y[k + sidx * m].im = im;
    }
  }
  memcpy(out, y, sizeof(fwc_cd) * (size_t)n);
  free(t);
  free(y);
}

static void general_axis(struct fwshim_plan_s* p, fwc_cd* data, int a) {
  long inner = 1, outer = 1;
  for (int b = a + 1; b < p->rank; ++b) inner *= p->n[b];
  for (int b = 0; b < a; ++b) outer *= p->n[b];
  const int na = p->n[a];
  fwc_cd* line = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)na);
  fwc_cd* res = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)na);
  for (long o = 0; o < outer; ++o)
    for (long in = 0; in < inner; ++in) {
      fwc_cd* base = data + o * inner * na + in;
      for (int j = 0; j < na; ++j) line[j] = base[(long)j * inner];
      if (p->pow2) {
        fwc_c2c(&p->ax[a], line, res, p->sign);
      } else {
        mixed_fft(line, na, 1, res, p->sign);
        memcpy(line, res, sizeof(fwc_cd) * (size_t)na);
      }
      for (int j = 0; j < na; ++j) base[(long)j * inner] = line[j];
    }
  free(line);
  free(res);
}

/* index of the multi-index (-k') mod n over axes 0..rank-2 for row r */
static long neg_row(const struct fwshim_plan_s* p, long r) {
  long idx[3] = {0, 0, 0};
  long rem = r;
  for (int a = p->rank - 2; a >= 0; --a) {
    idx[a] = rem % p->n[a];
    rem /= p->n[a];
  }
  long out = 0;
  for (int a = 0; a <= p->rank - 2; ++a) out = out * p->n[a] + (idx[a] == 0 ? 0 : p->n[a] - idx[a]);
  return out;
}

static void real_forward(struct fwshim_plan_s* p, fwc_cd* data) {
  const int d = p->rank, nl = p->n[d - 1], h = nl / 2;
  long rows = 1;
  for (int a = 0; a + 1 < d; ++a) rows *= p->n[a];
  double* x = (double*)malloc(sizeof(double) * (size_t)rows * nl);
  for (long i = 0; i < rows * nl; ++i) x[i] = data[i].re;
  fwc_cd* H = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)rows * (h + 1));
  fwc_realnd_forward(&p->real, x, H);
  for (long r = 0; r < rows; ++r) {
    const long rn = neg_row(p, r);
    for (int q = 0; q < nl; ++q) {
      if (q <= h) {
        data[r * nl + q] = H[r * (h + 1) + q];
      } else {
        const fwc_cd v = H[rn * (h + 1) + (nl - q)];
        data[r * nl + q].re = v.re;
        data[r * nl + q].im = -v.im;
      }
    }
  }
  free(x);
  free(H);
}

static int hermitian_consistent(const struct fwshim_plan_s* p, const fwc_cd* data) {
  const int d = p->rank, nl = p->n[d - 1], h = nl / 2;
  long rows = 1;
  for (int a = 0; a + 1 < d; ++a) rows *= p->n[a];
  for (long r = 0; r < rows; ++r) {
    const long rn = neg_row(p, r);
    for (int q = 1; q < h; ++q) {
      const fwc_cd a = data[r * nl + (nl - q)];
      const fwc_cd b = data[rn * nl + q];
      if (!(a.re == b.re) || !(a.im == -b.im)) return 0;
    }
  }
  return 1;
}

static void hermitian_backward(struct fwshim_plan_s* p, fwc_cd* data) {
  const int d = p->rank, nl = p->n[d - 1], h = nl / 2;
  long rows = 1;
  for (int a = 0; a + 1 < d; ++a) rows *= p->n[a];
  fwc_cd* H = (fwc_cd*)malloc(sizeof(fwc_cd) * (size_t)rows * (h + 1));
  for (long r = 0; r < rows; ++r)
    for (int q = 0; q <= h; ++q) H[r * (h + 1) + q] = data[r * nl + q];
  double* x = (double*)malloc(sizeof(double) * (size_t)rows * nl);
  double* i0 = (double*)malloc(sizeof(double) * (size_t)rows);
  double* ih = (double*)malloc(sizeof(double) * (size_t)rows);
  fwc_realnd_backward(&p->real, H, x, i0, ih);
  for (long r = 0; r < rows; ++r)
    for (int j = 0; j < nl; ++j) {
      data[r * nl + j].re = x[r * nl + j];
      data[r * nl + j].im = (j & 1) ? i0[r] - ih[r] : i0[r] + ih[r];
    }
  free(H);
  free(x);
  free(i0);
  free(ih);
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  long N = 1;
  for (int a = 0; a < p->rank; ++a) N *= p->n[a];
  if (out != in) memcpy(out, in, sizeof(fftw_complex) * (size_t)N);
  fwc_cd* data = (fwc_cd*)out;
  if (p->real_ok && p->sign == FFTW_FORWARD) {
    int real = 1;
    for (long i = 0; i < N && real; ++i) real = (data[i].im == 0.0);
    if (real) {
      __atomic_fetch_add(&g_real_fwd, 1, __ATOMIC_RELAXED);
      real_forward(p, data);
      return;
    }
  }
  if (p->real_ok && p->sign == FFTW_BACKWARD && hermitian_consistent(p, data)) {
    __atomic_fetch_add(&g_herm_bwd, 1, __ATOMIC_RELAXED);
    hermitian_backward(p, data);
    return;
  }
  __atomic_fetch_add(&g_general, 1, __ATOMIC_RELAXED);
  if (p->sign == FFTW_FORWARD)
    for (int a = p->rank - 1; a >= 0; --a) general_axis(p, data, a);
  else
    for (int a = 0; a < p->rank; ++a) general_axis(p, data, a);
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }
