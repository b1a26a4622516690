/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — see fw_oracle.h.
 *
 * Plain-C restatement of the fracwave hot path.  Every function cites the
 * reference lines it restates; the arithmetic is written in the same order as
 * the reference C++ (no contraction: built with -ffp-contract=off) so results
 * are bit-identical to the reference compiled against fwshim.
 */
#include "fw_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fwshim/fwcanon.h"

static _Thread_local char g_err[512];

const char* fwo_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

/* Grid::Grid validation (grid.cpp:35-58) + canonical-FFT support check */
static int check_grid(int d, const int* J, const double* lo, const double* hi) {
  if (d < 1 || d > 3) return fail(FWO_E_DIM_RANGE, "dimension must be 1, 2 or 3");
  for (int m = 0; m < d; ++m) {
    if (J[m] < 4 || J[m] % 2 != 0) return fail(FWO_E_ODD_SIZE, "point count must be even and >= 4");
    if (lo && hi && !(hi[m] > lo[m])) return fail(FWO_E_EMPTY_INTERVAL, "empty interval");
  }
  for (int m = 0; m < d; ++m)
    if (!fwc_is_pow2(J[m])) return fail(FWO_E_UNSUPPORTED, "canonical FFT needs power-of-two sizes");
  return FWO_OK;
}

static size_t total(int d, const int* J) {
  size_t N = 1;
  for (int m = 0; m < d; ++m) N *= (size_t)J[m];
  return N;
}

static size_t total_half(int d, const int* J) {
  return total(d, J) / (size_t)J[d - 1] * (size_t)(J[d - 1] / 2 + 1);
}

/* per-axis (base*k)^2 tables (grid.cpp:63-70) */
static double* axis_mu2(int d, const int* J, const double* lo, const double* hi) {
  size_t off = 0;
  for (int m = 0; m < d; ++m) off += (size_t)J[m];
  double* t = (double*)malloc(sizeof(double) * off);
  off = 0;
  for (int m = 0; m < d; ++m) {
    const double base = 2.0 * M_PI / (hi[m] - lo[m]);
    for (int p = 0; p < J[m]; ++p) {
      const int k = (p < J[m] / 2) ? p : p - J[m];
      t[off + p] = (base * k) * (base * k);
    }
    off += (size_t)J[m];
  }
  return t;
}

/* |mu|^2 at full-grid multi-index idx[] (grid.cpp:71-79: summed m = d-1 .. 0) */
static double mu2_at(int d, const int* J, const double* ax, const int* idx) {
  size_t off[3] = {0, 0, 0};
  for (int m = 1; m < d; ++m) off[m] = off[m - 1] + (size_t)J[m - 1];
  double v = 0.0;
  for (int m = d - 1; m >= 0; --m) v += ax[off[m] + idx[m]];
  return v;
}

int fwo_mu2(int d, const int* J, const double* lo, const double* hi, double* mu2) {
  int rc = check_grid(d, J, lo, hi);
  if (rc) return rc;
  double* ax = axis_mu2(d, J, lo, hi);
  const size_t N = total(d, J);
  for (size_t i = 0; i < N; ++i) {
    int idx[3] = {0, 0, 0};
    size_t rem = i;
    for (int m = d - 1; m >= 0; --m) {
      idx[m] = (int)(rem % (size_t)J[m]);
      rem /= (size_t)J[m];
    }
    mu2[i] = mu2_at(d, J, ax, idx);
  }
  free(ax);
  return FWO_OK;
}

/* |mu|^2 on the half spectrum [rows][J_last/2+1] */
static double* half_mu2(int d, const int* J, const double* lo, const double* hi) {
  double* ax = axis_mu2(d, J, lo, hi);
  const size_t Nh = total_half(d, J);
  const int hp1 = J[d - 1] / 2 + 1;
  double* out = (double*)malloc(sizeof(double) * Nh);
  for (size_t i = 0; i < Nh; ++i) {
    int idx[3] = {0, 0, 0};
    idx[d - 1] = (int)(i % (size_t)hp1);
    size_t rem = i / (size_t)hp1;
    for (int m = d - 2; m >= 0; --m) {
      idx[m] = (int)(rem % (size_t)J[m]);
      rem /= (size_t)J[m];
    }
    out[i] = mu2_at(d, J, ax, idx);
  }
  free(ax);
  return out;
}

int fwo_order_stats(const double* s, size_t N, const double* s0_override, double* s0,
                    double* smin, double* smax, int* constant_order) {
  /* std::min_element / max_element (orderfield.cpp:16-17) */
  double mn = s[0], mx = s[0];
  for (size_t i = 1; i < N; ++i) {
    if (s[i] < mn) mn = s[i];
    if (mx < s[i]) mx = s[i];
  }
  if (!(mn > 0.0) || !(mx < 2.0)) return fail(FWO_E_ORDER_RANGE, "order range outside (0, 2)");
  double z;
  if (s0_override) {
    z = *s0_override;
  } else if (mn == mx) {
    z = mn; /* orderfield.cpp:25-26 */
  } else {
    double sum = 0.0; /* serial sum in index order (orderfield.cpp:27-29) */
    for (size_t i = 0; i < N; ++i) sum += s[i];
    z = sum / (double)N;
  }
  const double dev = fmax(fabs(mn - z), fabs(mx - z));
  if (dev >= 1.0) return fail(FWO_E_DEVIATION, "max |s(x) - s0| >= 1; expansion would diverge");
  if (s0) *s0 = z;
  if (smin) *smin = mn;
  if (smax) *smax = mx;
  if (constant_order) *constant_order = (mx - mn <= 1e-14); /* orderfield.cpp:55-57 */
  return FWO_OK;
}

/* ------------------------------------------------------------------------- */
/* streaming operator: build_expansion tables regenerated per term            */

typedef struct {
  int d, J[3], M, constant_order;
  size_t N, Nh;
  double s0;
  fwc_realnd fft;
  double* mu2h;  /* half-spectrum |mu|^2 */
  double* base;  /* |mu|^{2 s0}, 0 at mu2 == 0 (flap.cpp:108-110) */
  double* logm;  /* log(mu2) where mu2 > 0 (flap.cpp:119) */
  double* dev1;  /* s - s0 (flap.cpp:127) */
} sop;

static void sop_free(sop* o) {
  fwc_realnd_free(&o->fft);
  free(o->mu2h);
  free(o->base);
  free(o->logm);
  free(o->dev1);
}

static int sop_init(sop* o, int d, const int* J, const double* lo, const double* hi,
                    const double* s, const double* s0_override, int M) {
  memset(o, 0, sizeof(*o));
  int rc = check_grid(d, J, lo, hi);
  if (rc) return rc;
  o->d = d;
  for (int m = 0; m < d; ++m) o->J[m] = J[m];
  o->N = total(d, J);
  o->Nh = total_half(d, J);
  double smin, smax;
  rc = fwo_order_stats(s, o->N, s0_override, &o->s0, &smin, &smax, &o->constant_order);
  if (rc) return rc;
  if (M < 0) return fail(FWO_E_NEGATIVE_M, "truncation count M must be >= 0");
  o->M = M;
  fwc_realnd_init(&o->fft, d, J);
  o->mu2h = half_mu2(d, J, lo, hi);
  o->base = (double*)malloc(sizeof(double) * o->Nh);
  o->logm = (double*)malloc(sizeof(double) * o->Nh);
  for (size_t k = 0; k < o->Nh; ++k) {
    const double m2 = o->mu2h[k];
    o->base[k] = m2 > 0.0 ? pow(m2, o->s0) : 0.0;
    o->logm[k] = m2 > 0.0 ? log(m2) : 0.0;
  }
  o->dev1 = (double*)malloc(sizeof(double) * o->N);
  for (size_t j = 0; j < o->N; ++j) o->dev1[j] = s[j] - o->s0;
  return FWO_OK;
}

/* apply_expansion (flap.cpp:38-92) */
static void sop_apply(const sop* o, const double* u, double* out, int m_first, double* residue) {
  const size_t N = o->N, Nh = o->Nh;
  const int nl = o->J[o->d - 1];
  const size_t rows = N / (size_t)nl;
  fwc_cd* H = (fwc_cd*)malloc(sizeof(fwc_cd) * Nh);
  fwc_cd* B = (fwc_cd*)malloc(sizeof(fwc_cd) * Nh);
  double* lw = (double*)calloc(Nh, sizeof(double));
  double* devm = (double*)malloc(sizeof(double) * N);
  double* x = (double*)malloc(sizeof(double) * N);
  double* i0 = (double*)malloc(sizeof(double) * rows);
  double* ih = (double*)malloc(sizeof(double) * rows);

  /* uhat = FFT(u) * (1/N)  (flap.cpp:46-50) */
  fwc_realnd_forward(&o->fft, u, H);
  const double inv = 1.0 / (double)N;
  for (size_t k = 0; k < Nh; ++k) {
    H[k].re *= inv;
    H[k].im *= inv;
  }
  const int m_last = o->constant_order ? 0 : o->M; /* flap.cpp:53 */
  for (size_t j = 0; j < N; ++j) out[j] = 0.0;
  double res = 0.0;
  for (int m = m_first; m <= m_last; ++m) {
    if (m >= 1) {
      /* log_weights recurrence (flap.cpp:115-122) */
      for (size_t k = 0; k < Nh; ++k) {
        if (o->mu2h[k] <= 0.0) continue;
        const double l = o->logm[k];
        lw[k] = (m == 1) ? l : lw[k] * l / m;
      }
      /* deviation_powers recurrence (flap.cpp:124-133) */
      if (m == 1)
        memcpy(devm, o->dev1, sizeof(double) * N);
      else
        for (size_t j = 0; j < N; ++j) devm[j] = devm[j] * o->dev1[j];
    }
    /* weight (flap.cpp:64-69) times uhat (flap.cpp:27) */
    for (size_t k = 0; k < Nh; ++k) {
      const double w = (m == 0) ? o->base[k] : o->base[k] * lw[k];
      B[k].re = w * H[k].re;
      B[k].im = w * H[k].im;
    }
    fwc_realnd_backward(&o->fft, B, x, i0, ih); /* flap.cpp:28 */
    for (size_t r = 0; r < rows; ++r) {       /* max |Im| (flap.cpp:32) */
      const double a = fabs(i0[r] + ih[r]), b = fabs(i0[r] - ih[r]);
      if (a > res) res = a;
      if (nl > 1 && b > res) res = b;
    }
    /* partial = 0 + devpow*re, then ascending-m reduction (flap.cpp:30-34, 82-89) */
    for (size_t j = 0; j < N; ++j) {
      double p = 0.0;
      p += (m == 0) ? x[j] : devm[j] * x[j];
      out[j] += p;
    }
  }
  if (residue) *residue = res;
  free(H);
  free(B);
  free(lw);
  free(devm);
  free(x);
  free(i0);
  free(ih);
}

int fwo_apply(int d, const int* J, const double* lo, const double* hi, const double* s,
              const double* s0_override, int M, int m_first, const double* u, double* out,
              double* imag_residue) {
  sop o;
  int rc = sop_init(&o, d, J, lo, hi, s, s0_override, M);
  if (rc) {
    sop_free(&o);
    return rc;
  }
  if (m_first >= 1 && o.constant_order) { /* flap.cpp:163-166 */
    for (size_t j = 0; j < o.N; ++j) out[j] = 0.0;
    if (imag_residue) *imag_residue = 0.0;
  } else {
    sop_apply(&o, u, out, m_first, imag_residue);
  }
  sop_free(&o);
  return FWO_OK;
}

int fwo_constant_order(int d, const int* J, const double* lo, const double* hi,
                       const double* u, double s, double* out) {
  if (!(s > 0.0) || !(s < 2.0)) return fail(FWO_E_ORDER_RANGE, "order s outside (0, 2)");
  int rc = check_grid(d, J, lo, hi);
  if (rc) return rc;
  fwc_realnd f;
  fwc_realnd_init(&f, d, J);
  const size_t N = total(d, J), Nh = total_half(d, J);
  double* m2 = half_mu2(d, J, lo, hi);
  fwc_cd* H = (fwc_cd*)malloc(sizeof(fwc_cd) * Nh);
  fwc_realnd_forward(&f, u, H); /* Grid::forward (grid.cpp:171-181) */
  const double inv = 1.0 / (double)N;
  for (size_t k = 0; k < Nh; ++k) {
    H[k].re *= inv;
    H[k].im *= inv;
    const double w = m2[k] > 0.0 ? pow(m2[k], s) : 0.0; /* flap.cpp:142-143 */
    H[k].re *= w;
    H[k].im *= w;
  }
  fwc_realnd_backward(&f, H, out, NULL, NULL); /* Grid::inverse (grid.cpp:183-197) */
  free(H);
  free(m2);
  fwc_realnd_free(&f);
  return FWO_OK;
}

/* ------------------------------------------------------------------------- */

int fwo_medium(int d, const int* J, const double* gamma, const double* c0, double omega0,
               double* c, double* eta, double* tau_coef) {
  const size_t N = total(d, J);
  for (size_t j = 0; j < N; ++j) /* seismic.cpp:14-19 */
    if (!(gamma[j] >= 0.0) || !(gamma[j] < 0.5))
      return fail(FWO_E_GAMMA_RANGE, "gamma outside [0, 0.5)");
  for (size_t j = 0; j < N; ++j) { /* seismic.cpp:30-39 */
    const double g = gamma[j];
    const double cg = c0[j];
    const double scale = pow(cg, 2.0 * g) * pow(omega0, -2.0 * g);
    c[j] = cg * cos(0.5 * M_PI * g);
    eta[j] = -scale * cos(M_PI * g);
    tau_coef[j] = -(scale / cg) * sin(M_PI * g);
  }
  return FWO_OK;
}

static double sup_norm(const double* f, size_t N) {
  double m = 0.0;
  for (size_t i = 0; i < N; ++i) m = fmax(m, fabs(f[i]));
  return m;
}

int fwo_seismic(int d, const int* J, const double* lo, const double* hi, const double* gamma,
                const double* c0, double omega0, int M, const double* phi, const double* psi,
                double tau, double blowup_factor, int nsteps, double* cur_out, double* prev_out,
                double* atten_prev_out, long* n_out) {
  int rc = check_grid(d, J, lo, hi);
  if (rc) return rc;
  const size_t N = total(d, J);
  double* c = (double*)malloc(sizeof(double) * N);
  double* eta = (double*)malloc(sizeof(double) * N);
  double* tc = (double*)malloc(sizeof(double) * N);
  rc = fwo_medium(d, J, gamma, c0, omega0, c, eta, tc);
  double* ord1 = (double*)malloc(sizeof(double) * N);
  double* ord2 = (double*)malloc(sizeof(double) * N);
  for (size_t j = 0; j < N && rc == FWO_OK; ++j) { /* seismic.cpp:37-38 */
    ord1[j] = 1.0 + gamma[j];
    ord2[j] = 0.5 + gamma[j];
  }
  sop A1, A2;
  memset(&A1, 0, sizeof(A1));
  memset(&A2, 0, sizeof(A2));
  if (rc == FWO_OK) rc = sop_init(&A1, d, J, lo, hi, ord1, NULL, M); /* seismic.cpp:41 */
  if (rc == FWO_OK) rc = sop_init(&A2, d, J, lo, hi, ord2, NULL, M); /* seismic.cpp:42 */
  double *prev = NULL, *cur = NULL, *ap = NULL, *l1 = NULL, *l2 = NULL, *nx = NULL;
  long n = 0;
  if (rc == FWO_OK) {
    prev = (double*)malloc(sizeof(double) * N);
    cur = (double*)malloc(sizeof(double) * N);
    ap = (double*)malloc(sizeof(double) * N);
    l1 = (double*)malloc(sizeof(double) * N);
    l2 = (double*)malloc(sizeof(double) * N);
    nx = (double*)malloc(sizeof(double) * N);
    /* constructor (seismic.cpp:85-109) */
    const double threshold = blowup_factor * fmax(sup_norm(phi, N), 1e-300);
    memcpy(prev, phi, sizeof(double) * N);
    sop_apply(&A1, phi, l1, 0, NULL);
    sop_apply(&A2, psi, l2, 0, NULL);
    for (size_t j = 0; j < N; ++j) {
      const double c2 = c[j] * c[j];
      cur[j] = phi[j] + tau * psi[j] + 0.5 * tau * tau * c2 * (eta[j] * l1[j] + tc[j] * l2[j]);
    }
    sop_apply(&A2, prev, ap, 0, NULL);
    n = 1;
    /* step() (seismic.cpp:111-133) */
    const double t2 = tau * tau;
    for (int s = 0; s < nsteps; ++s) {
      sop_apply(&A1, cur, l1, 0, NULL);
      sop_apply(&A2, cur, l2, 0, NULL);
      for (size_t j = 0; j < N; ++j) {
        const double c2 = c[j] * c[j];
        nx[j] = 2.0 * cur[j] - prev[j] + t2 * c2 * (eta[j] * l1[j] + tc[j] * (l2[j] - ap[j]) / tau);
      }
      ++n;
      const double sup = sup_norm(nx, N);
      if (!(sup <= threshold)) {
        snprintf(g_err, sizeof(g_err), "sup|u| = %g at step %ld", sup, n);
        rc = FWO_E_BLOWUP;
        break;
      }
      double* t = prev;
      prev = cur;
      cur = nx;
      nx = t;
      t = ap;
      ap = l2;
      l2 = t;
    }
    if (cur_out) memcpy(cur_out, cur, sizeof(double) * N);
    if (prev_out) memcpy(prev_out, prev, sizeof(double) * N);
    if (atten_prev_out) memcpy(atten_prev_out, ap, sizeof(double) * N);
  }
  if (n_out) *n_out = n;
  sop_free(&A1);
  sop_free(&A2);
  free(c); free(eta); free(tc); free(ord1); free(ord2);
  free(prev); free(cur); free(ap); free(l1); free(l2); free(nx);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* TSFP2 (stepping.cpp:106-131, 266-304)                                      */

static void osc_substep(fwc_cd* uh, fwc_cd* vh, double w, double dt) { /* stepping.cpp:106-117 */
  if (w == 0.0) {
    uh->re += dt * vh->re;
    uh->im += dt * vh->im;
    return;
  }
  const double c = cos(w * dt);
  const double s = sin(w * dt);
  const fwc_cd u0 = *uh, v0 = *vh;
  uh->re = u0.re * c + v0.re * (s / w);
  uh->im = u0.im * c + v0.im * (s / w);
  vh->re = -w * u0.re * s + v0.re * c;
  vh->im = -w * u0.im * s + v0.im * c;
}

int fwo_tsfp2(int d, const int* J, const double* lo, const double* hi, const double* s, int M,
              double kappa, int cubic, const double* phi, const double* psi, double tau,
              int nsteps, double* u_out, double* v_out) {
  sop A;
  int rc = sop_init(&A, d, J, lo, hi, s, NULL, M);
  if (rc) {
    sop_free(&A);
    return rc;
  }
  const size_t N = A.N, Nh = A.Nh;
  double* u = (double*)malloc(sizeof(double) * N);
  double* v = (double*)malloc(sizeof(double) * N);
  double* pert = (double*)malloc(sizeof(double) * N);
  double* w = (double*)malloc(sizeof(double) * Nh);
  fwc_cd* uh = (fwc_cd*)malloc(sizeof(fwc_cd) * Nh);
  fwc_cd* vh = (fwc_cd*)malloc(sizeof(fwc_cd) * Nh);
  memcpy(u, phi, sizeof(double) * N);
  memcpy(v, psi, sizeof(double) * N);
  const double threshold = 1e8 * fmax(sup_norm(phi, N), 1e-300); /* stepping.cpp:121 */
  for (size_t k = 0; k < Nh; ++k) /* stepping.cpp:125-131 */
    w[k] = A.mu2h[k] > 0.0 ? sqrt(kappa) * pow(A.mu2h[k], 0.5 * A.s0) : 0.0;
  const double inv = 1.0 / (double)N;
  const double half = 0.5 * tau;
  long n = 0;
  for (int st = 0; st < nsteps && rc == FWO_OK; ++st) {
    for (int flow = 0; flow < 2; ++flow) {
      if (flow == 1 && !(A.constant_order && !cubic)) { /* stepping.cpp:295-300 */
        if (A.constant_order)
          for (size_t j = 0; j < N; ++j) pert[j] = 0.0;
        else
          sop_apply(&A, u, pert, 1, NULL);
        for (size_t j = 0; j < N; ++j) {
          const double fu = cubic ? u[j] * u[j] * u[j] : 0.0;
          v[j] += tau * (-kappa * pert[j] + fu);
        }
      }
      /* oscillator_flow(tau/2) (stepping.cpp:271-291) */
      fwc_realnd_forward(&A.fft, u, uh);
      fwc_realnd_forward(&A.fft, v, vh);
      for (size_t k = 0; k < Nh; ++k) {
        uh[k].re *= inv;
        uh[k].im *= inv;
        vh[k].re *= inv;
        vh[k].im *= inv;
        osc_substep(&uh[k], &vh[k], w[k], half);
      }
      fwc_realnd_backward(&A.fft, uh, u, NULL, NULL);
      fwc_realnd_backward(&A.fft, vh, v, NULL, NULL);
    }
    ++n;
    if (!(sup_norm(u, N) <= threshold)) rc = fail(FWO_E_BLOWUP, "TSFP2 blow-up");
  }
  memcpy(u_out, u, sizeof(double) * N);
  memcpy(v_out, v, sizeof(double) * N);
  free(u); free(v); free(pert); free(w); free(uh); free(vh);
  sop_free(&A);
  return rc;
}

int fwo_rfftn(int d, const int* J, const double* x, double* H) {
  int rc = check_grid(d, J, NULL, NULL);
  if (rc) return rc;
  fwc_realnd f;
  fwc_realnd_init(&f, d, J);
  fwc_realnd_forward(&f, x, (fwc_cd*)H);
  fwc_realnd_free(&f);
  return FWO_OK;
}

int fwo_irfftn(int d, const int* J, const double* H, double* x) {
  int rc = check_grid(d, J, NULL, NULL);
  if (rc) return rc;
  fwc_realnd f;
  fwc_realnd_init(&f, d, J);
  const size_t Nh = total_half(d, J);
  fwc_cd* tmp = (fwc_cd*)malloc(sizeof(fwc_cd) * Nh);
  memcpy(tmp, H, sizeof(fwc_cd) * Nh);
  fwc_realnd_backward(&f, tmp, x, NULL, NULL);
  free(tmp);
  fwc_realnd_free(&f);
  return FWO_OK;
}
