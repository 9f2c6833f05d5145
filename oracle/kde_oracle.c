/*
 * kde_oracle.c — TEST INFRASTRUCTURE ONLY.  Plain, slow, single-threaded fp64 oracle for the
 * all-pairs kernel sums of arxiv 1505.01998 (Andrzejewski, Gramacki & Gramacki).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load this.
 * It shares no code, header, table or constant with the CUDA path (paper_1505_01998_b200/).
 *
 * Every function is the plain definition written out: direct i<j double loops, libm exp,
 * Horner for the Hermite polynomials ("Horner's method"), Neumaier-compensated
 * fp64 accumulation (P:524 discusses summation error; compensation makes the oracle's own
 * rounding negligible).  Citations: P:NNN = /root/reference/PAPER.md line NNN.
 *
 * Row-range entry points (i0 <= i < i1, all j > i) exist so that a harness can split one sum
 * over several threads and add the parts in a fixed order; they compute exactly the same terms.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define ORACLE_PI 3.14159265358979323846264338327950288

typedef struct { double s, c; } nsum;   /* Neumaier running sum: value = s + c */

static void nadd(nsum *a, double t) {
  double u = a->s + t;
  if (fabs(a->s) >= fabs(t)) a->c += (a->s - u) + t;
  else a->c += (t - u) + a->s;
  a->s = u;
}

/* Probabilists' Hermite polynomials He_r(u), as polynomials in u^2, by Horner.
 * He_4 = u^4 - 6u^2 + 3            (Eq. PLUGIN-Psi4Estimate)
 * He_6 = u^6 - 15u^4 + 45u^2 - 15  (Eq. PLUGIN-Psi6Estimate)
 * He_8 = u^8 - 28u^6 + 210u^4 - 420u^2 + 105 (next member of the same family; needed by
 *        Psi_8, BASELINE.json north_star "Psi_4/Psi_6/Psi_8").  Returns NAN for other r. */
double oracle_hermite(int r, double u) {
  double s = u * u;
  switch (r) {
    case 0: return 1.0;
    case 2: return s - 1.0;
    case 4: return (s - 6.0) * s + 3.0;
    case 6: return ((s - 15.0) * s + 45.0) * s - 15.0;
    case 8: return (((s - 28.0) * s + 210.0) * s - 420.0) * s + 105.0;
    default: return NAN;
  }
}

/* K^(r)(u) = d^r/du^r of the Gaussian kernel = He_r(u) exp(-u^2/2) / sqrt(2 pi)
 * (Gaussian kernel P:120 Eq. gaussian). */
double oracle_kernel_deriv(int r, double u) {
  return oracle_hermite(r, u) * exp(-0.5 * u * u) / sqrt(2.0 * ORACLE_PI);
}

/* Raw double sum  sum_{i0<=i<i1} sum_{j>i} K^(r)((x_i - x_j)/g)   (RR_fun). */
int oracle_psi_pairsum_rows(const double *x, int64_t n, int r, double g, int64_t i0, int64_t i1,
                            double *out) {
  if (!x || !out || n < 1 || g <= 0.0 || !(r == 4 || r == 6 || r == 8)) return 1;
  nsum a = {0.0, 0.0};
  for (int64_t i = i0; i < i1 && i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) nadd(&a, oracle_kernel_deriv(r, (x[i] - x[j]) / g));
  *out = a.s + a.c;
  return 0;
}

/* Psi_r-hat(g) = [2 sum_{i<j} K^(r)((X_i-X_j)/g) + n K^(r)(0)] / (n^2 g^(r+1)).
 * P:227-231 (Eq. 15) and P:243-247 (Eq. 17) typeset "2/(n^2 g^7) SS K + n K(0)", which is
 * dimensionally inconsistent; reading Z1: the n K(0) diagonal term sits inside the
 * bracket (the standard estimator, i.e. the full i,j double sum including i=j). */
int oracle_psi_r(const double *x, int64_t n, int r, double g, double *psi) {
  double S;
  if (!psi || n < 1) return 1;
  if (oracle_psi_pairsum_rows(x, n, r, g, 0, n, &S)) return 1;
  *psi = (2.0 * S + (double)n * oracle_kernel_deriv(r, 0.0)) /
         ((double)n * (double)n * pow(g, r + 1));
  return 0;
}

/* q = v^T M v for a d-vector v and a dense row-major d x d matrix M (plain double loop). */
static double qform(const double *v, const double *M, int d) {
  double q = 0.0;
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) q += v[a] * M[a * d + b] * v[b];
  return q;
}

/* LSCV_h raw sums over pairs in rows [i0,i1) (unmodified form, Eq. 24-27):
 *   out[0] = sum_{i<j} exp(-1/4 u^T Sigma^-1 u)   ((K*K)(u) without its constant)
 *   out[1] = sum_{i<j} exp(-1/2 u^T Sigma^-1 u)   (K(u) without its constant)
 * with u = (X_i - X_j)/h; X is d x n row-major (Eq. 19); Sinv row-major d x d.
 * Two separate exp calls, as written. */
int oracle_lscv_h_pairsums_rows(const double *X, int64_t n, int d, const double *Sinv, double h,
                                int64_t i0, int64_t i1, double *out) {
  if (!X || !Sinv || !out || n < 1 || d < 1 || d > 16 || !(h > 0.0)) return 1;
  nsum a = {0.0, 0.0}, b = {0.0, 0.0};
  double u[16];
  for (int64_t i = i0; i < i1 && i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      for (int k = 0; k < d; ++k) u[k] = (X[k * n + i] - X[k * n + j]) / h;
      double q = qform(u, Sinv, d);
      nadd(&a, exp(-0.25 * q));
      nadd(&b, exp(-0.5 * q));
    }
  out[0] = a.s + a.c;
  out[1] = b.s + b.c;
  return 0;
}

/* LSCV_H raw sums over pairs in rows [i0,i1) (Eq. 30-33):
 *   out[0] = sum_{i<j} exp(-1/4 (X_i-X_j)^T H^-1 (X_i-X_j)),  out[1] = same with -1/2. */
int oracle_lscv_H_pairsums_rows(const double *X, int64_t n, int d, const double *Hinv,
                                int64_t i0, int64_t i1, double *out) {
  if (!X || !Hinv || !out || n < 1 || d < 1 || d > 16) return 1;
  nsum a = {0.0, 0.0}, b = {0.0, 0.0};
  double v[16];
  for (int64_t i = i0; i < i1 && i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      for (int k = 0; k < d; ++k) v[k] = X[k * n + i] - X[k * n + j];
      double q = qform(v, Hinv, d);
      nadd(&a, exp(-0.25 * q));
      nadd(&b, exp(-0.5 * q));
    }
  out[0] = a.s + a.c;
  out[1] = b.s + b.c;
  return 0;
}

/* The paper's modified LSCV_h (Sec. 4.5, Eq. 36-41), step by step:
 * (1) precompute S(v) = v^T Sigma^-1 v for every pair i<j into a triangular buffer (Eq. 37),
 * (2) for each h, sum T~(v) = (K~*K~)(v) - 2 K~(v) over the buffer (Eq. 38-40), where
 *     K~(v) = (2pi)^{-d/2}|Sigma|^{-1/2} exp(-S/(2h^2)), (K~*K~)(v) = (4pi)^{-d/2}|Sigma|^{-1/2}
 *     exp(-S/(4h^2)), and form g(h) = h^-d [2 n^-2 sum T~ + n^-1 R(K)] (Eq. 41) with
 *     R(K) = (4pi)^{-d/2}|Sigma|^{-1/2} (reading Z2).  Buffer order: row-major over i<j.
 * Used to pin the paper's claim that (41) equals (24).  Returns 2 if the buffer is too big. */
int oracle_lscv_h_modified(const double *X, int64_t n, int d, const double *Sinv, double detS,
                           const double *h, int nh, double *g) {
  if (!X || !Sinv || !h || !g || n < 2 || d < 1 || d > 16 || nh < 1 || !(detS > 0.0)) return 1;
  int64_t np = n * (n - 1) / 2;
  if (np > (int64_t)1 << 27) return 2;
  double *S = (double *)malloc(sizeof(double) * (size_t)np);
  if (!S) return 2;
  double v[16];
  int64_t t = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      for (int k = 0; k < d; ++k) v[k] = X[k * n + i] - X[k * n + j];
      S[t++] = qform(v, Sinv, d);
    }
  double c4 = pow(4.0 * ORACLE_PI, -0.5 * d) / sqrt(detS);
  double c2 = pow(2.0 * ORACLE_PI, -0.5 * d) / sqrt(detS);
  for (int c = 0; c < nh; ++c) {
    nsum a = {0.0, 0.0};
    double hh = h[c] * h[c];
    for (int64_t k = 0; k < np; ++k)
      nadd(&a, c4 * exp(-0.25 * S[k] / hh) - 2.0 * c2 * exp(-0.5 * S[k] / hh));
    double sumT = a.s + a.c;
    g[c] = pow(h[c], -d) * (2.0 * sumT / ((double)n * (double)n) + c4 / (double)n);
  }
  free(S);
  return 0;
}

/* Sample moments (plain two-pass definitions, Eq. 11 / Eq. 20-23 read as the unbiased sample
 * (co)variance, reading Z10): mean[d], cov[d*d] row-major. */
int oracle_mean_cov(const double *X, int64_t n, int d, double *mean, double *cov) {
  if (!X || !mean || !cov || n < 2 || d < 1 || d > 16) return 1;
  for (int a = 0; a < d; ++a) {
    nsum s = {0.0, 0.0};
    for (int64_t i = 0; i < n; ++i) nadd(&s, X[a * n + i]);
    mean[a] = (s.s + s.c) / (double)n;
  }
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      nsum s = {0.0, 0.0};
      for (int64_t i = 0; i < n; ++i) nadd(&s, (X[a * n + i] - mean[a]) * (X[b * n + i] - mean[b]));
      cov[a * d + b] = (s.s + s.c) / (double)(n - 1);
    }
  return 0;
}

/* The upper-triangular tile grid enumerated column by column (column l holds rows q=0..l),
 * i.e. the numbering of Fig. bx2lq that Eq. 42-43 invert (Appendix A):
 * writes (l,q) for bx = 0 .. count-1 by plain enumeration (the definition, not the closed form). */
int oracle_tile_enumerate(int64_t count, int64_t *l, int64_t *q) {
  if (count < 0 || !l || !q) return 1;
  int64_t bx = 0;
  for (int64_t col = 0; bx < count; ++col)
    for (int64_t row = 0; row <= col && bx < count; ++row, ++bx) { l[bx] = col; q[bx] = row; }
  return 0;
}

/* KDE evaluation (Eq. kde-def-H, K_H, gaussian):
 *   fhat(y) = n^-1 sum_i |H|^{-1/2} (2 pi)^{-d/2} exp(-1/2 (y - X_i)^T H^-1 (y - X_i)),
 * for m query points Y (d x m row-major); Hinv row-major, detH = |H|.  Plain double loop. */
int oracle_kde_eval(const double *X, int64_t n, int d, const double *Y, int64_t m,
                    const double *Hinv, double detH, double *f) {
  if (!X || !Y || !Hinv || !f || n < 1 || m < 0 || d < 1 || d > 16 || !(detH > 0.0)) return 1;
  double v[16];
  const double c = pow(2.0 * ORACLE_PI, -0.5 * d) / sqrt(detH);
  for (int64_t q = 0; q < m; ++q) {
    nsum a = {0.0, 0.0};
    for (int64_t i = 0; i < n; ++i) {
      for (int k = 0; k < d; ++k) v[k] = Y[k * m + q] - X[k * n + i];
      nadd(&a, c * exp(-0.5 * qform(v, Hinv, d)));
    }
    f[q] = (a.s + a.c) / (double)n;
  }
  return 0;
}
