/*
 * oracle.c -- plain CPU oracle for RQLP / ERQLP / BRQLP (arXiv:1811.09334).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Shares no code with the CUDA product.
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -fPIC -shared oracle.c -lm
 *
 * Every function follows the paper's algorithm step by step in its order and notation; the
 * only parallelism is OpenMP over independent output rows/columns, which leaves each output's
 * summation order fixed (ascending index).  Pins: tests/test_oracle_pins.py.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define IDX(i, j, ld) ((size_t)(i) + (size_t)(j) * (size_t)(ld))

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of the following calls (bench.py's single-thread cpu_baseline sample); no arithmetic. */
void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ======================================================================================
 * Ω generator.  DESIGN.md §4: Philox4x64-10 (Salmon et al. SC'11), key = (seed, 0),
 * counter = (block, stream, 0, 0); uniforms u(x) = ((x>>12)+0.5)*2^-52; Box-Muller with both
 * outputs used; ln and sin/cos pinned to a fixed sequence of IEEE ops.
 * Alg.1 l.1 draws Ω Gaussian (reading R1).
 * ==================================================================================== */
static const uint64_t PHILOX_M0 = 0xD2E7470EE14C6C93ULL;
static const uint64_t PHILOX_M1 = 0xCA5A826395121157ULL;
static const uint64_t PHILOX_W0 = 0x9E3779B97F4A7C15ULL;
static const uint64_t PHILOX_W1 = 0xBB67AE8584CAA73BULL;

void orc_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
  uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint64_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
    unsigned __int128 p0 = (unsigned __int128)PHILOX_M0 * c0;
    unsigned __int128 p1 = (unsigned __int128)PHILOX_M1 * c2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

double orc_uniform(uint64_t x) { return ((double)(x >> 12) + 0.5) * 0x1p-52; }

/* ln(u), u in (0,1) normal: u = 2^e f, f in [sqrt(1/2), sqrt(2)); s = (f-1)/(f+1);
 * ln f = 2s + 2s s^2 P(s^2), P = atanh Taylor coefficients 1/3 .. 1/25 (Horner, fma);
 * ln u = e ln2_hi + (e ln2_lo + ln f).  Constants are the correctly rounded values. */
static const double LN_C[12] = {
    0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4,
    0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
    0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5, 0x1.47ae147ae147bp-5};
static const double LN2_HI = 0x1.62e42fee00000p-1;
static const double LN2_LO = 0x1.a39ef35793c76p-33;
static const double SQRT2 = 0x1.6a09e667f3bcdp+0;

double orc_ln(double u) {
  uint64_t bits;
  memcpy(&bits, &u, 8);
  int64_t e = (int64_t)((bits >> 52) & 0x7ff) - 1023;
  uint64_t mbits = (bits & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
  double f;
  memcpy(&f, &mbits, 8);
  if (f > SQRT2) {
    f = f * 0.5;
    e += 1;
  }
  double s = (f - 1.0) / (f + 1.0);
  double z = s * s;
  double P = LN_C[11];
  for (int i = 10; i >= 0; --i) P = fma(P, z, LN_C[i]);
  double t = s + s;
  double tz = t * z;
  double lnf = fma(tz, P, t);
  double ed = (double)e;
  double lo = fma(ed, LN2_LO, lnf);
  return fma(ed, LN2_HI, lo);
}

/* sin/cos(2*pi*u), u = (K+0.5) 2^-52, K = x>>12.  4u = q + r exactly with q = nearest integer
 * (integer arithmetic), phi = r*(pi/2) in [-pi/4, pi/4], Taylor polynomials to phi^19 / phi^20,
 * quadrant rotation by q mod 4. */
static const double SIN_C[9] = {-0x1.5555555555555p-3, 0x1.1111111111111p-7, -0x1.a01a01a01a01ap-13,
                                 0x1.71de3a556c734p-19, -0x1.ae64567f544e4p-26, 0x1.6124613a86d09p-33,
                                 -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49, -0x1.2f49b46814157p-57};
static const double COS_C[10] = {-0x1.0000000000000p-1, 0x1.5555555555555p-5, -0x1.6c16c16c16c17p-10,
                                  0x1.a01a01a01a01ap-16, -0x1.27e4fb7789f5cp-22, 0x1.1eed8eff8d898p-29,
                                  -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45, -0x1.6827863b97d97p-53,
                                  0x1.e542ba4020225p-62};
static const double PIO2 = 0x1.921fb54442d18p+0;

void orc_sincos_2pi(uint64_t x, double *sout, double *cout) {
  uint64_t K = x >> 12;                         /* u = (K + 0.5) 2^-52, 4u = (K + 0.5) 2^-50 */
  uint64_t q = (K + (1ULL << 49)) >> 50;        /* nearest integer to 4u (no ties possible) */
  int64_t rk = (int64_t)K - (int64_t)(q << 50); /* |rk| <= 2^49 */
  double r = ((double)rk + 0.5) * 0x1p-50;      /* exact, r in (-1/2, 1/2) */
  double phi = r * PIO2;
  double z = phi * phi;
  double S = SIN_C[8];
  for (int i = 7; i >= 0; --i) S = fma(S, z, SIN_C[i]);
  double sp = fma(phi * z, S, phi);
  double C = COS_C[9];
  for (int i = 8; i >= 0; --i) C = fma(C, z, COS_C[i]);
  double cp = fma(z, C, 1.0);
  switch (q & 3) {
    case 0: *sout = sp; *cout = cp; break;
    case 1: *sout = cp; *cout = -sp; break;
    case 2: *sout = -sp; *cout = -cp; break;
    default: *sout = -cp; *cout = sp; break;
  }
}

void orc_normal4(uint64_t seed, uint64_t stream, uint64_t block, double z[4]) {
  const uint64_t ctr[4] = {block, stream, 0, 0};
  const uint64_t key[2] = {seed, 0};
  uint64_t x[4];
  orc_philox4x64_10(ctr, key, x);
  for (int h = 0; h < 2; ++h) {
    double ua = orc_uniform(x[2 * h]);
    double rho = sqrt(-2.0 * orc_ln(ua));
    double s, c;
    orc_sincos_2pi(x[2 * h + 1], &s, &c);
    z[2 * h] = rho * c;
    z[2 * h + 1] = rho * s;
  }
}

void orc_gaussian(uint64_t seed, uint64_t stream, int64_t rows, int64_t cols, double *M, int64_t ld) {
  int64_t total = rows * cols;
  int64_t nblocks = (total + 3) / 4;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nblocks; ++b) {
    double z[4];
    orc_normal4(seed, stream, (uint64_t)b, z);
    for (int r = 0; r < 4; ++r) {
      int64_t t = 4 * b + r;
      if (t < total) M[IDX(t % rows, t / rows, ld)] = z[r];
    }
  }
}

/* ======================================================================================
 * Dense building blocks (plain loops; summation index ascending).
 * ==================================================================================== */
void orc_gemm_nn(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda, const double *B,
                 int64_t ldb, double *C, int64_t ldc) {
  const int64_t RB = 256;
  int64_t nrb = (m + RB - 1) / RB;
#pragma omp parallel for schedule(static)
  for (int64_t rb = 0; rb < nrb; ++rb) {
    int64_t i0 = rb * RB, i1 = i0 + RB < m ? i0 + RB : m;
    for (int64_t j = 0; j < n; ++j) {
      double *c = C + IDX(0, j, ldc);
      for (int64_t i = i0; i < i1; ++i) c[i] = 0.0;
      for (int64_t p = 0; p < k; ++p) {
        double b = B[IDX(p, j, ldb)];
        const double *a = A + IDX(0, p, lda);
        for (int64_t i = i0; i < i1; ++i) c[i] += a[i] * b;
      }
    }
  }
}

void orc_gemm_tn(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda, const double *B,
                 int64_t ldb, double *C, int64_t ldc) {
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      const double *a = A + IDX(0, i, lda), *b = B + IDX(0, j, ldb);
      double s = 0.0;
      for (int64_t p = 0; p < k; ++p) s += a[p] * b[p];
      C[IDX(i, j, ldc)] = s;
    }
}

void orc_gemm_nt(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda, const double *B,
                 int64_t ldb, double *C, int64_t ldc) {
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      double s = 0.0;
      for (int64_t p = 0; p < k; ++p) s += A[IDX(i, p, lda)] * B[IDX(j, p, ldb)];
      C[IDX(i, j, ldc)] = s;
    }
}

double orc_fro(int64_t m, int64_t n, const double *A, int64_t lda) {
  double *colsum = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += A[IDX(i, j, lda)] * A[IDX(i, j, lda)];
    colsum[j] = s;
  }
  double s = 0.0;
  for (int64_t j = 0; j < n; ++j) s += colsum[j];
  free(colsum);
  return sqrt(s);
}

static double norm2(int64_t len, const double *x) {
  double s = 0.0;
  for (int64_t i = 0; i < len; ++i) s += x[i] * x[i];
  return sqrt(s);
}

/* Householder reflector (LAPACK xLARFG without rescaling): x = [alpha; x2] (length len) is
 * overwritten by [beta; v2] with H = I - tau v v^T, v = [1; v2], H x = beta e1.
 * x2 == 0 gives tau = 0 (H = I) and beta = alpha (reading R21). */
static void house(int64_t len, double *x, double *tau) {
  double alpha = x[0];
  double xnorm = len > 1 ? norm2(len - 1, x + 1) : 0.0;
  if (xnorm == 0.0) {
    *tau = 0.0;
    return;
  }
  double beta = -copysign(sqrt(alpha * alpha + xnorm * xnorm), alpha);
  *tau = (beta - alpha) / beta;
  double scal = 1.0 / (alpha - beta);
  for (int64_t i = 1; i < len; ++i) x[i] *= scal;
  x[0] = beta;
}

/* c <- (I - tau v v^T) c on rows j..m-1, v = [1; V(j+1:m, j)]. */
static void apply_house(int64_t len, const double *v, double tau, double *c) {
  if (tau == 0.0) return;
  double w = c[0];
  for (int64_t i = 1; i < len; ++i) w += v[i] * c[i];
  w *= tau;
  c[0] -= w;
  for (int64_t i = 1; i < len; ++i) c[i] -= w * v[i];
}

/* Explicit thin Q (m x s) from reflectors stored below the diagonal of W (xORG2R order):
 * Q = H_0 H_1 ... H_{s-1} I(:, 0:s). */
static void form_q(int64_t m, int64_t s, const double *W, int64_t ldw, const double *tau, double *Q,
                   int64_t ldq) {
  for (int64_t j = 0; j < s; ++j)
    for (int64_t i = 0; i < m; ++i) Q[IDX(i, j, ldq)] = (i == j) ? 1.0 : 0.0;
  for (int64_t j = s - 1; j >= 0; --j) {
    const double *v = W + IDX(j, j, ldw);
#pragma omp parallel for schedule(static)
    for (int64_t c = j; c < s; ++c) apply_house(m - j, v, tau[j], Q + IDX(j, c, ldq));
  }
}

/* Core Householder QR with optional column pivoting, in place on W (m x n).
 * Pivoting (reading R5): at step j choose the remaining column with the
 * largest downdated norm, ties -> lowest ORIGINAL column index; swap; reflect; downdate the
 * norms with the xLAQP2 rule (tol3z = sqrt(2^-53)). */
static void qr_core(int64_t m, int64_t n, double *W, int64_t ldw, double *tau, int64_t *perm, int pivot,
                    int64_t steps) {
  int64_t s = m < n ? m : n;
  if (steps >= 0 && steps < s) s = steps; /* partial (truncated) factorisation */
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  double *vn1 = NULL, *vn2 = NULL;
  const double tol3z = sqrt(0x1p-53);
  if (pivot) {
    vn1 = (double *)malloc(sizeof(double) * (size_t)n);
    vn2 = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      vn1[i] = norm2(m, W + IDX(0, i, ldw));
      vn2[i] = vn1[i];
    }
  }
  for (int64_t j = 0; j < s; ++j) {
    if (pivot) {
      int64_t pv = j;
      for (int64_t i = j + 1; i < n; ++i)
        if (vn1[i] > vn1[pv] || (vn1[i] == vn1[pv] && perm[i] < perm[pv])) pv = i;
      if (pv != j) {
        for (int64_t r = 0; r < m; ++r) {
          double t = W[IDX(r, j, ldw)];
          W[IDX(r, j, ldw)] = W[IDX(r, pv, ldw)];
          W[IDX(r, pv, ldw)] = t;
        }
        int64_t tp = perm[j]; perm[j] = perm[pv]; perm[pv] = tp;
        double t1 = vn1[j]; vn1[j] = vn1[pv]; vn1[pv] = t1;
        double t2 = vn2[j]; vn2[j] = vn2[pv]; vn2[pv] = t2;
      }
    }
    double *v = W + IDX(j, j, ldw);
    house(m - j, v, &tau[j]);
    /* apply H_j to the trailing columns with v(0) = 1 temporarily */
    double beta = v[0];
    v[0] = 1.0;
#pragma omp parallel for schedule(static)
    for (int64_t c = j + 1; c < n; ++c) apply_house(m - j, v, tau[j], W + IDX(j, c, ldw));
    v[0] = beta;
    if (pivot) {
#pragma omp parallel for schedule(static)
      for (int64_t i = j + 1; i < n; ++i) {
        if (vn1[i] != 0.0) {
          double t = fabs(W[IDX(j, i, ldw)]) / vn1[i];
          t = 1.0 - t * t;
          t = t < 0.0 ? 0.0 : t;
          double r = vn1[i] / vn2[i];
          double t2 = t * r * r;
          if (t2 <= tol3z) {
            if (j + 1 < m) {
              vn1[i] = norm2(m - j - 1, W + IDX(j + 1, i, ldw));
              vn2[i] = vn1[i];
            } else {
              vn1[i] = 0.0;
              vn2[i] = 0.0;
            }
          } else {
            vn1[i] = vn1[i] * sqrt(t);
          }
        }
      }
    }
  }
  free(vn1);
  free(vn2);
}

/* Extract R (s x n upper trapezoidal) and explicit Q (m x s), then normalise R_ii >= 0. */
static void qr_outputs(int64_t m, int64_t n, int64_t s, const double *W, int64_t ldw, const double *tau,
                       double *Q, int64_t ldq, double *R, int64_t ldr) {
  if (Q) form_q(m, s, W, ldw, tau, Q, ldq);
  if (R)
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < s; ++i) R[IDX(i, j, ldr)] = (i <= j) ? W[IDX(i, j, ldw)] : 0.0;
  for (int64_t i = 0; i < s; ++i) {
    if (W[IDX(i, i, ldw)] < 0.0) {
      if (R)
        for (int64_t j = i; j < n; ++j) R[IDX(i, j, ldr)] = -R[IDX(i, j, ldr)];
      if (Q)
        for (int64_t r = 0; r < m; ++r) Q[IDX(r, i, ldq)] = -Q[IDX(r, i, ldq)];
    }
  }
}

int orc_hqr(int64_t m, int64_t n, const double *A, int64_t lda, double *Q, int64_t ldq, double *R,
            int64_t ldr) {
  if (m < 0) return -1;
  if (n < 0 || n > m) return -2;
  if (lda < (m > 1 ? m : 1)) return -4;
  double *W = (double *)malloc(sizeof(double) * (size_t)(m * n + 1));
  double *tau = (double *)malloc(sizeof(double) * (size_t)(n + 1));
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t j = 0; j < n; ++j) memcpy(W + IDX(0, j, m), A + IDX(0, j, lda), sizeof(double) * (size_t)m);
  qr_core(m, n, W, m, tau, perm, 0, -1);
  qr_outputs(m, n, n, W, m, tau, Q, ldq, R, ldr);
  free(W); free(tau); free(perm);
  return 0;
}

int orc_cpqr(int64_t m, int64_t n, const double *A, int64_t lda, double *Q, int64_t ldq, double *R,
             int64_t ldr, int64_t *perm) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  if (lda < (m > 1 ? m : 1)) return -4;
  int64_t s = m < n ? m : n;
  double *W = (double *)malloc(sizeof(double) * (size_t)(m * n + 1));
  double *tau = (double *)malloc(sizeof(double) * (size_t)(s + 1));
  for (int64_t j = 0; j < n; ++j) memcpy(W + IDX(0, j, m), A + IDX(0, j, lda), sizeof(double) * (size_t)m);
  qr_core(m, n, W, m, tau, perm, 1, -1);
  qr_outputs(m, n, s, W, m, tau, Q, ldq, R, ldr);
  free(W); free(tau);
  return 0;
}

int orc_cpqr_partial(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda, double *Q, int64_t ldq,
                     double *R, int64_t ldr, int64_t *perm) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  int64_t s = m < n ? m : n;
  if (k < 0 || k > s) return -3;
  if (lda < (m > 1 ? m : 1)) return -5;
  double *W = (double *)malloc(sizeof(double) * (size_t)(m * n + 1));
  double *tau = (double *)malloc(sizeof(double) * (size_t)(k + 1));
  for (int64_t j = 0; j < n; ++j) memcpy(W + IDX(0, j, m), A + IDX(0, j, lda), sizeof(double) * (size_t)m);
  qr_core(m, n, W, m, tau, perm, 1, k);
  qr_outputs(m, n, k, W, m, tau, Q, ldq, R, ldr);
  free(W); free(tau);
  return 0;
}

/* One-sided Jacobi (Hestenes) SVD, used only as a brute-force pin. */
int orc_svd_values(int64_t m, int64_t n, const double *A, int64_t lda, double *s) {
  int trans = m < n;
  int64_t r = trans ? n : m, c = trans ? m : n;
  double *U = (double *)malloc(sizeof(double) * (size_t)(r * c + 1));
  for (int64_t j = 0; j < c; ++j)
    for (int64_t i = 0; i < r; ++i) U[IDX(i, j, r)] = trans ? A[IDX(j, i, lda)] : A[IDX(i, j, lda)];
  int converged = 0;
  for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
    converged = 1;
    for (int64_t i = 0; i < c - 1; ++i)
      for (int64_t j = i + 1; j < c; ++j) {
        double *ui = U + IDX(0, i, r), *uj = U + IDX(0, j, r);
        double a = 0, b = 0, g = 0;
        for (int64_t t = 0; t < r; ++t) {
          a += ui[t] * ui[t];
          b += uj[t] * uj[t];
          g += ui[t] * uj[t];
        }
        if (g == 0.0 || fabs(g) <= 1e-15 * sqrt(a * b)) continue;
        converged = 0;
        double zeta = (b - a) / (2.0 * g);
        double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int64_t k = 0; k < r; ++k) {
          double x = ui[k], y = uj[k];
          ui[k] = cs * x - sn * y;
          uj[k] = sn * x + cs * y;
        }
      }
  }
  for (int64_t j = 0; j < c; ++j) s[j] = norm2(r, U + IDX(0, j, r));
  for (int64_t i = 1; i < c; ++i) { /* insertion sort, descending */
    double v = s[i];
    int64_t k = i - 1;
    while (k >= 0 && s[k] < v) {
      s[k + 1] = s[k];
      --k;
    }
    s[k + 1] = v;
  }
  free(U);
  return converged ? 0 : 1;
}

/* ======================================================================================
 * The method.
 * ==================================================================================== */
static double *dalloc(int64_t count) { return (double *)calloc((size_t)(count > 0 ? count : 1), sizeof(double)); }

static void transpose(int64_t m, int64_t n, const double *A, int64_t lda, double *B, int64_t ldb) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) B[IDX(j, i, ldb)] = A[IDX(i, j, lda)];
}

int orc_qlp_tail(int64_t l, int64_t n, const double *B, int64_t ldb, int d, double *QB, int64_t ldqb,
                 double *T, int64_t ldt, double *PB, int64_t ldpb, int64_t *piv0, int64_t *piv1,
                 int *t_is_upper) {
  if (l < 1) return -1;
  if (n < l) return -2;
  if (ldb < l) return -4;
  if (d < 0) return -5;
  /* Alg.1 l.5 / Alg.2 l.5: [Q0, R0, Π0] = cpqr(B) */
  double *Q0 = dalloc(l * l), *R0 = dalloc(l * n);
  int64_t *perm0 = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  orc_cpqr(l, n, B, ldb, Q0, l, R0, l, perm0);
  for (int64_t j = 0; j < l; ++j) piv0[j] = perm0[j];
  double *Rt = dalloc(n * l);
  transpose(l, n, R0, l, Rt, n); /* R0^T, n x l */
  double *P1 = dalloc(n * l);    /* the n x l right factor before the row scatter by Π0 */
  if (d == 0) {
    /* Alg.1 l.6: [Q1, L^T, Π1] = cpqr(R0^T) */
    double *Lt = dalloc(l * l);
    int64_t *perm1 = (int64_t *)malloc(sizeof(int64_t) * (size_t)l);
    orc_cpqr(n, l, Rt, n, P1, n, Lt, l, perm1);
    transpose(l, l, Lt, l, T, ldt); /* L = (L^T)^T, lower */
    /* Alg.1 l.7: Q_B = Q0 Π1 (columns of Q0 permuted by Π1) */
    for (int64_t t = 0; t < l; ++t) {
      piv1[t] = perm1[t];
      for (int64_t i = 0; i < l; ++i) QB[IDX(i, t, ldqb)] = Q0[IDX(i, perm1[t], l)];
    }
    *t_is_upper = 0;
    free(Lt);
    free(perm1);
  } else {
    /* Alg.2 l.6-8: [Q^(i), R^(i)] = qr([R^(i-1)]^T), i = 1..d.
     * Corrected assembly (reading R9): Q_B = Q^(0) Q^(2) ..., P_B = Π Q^(1) Q^(3) ...,
     * T = [R^(d)]^T (lower) for odd d, R^(d) (upper) for even d. */
    double *Rcur = dalloc(l * l), *Qi = dalloc(l * l), *tmp = dalloc((n > l ? n : l) * l);
    double *Qeven = dalloc(l * l);
    for (int64_t j = 0; j < l; ++j) memcpy(Qeven + IDX(0, j, l), Q0 + IDX(0, j, l), sizeof(double) * (size_t)l);
    orc_hqr(n, l, Rt, n, P1, n, Rcur, l); /* i = 1 on the n x l R0^T */
    for (int i = 2; i <= d; ++i) {
      double *Mt = dalloc(l * l), *Rn = dalloc(l * l);
      transpose(l, l, Rcur, l, Mt, l);
      orc_hqr(l, l, Mt, l, Qi, l, Rn, l);
      if (i % 2 == 0) {
        orc_gemm_nn(l, l, l, Qeven, l, Qi, l, tmp, l);
        for (int64_t j = 0; j < l; ++j) memcpy(Qeven + IDX(0, j, l), tmp + IDX(0, j, l), sizeof(double) * (size_t)l);
      } else {
        orc_gemm_nn(n, l, l, P1, n, Qi, l, tmp, n);
        for (int64_t j = 0; j < l; ++j) memcpy(P1 + IDX(0, j, n), tmp + IDX(0, j, n), sizeof(double) * (size_t)n);
      }
      memcpy(Rcur, Rn, sizeof(double) * (size_t)(l * l));
      free(Mt);
      free(Rn);
    }
    if (d % 2 == 1) {
      transpose(l, l, Rcur, l, T, ldt);
      *t_is_upper = 0;
    } else {
      for (int64_t j = 0; j < l; ++j)
        for (int64_t i = 0; i < l; ++i) T[IDX(i, j, ldt)] = Rcur[IDX(i, j, l)];
      *t_is_upper = 1;
    }
    for (int64_t j = 0; j < l; ++j) {
      piv1[j] = j;
      for (int64_t i = 0; i < l; ++i) QB[IDX(i, j, ldqb)] = Qeven[IDX(i, j, l)];
    }
    free(Rcur); free(Qi); free(tmp); free(Qeven);
  }
  /* P_B = Π0 P1: row perm0[i] of P_B is row i of P1 (Alg.1 l.7 "P = Π0 Q1") */
  for (int64_t j = 0; j < l; ++j)
    for (int64_t i = 0; i < n; ++i) PB[IDX(perm0[i], j, ldpb)] = P1[IDX(i, j, n)];
  free(Q0); free(R0); free(perm0); free(Rt); free(P1);
  return 0;
}

/* Range finder + q subspace iterations (reading R12):
 * Ω = RNG(seed, stream 0); Y = AΩ; V = qr(Y); repeat q: Z = A^T V; W = qr(Z); Y = AW; V = qr(Y). */
static void range_finder(int64_t m, int64_t n, int64_t l, int q, const double *A, int64_t lda, uint64_t seed,
                         double *V) {
  double *Om = dalloc(n * l), *Y = dalloc(m * l), *Z = dalloc(n * l), *W = dalloc(n * l);
  double *R = dalloc(l * l);
  orc_gaussian(seed, 0, n, l, Om, n);              /* Alg.1 l.1 */
  orc_gemm_nn(m, l, n, A, lda, Om, n, Y, m);       /* Alg.1 l.2: Y = AΩ */
  orc_hqr(m, l, Y, m, V, m, R, l);                 /* Alg.1 l.3: [V,~] = qr(Y) */
  for (int it = 0; it < q; ++it) {
    orc_gemm_tn(n, l, m, A, lda, V, m, Z, n);      /* Z = A^T V */
    orc_hqr(n, l, Z, n, W, n, R, l);               /* W = qr(Z) */
    orc_gemm_nn(m, l, n, A, lda, W, n, Y, m);      /* Y = A W */
    orc_hqr(m, l, Y, m, V, m, R, l);               /* V = qr(Y) */
  }
  free(Om); free(Y); free(Z); free(W); free(R);
}

int orc_rqlp(int64_t m, int64_t n, int k, int p, int q, int d, const double *A, int64_t lda, uint64_t seed,
             double *Q, int64_t ldq, double *T, int64_t ldt, double *P, int64_t ldp, int64_t *piv0,
             int64_t *piv1, int *t_is_upper, double *V_out, int64_t ldv, double *B_out, int64_t ldb) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (k < 2) return -3;  /* Alg.1 input: k >= 2 */
  if (p < 2) return -4;  /* p >= 2 */
  if (q < 0) return -5;
  if (d < 0) return -6;
  int64_t l = (int64_t)k + p;
  if (l > m || l > n) return -3;
  if (lda < m) return -8;
  double *V = dalloc(m * l), *B = dalloc(l * n), *QB = dalloc(l * l);
  range_finder(m, n, l, q, A, lda, seed, V);
  orc_gemm_tn(l, n, m, V, m, A, lda, B, l);        /* Alg.1 l.4: B = V^T A */
  orc_qlp_tail(l, n, B, l, d, QB, l, T, ldt, P, ldp, piv0, piv1, t_is_upper);
  orc_gemm_nn(m, l, l, V, m, QB, l, Q, ldq);       /* Q = V Q_B */
  if (V_out)
    for (int64_t j = 0; j < l; ++j) memcpy(V_out + IDX(0, j, ldv), V + IDX(0, j, m), sizeof(double) * (size_t)m);
  if (B_out)
    for (int64_t j = 0; j < n; ++j) memcpy(B_out + IDX(0, j, ldb), B + IDX(0, j, l), sizeof(double) * (size_t)l);
  free(V); free(B); free(QB);
  return 0;
}

/* V_j <- qr(V_j - Vprev (Vprev^T V_j))  (Alg.3 l.5, eq. (18)), applied twice
 * (reading R28: "twice is enough"; in exact arithmetic the second pass removes nothing
 * whenever V_j has a component outside span(Vprev), and it is what keeps V orthonormal when that
 * component is at the rounding level -- a block past rank(A), or past a spectral gap). */
static void reorth(int64_t m, int64_t nprev, int64_t bj, const double *Vprev, int64_t ldvp, double *Vj) {
  if (nprev == 0) return;
  double *C = dalloc(nprev * bj), *D = dalloc(m * bj), *R = dalloc(bj * bj);
  for (int pass = 0; pass < 2; ++pass) {
    orc_gemm_tn(nprev, bj, m, Vprev, ldvp, Vj, m, C, nprev);
    orc_gemm_nn(m, bj, nprev, Vprev, ldvp, C, nprev, D, m);
    for (int64_t i = 0; i < m * bj; ++i) D[i] = Vj[i] - D[i];
    orc_hqr(m, bj, D, m, Vj, m, R, bj);
  }
  free(C); free(D); free(R);
}

int orc_brqlp(int64_t m, int64_t n, int k, int p, int b, int q, const double *A, int64_t lda, uint64_t seed,
              double *Q, int64_t ldq, double *L, int64_t ldl, double *P, int64_t ldp, int64_t *piv0,
              int64_t *piv1, double *V_out, int64_t ldv) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (k < 2) return -3;
  if (p < 2) return -4;
  int64_t l = (int64_t)k + p;
  if (b < 1 || b > l) return -5;
  if (q < 0) return -6;
  if (l > m || l > n) return -3;
  if (lda < m) return -8;
  int64_t h = (l + b - 1) / b; /* ragged last block (reading R14) */
  double *Aw = dalloc(m * n);  /* working copy A^(j) (eq. (19)); A itself is never written */
  for (int64_t j = 0; j < n; ++j) memcpy(Aw + IDX(0, j, m), A + IDX(0, j, lda), sizeof(double) * (size_t)m);
  double *Om = dalloc(n * l), *Vall = dalloc(m * l);
  orc_gaussian(seed, 0, n, l, Om, n);                               /* Alg.3 l.1 */
  for (int64_t i = 0; i < l; ++i)
    for (int64_t j = 0; j < l; ++j) L[IDX(i, j, ldl)] = 0.0;
  for (int64_t blk = 0; blk < h; ++blk) {
    int64_t c0 = blk * b, bj = (c0 + b <= l) ? b : l - c0;
    double *Y = dalloc(m * bj), *Vj = Vall + IDX(0, c0, m), *R = dalloc(bj * bj);
    double *Z = dalloc(n * bj), *W = dalloc(n * bj), *Bj = dalloc(bj * n);
    orc_gemm_nn(m, bj, n, A, lda, Om + IDX(0, c0, n), n, Y, m);     /* l.3: Y_j = A Ω_j (original A, R15) */
    orc_hqr(m, bj, Y, m, Vj, m, R, bj);                             /* l.4 */
    reorth(m, c0, bj, Vall, m, Vj);                                 /* l.5 */
    for (int it = 0; it < q; ++it) {                                /* deflated power steps (R16) */
      orc_gemm_tn(n, bj, m, Aw, m, Vj, m, Z, n);
      orc_hqr(n, bj, Z, n, W, n, R, bj);
      orc_gemm_nn(m, bj, n, Aw, m, W, n, Y, m);
      orc_hqr(m, bj, Y, m, Vj, m, R, bj);
      reorth(m, c0, bj, Vall, m, Vj);
    }
    orc_gemm_tn(bj, n, m, Vj, m, Aw, m, Bj, bj);                    /* l.6: B_j = V_j^T A^(j-1) */
    /* l.7: A^(j) = A^(j-1) - V_j B_j */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c)
      for (int64_t t = 0; t < bj; ++t) {
        double bb = Bj[IDX(t, c, bj)];
        double *ac = Aw + IDX(0, c, m);
        const double *vt = Vj + IDX(0, t, m);
        for (int64_t i = 0; i < m; ++i) ac[i] -= vt[i] * bb;
      }
    /* l.8: [Q_B, L_j, P_B] = qlp(B_j) -- Stewart pivoted QLP */
    double *QB = dalloc(bj * bj), *Lj = dalloc(bj * bj);
    int tu;
    orc_qlp_tail(bj, n, Bj, bj, 0, QB, bj, Lj, bj, P + IDX(0, c0, ldp), ldp, piv0 + c0, piv1 + c0, &tu);
    orc_gemm_nn(m, bj, bj, Vj, m, QB, bj, Q + IDX(0, c0, ldq), ldq); /* l.9: Q_j = V_j Q_B */
    for (int64_t j = 0; j < bj; ++j)                                   /* l.11: L = blkdiag(L_j) */
      for (int64_t i = 0; i < bj; ++i) L[IDX(c0 + i, c0 + j, ldl)] = Lj[IDX(i, j, bj)];
    free(Y); free(R); free(Z); free(W); free(Bj); free(QB); free(Lj);
  }
  if (V_out)
    for (int64_t j = 0; j < l; ++j) memcpy(V_out + IDX(0, j, ldv), Vall + IDX(0, j, m), sizeof(double) * (size_t)m);
  free(Aw); free(Om); free(Vall);
  return 0;
}

int orc_autorank(int64_t m, int64_t n, int b, int l_max, int q, double eps, const double *A, int64_t lda,
                 uint64_t seed, double *Q, int64_t ldq, double *L, int64_t ldl, double *P, int64_t ldp,
                 int64_t *piv0, int64_t *piv1, int *l_out, double *err_out) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (b < 1) return -3;
  if (l_max < b || l_max > m || l_max > n) return -4;
  if (q < 0) return -5;
  if (!(eps >= 0.0)) return -6;
  if (lda < m) return -8;
  const int64_t l = l_max;
  double *Aw = dalloc(m * n);
  for (int64_t j = 0; j < n; ++j) memcpy(Aw + IDX(0, j, m), A + IDX(0, j, lda), sizeof(double) * (size_t)m);
  const double a2 = orc_fro(m, n, A, lda) * orc_fro(m, n, A, lda);   /* ||A||_F^2 */
  double *Om = dalloc(n * l), *Vall = dalloc(m * l);
  orc_gaussian(seed, 0, n, l, Om, n);
  for (int64_t i = 0; i < l; ++i)
    for (int64_t j = 0; j < l; ++j) L[IDX(i, j, ldl)] = 0.0;
  double b2 = 0.0;   /* sum_j ||B_j||_F^2 */
  int64_t used = 0;
  for (int64_t c0 = 0; c0 < l; c0 += b) {
    const int64_t bj = (c0 + b <= l) ? b : l - c0;
    double *Y = dalloc(m * bj), *Vj = Vall + IDX(0, c0, m), *R = dalloc(bj * bj);
    double *Z = dalloc(n * bj), *W = dalloc(n * bj), *Bj = dalloc(bj * n);
    orc_gemm_nn(m, bj, n, A, lda, Om + IDX(0, c0, n), n, Y, m);      /* Alg.3 l.3 (original A) */
    orc_hqr(m, bj, Y, m, Vj, m, R, bj);
    reorth(m, c0, bj, Vall, m, Vj);
    for (int it = 0; it < q; ++it) {
      orc_gemm_tn(n, bj, m, Aw, m, Vj, m, Z, n);
      orc_hqr(n, bj, Z, n, W, n, R, bj);
      orc_gemm_nn(m, bj, n, Aw, m, W, n, Y, m);
      orc_hqr(m, bj, Y, m, Vj, m, R, bj);
      reorth(m, c0, bj, Vall, m, Vj);
    }
    orc_gemm_tn(bj, n, m, Vj, m, Aw, m, Bj, bj);                     /* B_j = V_j^T A^(j-1) */
#pragma omp parallel for schedule(static)
    for (int64_t cc = 0; cc < n; ++cc)
      for (int64_t t = 0; t < bj; ++t) {
        double bb = Bj[IDX(t, cc, bj)];
        double *ac = Aw + IDX(0, cc, m);
        const double *vt = Vj + IDX(0, t, m);
        for (int64_t i = 0; i < m; ++i) ac[i] -= vt[i] * bb;
      }
    const double nb = orc_fro(bj, n, Bj, bj);
    b2 += nb * nb;
    double *QB = dalloc(bj * bj), *Lj = dalloc(bj * bj);
    int tu;
    orc_qlp_tail(bj, n, Bj, bj, 0, QB, bj, Lj, bj, P + IDX(0, c0, ldp), ldp, piv0 + c0, piv1 + c0, &tu);
    orc_gemm_nn(m, bj, bj, Vj, m, QB, bj, Q + IDX(0, c0, ldq), ldq);
    for (int64_t j = 0; j < bj; ++j)
      for (int64_t i = 0; i < bj; ++i) L[IDX(c0 + i, c0 + j, ldl)] = Lj[IDX(i, j, bj)];
    free(Y); free(R); free(Z); free(W); free(Bj); free(QB); free(Lj);
    used = c0 + bj;
    const double e2 = a2 - b2;   /* eq. (3): ||A - P_V A||_F^2 = ||A||_F^2 - ||B||_F^2 */
    if (err_out) *err_out = a2 > 0.0 ? sqrt(e2 > 0.0 ? e2 : 0.0) / sqrt(a2) : 0.0;
    if (e2 <= eps * eps * a2) break;
  }
  *l_out = (int)used;
  free(Aw); free(Om); free(Vall);
  return 0;
}

/* Truncated pivoted QLP (NEXT-3): Stewart's pivoted QLP truncated to rank l
 * as the paper describes it: "apply partial CPQR decomposition on the m-by-n
 * matrix A, i.e. A Π(:, 1:l) = Q R, and compute the full CPQR decomposition of the n-by-l matrix
 * [R11 R12]^T".  With [R11 R12]^T Π1 = P^ L^T: Q = Q_R Π1, L, P = Π0 P^ (eq. (1)). */
int orc_tqlp(int64_t m, int64_t n, int64_t l, const double *A, int64_t lda, double *Q, int64_t ldq, double *L,
             int64_t ldl, double *P, int64_t ldp, int64_t *piv0, int64_t *piv1) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (l < 1 || l > m || l > n) return -3;
  if (lda < m) return -5;
  double *QR = dalloc(m * l), *R = dalloc(l * n), *Rt = dalloc(n * l), *Ph = dalloc(n * l), *Lt = dalloc(l * l);
  int64_t *perm0 = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *perm1 = (int64_t *)malloc(sizeof(int64_t) * (size_t)l);
  orc_cpqr_partial(m, n, l, A, lda, QR, m, R, l, perm0);   /* A Π0(:, 1:l) = Q_R [R11 R12] */
  transpose(l, n, R, l, Rt, n);                              /* [R11 R12]^T, n x l */
  orc_cpqr(n, l, Rt, n, Ph, n, Lt, l, perm1);               /* [R11 R12]^T Π1 = P^ L^T */
  transpose(l, l, Lt, l, L, ldl);
  for (int64_t t = 0; t < l; ++t) {
    piv0[t] = perm0[t];
    piv1[t] = perm1[t];
    for (int64_t i = 0; i < m; ++i) Q[IDX(i, t, ldq)] = QR[IDX(i, perm1[t], m)];   /* Q = Q_R Π1 */
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t t = 0; t < l; ++t) P[IDX(perm0[i], t, ldp)] = Ph[IDX(i, t, n)];    /* P = Π0 P^ */
  free(QR); free(R); free(Rt); free(Ph); free(Lt); free(perm0); free(perm1);
  return 0;
}

double orc_residual(int64_t m, int64_t n, int64_t l, const double *A, int64_t lda, const double *Q, int64_t ldq,
                    const double *T, int64_t ldt, const double *P, int64_t ldp) {
  double *M = dalloc(l * n); /* M = T P^T  (l x n) */
  orc_gemm_nt(l, n, l, T, ldt, P, ldp, M, l);
  const int64_t RB = 64;
  int64_t nrb = (m + RB - 1) / RB;
  double *part = dalloc(nrb);
#pragma omp parallel for schedule(static)
  for (int64_t rb = 0; rb < nrb; ++rb) {
    int64_t i0 = rb * RB, i1 = i0 + RB < m ? i0 + RB : m;
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = i0; i < i1; ++i) {
        double x = 0.0;
        for (int64_t t = 0; t < l; ++t) x += Q[IDX(i, t, ldq)] * M[IDX(t, j, l)];
        double r = A[IDX(i, j, lda)] - x;
        s += r * r;
      }
    part[rb] = s;
  }
  double s = 0.0;
  for (int64_t rb = 0; rb < nrb; ++rb) s += part[rb];
  free(M);
  free(part);
  return sqrt(s);
}
