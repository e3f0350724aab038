/*
 * kp_oracle.c -- CPU restatement of the reference `kronphi` hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see kp_oracle.h).  Compiled with
 * -ffp-contract=off; every place where the reference's build (g++ -O3
 * -march=native, default -ffp-contract=fast) turns a multiply-add into an
 * FMA is written with an explicit fma() so the restatement follows the
 * reference's rounding as closely as plain C allows.
 *
 * The scalar-generic body lives in kp_oracle_impl.inc and is instantiated
 * twice: double (suffix _f64) and double _Complex (suffix _c128), mirroring
 * the reference's templates over T (inc/matrix.hpp:33, inc/tensor.hpp:22).
 */
#include "kp_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

const char* kpo_last_error(void) { return g_err; }

static int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

/* inc/matrix.hpp:17-21 */
static double factorial(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f *= i;
  return f;
}

/* inc/kernels.hpp:102-104: the k dimension is summed in KC=256 slices; a
 * slice's partial sums are folded into C with the alpha/beta convention of
 * compute_tile (inc/kernels.hpp:241-263). */
#define KPO_KC 256
/* inc/linsolve.hpp:22 */
#define KPO_LU_PANEL 64

/* inc/matrix_functions.hpp:20-35 */
static const double kPadeTheta[5] = {1.495585217958292e-2, 2.539398330063230e-1,
                                     9.504178996162932e-1, 2.097847961257068e0,
                                     5.371920351148152e0};
static const double kPade3[4] = {120., 60., 12., 1.};
static const double kPade5[6] = {30240., 15120., 3360., 420., 30., 1.};
static const double kPade7[8] = {17297280., 8648640., 1995840., 277200.,
                                 25200.,    1512.,    56.,      1.};
static const double kPade9[10] = {17643225600., 8821612800., 2075673600.,
                                  302702400.,   30270240.,   2162160.,
                                  110880.,      3960.,       90.,
                                  1.};
static const double kPade13[14] = {64764752532480000., 32382376266240000.,
                                   7771770303897600.,  1187353796428800.,
                                   129060195264000.,   10559470521600.,
                                   670442572800.,      33522128640.,
                                   1323241920.,        40840800.,
                                   960960.,            16380.,
                                   182.,               1.};
static const double* const kPadeCoeffs[5] = {kPade3, kPade5, kPade7, kPade9,
                                             kPade13};
static const int kPadeLen[5] = {4, 6, 8, 10, 14};

/* The reference TU is built with g++'s default -ffp-contract=fast, which
 * fuses several multiply-adds here; follow it for bitwise-equal nodes. */
#define KPO_CONTRACT __attribute__((optimize("fp-contract=fast")))

/* src/gll_rule.cpp:14-31: Legendre P_n(x), P'_n(x) by the 3-term recurrence */
KPO_CONTRACT static void legendre(int n, double x, double* p, double* dp) {
  double pm1 = 1.0, pm = x;
  if (n == 0) {
    *p = 1.0;
    *dp = 0.0;
    return;
  }
  for (int k = 1; k < n; ++k) {
    const double pk1 = ((2.0 * k + 1.0) * x * pm - k * pm1) / (k + 1.0);
    pm1 = pm;
    pm = pk1;
  }
  *p = pm;
  if (x == 1.0 || x == -1.0)
    *dp = 0.5 * n * (n + 1.0) * (x == 1.0 ? 1.0 : (n % 2 ? 1.0 : -1.0));
  else
    *dp = n * (x * pm - pm1) / (x * x - 1.0);
}

/* src/gll_rule.cpp:35-72: q-point Gauss-Legendre-Lobatto on [0,1]; interior
 * nodes are roots of P'_{q-1} by Newton from Chebyshev-Lobatto guesses. */
KPO_CONTRACT int kpo_gll_rule(int q, double* nodes, double* weights) {
  if (q < 2) return set_err(KPO_EINVAL, "gll_rule: need at least 2 nodes");
  const int n = q - 1;
  double* x = (double*)malloc(sizeof(double) * q);
  double* w = (double*)malloc(sizeof(double) * q);
  x[0] = -1.0;
  x[n] = 1.0;
  for (int i = 1; i < n; ++i) {
    double xi = -cos(M_PI * i / n);
    for (int iter = 0; iter < 100; ++iter) {
      double p, dp;
      legendre(n, xi, &p, &dp);
      const double g = dp;
      const double gp = (2.0 * xi * dp - n * (n + 1.0) * p) / (1.0 - xi * xi);
      const double step = g / gp;
      xi -= step;
      if (fabs(step) < 1e-15) break;
    }
    x[i] = xi;
  }
  for (int i = 0; i < q; ++i) {
    double p, dp;
    legendre(n, x[i], &p, &dp);
    w[i] = 2.0 / (n * (n + 1.0) * p * p);
  }
  for (int i = 0; i < q; ++i) {
    nodes[i] = 0.5 * (x[i] + 1.0);
    weights[i] = 0.5 * w[i];
  }
  nodes[0] = 0.0;
  nodes[q - 1] = 1.0;
  free(x);
  free(w);
  return KPO_OK;
}

/* src/problems.cpp:9-22 */
int kpo_fd_operator_1d(int n, double eps, double alpha, double* a) {
  if (n < 1) return set_err(KPO_EINVAL, "fd_operator_1d: need n >= 1");
  const double h = 1.0 / (n + 1);
  const double lo = eps / (h * h) - alpha / (2.0 * h);
  const double di = -2.0 * eps / (h * h);
  const double hi = eps / (h * h) + alpha / (2.0 * h);
  memset(a, 0, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i) {
    if (i > 0) a[i + (size_t)(i - 1) * n] = lo;
    a[i + (size_t)i * n] = di;
    if (i + 1 < n) a[i + (size_t)(i + 1) * n] = hi;
  }
  return KPO_OK;
}

/* New (not in the reference, which is Dirichlet-only): periodic
 * (1/h^2) circ(1,-2,1), the 1-D operator of the NLS config. */
int kpo_periodic_laplacian_1d(int n, double h, double* a) {
  if (n < 3) return set_err(KPO_EINVAL, "periodic_laplacian_1d: need n >= 3");
  const double c = 1.0 / (h * h);
  memset(a, 0, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i) {
    a[i + (size_t)i * n] = -2.0 * c;
    a[i + (size_t)((i + 1) % n) * n] = c;
    a[i + (size_t)((i + n - 1) % n) * n] = c;
  }
  return KPO_OK;
}

/* ======================= real instantiation ======================= */
#define SC double
#define SFX(name) name##_f64
#define ABSV(x) fabs(x)
#define ISFIN(x) isfinite(x)
#define MULADD(a, b, c) fma((a), (b), (c)) /* AVX2 _mm256_fmadd_pd */
#define IS_COMPLEX 0
#include "kp_oracle_impl.inc"
#undef SC
#undef SFX
#undef ABSV
#undef ISFIN
#undef MULADD
#undef IS_COMPLEX

/* ====================== complex instantiation ====================== */
#define SC double _Complex
#define SFX(name) name##_c128
#define ABSV(x) cabs(x)
#define ISFIN(x) (isfinite(creal(x)) && isfinite(cimag(x)))
#define MULADD(a, b, c) ((c) + (a) * (b)) /* generic micro-kernel, kernels.hpp:174-186 */
#define IS_COMPLEX 1
#include "kp_oracle_impl.inc"

/* real-only entry with the reference gemm_naive signature (kernels.hpp:56) */
void kpo_gemm_f64(int m, int n, int k, double alpha, const double* a, int lda,
                  const double* b, int ldb, int transb, double beta, double* c,
                  int ldc) {
  gemm_kc_f64(m, n, k, alpha, a, lda, b, ldb, transb, beta, c, ldc);
}
