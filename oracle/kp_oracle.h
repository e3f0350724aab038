/*
 * kp_oracle.h -- CPU restatement of the reference's direction-split phi path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker for the CUDA product
 * path; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product (paper_2304_02327_b200)
 * never links, imports or calls it.
 *
 * It restates, in plain C99, the algorithms of the reference C++ library
 * `kronphi` (arXiv 2304.02327, /root/reference/proj).  Every function cites
 * the reference file:line it follows (prefix inc/ = proj/include/kronphi/,
 * src/ = proj/src/).  Pinning: tests/test_oracle_pins.py checks this
 * restatement against the reference's own known-answer tests and against
 * golden vectors produced by the real reference (oracle/_ref, see
 * tests/golden/make_golden.py).
 *
 * Conventions (inc/tensor.hpp:1-2, inc/matrix.hpp:58-59): column-major,
 * first index fastest.  Complex data is interleaved (re, im) like
 * std::complex<double>.  Return value 0 = ok, nonzero = error with a message
 * in kpo_last_error() mirroring the reference exception text.
 */
#ifndef KP_ORACLE_H
#define KP_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
  KPO_OK = 0,
  KPO_EINVAL = 1,   /* std::invalid_argument */
  KPO_ERUNTIME = 2, /* std::runtime_error   */
  KPO_EDIVERGE = 3  /* DivergenceError       */
};

/* Method ids: inc/integrators.hpp:24-31 (same order). */
enum {
  KPO_LAWSON_EULER = 0,
  KPO_LAWSON2B = 1,
  KPO_EXP_EULER = 2,
  KPO_EXP_EULER_LS = 3,
  KPO_ETD2RK = 4,
  KPO_ROSENBROCK_EULER = 5 /* :166-194; Jacobian factors of the Riccati g only */
};

/* Closed set of pointwise nonlinearities g(t,u) (the reference takes a host
 * std::function, inc/integrators.hpp:60,112; these are the BASELINE configs'
 * g's plus the reference tests' square/const/zero g's). */
enum {
  KPO_G_ZERO = 0,        /* g = 0                          test_integrators.cpp:44-46 */
  KPO_G_SQUARE = 1,      /* g = u^2                        test_integrators.cpp:36-42 */
  KPO_G_CONST = 2,       /* g = p0                          test_integrators.cpp:177-181 */
  KPO_G_ALLEN_CAHN = 3,  /* g = u - u^3                    BASELINE configs 1,3 */
  KPO_G_BRUSSELATOR = 4, /* (a-(b+1)u+u^2 v, b u-u^2 v), species stacked as the
                            slowest mode of size 2; p0=a, p1=b   BASELINE config 4 */
  KPO_G_NLS = 5,         /* g = -i |u|^2 u (complex only)   BASELINE config 5 */
  KPO_G_ADR = 6,         /* 1/(1+u^2) + e^t psi_a - 1/(1+e^{2t} u0^2), aux = {psi_a, u0^2}
                            src/problems.cpp:101-115 */
  KPO_G_RICCATI = 7      /* C - (U b)(U^T b)^T on an n x n state, aux = {b, C}
                            src/problems.cpp:188-200, 263-276 */
};

typedef struct {
  int kind;
  double p[4];
  const double* aux[2];
} kpo_gfun;

const char* kpo_last_error(void);

/* inc/kernels.hpp:56-73 (gemm_naive semantics, column-major, op on B only) */
void kpo_gemm_f64(int m, int n, int k, double alpha, const double* a, int lda,
                  const double* b, int ldb, int transb, double beta, double* c,
                  int ldc);

/* ---- mode products: inc/mode_product.hpp ---- */
int kpo_mode_product_f64(const double* t, const int* dims, int d, int mode,
                         const double* m, int rows, int cols, double* out,
                         int accumulate);
int kpo_mode_product_c128(const double* t, const int* dims, int d, int mode,
                          const double* m, int rows, int cols, double* out,
                          int accumulate);
int kpo_tucker_f64(const double* t, const int* dims, int d,
                   const double* const* ms, const int* rows, double* out);
int kpo_tucker_c128(const double* t, const int* dims, int d,
                    const double* const* ms, const int* rows, double* out);
int kpo_kronsum_f64(const double* t, const int* dims, int d,
                    const double* const* as, double* out);
int kpo_kronsum_c128(const double* t, const int* dims, int d,
                     const double* const* as, double* out);

/* ---- matrix functions: inc/matrix_functions.hpp, src/gll_rule.cpp ---- */
int kpo_gll_rule(int q, double* nodes, double* weights);
int kpo_expm_f64(const double* x, int n, double* out);
int kpo_expm_c128(const double* x, int n, double* out);
/* phis: (ell_max+1) consecutive n*n matrices; forced_scaling < 0 = none */
int kpo_phiquad_f64(const double* x, int n, int ell_max, int q,
                    int forced_scaling, double* phis, int* scaling_exponent);
int kpo_phiquad_c128(const double* x, int n, int ell_max, int q,
                     int forced_scaling, double* phis, int* scaling_exponent);

/* ---- direction splitting: inc/split_phi.hpp ---- */
/* factors[mu] receives phi_ell(tau*A_mu) (n_mu x n_mu); returns prefactor */
int kpo_build_split_phi_f64(const double* const* as, const int* dims, int d,
                            double tau, int ell, int q, double* const* factors,
                            double* prefactor);
int kpo_build_split_phi_c128(const double* const* as, const int* dims, int d,
                             double tau, int ell, int q,
                             double* const* factors, double* prefactor);
int kpo_apply_split_phi_f64(const double* v, const int* dims, int d,
                            const double* const* factors, double prefactor,
                            double* out);
int kpo_apply_split_phi_c128(const double* v, const int* dims, int d,
                             const double* const* factors, double prefactor,
                             double* out);

/* ---- steppers and integrate: inc/integrators.hpp ---- */
/* g evaluation (the closed set above); gout has the shape of u */
int kpo_eval_g_f64(const kpo_gfun* g, double t, const double* u,
                   const int* dims, int d, double* gout);
int kpo_eval_g_c128(const kpo_gfun* g, double t, const double* u,
                    const int* dims, int d, double* gout);

/* One step.  f1/f2: for Lawson methods f1 = exp factors (f2 unused); for
 * ExpEuler f1 = phi1 factors; for ETD2RK f1 = phi1, f2 = phi2 factors.
 * pref1/pref2 are the split prefactors.  as = K factors. */
int kpo_step_f64(int method, const double* u, const int* dims, int d, double t,
                 double tau, const double* const* as, const double* const* f1,
                 double pref1, const double* const* f2, double pref2,
                 const kpo_gfun* g, double* out);
int kpo_step_c128(int method, const double* u, const int* dims, int d,
                  double t, double tau, const double* const* as,
                  const double* const* f1, double pref1,
                  const double* const* f2, double pref2, const kpo_gfun* g,
                  double* out);

/* inc/integrators.hpp:219-373, Split backend: precompute factors, run
 * n_steps, finite check per step.  *diverged_step receives the 1-based step
 * that went non-finite (KPO_EDIVERGE) or 0. */
int kpo_integrate_f64(int method, const double* u0, const int* dims, int d,
                      const double* const* as, const kpo_gfun* g, double t0,
                      double t_final, long n_steps, int q, double* u_final,
                      long* diverged_step);
int kpo_integrate_c128(int method, const double* u0, const int* dims, int d,
                       const double* const* as, const kpo_gfun* g, double t0,
                       double t_final, long n_steps, int q, double* u_final,
                       long* diverged_step);

/* ---- problems: src/problems.cpp:9-22 ---- */
int kpo_fd_operator_1d(int n, double eps, double alpha, double* out);
/* Periodic second difference scale*circ(1,-2,1)/h^2 (new; NLS config) */
int kpo_periodic_laplacian_1d(int n, double h, double* out);

#ifdef __cplusplus
}
#endif
#endif
