// ref_harness.cpp -- C-ABI shim over the REAL reference library (kronphi).
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile (`make ref`) against
// the reference's headers and its three translation units where they lie
// under /root/reference/proj (nothing is copied into this repo); the result
// is oracle/_ref/libkronphi_ref.so.  Exposes the same C signatures as the
// restatement (kp_oracle.h) with the prefix kpr_ so tests can run both on
// identical inputs, plus timing helpers used by bench.py's reference arm.
//
// The BASELINE configs' nonlinearities (Allen-Cahn, Brusselator, NLS) are not
// in the reference; they are supplied here as
// user g lambdas, exactly how a reference user would drive integrate().
// Complex stepping restates exp_euler_step / etd2rk_step
// (inc/integrators.hpp:134-164) over the reference's own complex kernels,
// because integrate() is double-only (inc/integrators.hpp:60,112).
#include <chrono>
#include <omp.h>
#include <complex>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "kronphi/integrators.hpp"
#include "kronphi/matrix_functions.hpp"
#include "kronphi/mode_product.hpp"
#include "kronphi/problems.hpp"
#include "kronphi/split_phi.hpp"
#include "kp_oracle.h"

using namespace kronphi;
using C = std::complex<double>;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return KPO_OK;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    return KPO_EDIVERGE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return KPO_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KPO_ERUNTIME;
  }
}

std::vector<int> vdims(const int* dims, int d) { return std::vector<int>(dims, dims + d); }
std::size_t numel(const int* dims, int d) {
  std::size_t n = 1;
  for (int i = 0; i < d; ++i) n *= std::size_t(dims[i]);
  return n;
}

template <typename T>
Tensor<T> to_tensor(const double* p, const int* dims, int d) {
  const T* tp = reinterpret_cast<const T*>(p);
  std::vector<T> v(tp, tp + numel(dims, d));
  return Tensor<T>(vdims(dims, d), v);
}
template <typename T>
Matrix<T> to_matrix(const double* p, int rows, int cols) {
  const T* tp = reinterpret_cast<const T*>(p);
  return Matrix<T>(rows, cols, std::vector<T>(tp, tp + std::size_t(rows) * cols));
}
template <typename T>
void from(const T* src, std::size_t n, double* dst) {
  std::memcpy(dst, src, sizeof(T) * n);
}

template <typename T>
std::vector<Matrix<T>> square_list(const double* const* as, const int* dims, int d) {
  std::vector<Matrix<T>> out;
  for (int mu = 0; mu < d; ++mu) out.push_back(to_matrix<T>(as[mu], dims[mu], dims[mu]));
  return out;
}

// g for the closed set (kp_oracle.h).  The reference has no such g's; they
// are user code, so the harness evaluates them with the restatement's g
// (compiled with -ffp-contract=off) to give every leg the same rounding.
GFun make_g(const kpo_gfun* g) {
  const kpo_gfun gg = *g;
  return [gg](double t, const Tensor<double>& u) {
    Tensor<double> o = Tensor<double>::no_init(u.dims());
    const int rc = kpo_eval_g_f64(&gg, t, u.data(), u.dims().data(), u.order(), o.data());
    if (rc) throw std::invalid_argument(kpo_last_error());
    return o;
  };
}

Tensor<C> g_complex(const kpo_gfun* g, const Tensor<C>& u) {
  Tensor<C> o = Tensor<C>::no_init(u.dims());
  const int rc = kpo_eval_g_c128(g, 0.0, reinterpret_cast<const double*>(u.data()),
                                 u.dims().data(), u.order(), reinterpret_cast<double*>(o.data()));
  if (rc) throw std::invalid_argument(kpo_last_error());
  return o;
}

Method to_method(int m) {
  switch (m) {
    case KPO_LAWSON_EULER: return Method::LawsonEuler;
    case KPO_LAWSON2B: return Method::Lawson2b;
    case KPO_EXP_EULER: return Method::ExpEuler;
    case KPO_EXP_EULER_LS: return Method::ExpEulerLinearSplit;
    case KPO_ETD2RK: return Method::ETD2RK;
  }
  throw std::invalid_argument("unknown method");
}

SplitPhi<C> split_of(const double* const* f, const int* dims, int d, double pref) {
  SplitPhi<C> sp;
  sp.factors = square_list<C>(f, dims, d);
  sp.prefactor = pref;
  return sp;
}

// Complex restatement of the step formulas over the reference kernels.
Tensor<C> step_c(int method, const Tensor<C>& u, double tau, const KroneckerSum<C>& k,
                 const kpo_gfun* g, const SplitPhi<C>& p1, const SplitPhi<C>& p2) {
  switch (method) {
    case KPO_LAWSON_EULER:
      return tucker(add_scaled(u, C(tau), g_complex(g, u)), p1.factors);
    case KPO_LAWSON2B: {
      const Tensor<C> gn = g_complex(g, u);
      const Tensor<C> stage = tucker(add_scaled(u, C(tau), gn), p1.factors);
      Tensor<C> out = tucker(add_scaled(u, C(0.5 * tau), gn), p1.factors);
      axpy(C(0.5 * tau), g_complex(g, stage), out);
      return out;
    }
    case KPO_EXP_EULER: {  // inc/integrators.hpp:134-141
      Tensor<C> r = kronsum_action(u, k);
      axpy(C(1), g_complex(g, u), r);
      return add_scaled(u, C(tau), apply_split_phi(p1, r));
    }
    case KPO_ETD2RK: {  // inc/integrators.hpp:153-164
      const Tensor<C> gn = g_complex(g, u);
      Tensor<C> r = kronsum_action(u, k);
      axpy(C(1), gn, r);
      const Tensor<C> stage = add_scaled(u, C(tau), apply_split_phi(p1, r));
      Tensor<C> dd = g_complex(g, stage);
      axpy(C(-1), gn, dd);
      return add_scaled(stage, C(tau), apply_split_phi(p2, dd));
    }
  }
  throw std::invalid_argument("complex step: unsupported method");
}

}  // namespace

extern "C" {

const char* kpr_last_error(void) { return g_err.c_str(); }

int kpr_num_threads(void) {
  int n = 1;
#pragma omp parallel
#pragma omp single
  n = omp_get_num_threads();
  return n;
}

void kpr_gemm_f64(int m, int n, int k, double alpha, const double* a, int lda,
                  const double* b, int ldb, int transb, double beta, double* c, int ldc) {
  gemm(m, n, k, alpha, a, lda, b, ldb, transb ? Op::transpose : Op::none, beta, c, ldc);
}

#define KPR_MODE_PRODUCT(SFX, T)                                                        \
  int kpr_mode_product_##SFX(const double* t, const int* dims, int d, int mode,         \
                             const double* m, int rows, int cols, double* out,          \
                             int accumulate) {                                          \
    return guard([&] {                                                                  \
      const Tensor<T> tt = to_tensor<T>(t, dims, d);                                    \
      const Matrix<T> mm = to_matrix<T>(m, rows, cols);                                 \
      std::vector<int> od = vdims(dims, d);                                             \
      if (mode >= 0 && mode < d) od[mode] = rows;                                       \
      Tensor<T> o = accumulate ? to_tensor<T>(out, od.data(), d) : Tensor<T>(od);       \
      mode_product_into(tt, mm, mode, o, accumulate != 0);                              \
      from(o.data(), o.size(), out);                                                    \
    });                                                                                 \
  }                                                                                     \
  int kpr_tucker_##SFX(const double* t, const int* dims, int d, const double* const* ms, \
                       const int* rows, double* out) {                                  \
    return guard([&] {                                                                  \
      std::vector<Matrix<T>> m;                                                         \
      for (int mu = 0; mu < d; ++mu) m.push_back(to_matrix<T>(ms[mu], rows[mu], dims[mu])); \
      const Tensor<T> o = tucker(to_tensor<T>(t, dims, d), m);                          \
      from(o.data(), o.size(), out);                                                    \
    });                                                                                 \
  }                                                                                     \
  int kpr_kronsum_##SFX(const double* t, const int* dims, int d, const double* const* as, \
                        double* out) {                                                  \
    return guard([&] {                                                                  \
      const KroneckerSum<T> k(square_list<T>(as, dims, d));                             \
      const Tensor<T> o = kronsum_action(to_tensor<T>(t, dims, d), k);                  \
      from(o.data(), o.size(), out);                                                    \
    });                                                                                 \
  }                                                                                     \
  int kpr_expm_##SFX(const double* x, int n, double* out) {                             \
    return guard([&] {                                                                  \
      const Matrix<T> e = expm(to_matrix<T>(x, n, n));                                  \
      from(e.data(), e.size(), out);                                                    \
    });                                                                                 \
  }                                                                                     \
  int kpr_phiquad_##SFX(const double* x, int n, int ell_max, int q, int forced,         \
                        double* phis, int* s_out) {                                     \
    return guard([&] {                                                                  \
      const auto tab = forced >= 0                                                      \
                           ? phiquad(to_matrix<T>(x, n, n), ell_max, gll_rule(q), forced) \
                           : phiquad(to_matrix<T>(x, n, n), ell_max, gll_rule(q));      \
      for (int j = 0; j <= ell_max; ++j)                                                \
        from(tab.phis[j].data(), tab.phis[j].size(), phis + (IS_C ? 2 : 1) * std::size_t(j) * n * n); \
      if (s_out) *s_out = tab.scaling_exponent;                                         \
    });                                                                                 \
  }                                                                                     \
  int kpr_build_split_phi_##SFX(const double* const* as, const int* dims, int d,        \
                                double tau, int ell, int q, double* const* factors,     \
                                double* prefactor) {                                    \
    return guard([&] {                                                                  \
      const KroneckerSum<T> k(square_list<T>(as, dims, d));                             \
      const SplitPhi<T> sp = build_split_phi(k, tau, ell, gll_rule(q));                 \
      for (int mu = 0; mu < d; ++mu)                                                    \
        from(sp.factors[mu].data(), sp.factors[mu].size(), factors[mu]);                \
      *prefactor = sp.prefactor;                                                        \
    });                                                                                 \
  }                                                                                     \
  int kpr_apply_split_phi_##SFX(const double* v, const int* dims, int d,                \
                                const double* const* factors, double prefactor,         \
                                double* out) {                                          \
    return guard([&] {                                                                  \
      SplitPhi<T> sp;                                                                   \
      sp.factors = square_list<T>(factors, dims, d);                                    \
      sp.prefactor = prefactor;                                                         \
      const Tensor<T> o = apply_split_phi(sp, to_tensor<T>(v, dims, d));                \
      from(o.data(), o.size(), out);                                                    \
    });                                                                                 \
  }

#define IS_C false
KPR_MODE_PRODUCT(f64, double)
#undef IS_C
#define IS_C true
KPR_MODE_PRODUCT(c128, C)
#undef IS_C

int kpr_gll_rule(int q, double* nodes, double* weights) {
  return guard([&] {
    const GLLRule r = gll_rule(q);
    for (int i = 0; i < q; ++i) {
      nodes[i] = r.nodes[i];
      weights[i] = r.weights[i];
    }
  });
}

int kpr_fd_operator_1d(int n, double eps, double alpha, double* out) {
  return guard([&] {
    const Matrix<double> a = fd_operator_1d(n, eps, alpha);
    from(a.data(), a.size(), out);
  });
}

int kpr_eval_g_f64(const kpo_gfun* g, double t, const double* u, const int* dims, int d,
                   double* gout) {
  return guard([&] {
    const Tensor<double> o = make_g(g)(t, to_tensor<double>(u, dims, d));
    from(o.data(), o.size(), gout);
  });
}

int kpr_step_f64(int method, const double* u, const int* dims, int d, double t, double tau,
                 const double* const* as, const double* const* f1, double pref1,
                 const double* const* f2, double pref2, const kpo_gfun* g, double* out) {
  return guard([&] {
    const Tensor<double> uu = to_tensor<double>(u, dims, d);
    const KroneckerSum<double> k(square_list<double>(as, dims, d));
    const GFun gf = make_g(g);
    Tensor<double> o;
    switch (method) {
      case KPO_LAWSON_EULER:
        o = lawson_euler_step(uu, t, tau, gf, square_list<double>(f1, dims, d));
        break;
      case KPO_LAWSON2B:
        o = lawson2b_step(uu, t, tau, gf, square_list<double>(f1, dims, d));
        break;
      case KPO_EXP_EULER: {
        SplitPhi<double> p1;
        p1.factors = square_list<double>(f1, dims, d);
        p1.prefactor = pref1;
        o = exp_euler_step(uu, t, tau, k, gf, p1);
        break;
      }
      case KPO_EXP_EULER_LS: {
        SplitPhi<double> p1;
        p1.factors = square_list<double>(f2, dims, d);
        p1.prefactor = pref2;
        o = exp_euler_linear_split_step(uu, t, tau, gf, square_list<double>(f1, dims, d), p1);
        break;
      }
      case KPO_ETD2RK: {
        SplitPhi<double> p1, p2;
        p1.factors = square_list<double>(f1, dims, d);
        p1.prefactor = pref1;
        p2.factors = square_list<double>(f2, dims, d);
        p2.prefactor = pref2;
        o = etd2rk_step(uu, t, tau, k, gf, p1, p2);
        break;
      }
      default:
        throw std::invalid_argument("step: unknown method");
    }
    from(o.data(), o.size(), out);
  });
}

int kpr_step_c128(int method, const double* u, const int* dims, int d, double t, double tau,
                  const double* const* as, const double* const* f1, double pref1,
                  const double* const* f2, double pref2, const kpo_gfun* g, double* out) {
  (void)t;
  return guard([&] {
    const KroneckerSum<C> k(square_list<C>(as, dims, d));
    const SplitPhi<C> p1 = split_of(f1, dims, d, pref1);
    const SplitPhi<C> p2 = method == KPO_ETD2RK ? split_of(f2, dims, d, pref2) : SplitPhi<C>{};
    const Tensor<C> o = step_c(method, to_tensor<C>(u, dims, d), tau, k, g, p1, p2);
    from(o.data(), o.size(), out);
  });
}

// integrate() on the Split backend (inc/integrators.hpp:219-373).
int kpr_integrate_f64(int method, const double* u0, const int* dims, int d,
                      const double* const* as, const kpo_gfun* g, double t0, double t_final,
                      long n_steps, int q, double* u_final, long* diverged_step) {
  if (diverged_step) *diverged_step = 0;
  return guard([&] {
    ProblemSpec p;
    p.K = KroneckerSum<double>(square_list<double>(as, dims, d));
    p.g = make_g(g);
    p.u0 = to_tensor<double>(u0, dims, d);
    p.t0 = t0;
    p.t_final = t_final;
    StepperConfig c;
    c.method = to_method(method);
    c.n_steps = n_steps;
    c.quad_nodes = q;
    try {
      const IntegrateResult r = integrate(p, c);
      from(r.final.data(), r.final.size(), u_final);
    } catch (const DivergenceError& e) {
      if (diverged_step) *diverged_step = e.step();
      throw;
    }
  });
}

// Complex integrate: the precompute of integrate() (inc/integrators.hpp:263-283)
// and its loop (:290-367) restated around the reference's complex kernels.
int kpr_integrate_c128(int method, const double* u0, const int* dims, int d,
                       const double* const* as, const kpo_gfun* g, double t0, double t_final,
                       long n_steps, int q, double* u_final, long* diverged_step) {
  if (diverged_step) *diverged_step = 0;
  return guard([&] {
    if (n_steps <= 0) throw std::invalid_argument("integrate: n_steps must be positive");
    const double tau = (t_final - t0) / double(n_steps);
    const GLLRule rule = gll_rule(q);
    const KroneckerSum<C> k(square_list<C>(as, dims, d));
    SplitPhi<C> p1, p2;
    switch (method) {
      case KPO_LAWSON_EULER:
      case KPO_LAWSON2B: p1 = build_split_phi(k, tau, 0, rule); break;
      case KPO_EXP_EULER: p1 = build_split_phi(k, tau, 1, rule); break;
      case KPO_ETD2RK:
        p1 = build_split_phi(k, tau, 1, rule);
        p2 = build_split_phi(k, tau, 2, rule);
        break;
      default: throw std::invalid_argument("complex integrate: unsupported method");
    }
    Tensor<C> u = to_tensor<C>(u0, dims, d);
    for (long n = 0; n < n_steps; ++n) {
      const double t = t0 + double(n) * tau;
      u = step_c(method, u, tau, k, g, p1, p2);
      if (!u.all_finite()) {
        if (diverged_step) *diverged_step = n + 1;
        throw DivergenceError(n + 1, t + tau);
      }
    }
    from(u.data(), u.size(), u_final);
  });
}

// The reference's own ADR experiment (src/problems.cpp:45-128 build_adr,
// run_adr's error measure src/bench_runner.cpp:181-203): integrate with the
// reference's g and report the final state and the relative inf-norm error
// against e^t u0.
int kpr_run_adr(int n1, int n2, int n3, int method, long n_steps, double* u_final,
                double* rel_err, double* seconds) {
  return guard([&] {
    const ADRProblem p = build_adr(n1, n2, n3);
    StepperConfig c;
    c.method = to_method(method);
    c.n_steps = n_steps;
    const IntegrateResult r = integrate(p.to_problem_spec(), c);
    from(r.final.data(), r.final.size(), u_final);
    const Tensor<double> ex = p.exact(1.0);
    *rel_err = diff_norm_inf(r.final, ex) / ex.norm_inf();
    if (seconds) *seconds = r.wallclock_s;
  });
}

// The reference's LQR Riccati problem (src/problems.cpp:130-284) through its
// own integrate() (Rosenbrock uses its jacobian_factors callback).
int kpr_run_riccati(int n_hat, int method, long n_steps, double t_final, double* u_final,
                    double* seconds) {
  return guard([&] {
    const RiccatiProblem p = build_riccati(n_hat);
    StepperConfig c;
    c.method = method == KPO_ROSENBROCK_EULER ? Method::RosenbrockEuler : to_method(method);
    c.n_steps = n_steps;
    const IntegrateResult r = integrate(p.to_problem_spec(t_final), c);
    from(r.final.data(), r.final.size(), u_final);
    if (seconds) *seconds = r.wallclock_s;
  });
}

// ---- timing helpers for bench.py's reference arm (steady_clock, in-process;
// inputs are built once outside the timed region) ----

// Seconds per tucker() call, best of `reps` after one warm-up call.
double kpr_time_tucker_f64(const double* t, const int* dims, int d, const double* const* ms,
                           int reps) {
  double best = 1e300;
  try {
    const Tensor<double> tt = to_tensor<double>(t, dims, d);
    std::vector<Matrix<double>> m;
    for (int mu = 0; mu < d; ++mu) m.push_back(to_matrix<double>(ms[mu], dims[mu], dims[mu]));
    volatile double sink = tucker(tt, m)[0];
    for (int r = 0; r < reps; ++r) {
      const auto a = std::chrono::steady_clock::now();
      const Tensor<double> o = tucker(tt, m);
      const auto b = std::chrono::steady_clock::now();
      sink = o[0];
      best = std::min(best, std::chrono::duration<double>(b - a).count());
    }
    (void)sink;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
  return best;
}

// Mean seconds per tucker() call over `steps` calls after `warmup` calls
// (bench.py --impl reference: only the reference's tucker() is inside the
// timed region; the input tensor and factors are converted once, outside).
double kpr_time_tucker_mean_f64(const double* t, const int* dims, int d, const double* const* ms,
                                int warmup, int steps) {
  try {
    const Tensor<double> tt = to_tensor<double>(t, dims, d);
    std::vector<Matrix<double>> m;
    for (int mu = 0; mu < d; ++mu) m.push_back(to_matrix<double>(ms[mu], dims[mu], dims[mu]));
    volatile double sink = 0.0;
    for (int r = 0; r < warmup; ++r) sink = tucker(tt, m)[0];
    const auto a = std::chrono::steady_clock::now();
    for (int r = 0; r < steps; ++r) sink = tucker(tt, m)[0];
    const auto b = std::chrono::steady_clock::now();
    (void)sink;
    return std::chrono::duration<double>(b - a).count() / std::max(1, steps);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// The reference's integrate() (Split backend) on n_steps steps; *loop_s =
// its IntegrateResult::loop_s (time loop only, factor build excluded) --
// the same quantity the device integrate reports.  Used for the integrator
// configs' same-run CPU baselines.
int kpr_time_integrate_f64(int method, const double* u0, const int* dims, int d,
                           const double* const* as, const kpo_gfun* g, double t0,
                           double t_final, long n_steps, int q, double* loop_s) {
  return guard([&] {
    ProblemSpec p;
    p.K = KroneckerSum<double>(square_list<double>(as, dims, d));
    p.g = make_g(g);
    p.u0 = to_tensor<double>(u0, dims, d);
    p.t0 = t0;
    p.t_final = t_final;
    StepperConfig c;
    c.method = to_method(method);
    c.n_steps = n_steps;
    c.quad_nodes = q;
    const IntegrateResult r = integrate(p, c);
    *loop_s = r.loop_s;
  });
}

// Complex counterpart: the restated loop of kpr_integrate_c128 over the
// reference's complex kernels; *loop_s = the time loop only.
int kpr_time_integrate_c128(int method, const double* u0, const int* dims, int d,
                            const double* const* as, const kpo_gfun* g, double t0,
                            double t_final, long n_steps, int q, double* loop_s) {
  return guard([&] {
    const double tau = (t_final - t0) / double(n_steps);
    const GLLRule rule = gll_rule(q);
    const KroneckerSum<C> k(square_list<C>(as, dims, d));
    SplitPhi<C> p1, p2;
    p1 = build_split_phi(k, tau, 1, rule);
    if (method == KPO_ETD2RK) p2 = build_split_phi(k, tau, 2, rule);
    else if (method != KPO_EXP_EULER)
      throw std::invalid_argument("complex integrate timing: exp_euler / etd2rk only");
    Tensor<C> u = to_tensor<C>(u0, dims, d);
    const auto a = std::chrono::steady_clock::now();
    for (long n = 0; n < n_steps; ++n) u = step_c(method, u, tau, k, g, p1, p2);
    const auto b = std::chrono::steady_clock::now();
    *loop_s = std::chrono::duration<double>(b - a).count();
  });
}

}  // extern "C"
