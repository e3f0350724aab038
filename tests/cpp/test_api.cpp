// C++ drop-in check: reference-style test cases written against the
// reference's headers/names ("kronphi/..."), compiled against
// include/kronphi_b200 and run on the GPU (tests/test_cpp_api.py).
// Cases restate /root/reference/proj/tests/test_tensor.cpp,
// test_matrix_functions.cpp, test_split_phi.cpp, test_integrators.cpp.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <vector>
#include <random>
#include <string>

#include "kronphi/integrators.hpp"
#include "kronphi/kernels.hpp"
#include "kronphi/linsolve.hpp"
#include "kronphi/problems.hpp"
#include "kronphi/matrix_functions.hpp"
#include "kronphi/mode_product.hpp"
#include "kronphi/split_phi.hpp"
#include "kronphi/tensor.hpp"

using namespace kronphi;

static int failures = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);          \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

static std::mt19937_64 rng(777);
static double urand() { return std::uniform_real_distribution<double>(-1, 1)(rng); }
static Tensor<double> random_tensor(std::vector<int> dims) {
  Tensor<double> t(std::move(dims));
  for (size_t i = 0; i < t.size(); ++i) t[i] = urand();
  return t;
}
static Matrix<double> random_matrix(int r, int c) {
  Matrix<double> m(r, c);
  for (size_t i = 0; i < m.size(); ++i) m.data()[i] = urand();
  return m;
}
static Matrix<double> random_stable(int n) {
  Matrix<double> m = random_matrix(n, n);
  const double s = m.norm1();
  for (int i = 0; i < n; ++i) m(i, i) -= s;
  return m;
}

int main() {
  {  // row permutation KAT (test_tensor.cpp:89-99)
    const Tensor<double> t({2, 2}, {1, 3, 2, 4});
    Matrix<double> m(2, 2);
    m(0, 1) = 1;
    m(1, 0) = 1;
    const Tensor<double> got = mode_product(t, m, 0);
    CHECK(got.at({0, 0}) == 3 && got.at({0, 1}) == 4 && got.at({1, 0}) == 1 && got.at({1, 1}) == 2);
  }
  {  // identity bit-exact (test_tensor.cpp:101-108)
    const Tensor<double> t = random_tensor({3, 4, 5});
    for (int mode = 0; mode < 3; ++mode)
      CHECK(diff_norm_inf(mode_product(t, Matrix<double>::identity(t.dim(mode)), mode), t) == 0.0);
  }
  {  // sizing error names the mode (test_tensor.cpp:118-124)
    const Tensor<double> t = random_tensor({3, 4, 5});
    bool ok = false;
    try {
      mode_product(t, random_matrix(6, 9), 1);
    } catch (const std::invalid_argument& e) {
      ok = std::string(e.what()).find("mode 1") != std::string::npos;
    }
    CHECK(ok);
  }
  {  // matvec (matrix.hpp:150-155) against the plain sum
    const Matrix<double> a = random_matrix(7, 5);
    std::vector<double> x(5), y(7, -1.0);
    for (int j = 0; j < 5; ++j) x[j] = 0.25 * (j + 1);
    matvec(a, x.data(), y.data());
    double worst = 0;
    for (int i = 0; i < 7; ++i) {
      double want = 0;
      for (int j = 0; j < 5; ++j) want += a(i, j) * x[j];
      worst = std::max(worst, std::abs(y[i] - want));
    }
    CHECK(worst < 1e-13);
  }
  {  // tucker in 2d is M1 T M2^T (test_tensor.cpp:159-169)
    const Tensor<double> t = random_tensor({3, 4});
    const Matrix<double> m1 = random_matrix(5, 3), m2 = random_matrix(6, 4);
    const Tensor<double> got = tucker(t, {m1, m2});
    const Matrix<double> tm(3, 4, vec(t));
    const Matrix<double> want = multiply(multiply(m1, tm), m2, Op::transpose);
    double worst = 0;
    for (int j = 0; j < 6; ++j)
      for (int i = 0; i < 5; ++i) worst = std::max(worst, std::abs(got.at({i, j}) - want(i, j)));
    CHECK(worst < 1e-13);
  }
  {  // kronsum zero factors (test_tensor.cpp:202-215)
    const Tensor<double> t3 = random_tensor({2, 3, 4});
    std::vector<Matrix<double>> zeros;
    for (int d : t3.dims()) zeros.push_back(Matrix<double>(d, d));
    CHECK(kronsum_action(t3, KroneckerSum<double>(zeros)).norm_inf() == 0.0);
  }
  {  // expm / phiquad closed forms (test_matrix_functions.cpp:56-80, :145-174)
    CHECK((expm(Matrix<double>(3, 3)) - Matrix<double>::identity(3)).norm1() == 0.0);
    Matrix<double> x(1, 1);
    x(0, 0) = 1.0;
    const auto tab = phiquad(x, 2);
    CHECK(std::abs(tab.phis[1](0, 0) - (std::exp(1.0) - 1.0)) < 1e-13);
    CHECK(std::abs(tab.phis[2](0, 0) - (std::exp(1.0) - 2.0)) < 1e-13);
    x(0, 0) = 2.0;
    CHECK(phiquad(x, 1).scaling_exponent == 2);
  }
  {  // prefactors (test_split_phi.cpp:66-75)
    const KroneckerSum<double> k3({random_stable(2), random_stable(3), random_stable(2)});
    CHECK(build_split_phi(k3, 0.1, 2).prefactor == 4.0);
    CHECK(build_split_phi(k3, 0.1, 1).prefactor == 1.0);
  }
  {  // etd2rk with K = 0 is the trapezoidal rule (test_integrators.cpp:282-296)
    const KroneckerSum<double> kz({Matrix<double>(2, 2)});
    const Tensor<double> u = random_tensor({2});
    const double tau = 0.21;
    const Tensor<double> got = etd2rk_step(u, 0.0, tau, kz, g_square(), build_split_phi(kz, tau, 1),
                                           build_split_phi(kz, tau, 2));
    for (int i = 0; i < 2; ++i) {
      const double g0 = u[i] * u[i], st = u[i] + tau * g0;
      CHECK(std::abs(got[i] - (st + tau * 0.5 * (st * st - g0))) < 1e-14);
    }
  }
  {  // integrate: one step equals the step function bitwise (test_integrators.cpp:350-371)
    ProblemSpec p;
    p.K = KroneckerSum<double>({random_stable(5), random_stable(6)});
    p.g = g_square();
    p.u0 = random_tensor({5, 6});
    p.t_final = 0.4;
    StepperConfig c;
    c.method = Method::ETD2RK;
    c.n_steps = 1;
    const auto r = integrate(p, c);
    const auto want = etd2rk_step(p.u0, 0.0, 0.4, p.K, p.g, build_split_phi(p.K, 0.4, 1),
                                  build_split_phi(p.K, 0.4, 2));
    CHECK(diff_norm_inf(r.final, want) == 0.0);
    CHECK(r.wallclock_s >= r.loop_s);
  }
  {  // divergence (test_integrators.cpp:404-422)
    ProblemSpec p;
    p.K = KroneckerSum<double>({Matrix<double>(2, 2)});
    p.g = g_square();
    p.u0 = Tensor<double>({2}, {1e100, 1e100});
    p.t_final = 10.0;
    StepperConfig c;
    c.method = Method::LawsonEuler;
    c.n_steps = 10;
    bool caught = false;
    try {
      integrate(p, c);
    } catch (const DivergenceError& e) {
      caught = e.step() >= 1 && std::string(e.what()).find("step") != std::string::npos;
    }
    CHECK(caught);
  }
  {  // complex tucker vs the nested-loop contraction
    using C = std::complex<double>;
    Tensor<C> t({3, 4});
    for (size_t i = 0; i < t.size(); ++i) t[i] = C(urand(), urand());
    Matrix<C> m(5, 3);
    for (size_t i = 0; i < m.size(); ++i) m.data()[i] = C(urand(), urand());
    const Tensor<C> got = mode_product(t, m, 0);
    double worst = 0;
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 5; ++i) {
        C acc{};
        for (int p = 0; p < 3; ++p) acc += m(i, p) * t.at({p, j});
        worst = std::max(worst, std::abs(got.at({i, j}) - acc));
      }
    CHECK(worst < 1e-14);
  }
  {  // Riccati (src/problems.cpp:130-284): Rosenbrock through integrate equals
     // the step loop with host-formed Jacobian factors A^T - (U b) b^T
    const RiccatiProblem pr = build_riccati(4);
    const int n = 16;
    CHECK(pr.a.rows() == n && pr.a_t(1, 0) == pr.a(0, 1));
    const ProblemSpec spec = pr.to_problem_spec(0.025);
    StepperConfig c;
    c.method = Method::RosenbrockEuler;
    c.n_steps = 6;
    const auto r = integrate(spec, c);
    Tensor<double> u = spec.u0;
    const double tau = 0.025 / 6;
    for (int s = 0; s < 6; ++s) {
      std::vector<double> w(n, 0.0);
      for (int p = 0; p < n; ++p)
        for (int i = 0; i < n; ++i) w[i] += u[i + size_t(p) * n] * pr.b[p];
      Matrix<double> j = pr.a_t;
      for (int jj = 0; jj < n; ++jj)
        for (int ii = 0; ii < n; ++ii) j(ii, jj) -= w[ii] * pr.b[jj];
      u = rosenbrock_euler_step(u, s * tau, tau, spec.K, spec.g, {j, j});
    }
    CHECK(diff_norm_inf(r.final, u) <= 1e-12 * u.norm_inf());
    c.method = Method::ETD2RK;
    const auto r2 = integrate(spec, c);
    CHECK(diff_norm_inf(r.final, r2.final) <= 1e-2 * r2.final.norm_inf());
    CHECK(parse_method("rosenbrock_euler") == Method::RosenbrockEuler);
  }
  {  // ADR (src/problems.cpp:45-128): second-order convergence to e^t u0
    const ADRProblem pr = build_adr(10, 11, 12);
    const ProblemSpec spec = pr.to_problem_spec();
    StepperConfig c;
    c.method = Method::ETD2RK;
    double err[2];
    for (int k = 0; k < 2; ++k) {
      c.n_steps = 20 << k;
      const auto r = integrate(spec, c);
      const Tensor<double> ex = pr.exact(1.0);
      err[k] = diff_norm_inf(r.final, ex) / ex.norm_inf();
    }
    CHECK(err[0] < 5e-3 && err[1] < err[0] / 3.0 && err[1] > err[0] / 5.0);
  }
  {  // gemm / gemm_batch_shared_b against the naive loops (kernels.hpp)
    std::mt19937_64 rg(7);
    std::uniform_real_distribution<double> ud(-1.0, 1.0);
    for (Op op : {Op::none, Op::transpose}) {
      const int m = 37, n = 29, k = 300;  // k spans two KC slices
      const int ldb = op == Op::none ? k : n, bcols = op == Op::none ? n : k;
      std::vector<double> a(size_t(m) * k), b(size_t(ldb) * bcols), c0(size_t(m) * n),
          c1;
      for (auto& x : a) x = ud(rg);
      for (auto& x : b) x = ud(rg);
      for (auto& x : c0) x = ud(rg);
      c1 = c0;
      gemm_naive(m, n, k, -1.5, a.data(), m, b.data(), ldb, op, 0.5, c0.data(), m);
      gemm(m, n, k, -1.5, a.data(), m, b.data(), ldb, op, 0.5, c1.data(), m);
      double err = 0.0;
      for (size_t i = 0; i < c0.size(); ++i) err = std::max(err, std::abs(c0[i] - c1[i]));
      CHECK(err < 1e-12);
    }
    using Cx = std::complex<double>;
    const int n = 40;
    std::vector<Cx> a(size_t(n) * n), b(size_t(n) * n), c0(size_t(n) * n), c1(size_t(n) * n);
    for (auto& x : a) x = Cx(ud(rg), ud(rg));
    for (auto& x : b) x = Cx(ud(rg), ud(rg));
    gemm_naive(n, n, n, Cx(1), a.data(), n, b.data(), n, Op::none, Cx(0), c0.data(), n);
    gemm(n, n, n, Cx(1), a.data(), n, b.data(), n, Op::none, Cx(0), c1.data(), n);
    double err = 0.0;
    for (size_t i = 0; i < c0.size(); ++i) err = std::max(err, std::abs(c0[i] - c1[i]));
    CHECK(err < 1e-12);
    // batched, shared B: 3 blocks of a 4-mode-like layout
    const int P = 6, nm = 5, q = 3;
    std::vector<double> t(size_t(P) * nm * q), mm(size_t(nm) * nm), o0(size_t(P) * nm * q),
        o1(size_t(P) * nm * q, 0.0);
    for (auto& x : t) x = ud(rg);
    for (auto& x : mm) x = ud(rg);
    for (int i = 0; i < q; ++i)
      gemm_naive(P, nm, nm, 1.0, t.data() + size_t(i) * P * nm, P, mm.data(), nm, Op::transpose,
                 0.0, o0.data() + size_t(i) * P * nm, P);
    gemm_batch_shared_b(P, nm, nm, 1.0, t.data(), P, size_t(P) * nm, mm.data(), nm,
                        Op::transpose, 0.0, o1.data(), P, size_t(P) * nm, q);
    err = 0.0;
    for (size_t i = 0; i < o0.size(); ++i) err = std::max(err, std::abs(o0[i] - o1[i]));
    CHECK(err < 1e-13);
  }
  {  // solve / lu_factor (linsolve.hpp): residual and the singular case
    std::mt19937_64 rg(9);
    std::uniform_real_distribution<double> ud(-1.0, 1.0);
    const int n = 150, nr = 3;
    Matrix<double> a(n, n), b(n, nr);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) a(i, j) = ud(rg) + (i == j ? 4.0 : 0.0);
    for (int j = 0; j < nr; ++j)
      for (int i = 0; i < n; ++i) b(i, j) = ud(rg);
    Matrix<double> x = solve(a, b);
    double res = 0.0;
    for (int j = 0; j < nr; ++j)
      for (int i = 0; i < n; ++i) {
        double s = -b(i, j);
        for (int p = 0; p < n; ++p) s += a(i, p) * x(p, j);
        res = std::max(res, std::abs(s));
      }
    CHECK(res < 1e-12);
    Matrix<double> sing(3, 3);
    bool threw = false;
    try {
      lu_factor(sing);
    } catch (const std::runtime_error&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // the native NCCL communicator at world size 1: the re-partition is the
     // identity and the halos wrap onto the rank itself
    Communicator comm(1, 0, Communicator::unique_id());
    const long long A = 3, B = 4, C = 2, S = 2, n = A * B * C * S;
    std::vector<double> h(n);
    for (long long i = 0; i < n; ++i) h[i] = 0.5 * double(i) - 3.0;
    detail::DevBuf x(h.data(), n * sizeof(double)), y(n * sizeof(double));
    comm.repartition(1, A, B, C, S, 1, x.d(), y.d());
    std::vector<double> got(n);
    y.download(got.data());
    CHECK(got == h);
    detail::DevBuf left(4 * sizeof(double)), right(4 * sizeof(double));
    comm.halo(x.d(), x.d() + 4, 4, left.d(), right.d());
    std::vector<double> l(4), r(4);
    left.download(l.data());
    right.download(r.data());
    CHECK(l[0] == h[4] && l[3] == h[7] && r[0] == h[0] && r[3] == h[3]);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
