// Reference-style integrator tests against the C++ drop-in, written the way
// /root/reference/proj/tests/test_integrators.cpp is (host lambda g's,
// ProblemSpec / StepperConfig / IntegrateResult, Backend::DenseOracle,
// trajectory sampling, DivergenceError), compiled against the
// reference-named headers include/kronphi/*.hpp and run on the GPU
// (tests/test_cpp_api.py).  The cases restate :84-110, :350-444 of that file.
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "kronphi/integrators.hpp"
#include "kronphi/problems.hpp"
#include "mini_doctest.h"

using namespace kronphi;

namespace {

std::mt19937_64 rng(555);

Matrix<double> random_stable(int n) {
  std::uniform_real_distribution<double> dist(-1, 1);
  Matrix<double> m(n, n);
  for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = dist(rng);
  const double shift = m.norm1();
  for (int i = 0; i < n; ++i) m(i, i) -= shift;
  return m;
}

Tensor<double> random_tensor(std::vector<int> dims) {
  std::uniform_real_distribution<double> dist(-1, 1);
  Tensor<double> t(std::move(dims));
  for (std::size_t i = 0; i < t.size(); ++i) t[i] = dist(rng);
  return t;
}

GFun square_g() {
  return [](double, const Tensor<double>& u) {
    Tensor<double> g(u.dims());
    for (std::size_t i = 0; i < u.size(); ++i) g[i] = u[i] * u[i];
    return g;
  };
}

// a small nonlinear 2-D Kronecker problem with a time-dependent host g
ProblemSpec small_problem() {
  ProblemSpec p;
  p.K = KroneckerSum<double>({random_stable(5), random_stable(6)});
  p.g = [](double t, const Tensor<double>& u) {
    Tensor<double> g(u.dims());
    for (std::size_t i = 0; i < u.size(); ++i) g[i] = 0.2 / (1.0 + u[i] * u[i]) + 0.1 * std::cos(t);
    return g;
  };
  p.u0 = random_tensor({5, 6});
  p.t0 = 0.0;
  p.t_final = 1.0;
  return p;
}

double rel_fro(const Tensor<double>& a, const Tensor<double>& b) {
  return diff_norm_fro(a, b) / b.norm_fro();
}

double slope(const std::vector<double>& x, const std::vector<double>& y) {
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  const double n = double(x.size());
  for (size_t i = 0; i < x.size(); ++i) {
    const double lx = std::log(x[i]), ly = std::log(y[i]);
    sx += lx;
    sy += ly;
    sxx += lx * lx;
    sxy += lx * ly;
  }
  return (n * sxy - sx * sy) / (n * sxx - sx * sx);
}

}  // namespace

TEST_CASE("trajectory sampling") {
  ProblemSpec p = small_problem();
  StepperConfig c;
  c.method = Method::LawsonEuler;
  c.n_steps = 20;
  c.sample_every = 5;
  const auto res = integrate(p, c);
  REQUIRE(res.trajectory.size() == 5);  // steps 0, 5, 10, 15, 20
  CHECK(res.trajectory.front().first == 0.0);
  CHECK(res.trajectory.back().first == doctest::Approx(1.0));
  CHECK(diff_norm_inf(res.trajectory.back().second, res.final) == 0.0);
  CHECK(res.wallclock_s >= res.loop_s);
}

TEST_CASE("trajectory sampling on the device path (device g)") {
  ProblemSpec p;
  p.K = KroneckerSum<double>({random_stable(8), random_stable(7), random_stable(6)});
  p.g = g_allen_cahn();
  p.u0 = random_tensor({8, 7, 6});
  p.t_final = 0.5;
  StepperConfig c;
  c.method = Method::ETD2RK;
  c.n_steps = 12;
  const auto plain = integrate(p, c);
  c.sample_every = 4;
  const auto res = integrate(p, c);
  REQUIRE(res.trajectory.size() == 4);  // steps 0, 4, 8, 12
  CHECK(res.trajectory[1].first == doctest::Approx(p.t0 + 4 * (0.5 / 12)));
  CHECK(diff_norm_inf(res.trajectory.back().second, res.final) == 0.0);
  CHECK(diff_norm_inf(res.final, plain.final) == 0.0);  // sampling does not change a bit
  CHECK(diff_norm_inf(res.trajectory.front().second, p.u0) == 0.0);
}

TEST_CASE("integrate with one step equals the single-step operation (host g)") {
  ProblemSpec p = small_problem();
  const double tau = 0.4;
  p.t_final = tau;
  const auto exps = build_split_phi(p.K, tau, 0).factors;
  const SplitPhi<double> phi1 = build_split_phi(p.K, tau, 1);
  const SplitPhi<double> phi2 = build_split_phi(p.K, tau, 2);
  StepperConfig c;
  c.n_steps = 1;
  c.method = Method::LawsonEuler;
  CHECK(diff_norm_inf(integrate(p, c).final, lawson_euler_step(p.u0, 0.0, tau, p.g, exps)) == 0.0);
  c.method = Method::Lawson2b;
  CHECK(diff_norm_inf(integrate(p, c).final, lawson2b_step(p.u0, 0.0, tau, p.g, exps)) == 0.0);
  c.method = Method::ExpEuler;
  CHECK(diff_norm_inf(integrate(p, c).final,
                      exp_euler_step(p.u0, 0.0, tau, p.K, p.g, phi1)) == 0.0);
  c.method = Method::ETD2RK;
  CHECK(diff_norm_inf(integrate(p, c).final,
                      etd2rk_step(p.u0, 0.0, tau, p.K, p.g, phi1, phi2)) == 0.0);
}

TEST_CASE("host g equals the same device g") {
  // Allen-Cahn as a host lambda vs the device KP_G_ALLEN_CAHN: the loop
  // structures differ (host round trips vs fused epilogues), the values agree
  ProblemSpec p;
  p.K = KroneckerSum<double>({random_stable(9), random_stable(8)});
  p.u0 = random_tensor({9, 8});
  p.t_final = 0.3;
  StepperConfig c;
  c.n_steps = 10;
  for (Method m : {Method::ExpEuler, Method::ETD2RK, Method::Lawson2b}) {
    c.method = m;
    p.g = g_allen_cahn();
    const auto dev = integrate(p, c);
    p.g = [](double, const Tensor<double>& u) {
      Tensor<double> g(u.dims());
      for (std::size_t i = 0; i < u.size(); ++i) g[i] = u[i] - u[i] * u[i] * u[i];
      return g;
    };
    const auto host = integrate(p, c);
    CHECK(rel_fro(host.final, dev.final) < 1e-13);
  }
}

TEST_CASE("backend equivalence: Lawson methods agree to roundoff") {
  ProblemSpec p = small_problem();
  for (Method m : {Method::LawsonEuler, Method::Lawson2b}) {
    StepperConfig c;
    c.method = m;
    c.n_steps = 20;
    const auto split = integrate(p, c);
    c.backend = Backend::DenseOracle;
    const auto dense = integrate(p, c);
    CHECK(rel_fro(split.final, dense.final) < 1e-12);
  }
}

TEST_CASE("backend equivalence: phi methods converge together at order >= 2") {
  ProblemSpec p = small_problem();
  for (Method m : {Method::ExpEuler, Method::ETD2RK}) {
    std::vector<double> taus, diffs;
    for (long n : {8L, 16L, 32L, 64L}) {
      StepperConfig c;
      c.method = m;
      c.n_steps = n;
      const auto split = integrate(p, c);
      c.backend = Backend::DenseOracle;
      const auto dense = integrate(p, c);
      taus.push_back(1.0 / double(n));
      diffs.push_back(rel_fro(split.final, dense.final));
    }
    CHECK(slope(taus, diffs) >= 1.9);
  }
}

TEST_CASE("divergence is reported with the step index") {
  ProblemSpec p;
  p.K = KroneckerSum<double>({Matrix<double>(2, 2)});
  p.g = square_g();
  p.u0 = Tensor<double>({2}, {1e100, 1e100});
  p.t_final = 10.0;
  StepperConfig c;
  c.method = Method::LawsonEuler;
  c.n_steps = 10;
  bool caught = false;
  try {
    integrate(p, c);
  } catch (const DivergenceError& e) {
    caught = true;
    CHECK(e.step() >= 1);
    CHECK(std::string(e.what()).find("step") != std::string::npos);
    CHECK(std::string(e.what()) == "state became non-finite at step 2 (t = 2.000000)");
  }
  CHECK(caught);
  // the device path reports the same step and message
  p.g = g_square();
  caught = false;
  try {
    integrate(p, c);
  } catch (const DivergenceError& e) {
    caught = true;
    CHECK(std::string(e.what()) == "state became non-finite at step 2 (t = 2.000000)");
  }
  CHECK(caught);
}

TEST_CASE("rosenbrock without a jacobian callback is a configuration error") {
  ProblemSpec p = small_problem();
  StepperConfig c;
  c.method = Method::RosenbrockEuler;
  c.n_steps = 4;
  CHECK_THROWS_AS(integrate(p, c), std::invalid_argument);
}

TEST_CASE("rosenbrock with the exact linear Jacobian is exponential Euler") {
  // g linear in u (g = 0.3 u): J = K + 0.3 I split as J_1 = A_1 + 0.3 I, J_2 = A_2
  ProblemSpec p = small_problem();
  p.g = [](double, const Tensor<double>& u) {
    Tensor<double> g(u.dims());
    for (std::size_t i = 0; i < u.size(); ++i) g[i] = 0.3 * u[i];
    return g;
  };
  const auto k = p.K;
  p.jacobian_factors = [k](const Tensor<double>&) {
    std::vector<Matrix<double>> j = k.factors;
    for (int i = 0; i < j[0].rows(); ++i) j[0](i, i) += 0.3;
    return j;
  };
  StepperConfig c;
  c.n_steps = 8;
  c.method = Method::RosenbrockEuler;
  const auto ros = integrate(p, c);
  CHECK(ros.final.all_finite());
  // one Rosenbrock step vs the step function with the same factors
  const auto one = rosenbrock_euler_step(p.u0, 0.0, 0.125, p.K, p.g, p.jacobian_factors(p.u0));
  ProblemSpec p1 = p;
  p1.t_final = 0.125;
  c.n_steps = 1;
  CHECK(diff_norm_inf(integrate(p1, c).final, one) == 0.0);
}

TEST_CASE("rosenbrock on the dense backend: one step differs from the split one at third order") {
  // g = 0.3 u with the exact Jacobian: the dense backend applies phi_1(tau J)
  // of the assembled Kronecker sum (inc/integrators.hpp:329-338), the split
  // backend the product of the per-direction phi_1's -- equal up to O(tau^3)
  ProblemSpec p = small_problem();
  p.g = [](double, const Tensor<double>& u) {
    Tensor<double> g(u.dims());
    for (std::size_t i = 0; i < u.size(); ++i) g[i] = 0.3 * u[i];
    return g;
  };
  const auto k = p.K;
  p.jacobian_factors = [k](const Tensor<double>&) {
    std::vector<Matrix<double>> j = k.factors;
    for (int i = 0; i < j[0].rows(); ++i) j[0](i, i) += 0.3;
    return j;
  };
  std::vector<double> taus, diffs;
  for (int e = 4; e <= 7; ++e) {
    const double tau = std::ldexp(1.0, -e);
    p.t_final = tau;
    StepperConfig c;
    c.n_steps = 1;
    c.method = Method::RosenbrockEuler;
    const auto split = integrate(p, c);
    c.backend = Backend::DenseOracle;
    const auto dense = integrate(p, c);
    CHECK(dense.final.all_finite());
    taus.push_back(tau);
    diffs.push_back(rel_fro(split.final, dense.final));
  }
  CHECK(slope(taus, diffs) >= 2.7);
  CHECK(slope(taus, diffs) <= 3.3);
}

TEST_CASE("riccati helpers: rhs, Jacobian factors, ARE residual (problems.hpp)") {
  const RiccatiProblem pr = build_riccati(6);
  const int n = pr.a.rows();
  // U = 0: the right-hand side is C, one Jacobian factor A^T serves both modes
  CHECK(diff_norm_inf(tensor_from_matrix(riccati_rhs(pr.u0, pr)), tensor_from_matrix(pr.c_mat)) == 0.0);
  CHECK(are_residual(pr.u0, pr) == doctest::Approx(pr.c_mat.norm_fro()).epsilon(1e-15));
  auto j0 = riccati_jacobian_factors(pr.u0, pr);
  CHECK(j0.size() == 2);
  CHECK(diff_norm_inf(tensor_from_matrix(j0[0]), tensor_from_matrix(pr.a_t)) == 0.0);
  // a symmetric U: J = A^T - (U b) b^T, and rhs = A^T U + U A + C - (U b)(U^T b)^T
  Matrix<double> u(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) u(i, j) = 0.01 * std::cos(0.3 * (i + 1)) * std::cos(0.3 * (j + 1)) + (i == j ? 0.02 : 0.0);
  std::vector<double> w(n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) w[i] += u(i, j) * pr.b[j];
  const auto js = riccati_jacobian_factors(u, pr);
  double ejac = 0.0, erhs = 0.0, scale = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      ejac = std::max(ejac, std::abs(js[0](i, j) - (pr.a_t(i, j) - w[i] * pr.b[j])));
  CHECK(ejac < 1e-12 * pr.a.norm1());
  const Matrix<double> rhs = riccati_rhs(u, pr);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      double v = pr.c_mat(i, j) - w[i] * w[j];
      for (int k = 0; k < n; ++k) v += pr.a_t(i, k) * u(k, j) + u(i, k) * pr.a(k, j);
      erhs = std::max(erhs, std::abs(rhs(i, j) - v));
      scale = std::max(scale, std::abs(v));
    }
  CHECK(erhs < 1e-12 * scale);
  CHECK_THROWS_AS(riccati_rhs(Matrix<double>(3, 3), pr), std::invalid_argument);
}

TEST_CASE("ADR problem: exact, source and g members (problems.hpp)") {
  const ADRProblem pr = build_adr(6, 7, 8);
  const ProblemSpec spec = pr.to_problem_spec();
  REQUIRE(bool(spec.exact));
  CHECK(diff_norm_inf(spec.exact(0.0), pr.u0) == 0.0);
  CHECK(diff_norm_inf(spec.exact(0.5), pr.exact(0.5)) == 0.0);
  // g(t, u) - 1/(1+u^2) = Psi(t, .), and the exact solution satisfies the ODE:
  // d/dt (e^t u0) = K e^t u0 + g(t, e^t u0) up to the FD truncation (exact for
  // this polynomial u0 with second-order differences)
  const double t = 0.3;
  const Tensor<double> u = pr.exact(t);
  const Tensor<double> g = pr.g(t, u), psi = pr.source(t);
  double e1 = 0.0;
  for (std::size_t r = 0; r < u.size(); ++r)
    e1 = std::max(e1, std::abs(g[r] - (1.0 / (1.0 + u[r] * u[r]) + psi[r])));
  CHECK(e1 < 1e-13);
  Tensor<double> rhs = kronsum_action(u, spec.K);
  axpy(1.0, g, rhs);
  CHECK(diff_norm_inf(rhs, u) < 1e-10 * u.norm_inf() + 1e-11);
}

TEST_CASE("shape mismatches are invalid_argument before any device work") {
  ProblemSpec p = small_problem();
  StepperConfig c;
  c.n_steps = 2;
  ProblemSpec bad = p;
  bad.K = KroneckerSum<double>({random_stable(5)});
  CHECK_THROWS_AS(integrate(bad, c), std::invalid_argument);
  bad = p;
  bad.K = KroneckerSum<double>({random_stable(5), random_stable(7)});
  CHECK_THROWS_AS(integrate(bad, c), std::invalid_argument);
  const auto phi1 = build_split_phi(p.K, 0.1, 1);
  CHECK_THROWS_AS(exp_euler_step(random_tensor({6, 5}), 0.0, 0.1, p.K, p.g, phi1),
                  std::invalid_argument);
}

TEST_CASE("method name round trip") {
  for (Method m : {Method::LawsonEuler, Method::Lawson2b, Method::ExpEuler,
                   Method::ExpEulerLinearSplit, Method::ETD2RK, Method::RosenbrockEuler})
    CHECK(parse_method(method_name(m)) == m);
}

TEST_CASE("problem spec carries the exact solution") {
  ProblemSpec p = small_problem();
  p.exact = [](double t) { return Tensor<double>({1}, {std::exp(t)}); };
  CHECK(p.exact(0.0)[0] == 1.0);
}

TEST_CASE("sharded integrate through a Communicator (world size 1) equals integrate") {
  ProblemSpec p;
  p.K = KroneckerSum<double>({fd_operator_1d(16, 0.01, 0.0), fd_operator_1d(12, 0.01, 0.0),
                              fd_operator_1d(8, 0.01, 0.0)});
  p.g = g_allen_cahn();
  p.u0 = random_tensor({16, 12, 8});
  p.t_final = 0.02;
  StepperConfig c;
  c.method = Method::ETD2RK;
  c.n_steps = 10;
  const auto single = integrate(p, c);
  Communicator comm(1, 0, Communicator::unique_id());
  ModeD used = ModeD::Measure;
  const auto sh = integrate(p, c, comm, ModeD::Measure, &used);
  CHECK(used == ModeD::AllToAll);  // one rank: the identity exchange
  CHECK(diff_norm_inf(sh.final, single.final) == 0.0);
}

int main() { return mini_doctest::run_all(); }
