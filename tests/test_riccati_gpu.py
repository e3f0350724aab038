"""The reference's second benchmark problem on the GPU: the LQR differential
Riccati equation U' = A^T U + U A + C + U B U (src/problems.cpp:130-284) in
Kronecker form K = {A^T, A^T} with the nonlocal g(U) = C - (U b)(U^T b)^T,
and Rosenbrock-Euler (inc/integrators.hpp:166-194) with the per-step Jacobian
factors J = A^T - w b^T rebuilt on the device (:212-250).  Parity with the
oracle (pinned to the reference on CPU, tests/test_oracle_pins.py) and with
the reference's own run_riccati build, plus the reference's observed-order
table (run_riccati, src/bench_runner.cpp:205-229)."""
import numpy as np
import pytest

from conftest import rel2

pytestmark = pytest.mark.gpu

ALL = ["lawson_euler", "lawson2b", "exp_euler", "exp_euler_ls", "etd2rk", "rosenbrock_euler"]


def _og(c):
    import pyoracle
    return pyoracle.gfun(pyoracle.G_RICCATI, aux=[c.b, c.c_mat])


@pytest.mark.parametrize("method", ALL)
def test_riccati_vs_oracle(kp, port, method):
    from paper_2304_02327_b200 import problems
    c = problems.riccati(6, n_steps=20, method=method)
    want = port.integrate(method, c.u0, c.K, _og(c), 0.0, c.t_final, 20)
    got = kp.integrate_config(method, c.u0, c.K, c.g, 0.0, c.t_final, 20)
    assert rel2(got, want) < 1e-11


@pytest.mark.parametrize("method", ["etd2rk", "rosenbrock_euler"])
def test_riccati_vs_reference(kp, ref, method):
    """n_hat = 12 (144 x 144 state, dense 144 x 144 factors): the device run
    against the reference's own build_riccati + integrate."""
    from paper_2304_02327_b200 import problems
    c = problems.riccati(12, n_steps=40)
    want, _ = ref.run_riccati(12, method, 40, 0.025)
    got = kp.integrate_config(method, c.u0, c.K, c.g, 0.0, 0.025, 40)
    assert rel2(got, want) < 1e-11


def test_riccati_g_bitwise(kp, port):
    """The control products' KC-sliced FMA chains and fma(-w_i, z_j, c_ij)
    reproduce the oracle's g bit for bit (n = 300 > KC = 256 exercises the
    slice boundary)."""
    from paper_2304_02327_b200 import problems
    import pyoracle
    c = problems.riccati(18)  # n = 324
    n = c.b.size
    r = np.random.default_rng(7)
    u = np.asfortranarray(r.standard_normal((n, n)))
    want = port.eval_g(_og(c), 0.0, u)
    got = kp.eval_g(c.g, 0.0, u)
    assert np.array_equal(got, want)
    assert pyoracle.G_RICCATI == kp.G_RICCATI


def test_rosenbrock_step_with_given_jacobians(kp, port):
    """rosenbrock_euler_step through the step API with caller Jacobian
    factors (one shared object -> one phi_1 build) and two distinct ones."""
    from paper_2304_02327_b200 import problems
    c = problems.riccati(5)
    n = c.b.size
    r = np.random.default_rng(3)
    u = np.asfortranarray(r.standard_normal((n, n)) * 0.1)
    tau = 1e-3
    j1 = np.asfortranarray(c.a_t - 0.3 * np.outer(r.standard_normal(n), c.b))
    j2 = np.asfortranarray(c.a_t - 0.2 * np.outer(r.standard_normal(n), c.b))
    for jac in ([j1, j1], [j1, j2]):
        want = port.step("rosenbrock_euler", u, 0.0, tau, c.K, jac, 1.0, None, 1.0, _og(c))
        got = kp.rosenbrock_euler_step(u, 0.0, tau, c.K, c.g, jac)
        assert rel2(got, want) < 1e-12


def test_rosenbrock_requires_riccati(kp):
    from paper_2304_02327_b200 import problems
    c = problems.riccati(4)
    with pytest.raises(kp.InvalidArgument, match="jacobian_factors"):
        kp.integrate_config("rosenbrock_euler", c.u0, c.K, kp.G.zero(), 0.0, 0.025, 3)


def test_riccati_order_table(kp):
    """The reference's run_riccati sweep at n_hat = 10: errors against an
    ETD2RK 4096-step solution at steps {30,65,100,135,170}; observed orders
    ~2 for both methods (PAPER.md's riccati_order table reports
    {2.05, 2.03, 2.02, 2.02} at n_hat = 30)."""
    from paper_2304_02327_b200 import problems
    c = problems.riccati(10)
    refsol = kp.integrate_config("etd2rk", c.u0, c.K, c.g, 0.0, 0.025, 4096)
    steps = [30, 65, 100, 135, 170]
    for m in ("rosenbrock_euler", "etd2rk"):
        errs = []
        for s in steps:
            u = kp.integrate_config(m, c.u0, c.K, c.g, 0.0, 0.025, s)
            errs.append(rel2(u, refsol))
        orders = [np.log(errs[i - 1] / errs[i]) / np.log(steps[i] / steps[i - 1])
                  for i in range(1, len(steps))]
        assert all(1.95 < o < 2.1 for o in orders), (m, orders)
