"""The round-2 boundary additions through the Python mirror (the C++ drop-in
has the same in tests/cpp/test_integrators_api.cpp): trajectory sampling
(StepperConfig.sample_every / IntegrateResult.trajectory,
inc/integrators.hpp:284-287,365-366), Backend::DenseOracle
(:243-262) and the DivergenceError message (:86-97)."""
import numpy as np
import pytest

from conftest import rel2, rng

pytestmark = pytest.mark.gpu


def stable(r, n):
    m = r.uniform(-1, 1, (n, n))
    m -= np.abs(m).sum(0).max() * np.eye(n)
    return np.asfortranarray(m)


def test_trajectory_sampling_device_path(kp):
    r = rng(31)
    K = [stable(r, 8), stable(r, 7), stable(r, 6)]
    u0 = np.asfortranarray(r.uniform(-1, 1, (8, 7, 6)))
    spec = kp.ProblemSpec(K, kp.G.allen_cahn(), u0, 0.0, 0.5)
    plain = kp.integrate(spec, kp.StepperConfig(kp.Method.ETD2RK, 12))
    res = kp.integrate(spec, kp.StepperConfig(kp.Method.ETD2RK, 12, sample_every=4))
    assert len(res.trajectory) == 4  # steps 0, 4, 8, 12
    assert res.trajectory[0][0] == 0.0 and np.array_equal(res.trajectory[0][1], u0)
    assert abs(res.trajectory[-1][0] - 0.5) < 1e-15
    assert np.array_equal(res.trajectory[-1][1], res.final)
    assert np.array_equal(res.final, plain.final)  # sampling does not change a bit
    # every sample equals the integrate of that many steps
    three = kp.integrate(kp.ProblemSpec(K, kp.G.allen_cahn(), u0, 0.0, 0.5 * 8 / 12),
                         kp.StepperConfig(kp.Method.ETD2RK, 8))
    assert rel2(res.trajectory[2][1], three.final) < 1e-14


def test_trajectory_sampling_every_step_complex(kp):
    from paper_2304_02327_b200 import problems
    c = problems.nls(n=16, n_steps=3)
    res = kp.integrate(kp.ProblemSpec(c.K, c.g, c.u0, 0.0, c.t_final),
                       kp.StepperConfig(kp.Method.ETD2RK, 3, sample_every=1))
    assert len(res.trajectory) == 4
    assert np.array_equal(res.trajectory[-1][1], res.final)


@pytest.mark.parametrize("method", ["lawson_euler", "lawson2b"])
def test_dense_oracle_lawson_agrees_to_roundoff(kp, method):
    # tests/test_integrators.cpp:373-384
    r = rng(5)
    K = [stable(r, 5), stable(r, 6)]
    u0 = np.asfortranarray(r.uniform(-1, 1, (5, 6)))
    spec = kp.ProblemSpec(K, kp.G.allen_cahn(), u0, 0.0, 1.0)
    m = kp.parse_method(method)
    split = kp.integrate(spec, kp.StepperConfig(m, 20))
    dense = kp.integrate(spec, kp.StepperConfig(m, 20, backend="dense_oracle"))
    assert rel2(split.final, dense.final) < 1e-12


def test_dense_oracle_phi_methods_converge_together(kp):
    # tests/test_integrators.cpp:386-402: split - dense = O(tau^2)
    r = rng(6)
    K = [stable(r, 5), stable(r, 6)]
    u0 = np.asfortranarray(r.uniform(-1, 1, (5, 6)))
    spec = kp.ProblemSpec(K, kp.G.allen_cahn(), u0, 0.0, 1.0)
    for m in (kp.Method.ExpEuler, kp.Method.ETD2RK):
        taus, diffs = [], []
        for n in (8, 16, 32, 64):
            a = kp.integrate(spec, kp.StepperConfig(m, n)).final
            b = kp.integrate(spec, kp.StepperConfig(m, n, backend="dense_oracle")).final
            taus.append(1.0 / n)
            diffs.append(rel2(a, b))
        assert np.polyfit(np.log(taus), np.log(diffs), 1)[0] >= 1.9


def test_divergence_message_is_the_references(kp):
    # tests/test_integrators.cpp:404-422 and the message of :86-97
    spec = kp.ProblemSpec([np.zeros((2, 2))], kp.G.square(), np.array([1e100, 1e100]), 0.0, 10.0)
    with pytest.raises(kp.DivergenceError) as e:
        kp.integrate(spec, kp.StepperConfig(kp.Method.LawsonEuler, 10))
    assert e.value.step == 2  # 1e100 -> 1e200 -> inf
    assert "state became non-finite at step 2 (t = 2.000000)" in str(e.value)
