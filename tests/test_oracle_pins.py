"""Pin the CPU oracle (oracle/kp_oracle.c, the restatement used as the GPU
checker) to the real reference: golden vectors produced by the reference
library itself (tests/golden/make_golden.py) and the reference's own
known-answer tests (tests/test_*.cpp of the reference).  CPU only."""
import math
import os

import numpy as np
import pytest

from conftest import ROOT, rel2, rng

GOLD = os.path.join(ROOT, "tests", "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def test_tucker_kronsum_bitwise(port):
    z = load("tucker_small.npz")
    ms = [z["m0"], z["m1"], z["m2"]]
    assert np.array_equal(port.tucker(z["t"], ms), z["tucker"])
    assert np.array_equal(port.kronsum(z["t"], ms), z["kronsum"])


def test_mode_product_kc_and_accumulate_bitwise(port):
    z = load("mode_product_kc.npz")
    assert np.array_equal(port.mode_product(z["t"], z["m"], 0), z["out"])
    z = load("mode_product_acc.npz")
    assert np.array_equal(port.mode_product(z["t"], z["m"], 1, out=z["base"]), z["out"])


def test_complex_tucker(port):
    z = load("tucker_c128.npz")
    ms = [z["m0"], z["m1"], z["m2"]]
    assert rel2(port.tucker(z["t"], ms), z["tucker"]) < 1e-15
    assert rel2(port.kronsum(z["t"], ms), z["kronsum"]) < 1e-15


def test_gll_bitwise(port):
    z = load("gll.npz")
    for q in range(2, 21):
        x, w = port.gll_rule(q)
        assert np.array_equal(x, z[f"x{q}"]) and np.array_equal(w, z[f"w{q}"])


def test_gll_closed_forms(port):
    # reference tests/test_matrix_functions.cpp:110-143
    x, w = port.gll_rule(2)
    assert list(x) == [0.0, 1.0] and abs(w[0] - 0.5) < 1e-15
    x, w = port.gll_rule(3)
    assert abs(x[1] - 0.5) < 1e-15 and abs(w[1] - 2 / 3) < 1e-14
    for q in range(2, 21):
        x, w = port.gll_rule(q)
        assert abs(w.sum() - 1) < 1e-14


def test_expm(port):
    z = load("expm.npz")
    for i in range(3):
        assert rel2(port.expm(z[f"x{i}"]), z[f"e{i}"]) < 1e-14
    assert rel2(port.expm(z["z"]), z["ez"]) < 1e-14


def test_phiquad(port):
    z = load("phiquad.npz")
    for tag in ("fd", "rn"):
        phis, s = port.phiquad(z[f"{tag}_x"], 2)
        assert s == int(z[f"{tag}_s"])
        for j in range(3):
            assert rel2(phis[j], z[f"{tag}_p{j}"]) < 1e-14


def test_phiquad_kats(port):
    # reference tests/test_matrix_functions.cpp:145-174
    phis, _ = port.phiquad(np.zeros((4, 4)), 2)
    for ell in range(3):
        assert np.abs(phis[ell] - np.eye(4) / math.factorial(ell)).max() < 1e-15
    phis, _ = port.phiquad(np.array([[1.0]]), 2)
    assert abs(phis[1][0, 0] - (math.e - 1)) < 1e-13 and abs(phis[2][0, 0] - (math.e - 2)) < 1e-13
    phis, s = port.phiquad(np.array([[2.0]]), 1)
    assert s == 2 and abs(phis[1][0, 0] - (math.e ** 2 - 1) / 2) < 1e-12


def test_split_phi(port):
    z = load("split_phi.npz")
    As = [z["A0"], z["A1"], z["A2"]]
    for ell in (0, 1, 2):
        fs, pref = port.build_split_phi(As, 0.02, ell)
        assert pref == float(z[f"pref{ell}"])
        for mu in range(3):
            assert rel2(fs[mu], z[f"f{ell}_{mu}"]) < 1e-14


def test_fd_operator_bitwise(port):
    z = load("fd.npz")
    assert np.array_equal(port.fd_operator_1d(7, 0.75, 0.1), z["a"])
    from paper_2304_02327_b200 import problems
    assert np.array_equal(problems.fd_operator_1d(7, 0.75, 0.1), z["a"])
    assert np.array_equal(problems.fd_operator_1d(5, 0.01), z["b"])


INTEGRATE_TAGS = ["ac2d", "ac3d", "ac2d_lawson", "ac2d_ls", "bru_etd", "bru_l2b", "nls_ee",
                  "nls_etd"]


def golden_case(z, tag):
    import pyoracle
    meta = z[f"{tag}_meta"]
    kind, tau, n_steps = int(meta[0]), float(meta[1]), int(meta[2])
    g = pyoracle.gfun(kind, *meta[3:7])
    As = []
    mu = 0
    while f"{tag}_A{mu}" in z:
        As.append(z[f"{tag}_A{mu}"])
        mu += 1
    return int(z[f"{tag}_method"]), z[f"{tag}_u0"], As, g, tau, n_steps, z[f"{tag}_out"]


@pytest.mark.parametrize("tag", INTEGRATE_TAGS)
def test_integrate(port, tag):
    z = load("integrate.npz")
    m, u0, As, g, tau, n, want = golden_case(z, tag)
    got = port.integrate(m, u0, As, g, 0.0, tau * n, n)
    assert rel2(got, want) < 1e-13


def test_restatement_vs_live_reference(port, ref):
    """Random shapes against the live reference when it is built here."""
    r = rng(42)
    for dims in [(3, 4), (2, 3, 4, 5), (17, 9, 6)]:
        t = np.asfortranarray(r.uniform(-1, 1, dims))
        ms = [np.asfortranarray(r.uniform(-1, 1, (n, n))) for n in dims]
        assert np.array_equal(port.tucker(t, ms), ref.tucker(t, ms))
        assert np.array_equal(port.kronsum(t, ms), ref.kronsum(t, ms))


def test_validation_messages(port):
    # reference tests/test_tensor.cpp:118-124
    import pyoracle
    t = np.zeros((3, 4, 5))
    with pytest.raises(pyoracle.InvalidArgument, match="mode 1"):
        port.mode_product(t, np.zeros((6, 9)), 1)
    with pytest.raises(pyoracle.InvalidArgument):
        port.mode_product(t, np.zeros((6, 9)), 7)


def test_divergence(port):
    import pyoracle
    with pytest.raises(pyoracle.Divergence, match="step"):
        port.integrate("lawson_euler", np.array([1e100, 1e100]), [np.zeros((2, 2))],
                       pyoracle.gfun(pyoracle.G_SQUARE), 0.0, 10.0, 10)


@pytest.mark.parametrize("method", ["etd2rk", "rosenbrock_euler", "exp_euler"])
def test_riccati_restatement_vs_live_reference(port, ref, method):
    """The Riccati problem data (problems.riccati restating build_riccati,
    src/problems.cpp:130-186), its g (:263-276) and the oracle's
    Rosenbrock-Euler (inc/integrators.hpp:166-194 with the Jacobian factors
    of :212-250) against the reference's own build + integrate.  ~1e-16:
    the residual difference is the reference's vectorised LU rounding inside
    phiquad (see test_phiquad)."""
    import pyoracle
    from paper_2304_02327_b200 import problems
    c = problems.riccati(6)
    g = pyoracle.gfun(pyoracle.G_RICCATI, aux=[c.b, c.c_mat])
    for steps in (1, 7):
        want, _ = ref.run_riccati(6, method, steps, 0.025)
        got = port.integrate(method, c.u0, c.K, g, 0.0, 0.025, steps)
        assert rel2(got, want) < 1e-14


def test_riccati_rosenbrock_needs_riccati_g(port):
    import pyoracle
    from paper_2304_02327_b200 import problems
    c = problems.riccati(3)
    with pytest.raises(pyoracle.InvalidArgument, match="jacobian_factors"):
        port.integrate("rosenbrock_euler", c.u0, c.K, pyoracle.gfun(pyoracle.G_ZERO), 0.0,
                       0.025, 2)
