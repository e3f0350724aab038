"""GPU parity of the device phi-factor builder (expm, phiquad, split phi)
against the CPU oracle, plus the reference's known-answer tests
(tests/test_matrix_functions.cpp, tests/test_split_phi.cpp).  Tolerance for
the phi tables: rel-1-norm <= 1e-12."""
import math

import numpy as np
import pytest

from conftest import rel2, rng

pytestmark = pytest.mark.gpu


def rel1(a, b):
    return float(np.abs(a - b).sum(0).max() / np.abs(b).sum(0).max())


def rand_norm(r, n, target, cplx=False):
    m = r.uniform(-1, 1, (n, n))
    if cplx:
        m = m + 1j * r.uniform(-1, 1, (n, n))
    m *= target / np.abs(m).sum(0).max()
    return np.asfortranarray(m)


@pytest.mark.parametrize("target", [0.01, 0.2, 0.9, 2.0, 5.0, 20.0, 800.0])
def test_expm_vs_oracle(kp, port, target):
    for n in (3, 8, 33, 70):
        x = rand_norm(rng(n), n, target)
        assert rel1(kp.expm(x), port.expm(x)) < 1e-12


def test_expm_kats(kp):
    # tests/test_matrix_functions.cpp:56-80
    assert np.array_equal(kp.expm(np.zeros((3, 3))), np.eye(3))
    e = kp.expm(np.diag([1.0, 2.0]))
    assert abs(e[0, 0] - math.e) < 1e-14 * math.e and abs(e[1, 1] - math.e ** 2) < 1e-14 * 8
    e = kp.expm(np.array([[0.0, 1.0], [0.0, 0.0]]))
    assert abs(e[0, 1] - 1.0) < 1e-15 and e[1, 0] == 0.0


def test_expm_complex(kp, port):
    # tests/test_matrix_functions.cpp:100-108: e^{i sigma_x}
    x = np.array([[0, 1j], [1j, 0]])
    e = kp.expm(x)
    assert abs(e[0, 0] - math.cos(1.0)) < 1e-14 and abs(e[0, 1] - 1j * math.sin(1.0)) < 1e-14
    for target in (0.3, 3.0, 40.0):
        z = rand_norm(rng(5), 12, target, True)
        assert rel1(kp.expm(z), port.expm(z)) < 1e-12


@pytest.mark.parametrize("n", [16, 64, 128, 256])
def test_phiquad_fd_operator(kp, port, n):
    """The sweep factors: phi_l(1e-3 * Laplacian), s = 3..9."""
    x = np.asfortranarray(port.fd_operator_1d(n, 1.0) * 1e-3)
    tab = kp.phiquad(x, 2)
    want, s = port.phiquad(x, 2)
    assert tab.scaling_exponent == s
    for j in range(3):
        assert rel1(tab.phis[j], want[j]) < 1e-12, j


def test_phiquad_random_and_forced(kp, port):
    r = rng(9)
    for n, target in [(10, 20.0), (7, 3.0), (40, 0.5), (65, 150.0)]:
        x = rand_norm(r, n, target)
        tab = kp.phiquad(x, 3)
        want, s = port.phiquad(x, 3)
        assert tab.scaling_exponent == s
        for j in range(4):
            assert rel1(tab.phis[j], want[j]) < 1e-12
        forced = kp.phiquad(x, 2, forced_scaling=s + 1)
        for j in range(3):
            assert rel1(forced.phis[j], tab.phis[j]) < 1e-11
    with pytest.raises(kp.InvalidArgument):
        kp.phiquad(rand_norm(r, 8, 6.0), 2, forced_scaling=0)


def test_phiquad_closed_forms(kp):
    # tests/test_matrix_functions.cpp:145-174
    tab = kp.phiquad(np.zeros((4, 4)), 2)
    for ell in range(3):
        assert np.abs(tab.phis[ell] - np.eye(4) / math.factorial(ell)).sum(0).max() < 1e-15
    tab = kp.phiquad(np.array([[1.0]]), 2)
    e = math.e
    assert abs(tab.phis[0][0, 0] - e) < 1e-13 * e
    assert abs(tab.phis[1][0, 0] - (e - 1)) < 1e-13
    assert abs(tab.phis[2][0, 0] - (e - 2)) < 1e-13
    tab = kp.phiquad(np.array([[2.0]]), 1)
    assert tab.scaling_exponent == 2
    assert abs(tab.phis[1][0, 0] - (e * e - 1) / 2) < 1e-13 * 4


def test_phiquad_complex(kp, port):
    """NLS factors: phi_l of (i/2) tau Laplacian (periodic)."""
    import pyoracle
    n = 64
    x = np.asfortranarray(0.5j * 1e-3 * pyoracle.periodic_laplacian_1d(n, 16.0 / 512))
    tab = kp.phiquad(x, 2)
    want, s = port.phiquad(x, 2)
    assert tab.scaling_exponent == s
    for j in range(3):
        assert rel1(tab.phis[j], want[j]) < 1e-12


def test_split_prefactors(kp):
    # tests/test_split_phi.cpp:66-75
    r = rng(3)
    k2 = [rand_norm(r, 3, 1.0), rand_norm(r, 4, 1.0)]
    k3 = [rand_norm(r, 2, 1.0), rand_norm(r, 3, 1.0), rand_norm(r, 2, 1.0)]
    assert kp.build_split_phi(k2, 0.1, 1).prefactor == 1.0
    assert kp.build_split_phi(k3, 0.1, 1).prefactor == 1.0
    assert kp.build_split_phi(k3, 0.1, 2).prefactor == 4.0
    assert kp.build_split_phi(k2, 0.1, 0).prefactor == 1.0
    assert kp.build_split_phi(k2, 0.1, 3).prefactor == 6.0
    with pytest.raises(kp.InvalidArgument):
        kp.build_split_phi(k2, 0.1, -1)


def test_split_vs_oracle_and_apply(kp, port):
    r = rng(4)
    As = [port.fd_operator_1d(n, 0.05) for n in (12, 20, 16)]
    v = np.asfortranarray(r.standard_normal((12, 20, 16)))
    for ell in (0, 1, 2):
        sp = kp.build_split_phi(As, 0.01, ell)
        fs, pref = port.build_split_phi(As, 0.01, ell)
        assert sp.prefactor == pref
        for a, b in zip(sp.factors, fs):
            assert rel1(a, b) < 1e-12
        got = kp.apply_split_phi(sp, v)
        want = port.apply_split_phi(v, fs, pref)
        assert rel2(got, want) < 1e-12


def test_tau_zero_gives_identity_over_factorial(kp):
    # tests/test_split_phi.cpp:77-87
    r = rng(5)
    k = [rand_norm(r, 3, 1.0), rand_norm(r, 4, 1.0)]
    for ell in (0, 1, 2):
        sp = kp.build_split_phi(k, 0.0, ell)
        for f in sp.factors:
            assert np.abs(f - np.eye(f.shape[0]) / math.factorial(ell)).sum(0).max() < 1e-15


@pytest.mark.parametrize("n", [70, 300, 900, 1700])
def test_cluster_lu_panel_bitwise(kp, n, monkeypatch):
    """The DSMEM cluster panel factorization (phi.cu lu_panel_cluster_kernel)
    and the one-CTA panel kernel produce bitwise identical expm (same
    arithmetic, different schedule); n = 1700 needs > 8 CTAs per panel.
    A matrix with repeated |entries| exercises the pivot tie rule."""
    r = rng(n)
    x = r.standard_normal((n, n)) * (3.0 / np.sqrt(n))
    x[:, 5] = np.round(x[:, 5] * 2) / 2  # ties in one pivot column
    x = np.asfortranarray(x)
    got = kp.expm(x)
    monkeypatch.setenv("KP_LU_PANEL", "simple")
    want = kp.expm(x)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("seed", range(4))
def test_phi_fuzz(kp, port, seed):
    """Random sizes 1..130 (every LU panel remainder, odd leading dimensions)
    and 1-norms 1e-3..300 (every Pade degree and scaling exponent): expm and the
    phi table against the oracle, same scaling exponent, <= 1e-12."""
    r = rng(7000 + seed)
    for _ in range(6):
        n = int(r.integers(1, 131))
        target = float(10.0 ** r.uniform(-3, 2.5))
        x = rand_norm(r, n, target)
        assert rel1(kp.expm(x), port.expm(x)) < 1e-12, (n, target)
        ell = int(r.integers(0, 4))
        tab = kp.phiquad(x, ell)
        want, s = port.phiquad(x, ell)
        assert tab.scaling_exponent == s, (n, target)
        for j in range(ell + 1):
            assert rel1(tab.phis[j], want[j]) < 1e-12, (n, target, j)
