"""The CUDA path against golden vectors produced by the real reference
(tests/golden/make_golden.py): no oracle in the loop."""
import os

import numpy as np
import pytest

from conftest import ROOT, rel2
from test_oracle_pins import INTEGRATE_TAGS, golden_case, load

pytestmark = pytest.mark.gpu


def test_tucker_kronsum(kp):
    z = load("tucker_small.npz")
    ms = [z["m0"], z["m1"], z["m2"]]
    assert rel2(kp.tucker(z["t"], ms), z["tucker"]) < 1e-12
    assert rel2(kp.kronsum_action(z["t"], ms), z["kronsum"]) < 1e-12
    z = load("mode_product_kc.npz")
    assert rel2(kp.mode_product(z["t"], z["m"], 0), z["out"]) < 1e-12
    z = load("mode_product_acc.npz")
    got = kp.mode_product_into(z["t"], z["m"], 1, np.asfortranarray(z["base"]).copy(order="F"),
                               accumulate=True)
    assert rel2(got, z["out"]) < 1e-12
    z = load("tucker_c128.npz")
    ms = [z["m0"], z["m1"], z["m2"]]
    assert rel2(kp.tucker(z["t"], ms), z["tucker"]) < 1e-12
    assert rel2(kp.kronsum_action(z["t"], ms), z["kronsum"]) < 1e-12


def test_matrix_functions(kp):
    z = load("expm.npz")
    for i in range(3):
        assert rel2(kp.expm(z[f"x{i}"]), z[f"e{i}"]) < 1e-12
    assert rel2(kp.expm(z["z"]), z["ez"]) < 1e-12
    z = load("phiquad.npz")
    for tag in ("fd", "rn"):
        tab = kp.phiquad(z[f"{tag}_x"], 2)
        assert tab.scaling_exponent == int(z[f"{tag}_s"])
        for j in range(3):
            assert rel2(tab.phis[j], z[f"{tag}_p{j}"]) < 1e-12
    z = load("split_phi.npz")
    As = [z["A0"], z["A1"], z["A2"]]
    for ell in (0, 1, 2):
        sp = kp.build_split_phi(As, 0.02, ell)
        assert sp.prefactor == float(z[f"pref{ell}"])
        for mu in range(3):
            assert rel2(sp.factors[mu], z[f"f{ell}_{mu}"]) < 1e-12


@pytest.mark.parametrize("tag", INTEGRATE_TAGS)
def test_integrate(kp, tag):
    z = load("integrate.npz")
    m, u0, As, g, tau, n, want = golden_case(z, tag)
    gg = kp.gfun(g.kind, *list(g.p))
    got = kp.integrate_config(m, u0, As, gg, 0.0, tau * n, n)
    assert rel2(got, want) < 1e-10
