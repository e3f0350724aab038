"""Randomized end-to-end parity: random small ragged shapes (odd extents take
the cp.async producer and the unvectorised epilogue stores), every method,
device g's, against the oracle's integrate (<= 1e-10, the north star's
end-to-end tolerance)."""
import numpy as np
import pytest

from conftest import rel2, rng

pytestmark = pytest.mark.gpu

METHODS = ["exp_euler", "etd2rk", "lawson2b", "lawson_euler", "exp_euler_ls"]


@pytest.mark.parametrize("seed", range(6))
def test_integrate_random_shapes(kp, port, seed):
    import pyoracle
    r = rng(900 + seed)
    for _ in range(4):
        d = int(r.integers(1, 4))
        dims = tuple(int(r.integers(2, 23)) for _ in range(d))
        method = METHODS[int(r.integers(0, len(METHODS)))]
        kind = int(r.integers(0, 3))
        K = [port.fd_operator_1d(n, float(r.uniform(0.005, 0.05)), float(r.uniform(0, 0.2)))
             for n in dims]
        u0 = np.asfortranarray(0.3 + 0.1 * r.uniform(-1, 1, dims))
        steps = int(r.integers(1, 7))
        T = steps * 1e-3
        if kind == 0:
            gk, gp = kp.G_ALLEN_CAHN, ()
            go = pyoracle.gfun(pyoracle.G_ALLEN_CAHN)
        elif kind == 1:
            gk, gp = kp.G_SQUARE, ()
            go = pyoracle.gfun(pyoracle.G_SQUARE)
        else:
            gk, gp = kp.G_ZERO, ()
            go = pyoracle.gfun(pyoracle.G_ZERO)
        got = kp.integrate_config(method, u0, K, kp.gfun(gk, *gp), 0.0, T, steps)
        want = port.integrate(method, u0, K, go, 0.0, T, steps)
        assert rel2(got, want) < 1e-10, (dims, method, kind, steps)
