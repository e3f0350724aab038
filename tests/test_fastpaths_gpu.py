"""The fast paths added for small cubes and the stencil are exact
re-schedules of the general ones: the fused mode-0/1 slice kernel
(fused01.cu, KP_FUSE01=0 disables), the line-marching stencil (banded.cu v2,
KP_BAND=v1 selects the one-entry-per-thread kernel) and the two-species
elementwise kernels.  Each must reproduce the general path BIT FOR BIT; the
general path is computed in a subprocess with the switch set (the switches
are read once per process).  Plus the usual oracle tolerance."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, rel2, rng

pytestmark = pytest.mark.gpu

_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + '/oracle')
import paper_2304_02327_b200 as kp
d = np.load({inp!r}, allow_pickle=True)
what = str(d['what'])
if what == 'tucker':
    out = kp.tucker(d['v'], list(d['ms']))
else:
    gk = int(d['gk'])
    out = kp.integrate_config(what, d['u0'], list(d['K']), kp.gfun(gk, *list(d['gp'])), 0.0,
                              float(d['T']), int(d['steps']))
np.save({outp!r}, out)
"""


def run_general(tmp_path, env, **arrays):
    inp = str(tmp_path / "in.npz")
    outp = str(tmp_path / "out.npy")
    np.savez(inp, **arrays)
    code = _CHILD.format(root=ROOT, inp=inp, outp=outp)
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(outp)


@pytest.mark.parametrize("dims", [(128, 128, 9), (64, 64, 5, 2), (128, 128, 128), (64, 64, 64),
                                  (128, 64, 256), (50, 30, 128), (64, 128, 130), (128, 128),
                                  (64, 64)])
def test_fused01_bitwise(kp, port, tmp_path, dims):
    r = rng(77)
    v = np.asfortranarray(r.standard_normal(dims))
    ms = [np.asfortranarray(r.uniform(-1, 1, (n, n))) for n in dims]
    got = kp.tucker(v, ms)
    want = run_general(tmp_path, {"KP_FUSE01": "0"}, what="tucker", v=v,
                       ms=np.array(ms, dtype=object))
    assert np.array_equal(got, want)
    if np.prod(dims) <= 64 ** 3 * 2:
        assert rel2(got, port.tucker(v, ms)) < 1e-12


def test_fused01_prefactor_and_phi(kp, port):
    """ETD2RK's phi_2 split carries the prefactor (l!)^(d-1) in mode 0's alpha."""
    n = 64
    A = port.fd_operator_1d(n, 1.0)
    fs, pref = port.build_split_phi([A, A, A], 1e-3, 2)
    v = np.asfortranarray(rng(5).standard_normal((n, n, n)))
    got = kp.tucker(pref * v, fs)
    want = port.tucker(pref * v, fs)
    assert rel2(got, want) < 1e-12


CASES = {
    # (method, u0 shape, K builder, g kind, g params, T, steps)
    "ac3d": ("etd2rk", (64, 64, 64), "ac", "G_ALLEN_CAHN", (), 5e-4 * 6, 6),
    # the config's cube: balanced single-wave GEMM tiles (gemm_dmma.cu B / C)
    "ac3d128": ("etd2rk", (128, 128, 128), "ac", "G_ALLEN_CAHN", (), 5e-4 * 3, 3),
    "ac3d128_l2b": ("lawson2b", (128, 128, 128), "ac", "G_ALLEN_CAHN", (), 5e-4 * 2, 2),
    "ac2d": ("exp_euler", (128, 128), "ac", "G_ALLEN_CAHN", (), 1e-3 * 8, 8),
    "ac2d_etd": ("etd2rk", (128, 128), "ac", "G_ALLEN_CAHN", (), 1e-3 * 8, 8),
    "ac2d_l2b": ("lawson2b", (64, 64), "ac", "G_ALLEN_CAHN", (), 1e-3 * 8, 8),
    "bru_etd": ("etd2rk", (32, 32, 32, 2), "bru", "G_BRUSSELATOR", (1.0, 3.0), 1e-3 * 5, 5),
    "bru_l2b": ("lawson2b", (32, 32, 32, 2), "bru", "G_BRUSSELATOR", (1.0, 3.0), 1e-3 * 5, 5),
    "nls": ("etd2rk", (24, 24, 24), "nls", "G_NLS", (), 1e-3 * 4, 4),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_integrate_fastpaths_bitwise(kp, port, tmp_path, case):
    import pyoracle
    method, shape, kb, gname, gp, T, steps = CASES[case]
    r = rng(11)
    if kb == "nls":
        n = shape[0]
        A = np.asfortranarray(0.5j * pyoracle.periodic_laplacian_1d(n, 16.0 / n))
        K = [A] * 3
        u0 = np.asfortranarray(np.exp(-0.1 * r.uniform(0, 4, shape)) * (1 + 0.1j))
    elif kb == "bru":
        n = shape[0]
        A = port.fd_operator_1d(n, 0.02)
        K = [A, A, A, np.zeros((2, 2), order="F")]
        u0 = np.asfortranarray(np.concatenate(
            [1 + 0.1 * r.uniform(-1, 1, shape[:3] + (1,)),
             3 + 0.1 * r.uniform(-1, 1, shape[:3] + (1,))], axis=3))
    else:
        A = port.fd_operator_1d(shape[0], 0.01)
        K = [A] * len(shape)
        u0 = np.asfortranarray(0.4 + 0.1 * r.uniform(-1, 1, shape))
    gk = getattr(kp, gname)
    got = kp.integrate_config(method, u0, K, kp.gfun(gk, *gp), 0.0, T, steps)
    want = run_general(tmp_path, {"KP_FUSE01": "0", "KP_BAND": "v1", "KP_GEMM_BAL": "0"},
                       what=method, u0=u0,
                       K=np.array(K, dtype=object), gk=gk, gp=np.array(gp, dtype=float),
                       T=T, steps=steps)
    assert np.array_equal(got, want)
