"""Generate golden vectors from the REAL reference library (oracle/_ref,
compiled from /root/reference/proj by `make -C oracle ref`).

Run here (the reference exists only in this container):
    python tests/golden/make_golden.py
Writes tests/golden/*.npz (small, committed).  The inputs are seeded numpy
data; each file stores inputs and the reference's outputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import pyoracle  # noqa: E402

R = pyoracle.Oracle("reference")


def save(name, **arrs):
    np.savez_compressed(os.path.join(HERE, name), **arrs)


def f(a):
    return np.asfortranarray(a)


def main():
    r = np.random.default_rng(20230517)
    # mu-mode products / Tucker / Kronecker sum (inc/mode_product.hpp)
    t = f(r.uniform(-1, 1, (5, 6, 7)))
    ms = [f(r.uniform(-1, 1, (k, k))) for k in (5, 6, 7)]
    save("tucker_small.npz", t=t, m0=ms[0], m1=ms[1], m2=ms[2], tucker=R.tucker(t, ms),
         kronsum=R.kronsum(t, ms), mp1=R.mode_product(t, f(r.uniform(-1, 1, (4, 6))), 1))
    # K > 256: two KC slices in the reference GEMM (inc/kernels.hpp:297)
    t = f(r.uniform(-1, 1, (260, 3, 2)))
    m = f(r.uniform(-1, 1, (260, 260)))
    save("mode_product_kc.npz", t=t, m=m, out=R.mode_product(t, m, 0))
    # accumulate (beta = 1) on an interior mode
    t = f(r.uniform(-1, 1, (4, 9, 3)))
    m = f(r.uniform(-1, 1, (9, 9)))
    base = f(r.uniform(-1, 1, (4, 9, 3)))
    save("mode_product_acc.npz", t=t, m=m, base=base, out=R.mode_product(t, m, 1, out=base))
    # complex
    t = f(r.uniform(-1, 1, (4, 5, 3)) + 1j * r.uniform(-1, 1, (4, 5, 3)))
    ms = [f(r.uniform(-1, 1, (k, k)) + 1j * r.uniform(-1, 1, (k, k))) for k in (4, 5, 3)]
    save("tucker_c128.npz", t=t, m0=ms[0], m1=ms[1], m2=ms[2], tucker=R.tucker(t, ms),
         kronsum=R.kronsum(t, ms))
    # GLL rules q = 2..20 (src/gll_rule.cpp)
    g = {}
    for q in range(2, 21):
        x, w = R.gll_rule(q)
        g[f"x{q}"] = x
        g[f"w{q}"] = w
    save("gll.npz", **g)
    # expm (inc/matrix_functions.hpp:76-95), norms 0.1 / 5 / 800
    ex = {}
    for i, target in enumerate((0.1, 5.0, 800.0)):
        x = r.uniform(-1, 1, (8, 8))
        x = f(x * target / np.abs(x).sum(0).max())
        ex[f"x{i}"] = x
        ex[f"e{i}"] = R.expm(x)
    z = f(r.uniform(-1, 1, (6, 6)) + 1j * r.uniform(-1, 1, (6, 6)))
    ex["z"] = z
    ex["ez"] = R.expm(z)
    save("expm.npz", **ex)
    # phiquad (inc/matrix_functions.hpp:146-199)
    ph = {}
    a = R.fd_operator_1d(32, 1.0)
    x = f(a * 1e-3)
    phis, s = R.phiquad(x, 2)
    ph.update(fd_x=x, fd_s=np.array(s), fd_p0=phis[0], fd_p1=phis[1], fd_p2=phis[2])
    x = r.uniform(-1, 1, (10, 10))
    x = f(x * 20.0 / np.abs(x).sum(0).max())
    phis, s = R.phiquad(x, 2)
    ph.update(rn_x=x, rn_s=np.array(s), rn_p0=phis[0], rn_p1=phis[1], rn_p2=phis[2])
    save("phiquad.npz", **ph)
    # build_split_phi (inc/split_phi.hpp:25-48)
    As = [R.fd_operator_1d(n, 0.05) for n in (6, 8, 5)]
    sp = {"A0": As[0], "A1": As[1], "A2": As[2]}
    for ell in (0, 1, 2):
        fs, pref = R.build_split_phi(As, 0.02, ell)
        sp[f"pref{ell}"] = np.array(pref)
        for mu in range(3):
            sp[f"f{ell}_{mu}"] = fs[mu]
    save("split_phi.npz", **sp)
    # fd_operator_1d (src/problems.cpp:9-22)
    save("fd.npz", a=R.fd_operator_1d(7, 0.75, 0.1), b=R.fd_operator_1d(5, 0.01, 0.0))
    # integrate (inc/integrators.hpp:219-373) on reduced BASELINE configs
    from paper_2304_02327_b200 import problems  # noqa: E402 (pure numpy builders)
    ints = {}

    def run(tag, cfg, method=None):
        m = method or cfg.method
        g = pyoracle.gfun(cfg.g.kind, *list(cfg.g.p))
        ints[f"{tag}_u0"] = cfg.u0
        for mu, a in enumerate(cfg.K):
            ints[f"{tag}_A{mu}"] = a
        ints[f"{tag}_meta"] = np.array([cfg.g.kind, cfg.tau, cfg.n_steps] + list(cfg.g.p))
        ints[f"{tag}_method"] = np.array(pyoracle.METHODS[m])
        ints[f"{tag}_out"] = R.integrate(m, cfg.u0, cfg.K, g, 0.0, cfg.t_final, cfg.n_steps)

    run("ac2d", problems.ac2d(n=24, n_steps=20))
    run("ac3d", problems.ac3d(n=10, n_steps=20))
    run("ac2d_lawson", problems.ac2d(n=16, n_steps=10), "lawson_euler")
    run("ac2d_ls", problems.ac2d(n=16, n_steps=10), "exp_euler_ls")
    run("bru_etd", problems.brusselator(n=6, n_steps=10, method="etd2rk"))
    run("bru_l2b", problems.brusselator(n=6, n_steps=10, method="lawson2b"))
    run("nls_ee", problems.nls(n=8, n_steps=5, method="exp_euler"))
    run("nls_etd", problems.nls(n=8, n_steps=5, method="etd2rk"))
    save("integrate.npz", **ints)
    print("golden vectors written:", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
