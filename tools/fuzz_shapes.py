"""One-off fuzz: random ragged shapes through mode_product / tucker / kronsum_action
(real and complex) against numpy, incl. extents 1-3 and K past the KC = 256 slice.
usage: fuzz_shapes.py [n_cases] [seed]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2304_02327_b200 as kp

ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 200
r = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
worst = 0.0
bad = 0


def mp_ref(t, m, mode):
    return np.asfortranarray(np.moveaxis(np.tensordot(m, t, axes=(1, mode)), 0, mode))


for case in range(ncase):
    d = int(r.integers(1, 5))
    big = r.random() < 0.15
    dims = [int(r.integers(1, 300 if (big and k == 0) else 40)) for k in range(d)]
    if np.prod(dims) > 3e6:
        continue
    cplx = r.random() < 0.3
    t = r.standard_normal(dims) + (1j * r.standard_normal(dims) if cplx else 0)
    t = np.asfortranarray(t)
    mode = int(r.integers(0, d))
    rows = int(r.integers(1, 50))
    m = r.standard_normal((rows, dims[mode])) + (1j * r.standard_normal((rows, dims[mode])) if cplx else 0)
    m = np.asfortranarray(m)
    try:
        got = kp.mode_product(t, m, mode)
        want = mp_ref(t, m, mode)
        e = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
        ms = [np.asfortranarray(r.standard_normal((n, n)) + (1j * r.standard_normal((n, n)) if cplx else 0))
              for n in dims]
        gt = kp.tucker(t, ms)
        wt = t
        for mu in range(d):
            wt = mp_ref(wt, ms[mu], mu)
        e2 = np.linalg.norm(gt - wt) / max(np.linalg.norm(wt), 1e-300)
        gk = kp.kronsum_action(t, ms)
        wk = sum(mp_ref(t, ms[mu], mu) for mu in range(d))
        e3 = np.linalg.norm(gk - wk) / max(np.linalg.norm(wk), 1e-300)
        w = max(e, e2, e3)
        worst = max(worst, w)
        if not (w < 1e-11):
            bad += 1
            print("BAD", dims, mode, rows, cplx, e, e2, e3, flush=True)
    except Exception as ex:
        bad += 1
        print("EXC", dims, mode, rows, cplx, repr(ex)[:200], flush=True)
print(f"cases {ncase} bad {bad} worst {worst:.3e}")
