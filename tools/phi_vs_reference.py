"""Device phi_l tables vs the REAL reference's phiquad (oracle/_ref, OpenMP on
the host cores) at the configs[1] d=2 sizes, where the scaling exponent s
reaches 13..19 (<= 1e-12 for s <= 11, report the value for
s ~ 19).  usage: phi_vs_reference.py n [n ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems
import pyoracle

ref = pyoracle.Oracle("reference")
for n in [int(a) for a in sys.argv[1:]]:
    X = np.asfortranarray(1e-3 * problems.fd_operator_1d(n, 1.0))
    t0 = time.perf_counter()
    tab = kp.phiquad(X, 1)
    t1 = time.perf_counter()
    rtab = ref.phiquad(X, 1)
    t2 = time.perf_counter()
    phis = [np.asarray(p) for p in tab.phis]
    rphis = rtab[0] if isinstance(rtab, tuple) else rtab
    rs = rtab[1] if isinstance(rtab, tuple) and len(rtab) > 1 else None
    errs = []
    for j in range(2):
        a, b = phis[j], np.asarray(rphis[j])
        errs.append(np.abs(a - b).sum(axis=0).max() / np.abs(b).sum(axis=0).max())
    print(f"n={n}: s={tab.scaling_exponent} (ref {rs}); rel-1-norm phi0 {errs[0]:.2e} phi1 "
          f"{errs[1]:.2e}; device {1e3 * (t1 - t0):.0f} ms (incl. transfers), reference "
          f"{t2 - t1:.1f} s on {ref.num_threads()} threads", flush=True)
