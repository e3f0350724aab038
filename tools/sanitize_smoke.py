"""Small run of every kernel family for compute-sanitizer (memcheck/racecheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems

r = np.random.default_rng(0)
for dims in [(5, 7, 3), (33, 17, 65), (40, 40, 40)]:
    t = np.asfortranarray(r.standard_normal(dims))
    ms = [np.asfortranarray(r.standard_normal((n + 1, n))) for n in dims]
    kp.tucker(t, ms)
    kp.kronsum_action(t, [np.asfortranarray(r.standard_normal((n, n))) for n in dims])
    kp.kronsum_action(t, [problems.fd_operator_1d(n, 0.1) for n in dims])
tc = np.asfortranarray(r.standard_normal((12, 10, 8)) + 1j * r.standard_normal((12, 10, 8)))
kp.tucker(tc, [np.asfortranarray(r.standard_normal((n, n)) + 0j) for n in tc.shape])
kp.phiquad(problems.fd_operator_1d(70, 1.0) * 1e-3, 2)
kp.expm(np.asfortranarray(r.standard_normal((9, 9)) * 3))
for cfg in (problems.ac2d(n=16, n_steps=3), problems.ac3d(n=12, n_steps=3),
            problems.brusselator(n=6, n_steps=2), problems.nls(n=8, n_steps=2)):
    kp.integrate_config(cfg.method, cfg.u0, cfg.K, cfg.g, 0.0, cfg.t_final, cfg.n_steps)
cfg = problems.brusselator(n=6, n_steps=2, method="lawson2b")
kp.integrate_config(cfg.method, cfg.u0, cfg.K, cfg.g, 0.0, cfg.t_final, cfg.n_steps)
print("sanitize smoke done")
