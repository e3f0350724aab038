"""Child process of tests/test_band_variants_gpu.py: banded Kronecker sums and
short integrations (the stencil with its fused g) under the current KP_BAND;
prints one sha256 per case."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems

out = []
r = np.random.default_rng(77)
# (300 / 260 / 270: rows straddling the reference's KC = 256 slice boundary)
for dims in [(64, 40, 30), (36, 24, 16), (130, 10, 9), (300, 6, 5), (8, 260, 3), (4, 4, 270)]:
    u = np.asfortranarray(r.standard_normal(dims))
    out.append(kp.kronsum_action(u, [problems.fd_operator_1d(n, 0.01) for n in dims]))
z = np.asfortranarray(r.standard_normal((32, 16, 24)) + 1j * r.standard_normal((32, 16, 24)))
out.append(kp.kronsum_action(z, [np.asfortranarray(0.5j * problems.periodic_laplacian_1d(n, 0.1))
                                 for n in z.shape]))
for c in (problems.ac3d(n=32, n_steps=6), problems.brusselator(n=16, n_steps=6),
          problems.nls(n=16, n_steps=4)):
    out.append(kp.integrate_config(c.method, c.u0, c.K, c.g, 0.0, c.t_final, c.n_steps))
for a in out:
    print(hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest())
