"""Child process of tests/test_gemm_tiles_gpu.py: mode products, Tucker
operators and complex products on seeded inputs under the current KP_GEMM_TILE
/ KP_TMA; prints one sha256 per case."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2304_02327_b200 as kp

r = np.random.default_rng(4242)
out = []
for shape in [(64, 64, 64), (130, 7, 66), (33, 65, 17), (128, 96, 40), (200, 200), (128, 128, 128),
              (160, 48, 30), (112, 80, 3)]:
    t = np.asfortranarray(r.standard_normal(shape))
    ms = [np.asfortranarray(r.standard_normal((n, n)) / n) for n in shape]
    out.append(kp.tucker(t, ms))
    for mode in range(len(shape)):
        m = np.asfortranarray(r.standard_normal((shape[mode] + 5, shape[mode])))
        out.append(kp.mode_product(t, m, mode))
z = np.asfortranarray(r.standard_normal((24, 20, 16)) + 1j * r.standard_normal((24, 20, 16)))
zs = [np.asfortranarray(r.standard_normal((n, n)) + 1j * r.standard_normal((n, n))) for n in z.shape]
out.append(kp.tucker(z, zs))
for a in out:
    print(hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest())
