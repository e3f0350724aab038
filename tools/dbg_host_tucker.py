import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import paper_2304_02327_b200 as kp
import pyoracle
port = pyoracle.Oracle("port")
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for n in (100, 64, 128, 36, 98):
    r = np.random.default_rng(n)
    t = np.asfortranarray(r.uniform(-1, 1, (n, n, n)))
    ms = [np.asfortranarray(r.uniform(-1, 1, (n, n))) for _ in range(3)]
    want = port.tucker(t, ms)
    hs = [rel(kp.tucker(t, ms), want) for _ in range(3)]
    dv = rel(kp.to_host(kp.tucker(kp.to_device(t), [kp.to_device(m) for m in ms])), want)
    modes = [rel(kp.mode_product(t, ms[m], m), port.mode_product(t, ms[m], m)) for m in range(3)]
    print(f"n={n}: host {['%.1e' % x for x in hs]} dev {dv:.1e} modes {['%.1e' % x for x in modes]}", flush=True)
    if max(modes) > 1e-12:
        for m in range(3):
            got = kp.mode_product(t, ms[m], m); w = port.mode_product(t, ms[m], m)
            bad = np.argwhere(np.abs(got - w) > 1e-10 * np.abs(w).max())
            if len(bad):
                print("  mode", m, "bad count", len(bad), "first", bad[:4].tolist(), "last", bad[-4:].tolist())
