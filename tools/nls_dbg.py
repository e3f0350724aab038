"""NLS (complex) path: GPU vs the real reference, a sequence of integrations
in one process.  usage: nls_dbg.py n steps method1,method2,..."""
import os
import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np
import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems
import pyoracle
ref = pyoracle.Oracle("reference")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


n, steps = int(sys.argv[1]), int(sys.argv[2])
for method in sys.argv[3].split(","):
    cfg = problems.nls(n=n, method=method, n_steps=steps)
    og = pyoracle.gfun(cfg.g.kind, *list(cfg.g.p))
    g = kp.integrate_config(method, cfg.u0, cfg.K, cfg.g, 0.0, cfg.t_final, cfg.n_steps)
    r = ref.integrate(method, cfg.u0, cfg.K, og, 0.0, cfg.t_final, cfg.n_steps)
    print(os.environ.get("TAG", ""), n, steps, method, "gpu-ref", rel(g, r), flush=True)
