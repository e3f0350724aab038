import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems
from paper_2304_02327_b200.integrators import _upload_factors
import pyoracle
port = pyoracle.Oracle("port")
c = problems.ac2d()
og = pyoracle.gfun(c.g.kind, *list(c.g.p))
want = port.integrate(c.method, c.u0, c.K, og, 0.0, c.t_final, c.n_steps)
def rel(a): return np.linalg.norm(a - want) / np.linalg.norm(want)
h = kp.integrate_config(c.method, c.u0, c.K, c.g, 0.0, c.t_final, c.n_steps)
print("host path", rel(h))
for warm in (False, True):
    ud = kp.to_device(c.u0); K = _upload_factors(c.K)
    spec = kp.ProblemSpec(K, c.g, ud, 0.0, c.t_final)
    if warm:
        kp.integrate(spec, kp.StepperConfig(kp.parse_method(c.method), 2, 12))
    try:
        r = kp.integrate(spec, kp.StepperConfig(kp.parse_method(c.method), c.n_steps, 12))
        print("device warm=%s" % warm, rel(kp.to_host(r.final)))
    except Exception as e:
        print("device warm=%s" % warm, "ERR", e)
