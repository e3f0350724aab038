"""A few Riccati steps (ncu / timing target).  usage: prof_riccati.py n_hat method steps"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_02327_b200 as kp  # noqa: E402
from paper_2304_02327_b200 import problems  # noqa: E402

nh = int(sys.argv[1])
m = sys.argv[2]
steps = int(sys.argv[3])
c = problems.riccati(nh, n_steps=steps)
kp.integrate_config(m, c.u0, c.K, c.g, 0.0, 0.025, 1)
t = time.perf_counter()
r = kp.integrate(kp.ProblemSpec(c.K, c.g, c.u0, 0.0, 0.025),
                 kp.StepperConfig(kp.parse_method(m), steps))
print("wall", time.perf_counter() - t, "loop", r.loop_s)
