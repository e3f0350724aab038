"""Run a few steps of one BASELINE integrator config (ncu launch-list target).
usage: prof_steps.py config [steps]   configs: see integrator_bench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200.integrators import _upload_factors
from integrator_bench import cfgs

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
c = cfgs(name)
spec = kp.ProblemSpec(_upload_factors(c.K), c.g, kp.to_device(c.u0), 0.0, c.t_final * steps / c.n_steps)
try:
    kp.integrate(spec, kp.StepperConfig(kp.parse_method(c.method), steps))
except kp.DivergenceError:
    pass
torch.cuda.synchronize()
print("ok", name, steps)
