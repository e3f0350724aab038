"""Time the BASELINE integrator configs on the GPU (device-resident state).
usage: integrator_bench.py [config ...]   configs: ac2d ac3d bru_etd bru_l2b nls_ee nls_etd"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems

FLOPS_PER_TUCKER = lambda dims, cplx: (8.0 if cplx else 2.0) * np.prod(dims) * sum(dims)


def cfgs(name):
    return {
        "ac2d": lambda: problems.ac2d(),
        "ac3d": lambda: problems.ac3d(),
        "bru_etd": lambda: problems.brusselator(method="etd2rk"),
        "bru_l2b": lambda: problems.brusselator(method="lawson2b"),
        "nls_ee": lambda: problems.nls(method="exp_euler"),
        "nls_etd": lambda: problems.nls(method="etd2rk"),
    }[name]()


def tuckers_per_step(method):
    """Tucker-equivalents per step, dense Kronecker sum counted as one
    (SURVEY.md 8(d)): ExpEuler 2, ETD2RK 3, Lawson2b 2."""
    return {"exp_euler": 2, "etd2rk": 3, "lawson2b": 2, "lawson_euler": 1, "exp_euler_ls": 2}[method]


def main():
    names = sys.argv[1:] or ["ac2d", "ac3d", "bru_etd", "bru_l2b", "nls_ee", "nls_etd"]
    ctx = kp.default_context(0)
    for name in names:
        c = cfgs(name)
        ud = kp.to_device(c.u0)
        from paper_2304_02327_b200.integrators import _upload_factors
        K = _upload_factors(c.K)
        spec = kp.ProblemSpec(K, c.g, ud, 0.0, c.t_final)
        cfg = kp.StepperConfig(kp.parse_method(c.method), c.n_steps)
        kp.integrate(spec, kp.StepperConfig(kp.parse_method(c.method), 2, 12))  # warm (tau*50)
        torch.cuda.synchronize()
        l0 = ctx.launches
        t0 = time.perf_counter()
        note = ""
        try:
            r = kp.integrate(spec, cfg)
        except kp.DivergenceError as e:  # BASELINE NLS config is split-unstable
            note = f" DIVERGED at step {e.step}"
            r = kp.IntegrateResult(None, 0.0, e.loop_s)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        cplx = np.iscomplexobj(c.u0)
        spatial = [d for d, a in zip(c.u0.shape, c.K) if a.any()]
        species = int(np.prod(c.u0.shape)) // int(np.prod(spatial))
        fl = tuckers_per_step(c.method) * species * FLOPS_PER_TUCKER(spatial, cplx)
        sps = c.n_steps / r.loop_s
        print(f"{name:8s} {c.method:9s} dims={list(c.u0.shape)} steps={c.n_steps} "
              f"loop={r.loop_s*1e3:9.2f} ms ({sps:9.1f} steps/s, {fl*sps/1e12:6.2f} TFLOP/s) "
              f"wall={wall*1e3:9.1f} ms launches={ctx.launches-l0}{note}", flush=True)


if __name__ == "__main__":
    main()
