"""Time one paper experiment several times in one process (first-call costs).
usage: paper_rerun.py tag [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems
import bench

tag = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for t, dims, method, steps, pub, lines in bench.PAPER_RUNS:
    if t != tag:
        continue
    c = problems.riccati(dims[0], n_steps=steps, method=method) if len(dims) == 1 else \
        problems.adr(*dims, n_steps=steps, method=method)
    kp.integrate_config(method, c.u0, c.K, c.g, 0.0, c.t_final, 2)
    for r in range(reps):
        t0 = time.perf_counter()
        res = kp.integrate(kp.ProblemSpec(c.K, c.g, c.u0, 0.0, c.t_final),
                           kp.StepperConfig(kp.parse_method(method), steps))
        print(f"{tag} rep {r}: wall {1e3 * (time.perf_counter() - t0):.1f} ms loop {1e3 * res.loop_s:.1f} ms",
              flush=True)
