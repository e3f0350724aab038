"""configs[1] in full: device phi_1 factor build + Tucker GFLOP/s for the d=3
cubes and the d=2 squares up to 8192^2, plus the phi-table recurrence check
(X phi_1 + I = phi_0, tests/test_matrix_functions.cpp:189-202 of the
reference) at the largest sizes where the CPU oracle cannot run."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems
from paper_2304_02327_b200._lib import check, ints, ptr_array


def run(d, n, reps):
    ctx = kp.default_context(0)
    s = torch.cuda.current_stream()
    ctx.set_stream(s.cuda_stream)
    A = kp.to_device(problems.fd_operator_1d(n, 1.0))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X = A * 1e-3
    tab = kp.phiquad(X, 1)
    torch.cuda.synchronize()
    build = time.perf_counter() - t0
    # recurrence invariant X phi_1 + I - phi_0 (relative 1-norm)
    lhs = X @ tab.phis[1] + torch.eye(n, dtype=torch.float64, device="cuda") - tab.phis[0]
    rec = (lhs.abs().sum(0).max() / tab.phis[0].abs().sum(0).max()).item()
    L = tab.phis[1]
    dims = [n] * d
    v = kp.fortran_empty(dims)
    v.normal_()
    out = kp.fortran_empty(dims)
    mp = ptr_array([L.data_ptr()] * d)

    def tk():
        check(ctx.lib.kp_tucker_f64(ctx.h, v.data_ptr(), ints(dims), d, mp, ints(dims), 1.0,
                                    out.data_ptr()))
    tk()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        tk()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.0 * n ** d * d * n
    print(f"d={d} n={n:5d}: phi build {build*1e3:9.1f} ms (s={tab.scaling_exponent}, recurrence "
          f"rel {rec:.1e}); tucker {ms:9.3f} ms = {fl/ms/1e9:6.2f} TFLOP/s", flush=True)


if __name__ == "__main__":
    for n in (64, 128, 256, 384, 512):
        run(3, n, 10)
    for n in (1024, 2048, 4096, 8192):
        run(2, n, 5 if n < 8192 else 3)
