"""Time the banded Kronecker-sum stencil (kp_kronsum_*, device tensors) at the
BASELINE shapes.  KP_BAND=v1 selects the one-entry-per-thread kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems


def main():
    ctx = kp.default_context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    out = {}
    for name, dims, cplx in [("ac3d", (128, 128, 128), False), ("bru", (256, 256, 256, 2), False),
                             ("nls", (512, 512, 512), True), ("ac2d", (128, 128), False)]:
        As = []
        for n in dims:
            if n == 2:
                As.append(np.zeros((2, 2), order="F"))
            elif cplx:
                As.append(np.asfortranarray(0.5j * problems.periodic_laplacian_1d(n, 1.0)))
            else:
                As.append(problems.fd_operator_1d(n, 0.01, 0.0))
        K = [kp.to_device(a) for a in As]
        g = torch.Generator(device="cuda").manual_seed(1)
        u = kp.fortran_empty(list(dims), torch.complex128 if cplx else None)
        u.copy_(torch.randn(u.shape, generator=g, device="cuda",
                            dtype=torch.complex128 if cplx else torch.float64))
        r = kp.kronsum_action(u, K)
        for _ in range(3):
            r = kp.kronsum_action(u, K)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            kp.kronsum_action(u, K)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        nbytes = 2 * u.numel() * u.element_size()
        print(f"{name:5s} dims={dims} {us:9.1f} us  {nbytes / us / 1e3:7.0f} GB/s (read u + write r)"
              f"  checksum {float(torch.sum(torch.abs(r)).item()):.17g}", flush=True)


if __name__ == "__main__":
    main()
