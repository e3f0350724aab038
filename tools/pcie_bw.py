"""PCIe bandwidth of this box with pinned host buffers: H2D alone, D2H alone,
and both directions at once (the e2e path's steady state)."""
import time

import torch

n = 1 << 27  # 1 GiB of float64
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


gb = n * 8 / 1e9
t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D {gb / t1:.1f} GB/s ({t1 * 1e3:.1f} ms/GiB), D2H {gb / t2:.1f} GB/s ({t2 * 1e3:.1f} ms), "
      f"both at once {t3 * 1e3:.1f} ms for 1 GiB each way ({gb / t3:.1f} GB/s per direction)")
