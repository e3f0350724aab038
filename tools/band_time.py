"""Time the banded Kronecker-sum stencil alone (pre-scanned bands, no host
sync: kp_kronsum_slab_banded_* on a one-rank slab with its two halo planes)
at the BASELINE shapes.  usage: band_time.py [ac3d bru nls] [reps=N]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems
from paper_2304_02327_b200._lib import check, ints

names = [a for a in sys.argv[1:] if "=" not in a] or ["ac3d", "bru", "nls"]
reps = int(dict(a.split("=") for a in sys.argv[1:] if "=" in a).get("reps", 20))
ctx = kp.default_context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
for name in names:
    dims, cplx = {"ac3d": ((128, 128, 128), False), "bru": ((256, 256, 256, 2), False),
                  "nls": ((512, 512, 512), True), "nls256": ((256, 256, 256), True)}[name]
    As = []
    for n in dims:
        if n == 2:
            As.append(np.zeros((2, 2), order="F"))
        elif cplx:
            As.append(np.asfortranarray(0.5j * problems.periodic_laplacian_1d(n, 1.0)))
        else:
            As.append(problems.fd_operator_1d(n, 0.01, 0.0))
    K = [kp.to_device(a) for a in As]
    bands = []
    for k in K:
        h = C.c_void_p()
        check(ctx.lib.kp_band_create(ctx.h, k.data_ptr(), k.shape[0], int(cplx), C.byref(h)))
        bands.append(h)
    arr = (C.c_void_p * len(bands))(*[b.value for b in bands])
    dt = torch.complex128 if cplx else torch.float64
    slab = len(dims) - (2 if name == "bru" else 1)
    ext = list(dims)
    ext[slab] += 2
    u = kp.fortran_empty(ext, dt)
    u.copy_(torch.randn(u.shape, device="cuda", dtype=dt))
    r = kp.fortran_empty(list(dims), dt)
    g = kp.gfun(kp.G_NLS) if cplx else (kp.gfun(kp.G_BRUSSELATOR, 1.0, 3.0) if name == "bru"
                                        else kp.gfun(kp.G_ALLEN_CAHN))
    f = ctx.lib.kp_kronsum_slab_banded_c128 if cplx else ctx.lib.kp_kronsum_slab_banded_f64
    def run():
        check(f(ctx.h, u.data_ptr(), ints(list(dims)), len(dims), arr, slab, 0, dims[slab],
                C.byref(g), r.data_ptr()))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    nbytes = 2 * r.numel() * r.element_size()
    print(f"{name:6s} {os.environ.get('KP_BAND', 'default'):8s} {us:9.1f} us  {nbytes / us / 1e3:7.0f} GB/s"
          f"  checksum {float(torch.sum(torch.abs(r)).item()):.17g}", flush=True)
