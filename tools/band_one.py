"""One banded Kronecker-sum launch with pre-scanned bands (ncu target).
usage: band_one.py {ac3d|bru|nls} [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems
from paper_2304_02327_b200._lib import check, ints
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = kp.default_context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
dims, cplx = {"ac3d": ((128, 128, 128), False), "bru": ((256, 256, 256, 2), False),
              "nls": ((512, 512, 512), True)}[name]
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
u = kp.fortran_empty(list(dims), dt)
u.copy_(torch.randn(u.shape, device="cuda", dtype=dt))
r = torch.empty_like(u)
g = kp.G.nls() if cplx else (kp.G.brusselator(1.0, 3.0) if name == "bru" else kp.G.allen_cahn())
f = ctx.lib.kp_kronsum_slab_banded_c128 if cplx else ctx.lib.kp_kronsum_slab_banded_f64
slab = len(dims) - (2 if name == "bru" else 1)
for _ in range(reps):  # slab mode = last spatial, k0 = 0, n_glob = n (halo planes are absent: P = 1)
    pass
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
# the unsharded path: kp_kronsum_* with device factors (band scan included once per call)
lib = ctx.lib
fk = lib.kp_kronsum_c128 if cplx else lib.kp_kronsum_f64
from paper_2304_02327_b200._lib import ptr_array
kp_ptrs = ptr_array([k.data_ptr() for k in K])
for _ in range(2):
    check(fk(ctx.h, u.data_ptr(), ints(list(dims)), len(dims), kp_ptrs, r.data_ptr()))
torch.cuda.synchronize()
print("ok")
