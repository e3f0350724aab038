"""Run one complex128 mode product a few times (ncu target).  usage: prof_mode_c.py n mode [reps]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200._lib import check, ints

n, mode = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ctx = kp.default_context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
dims = [n, n, n]
v = kp.fortran_empty(dims, torch.complex128)
v.copy_(torch.randn(v.shape, dtype=torch.complex128, device="cuda"))
m = kp.fortran_empty([n, n], torch.complex128)
m.copy_(torch.randn(m.shape, dtype=torch.complex128, device="cuda"))
out = kp.fortran_empty(dims, torch.complex128)
one = (C.c_double * 2)(1.0, 0.0)
zero = (C.c_double * 2)(0.0, 0.0)
for _ in range(reps):
    check(ctx.lib.kp_mode_product_c128(ctx.h, v.data_ptr(), ints(dims), 3, mode, m.data_ptr(), n,
                                       n, one, zero, out.data_ptr()))
torch.cuda.synchronize()
print("ok")
