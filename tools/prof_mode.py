"""Run one real mode product a few times (ncu target).  usage: prof_mode.py n mode [reps] [d]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_02327_b200 as kp
from paper_2304_02327_b200._lib import check, ints
n = int(sys.argv[1]); mode = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
d = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ctx = kp.default_context(0); ctx.set_stream(torch.cuda.current_stream().cuda_stream)
dims = [n] * d
v = kp.fortran_empty(dims); v.normal_(); m = kp.fortran_empty([n, n]); m.normal_(); out = kp.fortran_empty(dims)
for _ in range(reps):
    check(ctx.lib.kp_mode_product_f64(ctx.h, v.data_ptr(), ints(dims), d, mode, m.data_ptr(), n, n, 1.0, 0.0, out.data_ptr()))
torch.cuda.synchronize(); print("ok")
