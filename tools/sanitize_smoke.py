"""Small run of every kernel family for compute-sanitizer (memcheck/racecheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import problems

r = np.random.default_rng(0)
for dims in [(5, 7, 3), (33, 17, 65), (40, 40, 40)]:
    t = np.asfortranarray(r.standard_normal(dims))
    ms = [np.asfortranarray(r.standard_normal((n + 1, n))) for n in dims]
    kp.tucker(t, ms)
    kp.kronsum_action(t, [np.asfortranarray(r.standard_normal((n, n))) for n in dims])
    kp.kronsum_action(t, [problems.fd_operator_1d(n, 0.1) for n in dims])
tc = np.asfortranarray(r.standard_normal((12, 10, 8)) + 1j * r.standard_normal((12, 10, 8)))
kp.tucker(tc, [np.asfortranarray(r.standard_normal((n, n)) + 0j) for n in tc.shape])
kp.phiquad(problems.fd_operator_1d(70, 1.0) * 1e-3, 2)
kp.expm(np.asfortranarray(r.standard_normal((9, 9)) * 3))
for cfg in (problems.ac2d(n=16, n_steps=3), problems.ac3d(n=12, n_steps=3),
            problems.brusselator(n=6, n_steps=2), problems.nls(n=8, n_steps=2)):
    kp.integrate_config(cfg.method, cfg.u0, cfg.K, cfg.g, 0.0, cfg.t_final, cfg.n_steps)
cfg = problems.brusselator(n=6, n_steps=2, method="lawson2b")
kp.integrate_config(cfg.method, cfg.u0, cfg.K, cfg.g, 0.0, cfg.t_final, cfg.n_steps)
# round-1 late kernels: fused mode-0/1 slices, the GEMM / LU entry points,
# the repartition pack/unpack of the native communicator
import ctypes as C
import torch
from paper_2304_02327_b200._lib import check
for dims in [(64, 64, 6), (128, 128, 2)]:
    t = np.asfortranarray(r.standard_normal(dims))
    kp.tucker(t, [np.asfortranarray(r.standard_normal((n, n))) for n in dims])
ctx = kp.default_context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
a, b = kp.to_device(r.standard_normal((37, 29))), kp.to_device(r.standard_normal((29, 11)))
c = kp.to_device(r.standard_normal((37, 11)))
check(ctx.lib.kp_gemm_f64(ctx.h, 37, 11, 29, 1.0, a.data_ptr(), 37, b.data_ptr(), 29, 0, 0.5,
                          c.data_ptr(), 37))
ac = kp.to_device(r.standard_normal((9, 7)) + 1j * r.standard_normal((9, 7)))
bc = kp.to_device(r.standard_normal((5, 7)) + 1j * r.standard_normal((5, 7)))
cc = kp.to_device(np.zeros((9, 5), dtype=complex))
one = (C.c_double * 2)(1.0, 0.0)
check(ctx.lib.kp_gemm_c128(ctx.h, 9, 5, 7, one, ac.data_ptr(), 9, bc.data_ptr(), 5, 1, one,
                           cc.data_ptr(), 9))
m = kp.to_device(r.standard_normal((70, 70)) + 5 * np.eye(70))
rhs = kp.to_device(r.standard_normal((70, 2)))
piv = torch.zeros(70, dtype=torch.int32, device="cuda")
check(ctx.lib.kp_lu_factor_f64(ctx.h, m.data_ptr(), 70, piv.data_ptr()))
check(ctx.lib.kp_lu_solve_f64(ctx.h, m.data_ptr(), piv.data_ptr(), 70, rhs.data_ptr(), 2))
x = torch.randn(3 * 4 * 6 * 2 // 2, dtype=torch.float64, device="cuda")
send, out = torch.empty_like(x), torch.empty_like(x)
check(ctx.lib.kp_repartition_pack(ctx.h, 1, 2, 0, 3, 4, 6, 2, 1, x.data_ptr(), send.data_ptr()))
check(ctx.lib.kp_repartition_unpack(ctx.h, 1, 2, 0, 3, 4, 6, 2, 1, send.data_ptr(),
                                    out.data_ptr()))
torch.cuda.synchronize()
print("sanitize smoke done")
