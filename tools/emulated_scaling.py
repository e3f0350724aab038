"""The sharded algorithms with P ranks EMULATED on one GPU (all ranks' work
and all exchanges run on this device, the exchanges as device copies):
how much extra work the sharded step does at P = 1..8 relative to the
single-GPU one -- the pack / unpack / halo / scatter passes and the extra
launches a P-GPU run adds per GPU, summed over ranks.  (A real P-GPU run
divides the compute by P and moves the exchanged bytes over NVLink.)
usage: emulated_scaling.py [P ...]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import parallel, problems
from paper_2304_02327_b200._lib import check, ints, ptr_array
from paper_2304_02327_b200.integrators import _upload_factors

Ps = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
ctx = kp.default_context(0)
s = torch.cuda.current_stream()
ctx.set_stream(s.cuda_stream)
out = {}


def ev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


# the n = 512 Tucker, mode 3 sharded
n = 512
g = torch.Generator(device="cuda").manual_seed(3)
v = kp.fortran_empty([n, n, n])
v.copy_(torch.randn(v.shape, generator=g, device="cuda", dtype=torch.float64))
ms = [kp.fortran_empty([n, n]) for _ in range(3)]
for m in ms:
    m.copy_(torch.randn(m.shape, generator=g, device="cuda", dtype=torch.float64) / n)
mp = ptr_array([m.data_ptr() for m in ms])
o = kp.fortran_empty([n, n, n])
single = ev_time(lambda: check(ctx.lib.kp_tucker_f64(ctx.h, v.data_ptr(), ints([n] * 3), 3, mp,
                                                     ints([n] * 3), 1.0, o.data_ptr())), 3)
out["tucker512_single_ms"] = single
for P in Ps:
    nl = n // P
    slabs = [v[:, :, r * nl:(r + 1) * nl].clone(memory_format=torch.contiguous_format) for r in range(P)]
    slabs = [x.permute(2, 1, 0).contiguous().permute(2, 1, 0) for x in slabs]
    outs = [torch.empty_like(x) for x in slabs]
    arr = (C.c_void_p * P)(*[x.data_ptr() for x in slabs])
    oarr = (C.c_void_p * P)(*[x.data_ptr() for x in outs])
    for md in (1, 2, 3):
        t = ev_time(lambda: check(ctx.lib.kp_tucker_sharded_local_f64(
            ctx.h, P, C.cast(arr, C.c_void_p), ints([n, n, nl]), 3, mp, 1.0, md,
            C.cast(oarr, C.c_void_p))), 3)
        out[f"tucker512_P{P}_mode{md}_ms"] = t
        print(f"tucker n=512 P={P} mode_d={md}: {t:.2f} ms (single {single:.2f}; "
              f"+{100 * (t / single - 1):.1f} %)", flush=True)
    del slabs, outs
    torch.cuda.empty_cache()
del v, o
torch.cuda.empty_cache()

# the integrator configs 3 and 4, sharded
for name, builder, kw, nf in [("bru_etd", "brusselator", {"method": "etd2rk", "n_steps": 20}, 256),
                              ("nls_etd", "nls", {"method": "etd2rk", "n_steps": 6}, 512)]:
    c = getattr(problems, builder)(**kw)
    spec = kp.ProblemSpec(_upload_factors(c.K), c.g, kp.to_device(c.u0), 0.0, c.t_final)
    try:
        kp.integrate(spec, kp.StepperConfig(kp.parse_method(c.method), 2))
    except kp.DivergenceError:
        pass
    try:
        r = kp.integrate(spec, kp.StepperConfig(kp.parse_method(c.method), c.n_steps))
        single = r.loop_s / c.n_steps * 1e3
    except kp.DivergenceError as e:
        single = e.loop_s / c.n_steps * 1e3
    out[f"{name}_single_ms_per_step"] = single
    species = builder == "brusselator"
    for P in Ps:
        ax = c.u0.ndim - (2 if species else 1)
        nl = c.u0.shape[ax] // P
        hs = [np.asfortranarray(np.take(c.u0, range(q * nl, (q + 1) * nl), axis=ax))
              for q in range(P)]
        K = [kp.to_device(np.asarray(k)) for k in c.K]
        for md in ("alltoall", "reduce_scatter", "fused"):
            ds = [kp.to_device(h) for h in hs]
            try:
                parallel.native_sharded_integrate(kp, c.method, [d.clone() for d in ds],
                                                  list(hs[0].shape), K, c.g, 0.0, 2 * c.tau, 2,
                                                  mode_d=md)
                _, loop = parallel.native_sharded_integrate(kp, c.method, ds, list(hs[0].shape),
                                                            K, c.g, 0.0, c.t_final, c.n_steps,
                                                            mode_d=md)
            except kp.DivergenceError as e:
                loop = e.loop_s
            t = loop / c.n_steps * 1e3
            out[f"{name}_P{P}_{md}_ms_per_step"] = t
            print(f"{name} P={P} {md}: {t:.2f} ms/step (single {single:.2f}; "
                  f"+{100 * (t / single - 1):.1f} %)", flush=True)
            del ds
            torch.cuda.empty_cache()
print(json.dumps(out))
