"""d = 2 Tucker sweep (configs[1]'s matrix case) under the current KP_GEMM_TILE.
usage: d2_sweep.py [n ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_02327_b200 as kp
from paper_2304_02327_b200._lib import check, ints, ptr_array
ctx = kp.default_context(0)
s = torch.cuda.current_stream(); ctx.set_stream(s.cuda_stream)
for n in [int(x) for x in sys.argv[1:]] or [512, 1024, 2048, 4096]:
    dims = [n, n]
    v = kp.fortran_empty(dims); v.normal_()
    ms = [kp.fortran_empty([n, n]) for _ in range(2)]
    for m in ms: m.normal_()
    out = kp.fortran_empty(dims)
    mp = ptr_array([m.data_ptr() for m in ms])
    def tk():
        check(ctx.lib.kp_tucker_f64(ctx.h, v.data_ptr(), ints(dims), 2, mp, ints(dims), 1.0, out.data_ptr()))
    for _ in range(3): tk()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record(s)
    for _ in range(reps): tk()
    e1.record(s); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    print(f"d2 n={n} tile={os.environ.get('KP_GEMM_TILE', 'auto')}: {t:.3f} ms {2.0 * n**2 * 2 * n / t / 1e9:.1f} TFLOP/s", flush=True)
