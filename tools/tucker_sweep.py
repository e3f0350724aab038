import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_02327_b200 as kp
from paper_2304_02327_b200._lib import check, ints, ptr_array
ctx = kp.default_context(0)
s = torch.cuda.current_stream(); ctx.set_stream(s.cuda_stream)
print("peak", round(ctx.fp64_peak_tflops(),2), "tile", os.environ.get("KP_GEMM_TILE","auto"))
res = {}
sizes = [int(x) for x in sys.argv[1:]] or [64,128,256,384,512]
d2 = not sys.argv[1:]
for n in sizes:
    dims=[n,n,n]
    v = kp.fortran_empty(dims); v.normal_()
    ms = [kp.fortran_empty([n,n]) for _ in range(3)]
    for m in ms: m.normal_()
    out = kp.fortran_empty(dims)
    mp = ptr_array([m.data_ptr() for m in ms])
    def tk():
        check(ctx.lib.kp_tucker_f64(ctx.h, v.data_ptr(), ints(dims), 3, mp, ints(dims), 1.0, out.data_ptr()))
    def md(mode):
        check(ctx.lib.kp_mode_product_f64(ctx.h, v.data_ptr(), ints(dims), 3, mode, ms[0].data_ptr(), n, n, 1.0, 0.0, out.data_ptr()))
    def timeit(f, reps=10):
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps): f()
        e1.record(s); torch.cuda.synchronize()
        return e0.elapsed_time(e1)/reps
    t = timeit(tk)
    fl = 2.0*n**3*3*n
    modes = [timeit(lambda m=m: md(m)) for m in range(3)]
    print(f"n={n}: tucker {t:.3f} ms {fl/t/1e9:.1f} TFLOP/s; modes " + " ".join(f"{x:.3f}ms({2.0*n**4/x/1e9:.1f}TF)" for x in modes), flush=True)
# d=2
for n in ((1024, 2048, 4096) if d2 else ()):
    dims=[n,n]
    v = kp.fortran_empty(dims); v.normal_()
    ms = [kp.fortran_empty([n,n]) for _ in range(2)]
    for m in ms: m.normal_()
    out = kp.fortran_empty(dims)
    mp = ptr_array([m.data_ptr() for m in ms])
    def tk():
        check(ctx.lib.kp_tucker_f64(ctx.h, v.data_ptr(), ints(dims), 2, mp, ints(dims), 1.0, out.data_ptr()))
    for _ in range(2): tk()
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(s); 
    for _ in range(5): tk()
    e1.record(s); torch.cuda.synchronize()
    t=e0.elapsed_time(e1)/5
    print(f"d2 n={n}: {t:.3f} ms {2.0*n**2*2*n/t/1e9:.1f} TFLOP/s", flush=True)
