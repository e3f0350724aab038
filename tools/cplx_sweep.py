"""Complex128 Tucker operators (the NLS products) on the device: TFLOP/s (4M convention)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_02327_b200 as kp
ctx = kp.default_context(0)
s = torch.cuda.current_stream()
ctx.set_stream(s.cuda_stream)
for n in [int(x) for x in sys.argv[1:]] or [256, 512]:
    v = torch.randn((n, n, n), device="cuda", dtype=torch.complex128).permute(2, 1, 0).contiguous().permute(2, 1, 0)
    ms = [torch.randn((n, n), device="cuda", dtype=torch.complex128).t().contiguous().t() for _ in range(3)]
    for _ in range(2):
        kp.tucker(v, ms)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    reps = 3
    for _ in range(reps):
        kp.tucker(v, ms)
    e1.record(s)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    print(f"c n={n}: {t:.3f} ms {8.0 * n**3 * 3 * n / t / 1e9:.2f} TF", flush=True)
    del v, ms
