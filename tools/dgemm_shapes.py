"""cuBLAS DGEMM (torch) at the mode-product shapes of small cubes (reference point only)."""
import torch
for (m, n, k) in [(16384, 128, 128), (128, 16384, 128), (4096, 64, 64), (65536, 256, 256)]:
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(5):
        c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"cublas dgemm m={m} n={n} k={k}: {ms*1e3:.1f} us {2*m*n*k/ms/1e9:.1f} TFLOP/s")
