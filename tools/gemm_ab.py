"""A/B of the mode-product GEMM paths (run under the GPU).

  python tools/gemm_ab.py run OUT.npz      -- Tucker / mode products / complex
                                             products on seeded inputs with
                                             the current env (KP_GEMM, KP_TMA,
                                             KP_GEMM_TILE), outputs + timings
  python tools/gemm_ab.py cmp A.npz B.npz  -- bitwise comparison + timings
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(out):
    import torch
    import paper_2304_02327_b200 as kp
    from paper_2304_02327_b200._lib import check, ints, ptr_array
    ctx = kp.default_context(0)
    s = torch.cuda.current_stream()
    ctx.set_stream(s.cuda_stream)
    res = {}
    times = {}

    def timeit(f, reps):
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            f()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    g = torch.Generator(device="cuda")
    cases = [(3, 64), (3, 128), (3, 256), (3, 384), (3, 512), (2, 1024), (2, 2048), (2, 4096),
             (3, 100), (3, 33), (3, 130)]
    for d, n in cases:
        g.manual_seed(1000 + n)
        dims = [n] * d
        v = kp.fortran_empty(dims)
        v.copy_(torch.randn(v.shape, generator=g, device="cuda", dtype=torch.float64))
        ms = [kp.fortran_empty([n, n]) for _ in range(d)]
        for m in ms:
            m.copy_(torch.randn(m.shape, generator=g, device="cuda", dtype=torch.float64))
        o = kp.fortran_empty(dims)
        mp = ptr_array([m.data_ptr() for m in ms])

        def tk():
            check(ctx.lib.kp_tucker_f64(ctx.h, v.data_ptr(), ints(dims), d, mp, ints(dims), 1.0,
                                        o.data_ptr()))
        reps = 3 if n >= 2048 or n == 512 else 10
        t = timeit(tk, reps)
        fl = 2.0 * n ** d * d * n
        key = f"d{d}_n{n}"
        times[key] = (t, fl / t / 1e9)
        res[key] = o.cpu().numpy().ravel()[:: max(1, o.numel() // 2_000_000)].copy()
        print(f"{key}: {t:.3f} ms {fl / t / 1e9:.2f} TFLOP/s", flush=True)
        if d == 3 and n in (256, 512):
            for mode in range(3):
                def md(mode=mode):
                    check(ctx.lib.kp_mode_product_f64(ctx.h, v.data_ptr(), ints(dims), 3, mode,
                                                      ms[0].data_ptr(), n, n, 1.0, 0.0,
                                                      o.data_ptr()))
                t = timeit(md, reps)
                times[f"{key}_mode{mode}"] = (t, 2.0 * n ** 4 / t / 1e9)
                print(f"  mode {mode}: {t:.3f} ms {2.0 * n ** 4 / t / 1e9:.2f} TF", flush=True)
        del v, o, ms
    # complex
    for n in (64, 128, 256):
        g.manual_seed(7 + n)
        dims = [n] * 3
        v = torch.randn((n, n, n), generator=g, device="cuda", dtype=torch.complex128)
        v = v.permute(2, 1, 0).contiguous().permute(2, 1, 0)
        ms = [torch.randn((n, n), generator=g, device="cuda", dtype=torch.complex128).t()
              .contiguous().t() for _ in range(3)]
        got = kp.tucker(v, ms)
        torch.cuda.synchronize()
        t = timeit(lambda: kp.tucker(v, ms), 3)
        res[f"c_n{n}"] = torch.view_as_real(got).cpu().numpy().ravel()[::7].copy()
        times[f"c_n{n}"] = (t, 8.0 * n ** 3 * 3 * n / t / 1e9)
        print(f"c n={n}: {t:.3f} ms {8.0 * n ** 3 * 3 * n / t / 1e9:.2f} TF", flush=True)
    np.savez(out, **res, **{"t_" + k: np.array(v) for k, v in times.items()})


def cmp(a, b):
    A, B = np.load(a), np.load(b)
    for k in A.files:
        if k.startswith("t_"):
            continue
        same = np.array_equal(A[k], B[k])
        rel = float(np.linalg.norm(A[k] - B[k]) / max(np.linalg.norm(B[k]), 1e-300))
        ta, tb = A.get("t_" + k), B.get("t_" + k)
        print(f"{k:14s} bitwise={same} rel={rel:.2e}  A {ta[1]:.2f} TF  B {tb[1]:.2f} TF")
    for k in A.files:
        if k.startswith("t_") and "mode" in k:
            print(f"{k:20s} A {A[k][1]:.2f} TF  B {B[k][1]:.2f} TF")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        cmp(sys.argv[2], sys.argv[3])
