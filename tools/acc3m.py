import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2304_02327_b200 as kp
r = np.random.default_rng(5)
for dims, mode in [((48, 512, 40), 1), ((40, 36, 512), 2), ((96, 300, 20), 1)]:
    t = np.asfortranarray(r.standard_normal(dims) + 1j * r.standard_normal(dims))
    n = dims[mode]
    m = np.asfortranarray((r.standard_normal((n, n)) + 1j * r.standard_normal((n, n))) / np.sqrt(n))
    got = kp.mode_product(t, m, mode)
    tl = t.astype(np.clongdouble); ml = m.astype(np.clongdouble)
    want = np.moveaxis(np.tensordot(ml, tl, axes=(1, mode)), 0, mode)
    err = np.linalg.norm((got.astype(np.clongdouble) - want).ravel()) / np.linalg.norm(want.ravel())
    blas = np.moveaxis(np.tensordot(m, t, axes=(1, mode)), 0, mode)
    eb = np.linalg.norm((blas.astype(np.clongdouble) - want).ravel()) / np.linalg.norm(want.ravel())
    # componentwise on the imaginary part (3M's weak spot)
    ci = np.max(np.abs((got.imag.astype(np.longdouble) - want.imag))) / np.max(np.abs(want))
    print(dims, mode, f"3M rel-l2 vs long double {float(err):.2e}; numpy zgemm {float(eb):.2e}; max |d imag| / max|C| {float(ci):.2e}")
