"""The reference's GEMM cores and LU through the C ABI (kp_gemm_*,
kp_gemm_batch_shared_b_*, kp_lu_factor_f64 / kp_lu_solve_f64) against numpy,
the cases of the reference's tests/test_kernels.cpp: both ops, alpha/beta
accumulation, ragged sizes across KC=256 slices, complex, batched shared B,
the singular matrix."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def dev(kp, x):
    return kp.to_device(np.asfortranarray(x))


@pytest.fixture(autouse=True)
def torch_stream(kp):
    """kp_* calls ordered on torch's stream (the uploads / downloads run there)."""
    import torch
    kp.default_context(0).set_stream(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (37, 29, 300), (128, 64, 7), (5, 300, 513)])
@pytest.mark.parametrize("op", [0, 1])
def test_gemm_f64(kp, m, n, k, op):
    from paper_2304_02327_b200._lib import check
    ctx = kp.default_context(0)
    r = np.random.default_rng(m * 7 + n + k + op)
    a = r.uniform(-1, 1, (m, k))
    b = r.uniform(-1, 1, (k, n) if op == 0 else (n, k))
    c = r.uniform(-1, 1, (m, n))
    want = -1.5 * a @ (b if op == 0 else b.T) + 0.5 * c
    da, db, dc = dev(kp, a), dev(kp, b), dev(kp, c)
    check(ctx.lib.kp_gemm_f64(ctx.h, m, n, k, -1.5, da.data_ptr(), m, db.data_ptr(),
                              b.shape[0], op, 0.5, dc.data_ptr(), m))
    got = kp.to_host(dc)
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_gemm_c128_and_batched(kp):
    from paper_2304_02327_b200._lib import check
    ctx = kp.default_context(0)
    r = np.random.default_rng(3)
    m, n, k, q = 20, 17, 33, 4
    a = r.uniform(-1, 1, (m, k, q)) + 1j * r.uniform(-1, 1, (m, k, q))
    b = r.uniform(-1, 1, (n, k)) + 1j * r.uniform(-1, 1, (n, k))
    c = r.uniform(-1, 1, (m, n, q)) + 1j * r.uniform(-1, 1, (m, n, q))
    al, be = 0.5 - 0.25j, 1.0 + 0.5j
    want = np.stack([al * a[:, :, i] @ b.T + be * c[:, :, i] for i in range(q)], axis=2)
    da, db, dc = dev(kp, a), dev(kp, b), dev(kp, c)
    alpha = (C.c_double * 2)(al.real, al.imag)
    beta = (C.c_double * 2)(be.real, be.imag)
    check(ctx.lib.kp_gemm_batch_shared_b_c128(ctx.h, m, n, k, alpha, da.data_ptr(), m, m * k,
                                              db.data_ptr(), n, 1, beta, dc.data_ptr(), m, m * n,
                                              q))
    assert np.abs(kp.to_host(dc) - want).max() < 1e-12
    # real batched, Op::none
    ar = r.uniform(-1, 1, (m, k, q))
    br = r.uniform(-1, 1, (k, n))
    want = np.stack([ar[:, :, i] @ br for i in range(q)], axis=2)
    da, db, dc = dev(kp, ar), dev(kp, br), dev(kp, np.zeros((m, n, q)))
    check(ctx.lib.kp_gemm_batch_shared_b_f64(ctx.h, m, n, k, 1.0, da.data_ptr(), m, m * k,
                                             db.data_ptr(), k, 0, 0.0, dc.data_ptr(), m, m * n, q))
    assert np.abs(kp.to_host(dc) - want).max() < 1e-12


@pytest.mark.parametrize("n", [3, 64, 150, 700])
def test_lu_factor_solve(kp, n):
    import torch
    from paper_2304_02327_b200._lib import check
    ctx = kp.default_context(0)
    r = np.random.default_rng(n)
    a = r.uniform(-1, 1, (n, n)) + 4.0 * np.eye(n)
    b = r.uniform(-1, 1, (n, 3))
    da, db = dev(kp, a), dev(kp, b)
    piv = torch.zeros(n, dtype=torch.int32, device="cuda")
    check(ctx.lib.kp_lu_factor_f64(ctx.h, da.data_ptr(), n, piv.data_ptr()))
    check(ctx.lib.kp_lu_solve_f64(ctx.h, da.data_ptr(), piv.data_ptr(), n, db.data_ptr(), 3))
    x = kp.to_host(db)
    assert np.abs(a @ x - b).max() < 1e-11


def test_lu_singular_raises(kp):
    import torch
    from paper_2304_02327_b200._lib import check, KronphiError
    ctx = kp.default_context(0)
    da = dev(kp, np.zeros((4, 4)))
    piv = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(KronphiError, match="singular"):
        check(ctx.lib.kp_lu_factor_f64(ctx.h, da.data_ptr(), 4, piv.data_ptr()))


def test_invalid_arguments_raise(kp):
    """Validation errors of the late ABI entry points map to KP_EINVAL
    (std::invalid_argument in the C++ drop-in) with a message naming the
    problem -- the reference's error contract."""
    import torch
    from paper_2304_02327_b200._lib import check, InvalidArgument
    ctx = kp.default_context(0)
    a = torch.zeros(16, dtype=torch.float64, device="cuda")
    with pytest.raises(InvalidArgument, match="leading dimension"):
        check(ctx.lib.kp_gemm_f64(ctx.h, 4, 4, 4, 1.0, a.data_ptr(), 2, a.data_ptr(), 4, 0, 0.0,
                                  a.data_ptr(), 4))
    with pytest.raises(InvalidArgument, match="opb"):
        check(ctx.lib.kp_gemm_f64(ctx.h, 2, 2, 2, 1.0, a.data_ptr(), 2, a.data_ptr(), 2, 7, 0.0,
                                  a.data_ptr(), 2))
    with pytest.raises(InvalidArgument, match="divisible"):
        check(ctx.lib.kp_repartition_pack(ctx.h, 1, 3, 0, 2, 4, 4, 1, 1, a.data_ptr(),
                                          a.data_ptr()))
    with pytest.raises(InvalidArgument, match="dir"):
        check(ctx.lib.kp_repartition_pack(ctx.h, 3, 1, 0, 2, 2, 2, 1, 1, a.data_ptr(),
                                          a.data_ptr()))
    with pytest.raises(InvalidArgument, match="lu_solve"):
        check(ctx.lib.kp_lu_solve_f64(ctx.h, a.data_ptr(), None, 4, a.data_ptr(), 1))
