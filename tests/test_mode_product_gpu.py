"""GPU parity of the mu-mode product / Tucker / Kronecker-sum action against
the CPU oracle (oracle/kp_oracle.c, pinned to the reference), through the C
ABI.  Mirrors the reference's tests/test_tensor.cpp cases plus
BASELINE-size properties.  Tolerance: rel-l2 <= 1e-12 per Tucker operator
(BASELINE.json north_star)."""
import numpy as np
import pytest

from conftest import rel2, rng

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rand(r, shape, cplx=False):
    a = r.uniform(-1, 1, shape)
    if cplx:
        a = a + 1j * r.uniform(-1, 1, shape)
    return np.asfortranarray(a)


# ragged shapes hitting every tile-edge path and both B layouts
SHAPES = [(1,), (7,), (3, 4), (5, 1, 3), (2, 3, 4, 5), (17, 33, 9), (64, 64, 64),
          (130, 7, 66), (3, 129, 65), (200, 200), (1, 1, 300), (64, 1, 1)]


@pytest.mark.parametrize("shape", SHAPES)
def test_mode_product_vs_oracle(kp, port, shape):
    r = rng(hash(shape) % 1000)
    t = rand(r, shape)
    for mode in range(len(shape)):
        for rows in {shape[mode], shape[mode] + 3, max(1, shape[mode] - 1)}:
            m = rand(r, (rows, shape[mode]))
            got = kp.mode_product(t, m, mode)
            want = port.mode_product(t, m, mode)
            assert got.shape == want.shape
            assert rel2(got, want) < TOL, (shape, mode, rows)


@pytest.mark.parametrize("shape", [(5, 6, 7), (64, 32, 16), (33, 65, 17)])
def test_mode_product_accumulate(kp, port, shape):
    r = rng(7)
    t = rand(r, shape)
    for mode in range(len(shape)):
        m = rand(r, (shape[mode], shape[mode]))
        base = rand(r, shape)
        got = kp.mode_product_into(t, m, mode, base.copy(order="F"), accumulate=True)
        want = port.mode_product(t, m, mode, out=base)
        assert rel2(got, want) < TOL


def test_row_permutation_kat(kp):
    # tests/test_tensor.cpp:89-99
    t = np.asfortranarray(np.array([[1.0, 2.0], [3.0, 4.0]]))
    m = np.asfortranarray(np.array([[0.0, 1.0], [1.0, 0.0]]))
    got = kp.mode_product(t, m, 0)
    assert got.tolist() == [[3.0, 4.0], [1.0, 2.0]]


def test_identity_bit_exact(kp):
    # tests/test_tensor.cpp:101-108, :152-157
    r = rng(1)
    t = rand(r, (3, 4, 5))
    for mode in range(3):
        got = kp.mode_product(t, np.eye(t.shape[mode]), mode)
        assert np.array_equal(got, t)
    assert np.array_equal(kp.tucker(t, [np.eye(n) for n in t.shape]), t)


def test_permutation_tucker_bit_exact(kp):
    # tests/test_tensor.cpp:180-200
    r = rng(2)
    dims = (3, 4, 2)
    t = np.asfortranarray((np.arange(np.prod(dims)) % 23 - 11).reshape(dims, order="F") * 1.0)
    perms, maps = [], []
    for d in dims:
        p = r.permutation(d)
        pm = np.zeros((d, d))
        pm[p, np.arange(d)] = 1.0
        perms.append(np.asfortranarray(pm))
        maps.append(p)
    got = kp.tucker(t, perms)
    for k in range(dims[2]):
        for j in range(dims[1]):
            for i in range(dims[0]):
                assert got[maps[0][i], maps[1][j], maps[2][k]] == t[i, j, k]


def test_tucker_2d_is_m1_t_m2t(kp):
    # tests/test_tensor.cpp:159-169
    r = rng(3)
    t = rand(r, (3, 4))
    m1, m2 = rand(r, (5, 3)), rand(r, (6, 4))
    got = kp.tucker(t, [m1, m2])
    assert rel2(got, m1 @ t @ m2.T) < 1e-13


@pytest.mark.parametrize("n", [16, 64, 100, 128])
def test_tucker_cube_vs_oracle(kp, port, n):
    r = rng(n)
    t = rand(r, (n, n, n))
    ms = [rand(r, (n, n)) for _ in range(3)]
    assert rel2(kp.tucker(t, ms), port.tucker(t, ms)) < TOL


def test_tucker_nonsquare_factors(kp, port):
    r = rng(5)
    t = rand(r, (6, 10, 14))
    ms = [rand(r, (9, 6)), rand(r, (3, 10)), rand(r, (20, 14))]
    assert rel2(kp.tucker(t, ms), port.tucker(t, ms)) < TOL


def test_property_random_shapes(kp, port):
    # tests/test_tensor.cpp:233-260: 60 random shapes, d <= 4, N <= 500
    r = rng(777)
    done = 0
    while done < 60:
        d = 1 + int(r.integers(4))
        dims = tuple(int(x) for x in 1 + r.integers(6, size=d))
        if np.prod(dims) > 500:
            continue
        t = rand(r, dims)
        sq = [rand(r, (n, n)) for n in dims]
        assert rel2(kp.tucker(t, sq), port.tucker(t, sq)) < 1e-13
        assert rel2(kp.kronsum_action(t, sq), port.kronsum(t, sq)) < 1e-13
        done += 1


def test_kronsum_vs_oracle(kp, port):
    r = rng(11)
    for dims in [(6,), (2, 3, 4), (40, 30, 20), (64, 64, 64)]:
        t = rand(r, dims)
        As = [rand(r, (n, n)) for n in dims]
        assert rel2(kp.kronsum_action(t, As), port.kronsum(t, As)) < TOL


def test_kronsum_zero_factors(kp):
    t = rand(rng(4), (2, 3, 4))
    assert np.abs(kp.kronsum_action(t, [np.zeros((n, n)) for n in t.shape])).max() == 0.0


def test_sizing_error_names_mode(kp):
    # tests/test_tensor.cpp:118-124
    t = rand(rng(6), (3, 4, 5))
    with pytest.raises(kp.InvalidArgument, match="mode 1"):
        kp.mode_product(t, rand(rng(6), (6, 9)), 1)
    with pytest.raises(kp.InvalidArgument):
        kp.mode_product(t, rand(rng(6), (6, 9)), 7)
    with pytest.raises(kp.InvalidArgument):
        kp.KroneckerSum([rand(rng(6), (2, 3))])


@pytest.mark.parametrize("shape", [(3, 4), (5, 6, 7), (16, 8, 12), (40, 33, 21)])
def test_complex_mode_products(kp, port, shape):
    r = rng(21)
    t = rand(r, shape, True)
    for mode in range(len(shape)):
        m = rand(r, (shape[mode] + 1, shape[mode]), True)
        assert rel2(kp.mode_product(t, m, mode), port.mode_product(t, m, mode)) < TOL
    ms = [rand(r, (n, n), True) for n in shape]
    assert rel2(kp.tucker(t, ms), port.tucker(t, ms)) < TOL
    assert rel2(kp.kronsum_action(t, ms), port.kronsum(t, ms)) < TOL


def test_device_tensors_stay_on_device(kp, port):
    import torch
    r = rng(8)
    t = rand(r, (48, 40, 32))
    ms = [rand(r, (n, n)) for n in t.shape]
    td = kp.to_device(t)
    out = kp.tucker(td, [kp.to_device(m) for m in ms])
    assert out.is_cuda and out.dtype == torch.float64
    assert rel2(kp.to_host(out), port.tucker(t, ms)) < TOL


def test_launch_count_increments(kp):
    ctx = kp.default_context(0)
    before = ctx.launches
    t = rand(rng(9), (8, 8, 8))
    kp.tucker(t, [np.eye(8)] * 3)
    assert ctx.launches - before == 3


@pytest.mark.parametrize("n", [256])
def test_tucker_baseline_size_properties(kp, n):
    """At BASELINE size (n=256 here; 512 in the bench) check size-independent
    properties instead of a full oracle run: linearity in the tensor and the
    identity/permutation round trip."""
    import torch
    r = rng(12)
    t1 = kp.to_device(rand(r, (n, n, n)))
    t2 = kp.to_device(rand(r, (n, n, n)))
    ms = [kp.to_device(rand(r, (n, n))) for _ in range(3)]
    a, b = 0.37, -1.25
    lin = kp.tucker(a * t1 + b * t2, ms)
    want = a * kp.tucker(t1, ms) + b * kp.tucker(t2, ms)
    err = (torch.linalg.vector_norm(lin - want) / torch.linalg.vector_norm(want)).item()
    assert err < 1e-13
    perm = torch.randperm(n, generator=torch.Generator().manual_seed(0))
    pm = torch.zeros(n, n, dtype=torch.float64)
    pm[perm, torch.arange(n)] = 1.0
    fwd = kp.tucker(t1, [kp.to_device(pm.numpy())] * 3)
    back = kp.tucker(fwd, [kp.to_device(pm.numpy().T)] * 3)
    assert torch.equal(back, t1)


@pytest.mark.parametrize("dims", [(16, 12, 10), (300, 5, 4), (7, 260, 3), (64, 64, 64),
                                  (20, 20, 20, 2)])
def test_banded_kronsum_bitwise_vs_reference(kp, port, dims):
    """Tridiagonal / periodic factors take the stencil path (banded.cu), which
    follows the reference's dense FMA-chain rounding (incl. the KC=256 slices
    at n=260, 300): bit-identical to the reference's kronsum_action."""
    import pyoracle
    r = rng(31)
    t = rand(r, dims)
    As = []
    for mu, n in enumerate(dims):
        if n == 2:
            As.append(np.zeros((2, 2), order="F"))       # stacked-species factor
        elif mu % 2:
            As.append(port.fd_operator_1d(n, 0.3, 0.1))  # Dirichlet tridiagonal
        else:
            As.append(pyoracle.periodic_laplacian_1d(n, 0.7))  # periodic
    got = kp.kronsum_action(t, As)
    want = port.kronsum(t, As)
    assert np.array_equal(got, want)


def test_banded_kronsum_complex(kp, port):
    import pyoracle
    r = rng(32)
    t = rand(r, (24, 20, 18), True)
    As = [np.asfortranarray(0.5j * pyoracle.periodic_laplacian_1d(n, 0.5)) for n in t.shape]
    assert rel2(kp.kronsum_action(t, As), port.kronsum(t, As)) < 1e-15


@pytest.mark.parametrize("dims", [(40, 33, 70), (128, 128, 520)])
def test_host_tucker_stream_bitwise(kp, dims):
    """kp_host_tucker_stream_f64 (double-buffered upload/download overlap
    across tensors) returns, per tensor, exactly kp_host_tucker_f64's result."""
    import ctypes as C
    from paper_2304_02327_b200._lib import check, ints, ptr_array
    ctx = kp.default_context(0)
    r = np.random.default_rng(11)
    vs = [np.asfortranarray(r.standard_normal(dims)) for _ in range(5)]
    fs = [np.asfortranarray(r.standard_normal((n, n))) for n in dims]
    hptr = ptr_array([f.ctypes.data for f in fs])
    want = []
    for v in vs:
        o = np.zeros(dims, order="F")
        check(ctx.lib.kp_host_tucker_f64(ctx.h, v.ctypes.data, ints(list(dims)), 3, hptr,
                                         ints(list(dims)), 1.0, o.ctypes.data))
        want.append(o)
    outs = [np.zeros(dims, order="F") for _ in vs]
    ins_p = (C.c_void_p * 5)(*[v.ctypes.data for v in vs])
    outs_p = (C.c_void_p * 5)(*[o.ctypes.data for o in outs])
    check(ctx.lib.kp_host_tucker_stream_f64(ctx.h, 5, C.cast(ins_p, C.c_void_p),
                                            ints(list(dims)), 3, hptr, ints(list(dims)), 1.0,
                                            C.cast(outs_p, C.c_void_p)))
    for a, b in zip(outs, want):
        assert np.array_equal(a, b)


def _random_banded(r, n, kind):
    """kind 0: Dirichlet tridiagonal, 1: periodic tridiagonal, 2: bidiagonal (no
    diagonal), 3: diagonal only -- random values."""
    a = np.zeros((n, n), order="F")
    i = np.arange(n)
    if kind != 2:
        a[i, i] = r.standard_normal(n)
    if kind != 3 and n > 1:
        a[i[1:], i[:-1]] = r.standard_normal(n - 1)
        a[i[:-1], i[1:]] = r.standard_normal(n - 1)
    if kind == 1 and n > 2:
        a[0, n - 1] = r.standard_normal()
        a[n - 1, 0] = r.standard_normal()
    return a


@pytest.mark.parametrize("seed", range(8))
def test_banded_kronsum_fuzz_bitwise(kp, port, seed):
    """Random banded factors (every row pattern the stencil canonicalises or
    routes to its rare path), ragged extents incl. 1-3 and past the KC = 256
    slice, d = 1..4: bit-identical to the reference's dense kronsum_action."""
    r = rng(500 + seed)
    for _ in range(6):
        d = int(r.integers(1, 5))
        dims = [int(r.integers(1, 40)) for _ in range(d)]
        if r.random() < 0.5:
            dims[int(r.integers(0, d))] = int(r.integers(255, 300))
        while np.prod(dims) > 2e6:
            dims[int(np.argmax(dims))] //= 2
        t = rand(r, dims)
        As = [_random_banded(r, n, int(r.integers(0, 4))) for n in dims]
        got = kp.kronsum_action(t, As)
        want = port.kronsum(t, As)
        assert np.array_equal(got, want), (dims,)


@pytest.mark.parametrize("imag_only", [False, True])
def test_banded_kronsum_complex_fuzz(kp, port, imag_only):
    """Complex banded factors: general ones (the generic complex chain) and
    purely imaginary ones (the stencil's IMAG path: half the FP64 work, every
    value unchanged), periodic and Dirichlet, with a KC = 256 break."""
    r = rng(640 + int(imag_only))
    for dims in [(20, 17, 9), (258, 6, 5), (7, 270, 3), (5, 4, 262), (33, 12)]:
        t = rand(r, dims, True)
        As = []
        for n in dims:
            re = _random_banded(r, n, int(r.integers(0, 2)))
            im = _random_banded(r, n, int(r.integers(0, 2)))
            As.append(np.asfortranarray(1j * im if imag_only else re + 1j * im))
        assert rel2(kp.kronsum_action(t, As), port.kronsum(t, As)) < 1e-15, (dims,)
