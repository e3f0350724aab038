"""The native (C++) slab-sharded integrator, kp_integrate_sharded_* (stepper.cu
ShardedIntegrator).  On one GPU its P ranks run emulated in
one process (kp_integrate_sharded_local_*: the exchanges become device copies
between the ranks' buffers -- the same step sequence and data movement as a
P-GPU run); the NCCL communicator path runs at world size 1.
  * mode d by all-to-all pencil transposes: BITWISE equal to the single-GPU
    integrate (same inputs, same k order per entry);
  * mode d by partial products + reduce-scatter: rel-l2 <= 1e-12."""
import ctypes as C

import numpy as np
import pytest

from conftest import rel2, rng

pytestmark = pytest.mark.gpu


def config(name, method):
    from paper_2304_02327_b200 import problems
    if name == "ac3d":
        c = problems.ac3d(n=32, n_steps=12)
    elif name == "bru":
        c = problems.brusselator(n=16, n_steps=10, method=method)
    elif name == "nls":
        c = problems.nls(n=16, n_steps=8, method=method)
    elif name == "dense":  # non-banded factors: the dense Kronecker sum path
        r = rng(17)
        K = []
        for n in (12, 8, 8):
            a = r.uniform(-1, 1, (n, n))
            a -= np.abs(a).sum(0).max() * np.eye(n)
            K.append(np.asfortranarray(a))
        c = problems.ac3d(n=8, n_steps=6)
        c.u0 = np.asfortranarray(r.uniform(-1, 1, (12, 8, 8)))
        c.K = K
    c.method = method
    return c


def slabs_of(u0, P, species):
    ax = u0.ndim - (2 if species else 1)
    n = u0.shape[ax] // P
    return [np.asfortranarray(np.take(u0, range(r * n, (r + 1) * n), axis=ax)) for r in range(P)]


def run_native(kp, c, P, mode_d, comm=None):
    from paper_2304_02327_b200 import parallel
    species = c.g.kind == kp.G_BRUSSELATOR
    hs = slabs_of(c.u0, P, species)
    ds = [kp.to_device(h) for h in hs]
    used, loop = parallel.native_sharded_integrate(
        kp, c.method, ds, list(hs[0].shape), [kp.to_device(np.asarray(k)) for k in c.K], c.g,
        0.0, c.t_final, c.n_steps, comm=comm, mode_d=mode_d)
    ax = c.u0.ndim - (2 if species else 1)
    return np.concatenate([kp.to_host(x) for x in ds], axis=ax), used, loop


CASES = [("ac3d", "etd2rk"), ("ac3d", "exp_euler"), ("ac3d", "lawson2b"),
         ("ac3d", "lawson_euler"), ("bru", "etd2rk"), ("bru", "lawson2b"),
         ("nls", "etd2rk"), ("nls", "exp_euler"), ("dense", "etd2rk")]


@pytest.mark.parametrize("name,method", CASES)
@pytest.mark.parametrize("P", [1, 2, 4])
def test_native_sharded_alltoall_bitwise(kp, name, method, P):
    c = config(name, method)
    want = kp.integrate_config(c.method, c.u0, c.K, c.g, 0.0, c.t_final, c.n_steps)
    got, used, loop = run_native(kp, c, P, "alltoall")
    assert used == 1 and loop > 0
    assert np.array_equal(got, want), rel2(got, want)


@pytest.mark.parametrize("name,method", [c for c in CASES if c[0] != "dense"])
@pytest.mark.parametrize("P", [1, 2, 4])
def test_native_sharded_fused_bitwise(kp, name, method, P):
    """mode d 3: the mode products' epilogues store straight into the owning
    ranks' buffers (peer stores; here the emulated ranks' buffers), the plain
    re-partitions are scatter kernels -- the same values as the all-to-all:
    bitwise equal to the single-GPU integrate."""
    c = config(name, method)
    want = kp.integrate_config(c.method, c.u0, c.K, c.g, 0.0, c.t_final, c.n_steps)
    got, used, _ = run_native(kp, c, P, "fused")
    assert used == 3
    assert np.array_equal(got, want), rel2(got, want)


@pytest.mark.parametrize("name,method", [("ac3d", "etd2rk"), ("bru", "etd2rk"),
                                         ("nls", "etd2rk"), ("ac3d", "lawson2b"),
                                         ("ac3d", "exp_euler"), ("dense", "etd2rk")])
@pytest.mark.parametrize("P", [2, 4])
def test_native_sharded_reduce_scatter(kp, name, method, P):
    c = config(name, method)
    want = kp.integrate_config(c.method, c.u0, c.K, c.g, 0.0, c.t_final, c.n_steps)
    got, used, _ = run_native(kp, c, P, "reduce_scatter")
    assert used == 2
    assert rel2(got, want) < 1e-12


def test_native_sharded_auto_picks_one(kp):
    c = config("ac3d", "etd2rk")
    want = kp.integrate_config(c.method, c.u0, c.K, c.g, 0.0, c.t_final, c.n_steps)
    got, used, _ = run_native(kp, c, 2, "auto")
    assert used in (1, 2, 3)
    assert rel2(got, want) < 1e-12


def test_native_sharded_divergence_step(kp):
    """The 2-D NLS analogue of configs[4] diverges: the sharded
    run reports the single-GPU run's first non-finite step."""
    import pyoracle
    n = 64
    h = 2.0 / n
    A = np.asfortranarray(0.5j * pyoracle.periodic_laplacian_1d(n, h))
    r = rng(11)
    x = -1.0 + h * np.arange(n)
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = np.asfortranarray(np.exp(-(X * X + Y * Y) * 8.0) + 0.01 * (r.standard_normal((n, n)) +
                                                                    1j * r.standard_normal((n, n))))
    with pytest.raises(kp.DivergenceError) as e1:
        kp.integrate_config("exp_euler", u0, [A, A], kp.G.nls(), 0.0, 0.2, 200)
    from paper_2304_02327_b200 import problems
    c = problems.nls(n=8)
    c.u0, c.K, c.method, c.t_end, c.n_steps = u0, [A, A], "exp_euler", 0.2, 200
    with pytest.raises(kp.DivergenceError) as e2:
        run_native(kp, c, 2, "alltoall")
    assert e2.value.step == e1.value.step


class _OneRankComm:
    """kp_comm over NCCL at world size 1 (kp_comm_unique_id + kp_comm_create)."""

    def __init__(self, kp):
        ctx = kp.default_context(0)
        self.lib = ctx.lib
        uid = (C.c_char * 128)()
        assert self.lib.kp_comm_unique_id(uid) == 0
        h = C.c_void_p()
        assert self.lib.kp_comm_create(ctx.h, 1, 0, uid, C.byref(h)) == 0, \
            kp.last_error() if hasattr(kp, "last_error") else ""
        self.h = h

    def close(self):
        self.lib.kp_comm_destroy(self.h)


@pytest.mark.parametrize("name,method", [("ac3d", "etd2rk"), ("bru", "lawson2b"),
                                         ("nls", "etd2rk")])
def test_native_sharded_nccl_world1_bitwise(kp, name, method):
    c = config(name, method)
    want = kp.integrate_config(c.method, c.u0, c.K, c.g, 0.0, c.t_final, c.n_steps)
    comm = _OneRankComm(kp)
    try:
        got, used, _ = run_native(kp, c, 1, "auto", comm=comm)
    finally:
        comm.close()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("mode_d", [1, 2, 3])
def test_tucker_sharded_local(kp, P, mode_d):
    """kp_tucker_sharded_local_f64: mode 1 (all-to-all) gives each rank its
    pencil block of the single-GPU Tucker bitwise; mode 2 (reduce-scatter)
    its slab block within 1e-12."""
    import torch
    from paper_2304_02327_b200._lib import check, ints, ptr_array
    r = rng(99)
    n1, n2, n3 = 24, 16, 32
    v = np.asfortranarray(r.standard_normal((n1, n2, n3)))
    ms = [np.asfortranarray(r.standard_normal((n, n)) / n) for n in (n1, n2, n3)]
    want = kp.tucker(v, ms)
    ctx = kp.default_context(0)
    slabs = [kp.to_device(np.asfortranarray(v[:, :, k * n3 // P:(k + 1) * n3 // P]))
             for k in range(P)]
    outs = [kp.to_device(np.zeros_like(kp.to_host(s))) for s in slabs]
    md = [kp.to_device(m) for m in ms]
    arr = (C.c_void_p * P)(*[s.data_ptr() for s in slabs])
    oarr = (C.c_void_p * P)(*[o.data_ptr() for o in outs])
    check(ctx.lib.kp_tucker_sharded_local_f64(ctx.h, P, C.cast(arr, C.c_void_p),
                                              ints([n1, n2, n3 // P]), 3,
                                              ptr_array([m.data_ptr() for m in md]), 1.0,
                                              mode_d, C.cast(oarr, C.c_void_p)))
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        flat = kp.to_host(o).reshape(-1, order="F")
        if mode_d in (1, 3):  # pencil: (n1, n2/P, n3)
            blk = np.asfortranarray(want[:, k * n2 // P:(k + 1) * n2 // P, :])
            assert np.array_equal(flat, blk.reshape(-1, order="F"))
        else:            # slab: (n1, n2, n3/P)
            blk = np.asfortranarray(want[:, :, k * n3 // P:(k + 1) * n3 // P])
            assert rel2(flat, blk.reshape(-1, order="F")) < 1e-12


@pytest.mark.parametrize("seed", range(5))
def test_native_sharded_fuzz_shapes(kp, seed):
    """Random ragged slabs: mode extents with odd leading dimensions, P in
    {2, 3, 4} (modes d-1 and d divisible by P), banded and dense Kronecker
    sums, all-to-all and fused exchanges -- bitwise equal to one GPU."""
    from paper_2304_02327_b200 import problems
    r = rng(4100 + seed)
    for _ in range(3):
        P = int(r.integers(2, 5))
        dims = (int(r.integers(3, 20)), P * int(r.integers(1, 6)), P * int(r.integers(1, 6)))
        method = ["etd2rk", "exp_euler", "lawson2b", "lawson_euler"][int(r.integers(0, 4))]
        c = problems.ac3d(n=8, n_steps=int(r.integers(1, 5)))
        c.method = method
        c.u0 = np.asfortranarray(0.3 + 0.1 * r.uniform(-1, 1, dims))
        banded = r.random() < 0.5
        if banded:
            c.K = [problems.fd_operator_1d(n, 0.01, 0.05) for n in dims]
        else:
            c.K = []
            for n in dims:
                a = r.uniform(-1, 1, (n, n))
                a -= np.abs(a).sum(0).max() * np.eye(n)
                c.K.append(np.asfortranarray(a))
        want = kp.integrate_config(c.method, c.u0, c.K, c.g, 0.0, c.t_final, c.n_steps)
        # (the fused exchange is defined for banded factors and the phi methods)
        for md in ("alltoall", "fused") if banded else ("alltoall",):
            got, used, loop = run_native(kp, c, P, md)
            assert np.array_equal(got, want), (dims, P, method, md, rel2(got, want))
