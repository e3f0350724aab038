"""The sharded integrator's GPU backend at world size 1 (NCCL): the unfused
sharded step sequence must reproduce the fused single-GPU integrate bit for
bit (the property that makes P > 1 bit-identical as well, see
tests/test_parallel.py for the world-size-2 orchestration on CPU)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1():
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29571")
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("kronsum", ["banded", "dense"])
@pytest.mark.parametrize("case,method", [("ac3d", "etd2rk"), ("bru", "etd2rk"),
                                         ("bru", "lawson2b"), ("nls", "exp_euler")])
def test_sharded_p1_bitwise_equals_fused(kp, nccl1, case, method, kronsum):
    import torch
    from paper_2304_02327_b200 import parallel, problems
    if case == "ac3d":
        cfg = problems.ac3d(n=32, n_steps=6)
    elif case == "bru":
        cfg = problems.brusselator(n=16, n_steps=4, method=method)
    else:
        cfg = problems.nls(n=16, n_steps=4, method=method)
    cfg.method = method
    # both Kronecker-sum forms: the banded stencil (halo exchange when
    # sharded) and the dense one (pencil transposes when sharded)
    if kronsum == "dense":
        os.environ["KP_KRONSUM"] = "dense"
    try:
        want = kp.integrate_config(method, cfg.u0, cfg.K, cfg.g, 0.0, cfg.t_final, cfg.n_steps)
        be = parallel.CudaBackend(0)
        comm = parallel.Comm()
        K = [kp.to_device(k) for k in cfg.K]
        flat = kp.to_device(cfg.u0).permute(*reversed(range(cfg.u0.ndim))).reshape(-1)
        res = parallel.sharded_integrate(kp, be, comm, method, flat, list(cfg.u0.shape), K,
                                         cfg.g, 0.0, cfg.t_final, cfg.n_steps)
    finally:
        os.environ.pop("KP_KRONSUM", None)
    got = res.cpu().numpy().reshape(cfg.u0.shape, order="F")
    assert np.array_equal(got, want), np.abs(got - want).max()


@pytest.mark.parametrize("case,method,kronsum", [("ac3d", "etd2rk", "banded"),
                                                 ("ac3d", "exp_euler", "dense"),
                                                 ("ac2d", "exp_euler", "banded"),
                                                 ("bru", "lawson2b", "banded"),
                                                 ("bru", "etd2rk", "dense"),
                                                 ("nls", "etd2rk", "banded"),
                                                 ("ac3d", "lawson_euler", "banded")])
def test_peer_exchange_world2_one_gpu(kp, case, method, kronsum):
    """P = 2 processes on one GPU exchanging only through the fused peer
    stores (GEMM epilogue / scatter kernel into CUDA IPC buffers): the
    gathered result equals the single-GPU integrate bit for bit."""
    from conftest import ROOT, run_torchrun
    rc, out = run_torchrun(os.path.join(ROOT, "tests", "peer_worker.py"), [case, method, kronsum])
    assert rc == 0, out[-4000:]
    assert "PEER-OK" in out, out[-4000:]


def test_peer_exchange_p1_bitwise(kp):
    """PeerComm at P = 1 (no torch.distributed): the fused GEMM + exchange
    path reproduces the single-GPU integrate bit for bit."""
    from paper_2304_02327_b200 import parallel, problems
    cfg = problems.ac3d(n=24, n_steps=4)
    want = kp.integrate_config("etd2rk", cfg.u0, cfg.K, cfg.g, 0.0, cfg.t_final, cfg.n_steps)
    be = parallel.CudaBackend(0)
    comm = parallel.PeerComm(be)
    K = [kp.to_device(k) for k in cfg.K]
    flat = kp.to_device(cfg.u0).permute(*reversed(range(cfg.u0.ndim))).reshape(-1)
    res = parallel.sharded_integrate(kp, be, comm, "etd2rk", flat, list(cfg.u0.shape), K, cfg.g,
                                     0.0, cfg.t_final, cfg.n_steps)
    comm.close()
    got = res.cpu().numpy().reshape(cfg.u0.shape, order="F")
    assert np.array_equal(got, want)


@pytest.mark.parametrize("P,A,B,C,S,cplx", [(2, 6, 4, 8, 1, False), (3, 5, 6, 9, 2, False),
                                            (4, 3, 8, 4, 1, True), (2, 1, 2, 2, 2, True)])
def test_repartition_pack_unpack(kp, P, A, B, C, S, cplx):
    """kp_repartition_pack / _unpack (comm.cu, the local halves of
    kp_comm_repartition) with the all-to-all emulated between P simulated
    ranks on one GPU: slab -> pencil gives each rank exactly its pencil of
    the global tensor, and pencil -> slab restores the slabs bit for bit."""
    import torch
    from paper_2304_02327_b200._lib import check
    ctx = kp.default_context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    comps = 2 if cplx else 1
    dt = torch.complex128 if cplx else torch.float64
    g = torch.randn(S, C, B, A, dtype=dt, device="cuda")  # column-major (A, B, C, S)
    Cl, Bp = C // P, B // P
    slabs = [g[:, r * Cl:(r + 1) * Cl].contiguous().view(-1) for r in range(P)]
    pencils_want = [g[:, :, r * Bp:(r + 1) * Bp].contiguous().view(-1) for r in range(P)]

    def exchange(local, direction):
        sends = []
        for r in range(P):
            sb = torch.empty_like(local[r])
            check(ctx.lib.kp_repartition_pack(ctx.h, direction, P, r, A, B, C, S, comps,
                                              local[r].data_ptr(), sb.data_ptr()))
            sends.append(sb)
        blk = local[0].numel() // P
        outs = []
        for s in range(P):
            rb = torch.cat([sends[r][s * blk:(s + 1) * blk] for r in range(P)])
            ob = torch.empty_like(rb)
            check(ctx.lib.kp_repartition_unpack(ctx.h, direction, P, s, A, B, C, S, comps,
                                                rb.data_ptr(), ob.data_ptr()))
            outs.append(ob)
        return outs

    pencils = exchange(slabs, 1)
    for r in range(P):
        assert torch.equal(pencils[r], pencils_want[r]), r
    back = exchange(pencils, 2)
    for r in range(P):
        assert torch.equal(back[r], slabs[r]), r


@pytest.mark.parametrize("case,method,kronsum", [("ac3d", "etd2rk", "dense"),
                                                 ("bru", "etd2rk", "banded"),
                                                 ("nls", "exp_euler", "dense")])
def test_native_nccl_comm_p1_bitwise(kp, nccl1, case, method, kronsum):
    """The C ABI's own NCCL communicator (kp_comm_create from an ncclUniqueId,
    kp_comm_repartition, kp_comm_halo_f64) driving the sharded integrator at
    world size 1 reproduces the single-GPU integrate bit for bit."""
    from paper_2304_02327_b200 import parallel, problems
    if case == "ac3d":
        cfg = problems.ac3d(n=32, n_steps=4)
    elif case == "bru":
        cfg = problems.brusselator(n=16, n_steps=4, method=method)
    else:
        cfg = problems.nls(n=16, n_steps=4, method=method)
    cfg.method = method
    if kronsum == "dense":
        os.environ["KP_KRONSUM"] = "dense"
    try:
        want = kp.integrate_config(method, cfg.u0, cfg.K, cfg.g, 0.0, cfg.t_final, cfg.n_steps)
        be = parallel.CudaBackend(0)
        comm = parallel.NcclComm(be)
        K = [kp.to_device(k) for k in cfg.K]
        flat = kp.to_device(cfg.u0).permute(*reversed(range(cfg.u0.ndim))).reshape(-1)
        res = parallel.sharded_integrate(kp, be, comm, method, flat, list(cfg.u0.shape), K,
                                         cfg.g, 0.0, cfg.t_final, cfg.n_steps)
        comm.close()
    finally:
        os.environ.pop("KP_KRONSUM", None)
    got = res.cpu().numpy().reshape(cfg.u0.shape, order="F")
    assert np.array_equal(got, want), np.abs(got - want).max()


@pytest.mark.parametrize("case", ["ac", "bru", "nls"])
def test_mode_product_stage_matches_unfused(kp, case):
    """kp_mode_product_stage_* (ETD2RK's stage update in the last GEMM's
    epilogue, used by the sharded step) equals mode product -> fma -> two g
    evaluations -> subtraction, bit for bit."""
    import torch
    from paper_2304_02327_b200 import parallel, problems
    be = parallel.CudaBackend(0)
    r = np.random.default_rng(3)
    if case == "nls":
        dims, g = [12, 10, 8], problems.G.nls()
        mk = lambda s: torch.tensor(r.standard_normal(s) + 1j * r.standard_normal(s),
                                    device="cuda")
    elif case == "bru":
        dims, g = [10, 9, 8, 2], problems.G.brusselator(1.0, 3.0)
        mk = lambda s: torch.tensor(1 + 0.1 * r.standard_normal(s), device="cuda")
    else:
        dims, g = [10, 9, 8], problems.G.allen_cahn()
        mk = lambda s: torch.tensor(r.standard_normal(s), device="cuda")
    n = int(np.prod(dims))
    t, x = mk(n), mk(n)
    mode = 2
    m = mk(dims[mode] * dims[mode])
    tau = 1e-3
    out, dd = torch.empty_like(t), torch.empty_like(t)
    be.mode_product_stage(t, dims, mode, m.view(dims[mode], dims[mode]), 0.5, x, tau, g, out, dd)
    y = torch.empty_like(t)
    be.mode_product(t, dims, mode, m.view(dims[mode], dims[mode]), 0.5, 0.0, y)
    st = torch.empty_like(t)
    be.fma(tau, y, x, st)
    gs, gx = torch.empty_like(t), torch.empty_like(t)
    be.eval_g(g, st, dims, gs)
    be.eval_g(g, x, dims, gx)
    torch.cuda.synchronize()
    assert torch.equal(out, st)
    assert torch.equal(dd, gs - gx)
