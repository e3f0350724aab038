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
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "tests", "peer_worker.py"), case, method, kronsum]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
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
