"""Worker for tests/test_parallel_gpu.py::test_peer_exchange_world2_one_gpu:
P = 2 ranks (torch.distributed.run, gloo for the barrier and the IPC handle
exchange) that both run on cuda:0 and exchange data only through the fused
peer stores (parallel.PeerComm: GEMM epilogues and scatter kernels writing
into CUDA-IPC-mapped buffers).  No kernel waits on the other rank -- every
exchange is completed by a stream synchronize + host barrier -- so sharing
one GPU is safe.  Rank 0 checks the gathered result against the fused
single-GPU integrate bit for bit."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2304_02327_b200 as kp  # noqa: E402
from paper_2304_02327_b200 import parallel, problems  # noqa: E402


def main():
    case, method, kronsum = sys.argv[1], sys.argv[2], sys.argv[3]
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    if kronsum == "dense":
        os.environ["KP_KRONSUM"] = "dense"
    if case == "ac3d":
        cfg = problems.ac3d(n=16, n_steps=5)
    elif case == "ac2d":
        cfg = problems.ac2d(n=24, n_steps=5)
    elif case == "bru":
        cfg = problems.brusselator(n=12, n_steps=4, method=method)
    else:
        cfg = problems.nls(n=16, n_steps=3, method=method)
    species = 2 if case == "bru" else 1
    be = parallel.CudaBackend(0)
    comm = parallel.PeerComm(be)
    K = [kp.to_device(k) for k in cfg.K]
    sl = np.asfortranarray(parallel.local_slab(cfg.u0, P, rank, species))
    dims_local = list(sl.shape)
    flat = kp.to_device(sl).permute(*reversed(range(sl.ndim))).reshape(-1)
    res = parallel.sharded_integrate(kp, be, comm, method, flat, dims_local, K, cfg.g, 0.0,
                                     cfg.t_final, cfg.n_steps)
    mine = res.cpu().numpy().reshape(dims_local, order="F")
    slabs = [None] * P
    dist.all_gather_object(slabs, mine)
    comm.close()
    if rank == 0:
        axis = sl.ndim - 2 if species > 1 else sl.ndim - 1
        got = np.concatenate(slabs, axis=axis)
        want = kp.integrate_config(method, cfg.u0, cfg.K, cfg.g, 0.0, cfg.t_final, cfg.n_steps)
        ok = np.array_equal(got, want)
        print("PEER-OK" if ok else f"PEER-MISMATCH {np.abs(got - want).max()}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
