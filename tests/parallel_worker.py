"""Worker for tests/test_parallel.py (run under torch.distributed.run, gloo)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import pyoracle  # noqa: E402  (test infrastructure: the CPU backend below)
from paper_2304_02327_b200 import parallel, problems  # noqa: E402

port = pyoracle.Oracle("port")


class CpuBackend:
    """Oracle mode products (shape-independent rounding) + numpy elementwise."""

    def mode_product(self, t, dims, mode, m, alpha, beta, out):
        tt = t.numpy().reshape(dims, order="F")
        mm = m.numpy()
        od = list(dims)
        od[mode] = mm.shape[0]
        if alpha != 1.0:
            tt = tt * alpha  # powers of two (prefactor, folds of I/l!) in these tests
        if beta == 0.0:
            res = port.mode_product(tt, mm, mode)
        else:
            res = port.mode_product(tt, mm, mode, out=out.numpy().reshape(od, order="F"))
        out.copy_(torch.from_numpy(np.asarray(res).reshape(-1, order="F")))

    def eval_g(self, g, u, dims, out):
        og = pyoracle.gfun(g.kind, *list(g.p))
        res = port.eval_g(og, 0.0, u.numpy().reshape(dims, order="F"))
        out.copy_(torch.from_numpy(np.asarray(res).reshape(-1, order="F")))

    def fma(self, alpha, x, y, out):
        out.copy_(torch.from_numpy(np.asarray(alpha * x.numpy() + y.numpy())))


class KP:
    """CPU stand-in for the package's device factor builder (oracle build)."""

    @staticmethod
    def build_split_phi(K, tau, ell):
        fs, pref = port.build_split_phi([np.asarray(k) for k in K], tau, ell)

        class SP:
            pass
        sp = SP()
        sp.factors = [torch.from_numpy(np.asfortranarray(f)) for f in fs]
        sp.prefactor = pref
        return sp

    @staticmethod
    def to_host(t):
        return t.numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


class OneRank:
    P, rank = 1, 0

    def all_to_all(self, recv, send):
        recv.copy_(send)


def main():
    case, method = sys.argv[1], sys.argv[2]
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    comm = parallel.Comm()
    if case == "ac3d":
        cfg = problems.ac3d(n=8, n_steps=4)
    elif case == "ac2d":
        cfg = problems.ac2d(n=8, n_steps=4)
    elif case == "bru":
        cfg = problems.brusselator(n=4, n_steps=3, method=method)
    else:
        cfg = problems.nls(n=8, n_steps=3, method=method)
    cfg.method = method
    species = 2 if case == "bru" else 1
    K = [torch.from_numpy(np.asfortranarray(k)) for k in cfg.K]
    full = cfg.u0
    loc = np.asfortranarray(parallel.local_slab(full, P, rank, species))
    flat = torch.from_numpy(loc.reshape(-1, order="F").copy())
    be = CpuBackend()
    res = parallel.sharded_integrate(KP, be, comm, method, flat, list(loc.shape), K, cfg.g, 0.0,
                                     cfg.t_final, cfg.n_steps)
    parts = [torch.empty_like(res) for _ in range(P)]
    dist.all_gather(parts, res)
    if rank == 0:
        axis = full.ndim - 2 if species == 2 else full.ndim - 1
        glob = np.concatenate([p.numpy().reshape(loc.shape, order="F") for p in parts], axis=axis)
        one = parallel.sharded_integrate(KP, be, OneRank(), method,
                                         torch.from_numpy(full.reshape(-1, order="F").copy()),
                                         list(full.shape), K, cfg.g, 0.0, cfg.t_final,
                                         cfg.n_steps)
        one = one.numpy().reshape(full.shape, order="F")
        assert np.array_equal(glob, one), f"sharded != unsharded: {np.abs(glob - one).max()}"
        og = pyoracle.gfun(cfg.g.kind, *list(cfg.g.p))
        want = port.integrate(method, full, cfg.K, og, 0.0, cfg.t_final, cfg.n_steps)
        rel = np.linalg.norm(glob - want) / np.linalg.norm(want)
        assert rel < 1e-12, rel
        print("SHARDED-OK", case, method, rel)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
