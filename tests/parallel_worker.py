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

    def kronsum_slab(self, u_ext, dims, K, slab_mode, k0, n_glob, g, out):
        """numpy restatement of kp_kronsum_slab (rows' nonzeros in increasing
        column order; halo planes at local 0 and Cl+1 of the slab mode)."""
        d = len(dims)
        ext = list(dims)
        ext[slab_mode] += 2
        U = u_ext.numpy().reshape(ext, order="F")
        Cl = dims[slab_mode]
        interior = np.take(U, np.arange(1, Cl + 1), axis=slab_mode)
        R = None
        for mu in range(d):
            A = K[mu].numpy()
            if not A.any():
                continue
            term = np.zeros(dims, dtype=U.dtype)
            for i in range(dims[mu]):
                gi = i + k0 if mu == slab_mode else i
                acc = None
                for j in np.nonzero(A[gi])[0]:
                    if mu == slab_mode:
                        src = np.take(U, [(j - (k0 - 1)) % n_glob], axis=mu)
                    else:
                        src = np.take(interior, [j], axis=mu)
                    p = A[gi, j] * src
                    acc = p if acc is None else acc + p
                if acc is not None:
                    idx = [slice(None)] * d
                    idx[mu] = slice(i, i + 1)
                    term[tuple(idx)] = acc
            R = term if R is None else term + R
        if g is not None:
            og = pyoracle.gfun(g.kind, *list(g.p))
            R = R + port.eval_g(og, 0.0, np.asfortranarray(interior))
        out.copy_(torch.from_numpy(np.asfortranarray(R).reshape(-1, order="F")))


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
        one = parallel.sharded_integrate(KP, be, parallel.LocalComm(), method,
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
