"""Slab-sharded integrators across the GPUs of one node.

Partition: the last spatial mode n_d is split into P contiguous slabs (in the
column-major layout a slab is a contiguous run of n_d/P planes per species).
Modes 1..d-1 and the pointwise g are local.  Mode d needs every slab: the
state is re-partitioned along mode d-1 by an all-to-all "pencil transpose"
(torch.distributed over NCCL/NVLink on GPUs, gloo in the CPU tests), mode d
is applied locally, and the result goes back.  Every output entry is computed
from the same inputs in the same k order as on one GPU, so the sharded run is
bit-identical to the single-GPU one (tests/test_parallel.py checks this on
CPU with world size 2; the GPU backend reuses the single-GPU kernels).

Per step (unfused, same rounding as the fused single-GPU path), with the
configs' banded factors the Kronecker sum is the stencil pass of banded.cu on
the slab plus a one-plane halo exchange (batch_isend_irecv):
  ExpEuler : halo + 3 all-to-alls (Tucker in, u to pencil, result back)
  ETD2RK   : halo + 5 all-to-alls
  Lawson2b : 4 all-to-alls (two Tuckers, each in and out)
(dense factors: the Kronecker sum's last-mode term takes 2 more).  Each
all-to-all moves N_local (P-1)/P entries per rank; DESIGN.md 7 has the model.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

try:
    import torch
    import torch.distributed as dist
except Exception:  # pragma: no cover
    torch = None
    dist = None


# ------------------------------------------------------------------ layout

@dataclass
class Layout:
    """Column-major local tensor viewed as (A, B, C, S):
    A = prod(n_1..n_{d-2}), B = n_{d-1} (or its pencil share), C = n_d share,
    S = species (1 if none).  `slab` splits C, `pencil` splits B."""
    A: int
    B: int
    C: int
    S: int
    P: int

    @staticmethod
    def of(spatial, species, P):
        *lead, nb, nc = ([1] + list(spatial)) if len(spatial) == 1 else list(spatial)
        A = int(np.prod(lead)) if lead else 1
        if nc % P or nb % P:
            raise ValueError(f"slab sharding needs n_(d-1) and n_d divisible by P={P}")
        return Layout(A, nb, nc, species, P)

    def slab_dims(self, spatial, species):
        d = list(spatial[:-1]) + [spatial[-1] // self.P]
        return d + ([species] if species > 1 else [])

    def pencil_dims(self, spatial, species):
        d = list(spatial[:-2]) + [spatial[-2] // self.P, spatial[-1]]
        return d + ([species] if species > 1 else [])


def slab_to_pencil(x, lay: Layout, comm):
    """x: flat local slab (A, B, C/P... as column-major (A, B, Cl, S)) ->
    flat local pencil (A, B/P, C, S)."""
    if hasattr(comm, "repartition"):  # native: pack -> NCCL -> unpack (comm.cu)
        return comm.repartition(x, lay, 1)
    A, B, C, S, P = lay.A, lay.B, lay.C, lay.S, lay.P
    Cl, Bp = C // P, B // P
    send = x.view(S, Cl, P, Bp, A).permute(2, 0, 1, 3, 4).contiguous().view(-1)
    recv = torch.empty_like(send)
    comm.all_to_all(recv, send)
    return recv.view(P, S, Cl, Bp, A).permute(1, 0, 2, 3, 4).contiguous().view(-1)


def pencil_to_slab(y, lay: Layout, comm):
    if hasattr(comm, "repartition"):
        return comm.repartition(y, lay, 2)
    A, B, C, S, P = lay.A, lay.B, lay.C, lay.S, lay.P
    Cl, Bp = C // P, B // P
    send = y.view(S, P, Cl, Bp, A).permute(1, 0, 2, 3, 4).contiguous().view(-1)
    recv = torch.empty_like(send)
    comm.all_to_all(recv, send)
    return recv.view(P, S, Cl, Bp, A).permute(1, 2, 0, 3, 4).contiguous().view(-1)


def halo_extend(x, lay: Layout, comm):
    """Flat slab (A, B, C/P, S) -> flat (A, B, C/P + 2, S) with one halo plane
    of the sharded mode on each side: global planes k0-1 and k1 (periodic in
    the rank index; a Dirichlet factor never reads the wrapped plane)."""
    A, B, S, P = lay.A, lay.B, lay.S, lay.P
    Cl = lay.C // P
    xs = x.view(S, Cl, A * B)
    first = xs[:, 0, :].contiguous()
    last = xs[:, Cl - 1, :].contiguous()
    left, right = torch.empty_like(first), torch.empty_like(last)
    comm.exchange_halos(first, last, left, right)
    ext = torch.empty((S, Cl + 2, A * B), dtype=x.dtype, device=x.device)
    ext[:, 1:Cl + 1, :] = xs
    ext[:, 0, :] = left
    ext[:, Cl + 1, :] = right
    return ext.view(-1)


class Comm:
    """Equal-split all-to-all on a torch.distributed group (NCCL on GPUs)."""

    def __init__(self, group=None):
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_to_all(self, recv, send):
        if self.P == 1:
            recv.copy_(send)
            return
        if torch.is_complex(send):
            dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send),
                                   group=self.group)
        else:
            dist.all_to_all_single(recv, send, group=self.group)

    def exchange_halos(self, first, last, left, right):
        """left <- last plane of rank-1, right <- first plane of rank+1 (cyclic)."""
        if self.P == 1:
            left.copy_(last)
            right.copy_(first)
            return
        prev, nxt = (self.rank - 1) % self.P, (self.rank + 1) % self.P
        g = lambda r: dist.get_global_rank(self.group, r) if self.group is not None else r
        view = torch.view_as_real if torch.is_complex(first) else (lambda t: t)
        ops = [dist.P2POp(dist.isend, view(last), g(nxt), self.group, 0),
               dist.P2POp(dist.irecv, view(left), g(prev), self.group, 0),
               dist.P2POp(dist.isend, view(first), g(prev), self.group, 1),
               dist.P2POp(dist.irecv, view(right), g(nxt), self.group, 1)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()


class NcclComm:
    """The C ABI's own NCCL communicator (kp_comm_*, comm.cu): created from an
    ncclUniqueId that rank 0 generates and torch.distributed broadcasts (any
    side channel would do -- this is how a C++ host without Python runs the
    sharded path).  Re-partitions run as pack -> grouped ncclSend/Recv ->
    unpack on the context's stream, halos as grouped send/recv."""

    def __init__(self, backend, group=None):
        import ctypes as C
        self.be = backend
        self.lib, self.ctx = backend.ctx.lib, backend.ctx
        self.group = group
        self.P = dist.get_world_size(group) if dist and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist and dist.is_initialized() else 0
        uid = (C.c_char * 128)()
        if self.rank == 0:
            backend.check(self.lib.kp_comm_unique_id(uid))
        if self.P > 1:
            obj = [bytes(uid)]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
            C.memmove(uid, obj[0], 128)
        h = C.c_void_p()
        backend.check(self.lib.kp_comm_create(self.ctx.h, self.P, self.rank, uid, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.be.check(self.lib.kp_comm_destroy(self.h))
            self.h = None

    def all_to_all(self, recv, send):
        self.be._sync_stream()
        n = send.numel() * (2 if torch.is_complex(send) else 1)
        self.be.check(self.lib.kp_comm_alltoall_f64(self.ctx.h, self.h, send.data_ptr(),
                                                    recv.data_ptr(), n // self.P))

    def repartition(self, x, lay: Layout, direction):
        self.be._sync_stream()
        comps = 2 if torch.is_complex(x) else 1
        y = torch.empty_like(x)
        self.be.check(self.lib.kp_comm_repartition(self.ctx.h, self.h, direction, lay.A, lay.B,
                                                   lay.C, lay.S, comps, x.data_ptr(),
                                                   y.data_ptr()))
        return y

    def exchange_halos(self, first, last, left, right):
        self.be._sync_stream()
        n = first.numel() * (2 if torch.is_complex(first) else 1)
        self.be.check(self.lib.kp_comm_halo_f64(self.ctx.h, self.h, first.data_ptr(),
                                                last.data_ptr(), n, left.data_ptr(),
                                                right.data_ptr()))


class LocalComm:
    """World of one rank without torch.distributed (the unsharded reference
    run of the sharded code path)."""
    P, rank = 1, 0

    def all_to_all(self, recv, send):
        recv.copy_(send)

    def exchange_halos(self, first, last, left, right):
        left.copy_(last)
        right.copy_(first)


def scatter_destinations(lay: Layout, direction: int, rank: int):
    """Host restatement of the kp_scatter index map (exchange.cu /
    mode_product.cu scatter_ptr): for every entry of the rank's local tensor
    (slab for direction 1, pencil for 2), its destination rank and index in
    that rank's receive buffer.  Used by the tests to check the device map
    against slab_to_pencil / pencil_to_slab."""
    A, B, C, S, P = lay.A, lay.B, lay.C, lay.S, lay.P
    Bp, Cl = B // P, C // P
    if direction == 1:
        n = A * B * Cl * S
        e = np.arange(n, dtype=np.int64)
        a, t = e % A, e // A
        b, t = t % B, t // B
        cl, sp = t % Cl, t // Cl
        s = b // Bp
        idx = a + A * ((b - s * Bp) + Bp * (rank * Cl + cl + C * sp))
    else:
        n = A * Bp * C * S
        e = np.arange(n, dtype=np.int64)
        a, t = e % A, e // A
        bl, t = t % Bp, t // Bp
        c, sp = t % C, t // C
        s = c // Cl
        idx = a + A * ((rank * Bp + bl) + B * ((c - s * Cl) + Cl * sp))
    return s, idx


class _DevArray:
    """__cuda_array_interface__ view of a raw device pointer (IPC mappings)."""

    def __init__(self, ptr, n, cplx):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<c16" if cplx else "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


class PeerComm:
    """The exchange of the sharded integrators as device-initiated stores
    into peer memory instead of collectives (include/kronphi_b200.h,
    kp_scatter).  Every exchange site owns a receive buffer per rank,
    allocated once (cudaMalloc), shared through CUDA IPC (handles exchanged
    with torch.distributed) and mapped into every other rank; producers store
    into the owners' buffers -- from a GEMM epilogue (`mode_product_to`) or a
    scatter kernel (`slab_to_pencil` / `pencil_to_slab`) -- then every rank
    synchronizes its stream and meets the others at a barrier before reading.
    No kernel waits on another rank, so ranks may even share one GPU (the
    tests run P = 2 on one device).  `group` carries only the barrier and the
    handle exchange (gloo or NCCL)."""

    fused = True

    def __init__(self, backend, group=None):
        from ._lib import Scatter, check
        self.be = backend
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self._Scatter, self._check = Scatter, check
        self.slots = {}  # name -> (nbytes, own ptr, [peer ptrs], opened ptrs)

    # -- buffers ------------------------------------------------------------
    def _slot(self, name, nbytes):
        import ctypes as C
        lib, ctx = self.be.ctx.lib, self.be.ctx
        cur = self.slots.get(name)
        if cur is not None and cur[0] >= nbytes:
            return cur
        if cur is not None:
            self._release(name)
        own = C.c_void_p()
        self._check(lib.kp_malloc(ctx.h, max(int(nbytes), 16), C.byref(own)))
        h = (C.c_char * 64)()
        self._check(lib.kp_ipc_get_handle(own, h))
        handles = [None] * self.P
        if self.P > 1:
            dist.all_gather_object(handles, bytes(h), group=self.group)
        else:
            handles[0] = bytes(h)
        peers, opened = [], []
        for r in range(self.P):
            if r == self.rank:
                peers.append(own.value)
                continue
            p = C.c_void_p()
            hb = (C.c_char * 64).from_buffer_copy(handles[r])
            self._check(lib.kp_ipc_open_handle(hb, C.byref(p)))
            peers.append(p.value)
            opened.append(p.value)
        self.slots[name] = (int(nbytes), own.value, peers, opened)
        return self.slots[name]

    def _release(self, name):
        lib, ctx = self.be.ctx.lib, self.be.ctx
        nbytes, own, peers, opened = self.slots.pop(name)
        torch.cuda.synchronize(self.be.device)
        self.barrier()
        for p in opened:
            lib.kp_ipc_close_handle(p)
        self.barrier()
        lib.kp_free(ctx.h, own)

    def close(self):
        for name in list(self.slots):
            self._release(name)

    def barrier(self):
        """All ranks' stores into the receive buffers are complete."""
        torch.cuda.current_stream(self.be.device).synchronize()
        if self.P > 1:
            dist.barrier(group=self.group)

    def _desc(self, lay, direction, peers):
        import ctypes as C
        arr = (C.c_void_p * self.P)(*peers)
        sc = self._Scatter(direction, self.P, self.rank, lay.A, lay.B, lay.C, lay.S,
                           C.cast(arr, C.c_void_p))
        sc._keep = arr
        return sc

    def _view(self, name, n, like):
        _, own, _, _ = self.slots[name]
        return torch.as_tensor(_DevArray(own, n, torch.is_complex(like)), device=like.device)

    # -- exchanges ----------------------------------------------------------
    def _transpose(self, x, lay, direction, name):
        import ctypes as C
        cplx = torch.is_complex(x)
        n = x.numel()
        slot = self._slot(name, n * x.element_size())
        sc = self._desc(lay, direction, slot[2])
        self.be._sync_stream()
        self._check(self.be.ctx.lib.kp_scatter_copy(self.be.ctx.h, x.data_ptr(), n,
                                                    2 if cplx else 1, C.byref(sc)))
        self.barrier()
        return self._view(name, n, x)

    def slab_to_pencil(self, x, lay, name):
        return self._transpose(x, lay, 1, name)

    def pencil_to_slab(self, y, lay, name):
        return self._transpose(y, lay, 2, name)

    def mode_product_to(self, t, dims, mode, m, alpha, lay, direction, name, x=None, gamma=0.0):
        """fma(gamma, alpha (t x_mode m), x) with every entry stored at its
        owner in the other layout (one kernel: GEMM + exchange); returns this
        rank's received tensor (flat)."""
        import ctypes as C
        cplx = torch.is_complex(t)
        n_out = 1
        for i, v in enumerate(dims):
            n_out *= (m.shape[0] if i == mode else v)
        esz = 16 if cplx else 8
        slot = self._slot(name, n_out * esz)
        sc = self._desc(lay, direction, slot[2])
        self.be._sync_stream()
        lib = self.be.ctx.lib
        f = lib.kp_mode_product_scatter_c128 if cplx else lib.kp_mode_product_scatter_f64
        self._check(f(self.be.ctx.h, t.data_ptr(), self.be.ints(dims), len(dims), mode,
                      m.data_ptr(), m.shape[0], float(alpha),
                      x.data_ptr() if x is not None else None, float(gamma), C.byref(sc)))
        self.barrier()
        return self._view(name, n_out, t)

    def exchange_halos(self, first, last, left, right):
        """left <- last plane of rank-1, right <- first plane of rank+1 (cyclic),
        as peer copies into the neighbours' halo buffers (raw device pointers:
        the peers' buffers may live on other GPUs)."""
        n = first.numel()
        esz = first.element_size()
        slot = self._slot("halo", 2 * n * esz)
        prev, nxt = (self.rank - 1) % self.P, (self.rank + 1) % self.P
        lib, h = self.be.ctx.lib, self.be.ctx.h
        lastc, firstc = last.contiguous(), first.contiguous()
        self.be._sync_stream()
        # my last plane -> next rank's left halo (offset 0); first -> prev's right (offset n)
        self._check(lib.kp_copy(h, slot[2][nxt], lastc.data_ptr(), n * esz))
        self._check(lib.kp_copy(h, slot[2][prev] + n * esz, firstc.data_ptr(), n * esz))
        self.barrier()
        mine = self._view("halo", 2 * n, first)
        left.copy_(mine[:n].view(left.shape))
        right.copy_(mine[n:].view(right.shape))
        self.barrier()  # the halo buffer is free again


# ----------------------------------------------------------------- backends

class CudaBackend:
    """Local compute through the C ABI (the single-GPU kernels)."""

    def __init__(self, device=None):
        from . import _lib
        from ._lib import check, ints
        self.check, self.ints = check, ints
        dev = torch.cuda.current_device() if device is None else device
        self.ctx = _lib.default_context(dev)
        self.device = torch.device("cuda", dev)

    def _sync_stream(self):
        self.ctx.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def mode_product(self, t, dims, mode, m, alpha, beta, out):
        import ctypes as C
        self._sync_stream()
        lib = self.ctx.lib
        if torch.is_complex(t):
            a2 = (C.c_double * 2)(alpha, 0.0)
            b2 = (C.c_double * 2)(beta, 0.0)
            self.check(lib.kp_mode_product_c128(self.ctx.h, t.data_ptr(), self.ints(dims),
                                                len(dims), mode, m.data_ptr(), m.shape[0],
                                                m.shape[1], a2, b2, out.data_ptr()))
        else:
            self.check(lib.kp_mode_product_f64(self.ctx.h, t.data_ptr(), self.ints(dims),
                                               len(dims), mode, m.data_ptr(), m.shape[0],
                                               m.shape[1], float(alpha), float(beta),
                                               out.data_ptr()))

    def mark_nonfinite(self, x, bad, step):
        """atomicMin(bad, step) on the device if x has a non-finite entry."""
        self._sync_stream()
        n = x.numel() * (2 if torch.is_complex(x) else 1)
        self.check(self.ctx.lib.kp_mark_nonfinite_f64(self.ctx.h, n, x.data_ptr(),
                                                      bad.data_ptr(), int(step)))

    def mode_product_stage(self, t, dims, mode, m, alpha, x, gamma, g, out, d_out):
        """out = fma(gamma, alpha * (t x_mode m), x); d_out = g(out) - g(x) in the
        same epilogue (kp_mode_product_stage_*)."""
        import ctypes as C
        self._sync_stream()
        f = self.ctx.lib.kp_mode_product_stage_c128 if torch.is_complex(t) else \
            self.ctx.lib.kp_mode_product_stage_f64
        self.check(f(self.ctx.h, t.data_ptr(), self.ints(dims), len(dims), mode, m.data_ptr(),
                     m.shape[0], float(alpha), x.data_ptr(), float(gamma), C.byref(g), 0.0, 0.0,
                     out.data_ptr(), d_out.data_ptr()))

    def eval_g(self, g, u, dims, out):
        import ctypes as C
        self._sync_stream()
        f = self.ctx.lib.kp_eval_g_c128 if torch.is_complex(u) else self.ctx.lib.kp_eval_g_f64
        self.check(f(self.ctx.h, C.byref(g), 0.0, u.data_ptr(), self.ints(dims), len(dims),
                     out.data_ptr()))

    def kronsum_slab(self, u_ext, dims, K, slab_mode, k0, n_glob, g, out):
        """r = K u + g(u) on a slab with halo planes.  The factors' band
        structures are scanned once per factor set (kp_band_create, cached
        with a reference to the factor tensors) and every step calls
        kp_kronsum_slab_banded_*, which never syncs the host."""
        import ctypes as C
        self._sync_stream()
        cplx = torch.is_complex(u_ext)
        key = (cplx,) + tuple((k.data_ptr(), k.numel()) for k in K)
        cache = self.__dict__.setdefault("_bands", {})
        if key not in cache:
            hs = []
            for k in K:
                h = C.c_void_p()
                self.check(self.ctx.lib.kp_band_create(self.ctx.h, k.data_ptr(), k.shape[0],
                                                       int(cplx), C.byref(h)))
                hs.append(h)
            cache[key] = (list(K), hs, (C.c_void_p * len(hs))(*[h.value for h in hs]))
        _, _, arr = cache[key]
        f = self.ctx.lib.kp_kronsum_slab_banded_c128 if cplx else \
            self.ctx.lib.kp_kronsum_slab_banded_f64
        self.check(f(self.ctx.h, u_ext.data_ptr(), self.ints(dims), len(dims),
                     C.cast(arr, C.c_void_p), slab_mode, k0, n_glob,
                     C.cast(C.byref(g), C.c_void_p) if g is not None else None, out.data_ptr()))

    def release_bands(self):
        for _, hs, _ in self.__dict__.pop("_bands", {}).values():
            for h in hs:
                self.ctx.lib.kp_band_destroy(h)

    def fma(self, alpha, x, y, out):
        """out = fma(alpha, x, y) elementwise (componentwise for complex)."""
        self._sync_stream()
        n = x.numel() * (2 if torch.is_complex(x) else 1)
        self.check(self.ctx.lib.kp_add_scaled_f64(self.ctx.h, n, y.data_ptr(), float(alpha),
                                                  x.data_ptr(), out.data_ptr()))


# --------------------------------------------------------------- integrator

class ShardedIntegrator:
    """integrate() (inc/integrators.hpp:219-373) with the state slab-sharded
    along the last spatial mode.  `factors`: dict method-part -> list of
    (n x n) torch tensors on this rank's device, identical on every rank."""

    def __init__(self, backend, comm, method, spatial, species, K, g, tau, f1, pref1, f2=None,
                 pref2=1.0, fold1=1.0, fold2=1.0, K_all=None, banded=False):
        self.K_all = K_all if K_all is not None else K
        self.banded = banded
        self.be, self.comm = backend, comm
        self.method = method
        self.spatial = list(spatial)
        self.S = species
        self.K = K
        self.g = g
        self.tau = tau
        self.t0 = 0.0
        self.f1, self.f2 = f1, f2
        self.pref1, self.pref2 = pref1, pref2
        self.fold1, self.fold2 = fold1, fold2
        self.lay = Layout.of(self.spatial, species, comm.P)
        self.sd = self.lay.slab_dims(self.spatial, species)
        self.pd = self.lay.pencil_dims(self.spatial, species)
        self.d = len(self.spatial)

    @property
    def fused(self):
        return getattr(self.comm, "fused", False)

    def to_pencil(self, x, site):
        if self.fused:
            return self.comm.slab_to_pencil(x, self.lay, site)
        return slab_to_pencil(x, self.lay, self.comm)

    def to_slab(self, y, site):
        if self.fused:
            return self.comm.pencil_to_slab(y, self.lay, site)
        return pencil_to_slab(y, self.lay, self.comm)

    # y = ((pref x) x_1 F_1 ... x_d F_d) * fold ; x in slab layout, y in pencil
    # layout -- or, with `to_slab_x`, fma(gamma, y, x2) returned in slab layout
    # (the final update of a step, fused into the last GEMM's epilogue)
    def tucker(self, x, fs, pref, fold, site="t", final=None, stage=None):
        d = self.d
        cur, dims = x, self.sd
        for mu in range(d - 1):
            alpha = pref if mu == 0 else 1.0
            if self.fused and mu == d - 2:
                # GEMM + slab -> pencil exchange in one kernel
                cp = self.comm.mode_product_to(cur, dims, mu, fs[mu], alpha, self.lay, 1, site)
                break
            out = torch.empty_like(cur)
            self.be.mode_product(cur, dims, mu, fs[mu], alpha, 0.0, out)
            cur = out
        else:
            cp = None
        if cp is None:
            cp = slab_to_pencil(cur, self.lay, self.comm) if not self.fused else \
                self.comm.slab_to_pencil(cur, self.lay, site)
        alpha = (pref if d == 1 else 1.0) * fold
        if final is not None:
            x2, gamma, fsite = final
            if self.fused:  # last mode + fma + pencil -> slab exchange in one kernel
                return self.comm.mode_product_to(cp, self.pd, d - 1, fs[d - 1], alpha, self.lay,
                                                 2, fsite, x=x2, gamma=gamma)
            y = torch.empty_like(cp)
            self.be.mode_product(cp, self.pd, d - 1, fs[d - 1], alpha, 0.0, y)
            out = torch.empty_like(y)
            if x2 is None:
                out = y
            else:
                self.be.fma(gamma, y, x2, out)
            return pencil_to_slab(out, self.lay, self.comm)
        out = torch.empty_like(cp)
        if stage is not None:  # (stage, g(stage) - g(x2)), both pencil layout
            x2, gamma = stage
            dp = torch.empty_like(cp)
            self.be.mode_product_stage(cp, self.pd, d - 1, fs[d - 1], alpha, x2, gamma, self.g,
                                       out, dp)
            return out, dp
        self.be.mode_product(cp, self.pd, d - 1, fs[d - 1], alpha, 0.0, out)
        return out  # pencil layout

    # r = K u + g(u); u in slab layout (and u_p = its pencil copy); r in pencil layout
    def kronsum_g(self, u, u_p):
        d = self.d
        r = torch.empty_like(u)
        for mu in range(d - 1):
            self.be.mode_product(u, self.sd, mu, self.K[mu], 1.0, 0.0 if mu == 0 else 1.0, r)
        r_p = self.to_pencil(r, "kr") if d > 1 else r
        self.be.mode_product(u_p, self.pd, d - 1, self.K[d - 1], 1.0, 1.0 if d > 1 else 0.0, r_p)
        gu = torch.empty_like(u_p)
        self.be.eval_g(self.g, u_p, self.pd, gu)
        return r_p + gu  # exact IEEE add, as the fused EPI_ADD_G

    def kronsum_g_banded(self, u):
        """r = K u + g(u) in slab layout: banded stencil with a one-plane
        halo exchange instead of transposes (banded.cu, same rounding as the
        single-GPU path)."""
        ext = halo_extend(u, self.lay, self.comm)
        r = torch.empty_like(u)
        k0 = self.comm.rank * (self.spatial[-1] // self.comm.P)
        self.be.kronsum_slab(ext, self.sd, self.K_all, self.d - 1, k0, self.spatial[-1], self.g,
                             r)
        return r

    def step(self, u):
        """u (slab) -> u' (slab)."""
        tau = self.tau
        m = self.method
        if m in ("exp_euler", "etd2rk"):
            u_p = self.to_pencil(u, "u_p")
            if self.banded:
                r = self.kronsum_g_banded(u)
            else:
                r_p = self.kronsum_g(u, u_p)
                r = self.to_slab(r_p, "r")
            if m == "exp_euler":  # u + tau*SP1(r), back in slab layout
                return self.tucker(r, self.f1, self.pref1, self.fold1, "t1",
                                   final=(u_p, tau, "u"))
            if hasattr(self.be, "mode_product_stage"):
                # stage = u + tau*SP1(r) and g(stage) - g(u) in the last GEMM's epilogue
                stage, dp = self.tucker(r, self.f1, self.pref1, self.fold1, "t1",
                                        stage=(u_p, tau))
                dd = self.to_slab(dp, "dd")
            else:
                y1 = self.tucker(r, self.f1, self.pref1, self.fold1, "t1")   # pencil
                stage = torch.empty_like(y1)
                self.be.fma(tau, y1, u_p, stage)                              # u + tau*SP1(r)
                gs, gu = torch.empty_like(stage), torch.empty_like(stage)
                self.be.eval_g(self.g, stage, self.pd, gs)
                self.be.eval_g(self.g, u_p, self.pd, gu)
                dd = self.to_slab(gs - gu, "dd")
            # stage + tau*SP2(d), back in slab layout
            return self.tucker(dd, self.f2, self.pref2, self.fold2, "t2", final=(stage, tau, "u"))
        if m in ("lawson_euler", "lawson2b"):
            gn = torch.empty_like(u)
            self.be.eval_g(self.g, u, self.sd, gn)
            w = torch.empty_like(u)
            self.be.fma(tau, gn, u, w)
            if m == "lawson_euler":
                return self.tucker(w, self.f1, 1.0, self.fold1, "t1", final=(None, 0.0, "u"))
            stage = self.tucker(w, self.f1, 1.0, self.fold1, "t1")
            w2 = torch.empty_like(u)
            self.be.fma(0.5 * tau, gn, u, w2)
            out = self.tucker(w2, self.f1, 1.0, self.fold1, "t2")
            gs = torch.empty_like(stage)
            self.be.eval_g(self.g, stage, self.pd, gs)
            res = torch.empty_like(out)
            self.be.fma(0.5 * tau, gs, out, res)
            return self.to_slab(res, "u")
        raise ValueError(f"sharded integrate: unsupported method {m}")

    def run(self, u, n_steps):
        """n_steps steps; like the single-GPU loop it runs to the end and then
        reports the first non-finite step (DivergenceError(step))."""
        first_bad = 0
        mark = getattr(self.be, "mark_nonfinite", None)
        if mark is not None:  # device flag, no host sync per step
            big = 2 ** 31 - 1
            bad = torch.full((1,), big, dtype=torch.int32, device=u.device)
            for k in range(n_steps):
                u = self.step(u)
                mark(u, bad, k + 1)
            if self.comm.P > 1:  # first bad step over ranks
                vals = bad.to(torch.float64)
                dist.all_reduce(vals, op=dist.ReduceOp.MIN)
                bad.copy_(vals.to(torch.int32))
            b = int(bad.item())
            first_bad = 0 if b == big else b
        else:
            flag = torch.zeros(1, dtype=torch.float64, device=u.device)
            for k in range(n_steps):
                u = self.step(u)
                if not first_bad:
                    flag.fill_(0.0 if bool(torch.isfinite(u).all()) else float(k + 1))
                    if self.comm.P > 1:
                        # first bad step over ranks: any rank's nonzero flag, smallest k
                        vals = torch.where(flag > 0, flag, torch.full_like(flag, 1e300))
                        dist.all_reduce(vals, op=dist.ReduceOp.MIN)
                        flag.copy_(torch.where(vals < 1e299, vals, torch.zeros_like(vals)))
                    first_bad = int(flag.item())
        if self.fused:
            u = u.clone()  # the result lives in an exchange buffer
        if first_bad:
            from ._lib import DivergenceError
            raise DivergenceError(3, f"state became non-finite at step {first_bad} "
                                     f"(t = {self.t0 + first_bad * self.tau:f})", first_bad)
        return u


# ------------------------------------------------------------ factor set-up

def split_factors(kp, K, tau, ell):
    """Device build of phi_ell(tau A_mu) (build_split_phi) and the scalar
    folding of factors that are exactly c*I (the stacked species mode)."""
    sp = kp.build_split_phi(K, tau, ell)
    fs, fold, active = [], 1.0, []
    for f in sp.factors:
        h = kp.to_host(f) if hasattr(f, "is_cuda") else np.asarray(f)
        n = h.shape[0]
        if n <= 64 and np.array_equal(h, h[0, 0] * np.eye(n)):
            fold *= float(np.real(h[0, 0]))
            active.append(False)
        else:
            active.append(True)
        fs.append(f)
    return fs, sp.prefactor, fold, active


def local_slab(x_global, P, rank, species):
    """The rank's slab of a global column-major tensor (torch or numpy)."""
    if species > 1:
        n = x_global.shape[-2] // P
        return x_global[..., rank * n:(rank + 1) * n, :]
    n = x_global.shape[-1] // P
    return x_global[..., rank * n:(rank + 1) * n]


def make_sharded_integrator(kp, backend, comm, method, dims_local, K, g, t0, t_final,
                            n_steps):
    """Factor set-up (on every rank, single-GPU device builder) for a slab-
    sharded integrate.  dims_local: this rank's slab dims (the last spatial
    mode holds n_d/P planes; a stacked Brusselator keeps its species mode
    last).  K = all factors as the reference takes them (including the zero
    2x2 species factor)."""
    tau = (t_final - t0) / float(n_steps)
    # the sharded kernels evaluate g at slab-local indices with no step clock:
    # time-dependent or nonlocal g's (ADR, Riccati) would be silently wrong
    kind = getattr(g, "kind", None)
    if kind in (getattr(kp, "G_ADR", -1), getattr(kp, "G_RICCATI", -1)):
        raise kp.InvalidArgument(1, "sharded integrate: the ADR and Riccati g's are not "
                                    "supported (time-dependent / nonlocal)")
    k_last = kp.to_host(K[-1])
    species = 2 if (len(K) >= 2 and k_last.shape[0] == 2 and not np.any(k_last)) else 1
    spatial_K = list(K[:-1]) if species == 2 else list(K)
    d = len(spatial_K)
    spatial = list(dims_local[:d])
    spatial[-1] *= comm.P
    f2, p2, fold2 = None, 1.0, 1.0
    if method in ("lawson_euler", "lawson2b"):
        f1, p1, fold1, _ = split_factors(kp, K, tau, 0)
    elif method == "exp_euler":
        f1, p1, fold1, _ = split_factors(kp, K, tau, 1)
    elif method == "etd2rk":
        f1, p1, fold1, _ = split_factors(kp, K, tau, 1)
        f2, p2, fold2, _ = split_factors(kp, K, tau, 2)
    else:
        raise ValueError(f"sharded integrate: unsupported method {method}")
    banded = hasattr(backend, "kronsum_slab") and banded_kronsum_enabled() and \
        all(_is_banded(kp.to_host(k)) for k in K)
    it = ShardedIntegrator(backend, comm, method, spatial, species, spatial_K, g, tau,
                           f1[:d], p1, f2[:d] if f2 else None, p2, fold1, fold2,
                           K_all=list(K), banded=banded)
    it.t0 = t0
    return it


def banded_kronsum_enabled():
    import os
    return os.environ.get("KP_KRONSUM", "") != "dense"


def _is_banded(a):
    """At most three nonzeros per row (the stencil form of banded.cu)."""
    return bool(np.all(np.count_nonzero(np.asarray(a), axis=1) <= 3))


def sharded_integrate(kp, backend, comm, method, u_local, dims_local, K, g, t0, t_final,
                      n_steps):
    """Slab-sharded integrate of this rank's slab (a FLAT torch tensor in
    column-major order with local dims `dims_local`); returns the final slab."""
    it = make_sharded_integrator(kp, backend, comm, method, dims_local, K, g, t0, t_final,
                                 n_steps)
    try:
        return it.run(u_local, n_steps)
    finally:
        rel = getattr(backend, "release_bands", None)
        if rel is not None:
            rel()


# ------------------------------------------- the native sharded integrator

MODE_D = {"auto": 0, "alltoall": 1, "reduce_scatter": 2, "fused": 3}


def native_sharded_integrate(kp, method, u_slabs, dims_local, K, g, t0, t_final, n_steps,
                             comm=None, mode_d="alltoall", q=12):
    """The C++ slab-sharded integrator (stepper.cu ShardedIntegrator,
    kp_integrate_sharded_*).  u_slabs: list of this process's slabs (flat or
    shaped CUDA tensors, column-major data, updated in place) -- one slab
    with `comm` (a NcclComm over the job's ranks), or all P slabs with
    comm=None (the P ranks emulated in this process on one GPU).  K: the full
    factors (device tensors).  Returns (mode_used, loop_seconds); raises
    DivergenceError like integrate()."""
    import ctypes as C
    from ._lib import check, ints, ptr_array
    from .integrators import _upload_factors, parse_method
    cplx = torch.is_complex(u_slabs[0])
    ctx = kp.default_context(u_slabs[0].device.index or 0)
    fs = _upload_factors(K)
    fs = [f.to(torch.complex128 if cplx else torch.float64) for f in fs]
    m = parse_method(method) if isinstance(method, str) else int(method)
    used = C.c_int(0)
    dv = C.c_long(0)
    loop = C.c_double(0.0)
    md = MODE_D.get(mode_d, mode_d)
    torch.cuda.current_stream(u_slabs[0].device).synchronize()
    if comm is not None:
        f = ctx.lib.kp_integrate_sharded_c128 if cplx else ctx.lib.kp_integrate_sharded_f64
        rc = f(ctx.h, comm.h, int(m), u_slabs[0].data_ptr(), ints(dims_local), len(dims_local),
               ptr_array([x.data_ptr() for x in fs]), C.byref(g), float(t0), float(t_final),
               int(n_steps), int(q), int(md), C.byref(used), C.byref(dv), C.byref(loop))
    else:
        f = ctx.lib.kp_integrate_sharded_local_c128 if cplx else \
            ctx.lib.kp_integrate_sharded_local_f64
        arr = (C.c_void_p * len(u_slabs))(*[x.data_ptr() for x in u_slabs])
        rc = f(ctx.h, len(u_slabs), int(m), C.cast(arr, C.c_void_p), ints(dims_local),
               len(dims_local), ptr_array([x.data_ptr() for x in fs]), C.byref(g), float(t0),
               float(t_final), int(n_steps), int(q), int(md), C.byref(used), C.byref(dv),
               C.byref(loop))
    try:
        check(rc, step=dv.value)
    except Exception as e:
        e.loop_s = loop.value
        raise
    return used.value, loop.value
