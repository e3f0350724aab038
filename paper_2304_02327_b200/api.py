"""Python mirror of the reference's hot-path API (inc/mode_product.hpp,
inc/split_phi.hpp, inc/matrix_functions.hpp, inc/integrators.hpp) on top of
the C ABI.

Arrays follow the reference's storage convention: column-major, first index
fastest (inc/tensor.hpp:1-2).  Two kinds of operands are accepted:

* numpy arrays (host): Fortran-ordered float64/complex128.  Calls go through
  the ``kp_host_*`` entry points: H2D, device compute, D2H -- the drop-in path.
* torch CUDA tensors (device): float64/complex128 with column-major strides
  (see :func:`fortran_empty`); calls are stream-ordered on torch's current
  stream and never leave the device.

Errors raise the reference's exception taxonomy: :class:`InvalidArgument`
(std::invalid_argument, with the reference's messages), :class:`KronphiError`
(std::runtime_error) and :class:`DivergenceError`.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _lib
from ._lib import (DivergenceError, InvalidArgument, KronphiError, check, default_context, ints,
                   ptr_array)

try:  # torch is plumbing for device memory/streams only
    import torch
except Exception:  # pragma: no cover
    torch = None


# ---------------------------------------------------------------- helpers

def _is_torch(x):
    return torch is not None and isinstance(x, torch.Tensor)


def _is_cplx(x):
    if _is_torch(x):
        return x.dtype == torch.complex128
    return np.iscomplexobj(x)


def fortran_empty(dims, dtype=None, device="cuda"):
    """Uninitialised torch tensor of shape ``dims`` with column-major strides."""
    dtype = dtype or torch.float64
    base = torch.empty(tuple(reversed([int(d) for d in dims])), dtype=dtype, device=device)
    return base.permute(*reversed(range(len(dims))))


def fortran_zeros(dims, dtype=None, device="cuda"):
    t = fortran_empty(dims, dtype, device)
    t.zero_()
    return t


def to_device(a, device="cuda"):
    """numpy (any order) -> column-major torch CUDA tensor."""
    a = np.asarray(a)
    dt = torch.complex128 if np.iscomplexobj(a) else torch.float64
    t = fortran_empty(a.shape, dt, device)
    t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return t


def to_host(t):
    return np.asfortranarray(t.detach().cpu().numpy())


def _check_fortran_torch(t, what):
    if not t.is_cuda:
        raise InvalidArgument(1, f"{what}: torch tensors must live on a CUDA device")
    if t.dtype not in (torch.float64, torch.complex128):
        raise InvalidArgument(1, f"{what}: dtype must be float64 or complex128")
    exp = 1
    for dim, st in zip(t.shape, t.stride()):
        if dim > 1 and st != exp:
            raise InvalidArgument(1, f"{what}: tensor must be column-major (first index fastest)")
        exp *= dim


def _host(a, cplx):
    a = np.asarray(a)
    if a.ndim == 0:
        raise InvalidArgument(1, "Tensor: empty dims")
    return np.asfortranarray(a, dtype=np.complex128 if cplx else np.float64)


def _ctx_for(t):
    ctx = default_context(t.device.index if _is_torch(t) and t.device.index is not None else 0)
    if _is_torch(t):
        ctx.set_stream(torch.cuda.current_stream(t.device).cuda_stream)
    return ctx


def _dims(x):
    return list(x.shape)


# ------------------------------------------------------- Kronecker sum type

class KroneckerSum:
    """Ordered factor list [A_1..A_d] for A_d (+) ... (+) A_1, never assembled
    (inc/mode_product.hpp:21-41)."""

    def __init__(self, factors):
        factors = list(factors)
        if not factors:
            raise InvalidArgument(1, "KroneckerSum: needs at least one factor")
        for mu, f in enumerate(factors):
            if f.ndim != 2 or f.shape[0] != f.shape[1]:
                raise InvalidArgument(1, f"KroneckerSum: factor {mu} is not square")
        self.factors = factors

    def order(self):
        return len(self.factors)

    def dims(self):
        return [int(f.shape[0]) for f in self.factors]


# ---------------------------------------------------------- mode products

def mode_product_into(t, m, mode, out, accumulate=False):
    """out (+)= t x_mode m  (inc/mode_product.hpp:61-87)."""
    cplx = _is_cplx(t) or _is_cplx(m)
    if _is_torch(t):
        for x, w in ((t, "mode_product"), (m, "mode_product"), (out, "mode_product")):
            _check_fortran_torch(x, w)
        ctx = _ctx_for(t)
        if cplx:
            one = (C.c_double * 2)(1.0, 0.0)
            beta = (C.c_double * 2)(1.0 if accumulate else 0.0, 0.0)
            check(ctx.lib.kp_mode_product_c128(ctx.h, t.data_ptr(), ints(_dims(t)), t.ndim, mode,
                                               m.data_ptr(), m.shape[0], m.shape[1], one, beta,
                                               out.data_ptr()))
        else:
            check(ctx.lib.kp_mode_product_f64(ctx.h, t.data_ptr(), ints(_dims(t)), t.ndim, mode,
                                              m.data_ptr(), m.shape[0], m.shape[1], 1.0,
                                              1.0 if accumulate else 0.0, out.data_ptr()))
        return out
    if cplx:
        # host complex: route through the device tensors
        td, md = to_device(t), to_device(m)
        od = to_device(out) if accumulate else fortran_zeros(out.shape, torch.complex128)
        mode_product_into(td, md, mode, od, accumulate)
        out[...] = to_host(od)
        return out
    th, mh = _host(t, False), _host(m, False)
    if not (isinstance(out, np.ndarray) and out.flags.f_contiguous and out.dtype == np.float64):
        raise InvalidArgument(1, "mode_product_into: out must be a Fortran-ordered float64 array")
    ctx = default_context(0)
    check(ctx.lib.kp_host_mode_product_f64(ctx.h, th.ctypes.data, ints(th.shape), th.ndim, mode,
                                           mh.ctypes.data, mh.shape[0], mh.shape[1], 1.0,
                                           1.0 if accumulate else 0.0, out.ctypes.data))
    return out


def _check_mode(dims, mode, cols):
    if mode < 0 or mode >= len(dims):
        raise InvalidArgument(1, f"mode_product: mode {mode} out of range for order {len(dims)}")
    if cols != dims[mode]:
        raise InvalidArgument(1, f"mode_product: size mismatch on mode {mode}: matrix has {cols} "
                                 f"columns, tensor dim is {dims[mode]}")


def mode_product(t, m, mode):
    """t x_mode m as a new tensor (inc/mode_product.hpp:89-97)."""
    dims = _dims(t)
    _check_mode(dims, mode, m.shape[1])
    od = dims.copy()
    od[mode] = m.shape[0]
    cplx = _is_cplx(t) or _is_cplx(m)
    if _is_torch(t):
        out = fortran_empty(od, torch.complex128 if cplx else torch.float64, t.device)
    else:
        out = np.zeros(od, order="F", dtype=np.complex128 if cplx else np.float64)
    return mode_product_into(t, m, mode, out)


def _tucker(t, ms, prefactor):
    cplx = _is_cplx(t) or any(_is_cplx(m) for m in ms)
    rows = [int(m.shape[0]) for m in ms]
    dims = _dims(t)
    if _is_torch(t):
        dt = torch.complex128 if cplx else torch.float64
        t = t.to(dt) if t.dtype != dt else t
        ms = [m.to(dt) if m.dtype != dt else m for m in ms]
        for x in [t] + ms:
            _check_fortran_torch(x, "tucker")
        ctx = _ctx_for(t)
        out = fortran_empty(rows, dt, t.device)
        f = ctx.lib.kp_tucker_c128 if cplx else ctx.lib.kp_tucker_f64
        check(f(ctx.h, t.data_ptr(), ints(dims), len(dims), ptr_array([m.data_ptr() for m in ms]),
                ints(rows), float(prefactor), out.data_ptr()))
        return out
    th = _host(t, cplx)
    mh = [_host(m, cplx) for m in ms]
    out = np.zeros(rows, order="F", dtype=th.dtype)
    ctx = default_context(0)
    f = ctx.lib.kp_host_tucker_c128 if cplx else ctx.lib.kp_host_tucker_f64
    check(f(ctx.h, th.ctypes.data, ints(dims), len(dims), ptr_array([m.ctypes.data for m in mh]),
            ints(rows), float(prefactor), out.ctypes.data))
    return out


def tucker(t, ms: Sequence):
    """t x_1 ms[0] x_2 ... x_d ms[d-1] (inc/mode_product.hpp:101-108)."""
    ms = list(ms)
    if len(ms) != t.ndim:
        raise InvalidArgument(1, "tucker: expected one factor per mode")
    for mu, m in enumerate(ms):
        _check_mode(_dims(t), mu, m.shape[1])
    return _tucker(t, ms, 1.0)


def kronsum_action(t, k):
    """sum_mu t x_mu A_mu (inc/mode_product.hpp:111-121)."""
    if not isinstance(k, KroneckerSum):
        k = KroneckerSum(k)
    if k.order() != t.ndim:
        raise InvalidArgument(1, "kronsum_action: expected one factor per mode")
    dims = _dims(t)
    for mu, a in enumerate(k.factors):
        _check_mode(dims, mu, a.shape[1])
    cplx = _is_cplx(t) or any(_is_cplx(a) for a in k.factors)
    if _is_torch(t):
        dt = torch.complex128 if cplx else torch.float64
        t = t.to(dt) if t.dtype != dt else t
        fs = [a.to(dt) if a.dtype != dt else a for a in k.factors]
        for x in [t] + fs:
            _check_fortran_torch(x, "kronsum_action")
        ctx = _ctx_for(t)
        out = fortran_empty(dims, dt, t.device)
        f = ctx.lib.kp_kronsum_c128 if cplx else ctx.lib.kp_kronsum_f64
        check(f(ctx.h, t.data_ptr(), ints(dims), len(dims), ptr_array([a.data_ptr() for a in fs]),
                out.data_ptr()))
        return out
    if cplx:
        return to_host(kronsum_action(to_device(t), KroneckerSum([to_device(a) for a in k.factors])))
    th = _host(t, False)
    fs = [_host(a, False) for a in k.factors]
    out = np.zeros(dims, order="F")
    ctx = default_context(0)
    check(ctx.lib.kp_host_kronsum_f64(ctx.h, th.ctypes.data, ints(dims), len(dims),
                                      ptr_array([a.ctypes.data for a in fs]), out.ctypes.data))
    return out
