"""ctypes binding of libkronphi_b200.so (the C ABI in include/kronphi_b200.h).

The shared library is built in-tree by ``make -C paper_2304_02327_b200``
(``__graft_entry__.build()``).  There is no fallback: if the library or a
CUDA device is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# KP_LIB: another build of the same library (A/B measurements of two builds
# on one GPU box); the default is the in-tree build
LIB_PATH = os.environ.get("KP_LIB") or os.path.join(HERE, "lib", "libkronphi_b200.so")

KP_OK, KP_EINVAL, KP_ERUNTIME, KP_EDIVERGE, KP_ECUDA = range(5)
LAWSON_EULER, LAWSON2B, EXP_EULER, EXP_EULER_LS, ETD2RK = range(5)
G_ZERO, G_SQUARE, G_CONST, G_ALLEN_CAHN, G_BRUSSELATOR, G_NLS, G_ADR, G_RICCATI = range(8)


class KronphiError(RuntimeError):
    """Base class; ``code`` is the kp status code."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(KronphiError, ValueError):
    """std::invalid_argument in the reference (sizing/validation errors)."""


class CudaError(KronphiError):
    pass


class DivergenceError(KronphiError):
    """kronphi::DivergenceError (inc/integrators.hpp:86-97)."""

    def __init__(self, code, msg, step=0):
        super().__init__(code, msg)
        self.step = step


class GFun(C.Structure):
    """kp_gfun (include/kronphi_b200.h): nonlinearity id, parameters, device
    auxiliary fields (ADR) and the integrators' step-counter time hook."""
    _fields_ = [("kind", C.c_int), ("p", C.c_double * 4), ("aux", C.c_void_p * 2),
                ("step_ctr", C.c_void_p), ("t0", C.c_double), ("tau", C.c_double)]


class Scatter(C.Structure):
    """kp_scatter (include/kronphi_b200.h): the slab <-> pencil destination
    map of the fused exchange and the peer receive buffers."""
    _fields_ = [("dir", C.c_int), ("P", C.c_int), ("rank", C.c_int), ("A", C.c_longlong),
                ("B", C.c_longlong), ("C", C.c_longlong), ("S", C.c_longlong),
                ("peers", C.c_void_p)]


_D, _I, _L, _SZ = C.c_double, C.c_int, C.c_long, C.c_size_t
_PD, _PI, _VP = C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_void_p
_PPD = C.POINTER(C.POINTER(C.c_double))
_CTX = C.c_void_p

_SIGS = {
    "kp_last_error": (C.c_char_p, []),
    "kp_ctx_create": (_I, [_I, C.POINTER(_CTX)]),
    "kp_ctx_destroy": (_I, [_CTX]),
    "kp_ctx_set_stream": (_I, [_CTX, _VP]),
    "kp_ctx_use_own_stream": (_I, [_CTX]),
    "kp_ctx_get_stream": (_VP, [_CTX]),
    "kp_ctx_synchronize": (_I, [_CTX]),
    "kp_ctx_launch_count": (C.c_ulonglong, [_CTX]),
    "kp_malloc": (_I, [_CTX, _SZ, C.POINTER(_VP)]),
    "kp_mode_product_scatter_f64": (_I, [_CTX, _VP, _PI, _I, _I, _VP, _I, _D, _VP, _D,
                                         C.POINTER(Scatter)]),
    "kp_mode_product_scatter_c128": (_I, [_CTX, _VP, _PI, _I, _I, _VP, _I, _D, _VP, _D,
                                          C.POINTER(Scatter)]),
    "kp_scatter_copy": (_I, [_CTX, _VP, C.c_longlong, _I, C.POINTER(Scatter)]),
    "kp_ipc_get_handle": (_I, [_VP, _VP]),
    "kp_ipc_open_handle": (_I, [_VP, C.POINTER(_VP)]),
    "kp_ipc_close_handle": (_I, [_VP]),
    "kp_mode_product_stage_f64": (_I, [_CTX, _VP, _PI, _I, _I, _VP, _I, _D, _VP, _D, _VP, _D,
                                       _D, _VP, _VP]),
    "kp_mode_product_stage_c128": (_I, [_CTX, _VP, _PI, _I, _I, _VP, _I, _D, _VP, _D, _VP, _D,
                                        _D, _VP, _VP]),
    "kp_gemm_f64": (_I, [_CTX, _I, _I, _I, _D, _VP, _I, _VP, _I, _I, _D, _VP, _I]),
    "kp_gemm_c128": (_I, [_CTX, _I, _I, _I, _VP, _VP, _I, _VP, _I, _I, _VP, _VP, _I]),
    "kp_gemm_batch_shared_b_f64": (_I, [_CTX, _I, _I, _I, _D, _VP, _I, C.c_longlong, _VP, _I, _I,
                                        _D, _VP, _I, C.c_longlong, _I]),
    "kp_gemm_batch_shared_b_c128": (_I, [_CTX, _I, _I, _I, _VP, _VP, _I, C.c_longlong, _VP, _I,
                                         _I, _VP, _VP, _I, C.c_longlong, _I]),
    "kp_lu_factor_f64": (_I, [_CTX, _VP, _I, _VP]),
    "kp_lu_solve_f64": (_I, [_CTX, _VP, _VP, _I, _VP, _I]),
    "kp_band_create": (_I, [_CTX, _VP, _I, _I, C.POINTER(_VP)]),
    "kp_band_destroy": (_I, [_VP]),
    "kp_kronsum_slab_banded_f64": (_I, [_CTX, _VP, _PI, _I, _VP, _I, _I, _I, C.c_void_p, _VP]),
    "kp_kronsum_slab_banded_c128": (_I, [_CTX, _VP, _PI, _I, _VP, _I, _I, _I, C.c_void_p, _VP]),
    "kp_comm_unique_id": (_I, [_VP]),
    "kp_comm_create": (_I, [_CTX, _I, _I, _VP, C.POINTER(_VP)]),
    "kp_comm_destroy": (_I, [_VP]),
    "kp_comm_alltoall_f64": (_I, [_CTX, _VP, _VP, _VP, C.c_longlong]),
    "kp_comm_repartition": (_I, [_CTX, _VP, _I, C.c_longlong, C.c_longlong, C.c_longlong,
                                 C.c_longlong, _I, _VP, _VP]),
    "kp_repartition_pack": (_I, [_CTX, _I, _I, _I, C.c_longlong, C.c_longlong, C.c_longlong,
                                 C.c_longlong, _I, _VP, _VP]),
    "kp_repartition_unpack": (_I, [_CTX, _I, _I, _I, C.c_longlong, C.c_longlong, C.c_longlong,
                                   C.c_longlong, _I, _VP, _VP]),
    "kp_comm_halo_f64": (_I, [_CTX, _VP, _VP, _VP, C.c_longlong, _VP, _VP]),
    "kp_free": (_I, [_CTX, _VP]),
    "kp_upload": (_I, [_CTX, _VP, _VP, _SZ]),
    "kp_download": (_I, [_CTX, _VP, _VP, _SZ]),
    "kp_memset": (_I, [_CTX, _VP, _I, _SZ]),
    "kp_copy": (_I, [_CTX, _VP, _VP, _SZ]),
    "kp_mode_product_f64": (_I, [_CTX, _VP, _PI, _I, _I, _VP, _I, _I, _D, _D, _VP]),
    "kp_mode_product_c128": (_I, [_CTX, _VP, _PI, _I, _I, _VP, _I, _I, _PD, _PD, _VP]),
    "kp_tucker_f64": (_I, [_CTX, _VP, _PI, _I, _PPD, _PI, _D, _VP]),
    "kp_tucker_c128": (_I, [_CTX, _VP, _PI, _I, _PPD, _PI, _D, _VP]),
    "kp_kronsum_f64": (_I, [_CTX, _VP, _PI, _I, _PPD, _VP]),
    "kp_kronsum_c128": (_I, [_CTX, _VP, _PI, _I, _PPD, _VP]),
    "kp_kronsum_slab_f64": (_I, [_CTX, _VP, _PI, _I, _PPD, _I, _I, _I, C.c_void_p, _VP]),
    "kp_kronsum_slab_c128": (_I, [_CTX, _VP, _PI, _I, _PPD, _I, _I, _I, C.c_void_p, _VP]),
    "kp_host_mode_product_f64": (_I, [_CTX, _VP, _PI, _I, _I, _VP, _I, _I, _D, _D, _VP]),
    "kp_host_tucker_f64": (_I, [_CTX, _VP, _PI, _I, _PPD, _PI, _D, _VP]),
    "kp_host_tucker_stream_f64": (_I, [_CTX, _I, _VP, _PI, _I, _PPD, _PI, _D, _VP]),
    "kp_host_tucker_c128": (_I, [_CTX, _VP, _PI, _I, _PPD, _PI, _D, _VP]),
    "kp_host_kronsum_f64": (_I, [_CTX, _VP, _PI, _I, _PPD, _VP]),
    "kp_axpy_f64": (_I, [_CTX, _SZ, _D, _VP, _VP]),
    "kp_add_scaled_f64": (_I, [_CTX, _SZ, _VP, _D, _VP, _VP]),
    "kp_eval_g_f64": (_I, [_CTX, C.POINTER(GFun), _D, _VP, _PI, _I, _VP]),
    "kp_eval_g_c128": (_I, [_CTX, C.POINTER(GFun), _D, _VP, _PI, _I, _VP]),
    "kp_riccati_jacobian_factors_f64": (_I, [_CTX, C.POINTER(GFun), _VP, _VP, _I, _VP, _VP, _PI]),
    "kp_all_finite_f64": (_I, [_CTX, _SZ, _VP, _PI]),
    "kp_mark_nonfinite_f64": (_I, [_CTX, _SZ, _VP, _VP, _I]),
    "kp_measure_fp64_peak": (_I, [_CTX, _PD]),
}

# Every symbol include/kronphi_b200.h declares (checked by tests/test_abi.py).
EXPORTS = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load():
    """Load the shared library (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} not built; run `make -C {HERE}` or __graft_entry__.build()")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            for extra in _EXTRA_SIGS:
                name, res, args = extra
                if hasattr(lib, name):
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
            _lib = lib
        return _lib


_EXTRA_SIGS = []


def register(name, res, args):
    """Register the signature of an additional entry point (used by modules
    that bind later-added parts of the ABI)."""
    _EXTRA_SIGS.append((name, res, args))
    if _lib is not None and hasattr(_lib, name):
        fn = getattr(_lib, name)
        fn.restype = res
        fn.argtypes = args


def check(rc, step=0):
    if rc == KP_OK:
        return
    msg = load().kp_last_error().decode(errors="replace")
    if rc == KP_EINVAL:
        raise InvalidArgument(rc, msg)
    if rc == KP_EDIVERGE:
        raise DivergenceError(rc, msg, step)
    if rc == KP_ECUDA:
        raise CudaError(rc, msg)
    raise KronphiError(rc, msg)


def ints(xs):
    xs = [int(x) for x in xs]
    return (C.c_int * len(xs))(*xs)


def ptr_array(ptrs):
    return (C.POINTER(C.c_double) * len(ptrs))(*[C.cast(C.c_void_p(int(p)), _PD) for p in ptrs])


class Context:
    """Owns a kp_ctx (device, stream, workspace).  One per device per thread
    of use; not thread-safe (see include/kronphi_b200.h)."""

    def __init__(self, device=0):
        self.lib = load()
        h = _CTX()
        check(self.lib.kp_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = int(device)

    def close(self):
        if getattr(self, "h", None):
            self.lib.kp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle):
        check(self.lib.kp_ctx_set_stream(self.h, stream_handle))

    def synchronize(self):
        check(self.lib.kp_ctx_synchronize(self.h))

    @property
    def launches(self):
        return int(self.lib.kp_ctx_launch_count(self.h))

    def fp64_peak_tflops(self):
        v = C.c_double(0)
        check(self.lib.kp_measure_fp64_peak(self.h, C.byref(v)))
        return v.value


_ctxs = {}


def default_context(device=0):
    c = _ctxs.get(device)
    if c is None:
        c = Context(device)
        _ctxs[device] = c
    return c
