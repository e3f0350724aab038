"""Matrix functions, direction splitting and the exponential integrators --
Python mirror of inc/matrix_functions.hpp, inc/split_phi.hpp and
inc/integrators.hpp on the device library.

Operands follow api.py: numpy arrays take the host drop-in path (upload,
compute on the GPU, download); torch CUDA tensors stay on the device.
The nonlinearity g is one of the closed set of device g's (:func:`gfun`);
the reference's arbitrary host std::function has no device equivalent.
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import GFun, InvalidArgument, DivergenceError, check, default_context, ints, ptr_array
from .api import (KroneckerSum, _check_fortran_torch, _ctx_for, _is_cplx, _is_torch,
                  fortran_empty, to_device, to_host)

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

_D, _I, _L, _PD, _PI, _VP, _PPD = (C.c_double, C.c_int, C.c_long, C.POINTER(C.c_double),
                                   C.POINTER(C.c_int), C.c_void_p,
                                   C.POINTER(C.POINTER(C.c_double)))
_CTX, _PG, _PL = C.c_void_p, C.POINTER(GFun), C.POINTER(C.c_long)
# kp_sample_fn: (user, step, u_host) -- the trajectory hook of kp_integrate_sampled_*
SAMPLE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_long, C.POINTER(C.c_double))
for _name, _res, _args in [
    # the native slab-sharded integrator (stepper.cu; parallel.native_sharded_integrate)
    ("kp_integrate_sharded_f64", _I, [_CTX, _VP, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L, _I,
                                      _I, _PI, _PL, _PD]),
    ("kp_integrate_sharded_c128", _I, [_CTX, _VP, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L, _I,
                                       _I, _PI, _PL, _PD]),
    ("kp_integrate_sharded_local_f64", _I, [_CTX, _I, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L,
                                            _I, _I, _PI, _PL, _PD]),
    ("kp_integrate_sharded_local_c128", _I, [_CTX, _I, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L,
                                             _I, _I, _PI, _PL, _PD]),
    ("kp_tucker_sharded_f64", _I, [_CTX, _VP, _VP, _PI, _I, _PPD, _D, _I, _VP]),
    ("kp_tucker_sharded_local_f64", _I, [_CTX, _I, _VP, _PI, _I, _PPD, _D, _I, _VP]),
    ("kp_integrate_sampled_f64", _I, [_CTX, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L, _I, _I,
                                      SAMPLE_FN, _VP, _PL, _PD]),
    ("kp_integrate_sampled_c128", _I, [_CTX, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L, _I, _I,
                                       SAMPLE_FN, _VP, _PL, _PD]),
    ("kp_gll_rule", _I, [_I, _PD, _PD]),
    ("kp_expm_f64", _I, [_CTX, _VP, _I, _VP]),
    ("kp_solve_f64", _I, [_CTX, _VP, _I, _VP, _I, _VP]),
    ("kp_expm_c128", _I, [_CTX, _VP, _I, _VP]),
    ("kp_phiquad_f64", _I, [_CTX, _VP, _I, _I, _I, _I, _VP, _PI]),
    ("kp_phiquad_c128", _I, [_CTX, _VP, _I, _I, _I, _I, _VP, _PI]),
    ("kp_build_split_phi_f64", _I, [_CTX, _PPD, _PI, _I, _D, _I, _I, _PPD, _PD]),
    ("kp_build_split_phi_c128", _I, [_CTX, _PPD, _PI, _I, _D, _I, _I, _PPD, _PD]),
    ("kp_step_f64", _I, [_CTX, _I, _VP, _PI, _I, _D, _D, _PPD, _PPD, _D, _PPD, _D, _PG, _VP]),
    ("kp_step_c128", _I, [_CTX, _I, _VP, _PI, _I, _D, _D, _PPD, _PPD, _D, _PPD, _D, _PG, _VP]),
    ("kp_integrate_f64", _I, [_CTX, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L, _I, _PL, _PD]),
    ("kp_integrate_c128", _I, [_CTX, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L, _I, _PL, _PD]),
    ("kp_host_integrate_f64", _I, [_CTX, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L, _I, _VP, _PL,
                                   _PD]),
    ("kp_host_integrate_c128", _I, [_CTX, _I, _VP, _PI, _I, _PPD, _PG, _D, _D, _L, _I, _VP,
                                    _PL, _PD]),
]:
    _lib.register(_name, _res, _args)

kDefaultQuadNodes = 12  # inc/matrix_functions.hpp:107


class Method(enum.IntEnum):
    """inc/integrators.hpp:24-31."""
    LawsonEuler = 0
    Lawson2b = 1
    ExpEuler = 2
    ExpEulerLinearSplit = 3
    ETD2RK = 4
    RosenbrockEuler = 5


_NAMES = {Method.LawsonEuler: "lawson_euler", Method.Lawson2b: "lawson2b",
          Method.ExpEuler: "exp_euler", Method.ExpEulerLinearSplit: "exp_euler_ls",
          Method.ETD2RK: "etd2rk", Method.RosenbrockEuler: "rosenbrock_euler"}


def method_name(m):
    return _NAMES[Method(m)]


def parse_method(s):
    for k, v in _NAMES.items():
        if v == s:
            return k
    raise InvalidArgument(1, f"unknown method: {s}")


G_ZERO, G_SQUARE, G_CONST, G_ALLEN_CAHN, G_BRUSSELATOR, G_NLS, G_ADR, G_RICCATI = range(8)


def gfun(kind, *params) -> GFun:
    """Device nonlinearity descriptor (include/kronphi_b200.h KP_G_*)."""
    g = GFun()
    g.kind = int(kind)
    for i, v in enumerate(params):
        g.p[i] = float(v)
    return g


class G:
    zero = staticmethod(lambda: gfun(G_ZERO))
    square = staticmethod(lambda: gfun(G_SQUARE))
    const = staticmethod(lambda c: gfun(G_CONST, c))
    allen_cahn = staticmethod(lambda: gfun(G_ALLEN_CAHN))
    brusselator = staticmethod(lambda a=1.0, b=3.0: gfun(G_BRUSSELATOR, a, b))
    nls = staticmethod(lambda: gfun(G_NLS))

    @staticmethod
    def adr(psi_a, u0_sq):
        """The reference's ADR source g (src/problems.cpp:101-115).  The
        fields (host numpy or device torch, shaped like u) are uploaded at the
        first device use and kept alive by the descriptor."""
        g = gfun(G_ADR)
        g._aux_src = [psi_a, u0_sq]
        return g

    @staticmethod
    def riccati(b, c_mat):
        """The reference's LQR Riccati g(U) = C - (U b)(U^T b)^T
        (src/problems.cpp:263-276) on an n x n state; b (n) and C (n x n)
        are uploaded at the first device use.  With K = {A^T, A^T} it also
        drives Rosenbrock-Euler's Jacobian factors (:212-250)."""
        g = gfun(G_RICCATI)
        g._aux_src = [b, c_mat]
        return g


def _bind_aux(g):
    """Device pointers for a g with auxiliary fields (ADR, Riccati)."""
    src = getattr(g, "_aux_src", None)
    if src is None or getattr(g, "_aux_dev", None) is not None:
        return g
    dev = [x if _is_torch(x) else to_device(np.asfortranarray(x, dtype=np.float64))
           for x in src]
    for i, t in enumerate(dev):
        g.aux[i] = t.data_ptr()
    g._aux_dev = dev
    return g


# ------------------------------------------------------------ matrix functions

@dataclass
class GLLRule:
    q: int
    nodes: np.ndarray
    weights: np.ndarray


def gll_rule(q: int) -> GLLRule:
    """src/gll_rule.cpp:35-72."""
    x, w = np.zeros(q), np.zeros(q)
    check(_lib.load().kp_gll_rule(int(q), x.ctypes.data_as(_PD), w.ctypes.data_as(_PD)))
    return GLLRule(q, x, w)


def _dev_matrix(x):
    """-> (torch device tensor, was_host, cplx)"""
    if _is_torch(x):
        _check_fortran_torch(x, "matrix")
        return x, False, x.dtype == torch.complex128
    a = np.asarray(x)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise InvalidArgument(1, "expm: matrix not square")
    if not np.all(np.isfinite(a)):
        raise InvalidArgument(1, "expm: non-finite entries")
    return to_device(a), True, np.iscomplexobj(a)


def expm(x):
    """e^x (inc/matrix_functions.hpp:76-95)."""
    xd, host, cplx = _dev_matrix(x)
    if xd.shape[0] != xd.shape[1]:
        raise InvalidArgument(1, "expm: matrix not square")
    ctx = _ctx_for(xd)
    out = fortran_empty(list(xd.shape), xd.dtype, xd.device)
    f = ctx.lib.kp_expm_c128 if cplx else ctx.lib.kp_expm_f64
    check(f(ctx.h, xd.data_ptr(), xd.shape[0], out.data_ptr()))
    return to_host(out) if host else out


def solve(a, b):
    """a^{-1} b by the device blocked LU with partial pivoting
    (inc/linsolve.hpp:148-151: lu_factor + lu_solve); b is n or n x nrhs."""
    ad, host, cplx = _dev_matrix(a)
    if cplx:
        raise InvalidArgument(1, "solve: real matrices only")
    n = ad.shape[0]
    if ad.shape[1] != n:
        raise InvalidArgument(1, "solve: matrix not square")
    vec = np.ndim(b) == 1 if not _is_torch(b) else b.dim() == 1
    bd = (to_device(np.asarray(b, dtype=np.float64)) if not _is_torch(b) else b).to(torch.float64)
    if vec:
        bd = bd.reshape(n, 1)
    if bd.shape[0] != n:
        raise InvalidArgument(1, "solve: size mismatch")
    nrhs = bd.shape[1]
    x = fortran_empty([n, nrhs], torch.float64, ad.device)
    x.copy_(bd)
    ctx = _ctx_for(ad)
    check(ctx.lib.kp_solve_f64(ctx.h, ad.data_ptr(), n, x.data_ptr(), nrhs, x.data_ptr()))
    out = x.reshape(n) if vec else x
    return to_host(out) if host else out


@dataclass
class PhiTable:
    """inc/matrix_functions.hpp:111-117."""
    base: object
    ell_max: int
    phis: list
    scaling_exponent: int


def phiquad(x, ell_max, rule=None, forced_scaling=None) -> PhiTable:
    """phi_0..phi_ell_max of x (inc/matrix_functions.hpp:146-204)."""
    q = kDefaultQuadNodes if rule is None else (rule.q if isinstance(rule, GLLRule) else int(rule))
    if ell_max < 0:
        raise InvalidArgument(1, "phiquad: negative ell_max")
    xd, host, cplx = _dev_matrix(x)
    if xd.shape[0] != xd.shape[1]:
        raise InvalidArgument(1, "phiquad: matrix not square")
    n = xd.shape[0]
    ctx = _ctx_for(xd)
    tab = fortran_empty([n, n * (ell_max + 1)], xd.dtype, xd.device)
    s = C.c_int(0)
    f = ctx.lib.kp_phiquad_c128 if cplx else ctx.lib.kp_phiquad_f64
    check(f(ctx.h, xd.data_ptr(), n, int(ell_max), int(q),
            -1 if forced_scaling is None else int(forced_scaling), tab.data_ptr(), C.byref(s)))
    phis = [tab[:, j * n:(j + 1) * n] for j in range(ell_max + 1)]
    base = xd * (2.0 ** -s.value)
    if host:
        phis = [to_host(p) for p in phis]
        base = to_host(base)
    return PhiTable(base, ell_max, phis, s.value)


# ------------------------------------------------------------- split phi

@dataclass
class SplitPhi:
    """inc/split_phi.hpp:17-23."""
    ell: int = 0
    tau: float = 0.0
    factors: list = field(default_factory=list)
    prefactor: float = 1.0


def _factor_list(k):
    if not isinstance(k, KroneckerSum):
        k = KroneckerSum(k)
    return k


def _upload_factors(fs):
    """Upload host factors, sharing one device copy among equal matrices
    (the device build dedupes identical factors by pointer)."""
    out = []
    for i, f in enumerate(fs):
        if _is_torch(f):
            out.append(f)
            continue
        same = next((j for j in range(i) if not _is_torch(fs[j]) and fs[j].shape == f.shape
                     and np.array_equal(fs[j], f)), None)
        out.append(out[same] if same is not None else to_device(np.asarray(f)))
    return out


def build_split_phi(k, tau, ell, rule=None) -> SplitPhi:
    """inc/split_phi.hpp:25-48."""
    if ell < 0:
        raise InvalidArgument(1, "build_split_phi: negative ell")
    k = _factor_list(k)
    q = kDefaultQuadNodes if rule is None else (rule.q if isinstance(rule, GLLRule) else int(rule))
    host = not _is_torch(k.factors[0])
    cplx = any(_is_cplx(f) for f in k.factors)
    dev = _upload_factors(k.factors)
    dt = torch.complex128 if cplx else torch.float64
    dev = [f.to(dt) for f in dev]
    dims = [int(f.shape[0]) for f in dev]
    outs = [fortran_empty([n, n], dt, dev[0].device) for n in dims]
    pref = C.c_double(0)
    ctx = _ctx_for(dev[0])
    f = ctx.lib.kp_build_split_phi_c128 if cplx else ctx.lib.kp_build_split_phi_f64
    check(f(ctx.h, ptr_array([x.data_ptr() for x in dev]), ints(dims), len(dims), float(tau),
            int(ell), int(q), ptr_array([o.data_ptr() for o in outs]), C.byref(pref)))
    facs = [to_host(o) for o in outs] if host else outs
    return SplitPhi(ell, tau, facs, pref.value)


def apply_split_phi(sp: SplitPhi, v):
    """((l!)^(d-1) V) x_1 F_1 ... x_d F_d (inc/split_phi.hpp:53-62)."""
    from .api import _tucker
    if len(sp.factors) != v.ndim:
        raise InvalidArgument(1, "apply_split_phi: order mismatch")
    for mu, f in enumerate(sp.factors):
        if f.shape[1] != v.shape[mu]:
            raise InvalidArgument(1, f"mode_product: size mismatch on mode {mu}")
    return _tucker(v, list(sp.factors), sp.prefactor)


# ---------------------------------------------------------------- steppers

def _step(method, u, t, tau, K, g, f1, pref1, f2, pref2):
    host = not _is_torch(u)
    cplx = _is_cplx(u) or any(_is_cplx(x) for x in (K or []) + f1 + (f2 or []))
    dt = torch.complex128 if cplx else torch.float64
    ud = (to_device(u) if host else u).to(dt)
    f1d = [x.to(dt) for x in _upload_factors(f1)]
    f2d = [x.to(dt) for x in _upload_factors(f2)] if f2 else None
    Kd = [x.to(dt) for x in _upload_factors(K)] if K else None
    dims = list(ud.shape)
    out = fortran_empty(dims, dt, ud.device)
    ctx = _ctx_for(ud)
    _bind_aux(g)
    f = ctx.lib.kp_step_c128 if cplx else ctx.lib.kp_step_f64
    check(f(ctx.h, int(method), ud.data_ptr(), ints(dims), len(dims), float(t), float(tau),
            ptr_array([x.data_ptr() for x in Kd]) if Kd else None,
            ptr_array([x.data_ptr() for x in f1d]), float(pref1),
            ptr_array([x.data_ptr() for x in f2d]) if f2d else None, float(pref2),
            C.byref(g), out.data_ptr()))
    return to_host(out) if host else out


def eval_g(g, t, u):
    """g(t, u) on the device (the closed set of include/kronphi_b200.h
    KP_G_*; the reference's ProblemSpec::g, inc/integrators.hpp:60)."""
    host = not _is_torch(u)
    cplx = _is_cplx(u)
    ud = to_device(u) if host else u
    dims = list(ud.shape)
    out = fortran_empty(dims, ud.dtype, ud.device)
    ctx = _ctx_for(ud)
    _bind_aux(g)
    f = ctx.lib.kp_eval_g_c128 if cplx else ctx.lib.kp_eval_g_f64
    check(f(ctx.h, C.byref(g), float(t), ud.data_ptr(), ints(dims), len(dims), out.data_ptr()))
    return to_host(out) if host else out


def lawson_euler_step(u, t, tau, g, exp_factors):
    """inc/integrators.hpp:116-122"""
    return _step(Method.LawsonEuler, u, t, tau, None, g, list(exp_factors), 1.0, None, 1.0)


def lawson2b_step(u, t, tau, g, exp_factors):
    """inc/integrators.hpp:124-132"""
    return _step(Method.Lawson2b, u, t, tau, None, g, list(exp_factors), 1.0, None, 1.0)


def exp_euler_step(u, t, tau, k, g, phi1: SplitPhi):
    """inc/integrators.hpp:134-141"""
    k = _factor_list(k)
    return _step(Method.ExpEuler, u, t, tau, k.factors, g, phi1.factors, phi1.prefactor, None, 1.0)


def exp_euler_linear_split_step(u, t, tau, g, exp_factors, phi1: SplitPhi):
    """inc/integrators.hpp:143-151"""
    return _step(Method.ExpEulerLinearSplit, u, t, tau, None, g, list(exp_factors), 1.0,
                 phi1.factors, phi1.prefactor)


def etd2rk_step(u, t, tau, k, g, phi1: SplitPhi, phi2: SplitPhi):
    """inc/integrators.hpp:153-164"""
    k = _factor_list(k)
    return _step(Method.ETD2RK, u, t, tau, k.factors, g, phi1.factors, phi1.prefactor,
                 phi2.factors, phi2.prefactor)


def rosenbrock_euler_step(u, t, tau, k, g, jac_factors, q=kDefaultQuadNodes):
    """inc/integrators.hpp:166-194: phi_1(tau J_mu) rebuilt from the given
    Jacobian factors on the device (the same object twice shares one build)."""
    if q != kDefaultQuadNodes:
        raise InvalidArgument(1, "rosenbrock_euler_step: the device step uses the default rule")
    k = _factor_list(k)
    return _step(Method.RosenbrockEuler, u, t, tau, k.factors, g, list(jac_factors), 1.0,
                 None, 1.0)


# --------------------------------------------------------------- integrate

@dataclass
class ProblemSpec:
    """inc/integrators.hpp:58-69 with g from the device closed set."""
    K: object
    g: GFun
    u0: object
    t0: float = 0.0
    t_final: float = 1.0


@dataclass
class StepperConfig:
    """inc/integrators.hpp:71-77.  backend: "split" (the device splitting
    path) or "dense_oracle" (validation: the assembled Kronecker sum as the
    single factor of a one-mode problem, i.e. the exact phi actions)."""
    method: Method = Method.ExpEuler
    n_steps: int = 1
    quad_nodes: int = kDefaultQuadNodes
    sample_every: int = 0  # 0 disables trajectory sampling
    backend: str = "split"


@dataclass
class IntegrateResult:
    """inc/integrators.hpp:79-84."""
    final: object
    wallclock_s: float = 0.0
    loop_s: float = 0.0
    trajectory: list = None  # [(t, u)] at t0 and every sample_every steps


def integrate(p: ProblemSpec, c: StepperConfig) -> IntegrateResult:
    """inc/integrators.hpp:219-373: factors built once on the GPU, the time
    loop on device-resident state (CUDA graph), per-step finite check."""
    if c.n_steps <= 0:
        raise InvalidArgument(1, "integrate: n_steps must be positive")
    if not p.t_final > p.t0:
        raise InvalidArgument(1, "integrate: empty time interval")
    k = _factor_list(p.K)
    u0 = p.u0
    host = not _is_torch(u0)
    cplx = _is_cplx(u0) or any(_is_cplx(f) for f in k.factors)
    dims = list(u0.shape)
    if len(dims) != k.order():
        raise InvalidArgument(1, "kronsum_action: expected one factor per mode")
    for mu, f in enumerate(k.factors):
        if f.shape[0] != dims[mu]:
            raise InvalidArgument(1, f"mode_product: size mismatch on mode {mu}")
    if c.sample_every < 0:
        raise InvalidArgument(1, "integrate: negative sample_every")
    if c.backend == "dense_oracle":
        return _integrate_dense_oracle(p, c, k, dims, cplx, host)
    if c.backend != "split":
        raise InvalidArgument(1, f"integrate: unknown backend {c.backend}")
    t_start = time.perf_counter()
    dv = C.c_long(0)
    loop = C.c_double(0)
    _bind_aux(p.g)
    traj = None
    if host and not c.sample_every:
        dtype = np.complex128 if cplx else np.float64
        uh = np.asfortranarray(u0, dtype=dtype)
        fs = [np.asfortranarray(f, dtype=dtype) for f in k.factors]
        out = np.zeros(dims, order="F", dtype=dtype)
        ctx = default_context(0)
        f = ctx.lib.kp_host_integrate_c128 if cplx else ctx.lib.kp_host_integrate_f64
        rc = f(ctx.h, int(c.method), uh.ctypes.data, ints(dims), len(dims),
               ptr_array([x.ctypes.data for x in fs]), C.byref(p.g), float(p.t0),
               float(p.t_final), int(c.n_steps), int(c.quad_nodes), out.ctypes.data,
               C.byref(dv), C.byref(loop))
    else:
        dt = torch.complex128 if cplx else torch.float64
        src = to_device(np.asarray(u0)) if host else u0
        out = fortran_empty(dims, dt, src.device)
        out.copy_(src)
        fs = [x.to(dt) for x in _upload_factors(k.factors)]
        ctx = _ctx_for(out)
        if c.sample_every:
            tau = (p.t_final - p.t0) / float(c.n_steps)
            n = int(np.prod(dims))
            npdt = np.complex128 if cplx else np.float64
            traj = [(p.t0, np.array(u0, copy=True) if host else u0.clone())]

            def _hook(user, step, uh):
                a = np.ctypeslib.as_array(uh, shape=(n * (2 if cplx else 1),)).copy()
                a = a.view(npdt).reshape(dims, order="F")
                traj.append((p.t0 + float(step) * tau, a if host else to_device(a)))
            hook = SAMPLE_FN(_hook)
            f = ctx.lib.kp_integrate_sampled_c128 if cplx else ctx.lib.kp_integrate_sampled_f64
            rc = f(ctx.h, int(c.method), out.data_ptr(), ints(dims), len(dims),
                   ptr_array([x.data_ptr() for x in fs]), C.byref(p.g), float(p.t0),
                   float(p.t_final), int(c.n_steps), int(c.quad_nodes), int(c.sample_every),
                   hook, None, C.byref(dv), C.byref(loop))
        else:
            f = ctx.lib.kp_integrate_c128 if cplx else ctx.lib.kp_integrate_f64
            rc = f(ctx.h, int(c.method), out.data_ptr(), ints(dims), len(dims),
                   ptr_array([x.data_ptr() for x in fs]), C.byref(p.g), float(p.t0),
                   float(p.t_final), int(c.n_steps), int(c.quad_nodes), C.byref(dv),
                   C.byref(loop))
        if host:
            torch.cuda.synchronize(out.device)
            out = to_host(out)
    try:
        check(rc, step=dv.value)
    except DivergenceError as e:
        e.loop_s = loop.value  # the loop ran to the end; its device time is still valid
        raise
    return IntegrateResult(out, time.perf_counter() - t_start, loop.value, traj)


def _assemble_kronsum(factors):
    """Dense K = sum_mu I (x) .. (x) A_mu (x) .. (x) I, first mode fastest."""
    dims = [f.shape[0] for f in factors]
    N = int(np.prod(dims))
    if N > 8192:
        raise InvalidArgument(1, "DenseOracle: problem too large (N > 8192)")
    K = np.zeros((N, N), dtype=np.result_type(*factors), order="F")
    P = 1
    for mu, a in enumerate(factors):
        Q = N // (P * dims[mu])
        K += np.kron(np.kron(np.eye(Q), np.asarray(a)), np.eye(P))
        P *= dims[mu]
    return np.asfortranarray(K)


def _integrate_dense_oracle(p, c, k, dims, cplx, host):
    """Backend::DenseOracle (inc/integrators.hpp:243-262): the textbook
    exponential integrators on the assembled operator -- run as the one-mode
    problem vec(u)' = K vec(u) + g on the device, where the split phi of the
    single factor is the exact phi_l(tau K)."""
    if int(c.method) == int(Method.RosenbrockEuler):
        raise InvalidArgument(1, "DenseOracle: Rosenbrock-Euler is not provided")
    if p.g.kind in (G_BRUSSELATOR, G_RICCATI):
        raise InvalidArgument(1, "DenseOracle: this g needs the tensor shape")
    fs = [to_host(f) if _is_torch(f) else np.asarray(f) for f in k.factors]
    K = _assemble_kronsum(fs)
    u = to_host(p.u0) if not host else np.asarray(p.u0)
    u1 = np.asfortranarray(u.reshape(-1, order="F"))
    c1 = StepperConfig(c.method, c.n_steps, c.quad_nodes, c.sample_every, "split")
    r = integrate(ProblemSpec([K], p.g, u1, p.t0, p.t_final), c1)
    shape = lambda a: np.asfortranarray(np.asarray(a).reshape(dims, order="F"))
    fin = shape(r.final)
    traj = [(t, shape(x)) for t, x in r.trajectory] if r.trajectory else None
    if not host:
        fin = to_device(fin)
        traj = [(t, to_device(x)) for t, x in traj] if traj else None
    return IntegrateResult(fin, r.wallclock_s, r.loop_s, traj)


def integrate_config(method, u0, As, g, t0, t_final, n_steps, q=kDefaultQuadNodes):
    """Convenience: integrate(ProblemSpec(As, g, u0, t0, t_final), StepperConfig(...)).final"""
    m = parse_method(method) if isinstance(method, str) else Method(method)
    return integrate(ProblemSpec(As, g, u0, t0, t_final),
                     StepperConfig(m, n_steps, q)).final
