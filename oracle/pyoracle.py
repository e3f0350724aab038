"""ctypes wrapper over the CPU oracle libraries.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.

Two interchangeable backends with one numpy API:
  * ``Oracle("port")``      -- oracle/lib/libkp_oracle.so, the plain-C
                               restatement (kp_oracle.c), always present;
  * ``Oracle("reference")`` -- oracle/_ref/libkronphi_ref.so, the real
                               reference library compiled from
                               /root/reference/proj by ``make -C oracle ref``.

All arrays are numpy, column-major (Fortran order) like the reference's
Tensor/Matrix (inc/tensor.hpp:1-2); complex arrays are complex128.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "lib", "libkp_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libkronphi_ref.so")

# kp_oracle.h enums
LAWSON_EULER, LAWSON2B, EXP_EULER, EXP_EULER_LS, ETD2RK = range(5)
METHODS = {"lawson_euler": LAWSON_EULER, "lawson2b": LAWSON2B, "exp_euler": EXP_EULER,
           "exp_euler_ls": EXP_EULER_LS, "etd2rk": ETD2RK,
           "rosenbrock_euler": 5}
G_ZERO, G_SQUARE, G_CONST, G_ALLEN_CAHN, G_BRUSSELATOR, G_NLS = range(6)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(OracleError, ValueError):
    pass


class Divergence(OracleError):
    pass


class GFun(C.Structure):
    _fields_ = [("kind", C.c_int), ("p", C.c_double * 4), ("aux", C.c_void_p * 2)]


G_ADR = 6
G_RICCATI = 7  # aux = (b, C) on an n x n state, src/problems.cpp:188-200, 263-276


def gfun(kind, *params, aux=None):
    """aux: host arrays (ADR: psi_a, u0^2), kept alive on the descriptor."""
    g = GFun()
    g.kind = kind
    for i, v in enumerate(params):
        g.p[i] = v
    if aux is not None:
        g._keep = [np.asfortranarray(a, dtype=np.float64) for a in aux]
        for i, a in enumerate(g._keep):
            g.aux[i] = a.ctypes.data
    return g


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ints(xs):
    return (C.c_int * len(xs))(*xs)


def _ptrs(arrs):
    return (C.POINTER(C.c_double) * len(arrs))(*[_dp(a) for a in arrs])


def _f(a, cplx):
    return np.asfortranarray(a, dtype=np.complex128 if cplx else np.float64)


def available(kind):
    return os.path.exists(REF_LIB if kind == "reference" else PORT_LIB)


class Oracle:
    def __init__(self, kind="port"):
        self.kind = kind
        path = REF_LIB if kind == "reference" else PORT_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle"
                                    f"{' ref' if kind == 'reference' else ''})")
        self.lib = C.CDLL(path)
        self.p = "kpr_" if kind == "reference" else "kpo_"
        self.fn("last_error").restype = C.c_char_p
        D, I, L, PD, PI, PP = (C.c_double, C.c_int, C.c_long, C.POINTER(C.c_double),
                               C.POINTER(C.c_int), C.POINTER(C.POINTER(C.c_double)))
        PG = C.POINTER(GFun)
        sig = {
            "mode_product": [PD, PI, I, I, PD, I, I, PD, I],
            "tucker": [PD, PI, I, PP, PI, PD],
            "kronsum": [PD, PI, I, PP, PD],
            "expm": [PD, I, PD],
            "phiquad": [PD, I, I, I, I, PD, PI],
            "build_split_phi": [PP, PI, I, D, I, I, PP, PD],
            "apply_split_phi": [PD, PI, I, PP, D, PD],
            "eval_g": [PG, D, PD, PI, I, PD],
            "step": [I, PD, PI, I, D, D, PP, PP, D, PP, D, PG, PD],
            "integrate": [I, PD, PI, I, PP, PG, D, D, L, I, PD, C.POINTER(C.c_long)],
        }
        for name, args in sig.items():
            for sfx in ("_f64", "_c128"):
                if hasattr(self.lib, self.p + name + sfx):
                    self.fn(name + sfx).argtypes = args
        self.fn("gll_rule").argtypes = [I, PD, PD]
        self.fn("fd_operator_1d").argtypes = [I, D, D, PD]

    def fn(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc:
            msg = self.fn("last_error")().decode()
            if rc == 1:
                raise InvalidArgument(rc, msg)
            if rc == 3:
                raise Divergence(rc, msg)
            raise OracleError(rc, msg)

    # ---- tensor ops ----
    def mode_product(self, t, m, mode, out=None):
        cplx = np.iscomplexobj(t) or np.iscomplexobj(m)
        t, m = _f(t, cplx), _f(m, cplx)
        dims = list(t.shape)
        od = dims.copy()
        if 0 <= mode < len(dims):
            od[mode] = m.shape[0]
        acc = out is not None
        o = _f(out, cplx).copy(order="F") if acc else np.zeros(od, order="F",
                                                                dtype=t.dtype)
        f = self.fn("mode_product_c128" if cplx else "mode_product_f64")
        self._check(f(_dp(t), _ints(dims), len(dims), mode, _dp(m), m.shape[0], m.shape[1],
                      _dp(o), int(acc)))
        return o

    def tucker(self, t, ms):
        cplx = np.iscomplexobj(t) or any(np.iscomplexobj(m) for m in ms)
        t = _f(t, cplx)
        ms = [_f(m, cplx) for m in ms]
        rows = [m.shape[0] for m in ms]
        o = np.zeros(rows, order="F", dtype=t.dtype)
        f = self.fn("tucker_c128" if cplx else "tucker_f64")
        self._check(f(_dp(t), _ints(list(t.shape)), t.ndim, _ptrs(ms), _ints(rows), _dp(o)))
        return o

    def kronsum(self, t, As):
        cplx = np.iscomplexobj(t) or any(np.iscomplexobj(a) for a in As)
        t = _f(t, cplx)
        As = [_f(a, cplx) for a in As]
        o = np.zeros(t.shape, order="F", dtype=t.dtype)
        f = self.fn("kronsum_c128" if cplx else "kronsum_f64")
        self._check(f(_dp(t), _ints(list(t.shape)), t.ndim, _ptrs(As), _dp(o)))
        return o

    # ---- matrix functions ----
    def gll_rule(self, q):
        x = np.zeros(q)
        w = np.zeros(q)
        self._check(self.fn("gll_rule")(q, _dp(x), _dp(w)))
        return x, w

    def expm(self, x):
        cplx = np.iscomplexobj(x)
        x = _f(x, cplx)
        o = np.zeros_like(x, order="F")
        self._check(self.fn("expm_c128" if cplx else "expm_f64")(_dp(x), x.shape[0], _dp(o)))
        return o

    def phiquad(self, x, ell_max, q=12, forced_scaling=None):
        cplx = np.iscomplexobj(x)
        x = _f(x, cplx)
        n = x.shape[0]
        phis = np.zeros((n, n, ell_max + 1), order="F", dtype=x.dtype)
        s = C.c_int(0)
        f = self.fn("phiquad_c128" if cplx else "phiquad_f64")
        self._check(f(_dp(x), n, ell_max, q, -1 if forced_scaling is None else forced_scaling,
                      _dp(phis), C.byref(s)))
        return [np.asfortranarray(phis[:, :, j]) for j in range(ell_max + 1)], s.value

    def build_split_phi(self, As, tau, ell, q=12):
        cplx = any(np.iscomplexobj(a) for a in As)
        As = [_f(a, cplx) for a in As]
        dims = [a.shape[0] for a in As]
        fs = [np.zeros_like(a, order="F") for a in As]
        pref = C.c_double(0)
        f = self.fn("build_split_phi_c128" if cplx else "build_split_phi_f64")
        self._check(f(_ptrs(As), _ints(dims), len(As), tau, ell, q, _ptrs(fs), C.byref(pref)))
        return fs, pref.value

    def apply_split_phi(self, v, factors, prefactor):
        cplx = np.iscomplexobj(v) or any(np.iscomplexobj(a) for a in factors)
        v = _f(v, cplx)
        fs = [_f(a, cplx) for a in factors]
        o = np.zeros(v.shape, order="F", dtype=v.dtype)
        f = self.fn("apply_split_phi_c128" if cplx else "apply_split_phi_f64")
        self._check(f(_dp(v), _ints(list(v.shape)), v.ndim, _ptrs(fs), prefactor, _dp(o)))
        return o

    # ---- steppers ----
    def eval_g(self, g, t, u):
        cplx = np.iscomplexobj(u)
        u = _f(u, cplx)
        o = np.zeros_like(u, order="F")
        f = self.fn("eval_g_c128" if cplx else "eval_g_f64")
        self._check(f(C.byref(g), t, _dp(u), _ints(list(u.shape)), u.ndim, _dp(o)))
        return o

    def step(self, method, u, t, tau, As, f1, pref1, f2, pref2, g):
        cplx = np.iscomplexobj(u) or any(np.iscomplexobj(a) for a in As)
        u = _f(u, cplx)
        As = [_f(a, cplx) for a in As]
        f1 = [_f(a, cplx) for a in f1]
        f2 = [_f(a, cplx) for a in (f2 if f2 is not None else f1)]
        o = np.zeros(u.shape, order="F", dtype=u.dtype)
        f = self.fn("step_c128" if cplx else "step_f64")
        self._check(f(METHODS.get(method, method), _dp(u), _ints(list(u.shape)), u.ndim, t, tau,
                      _ptrs(As), _ptrs(f1), pref1, _ptrs(f2), pref2, C.byref(g), _dp(o)))
        return o

    def integrate(self, method, u0, As, g, t0, t_final, n_steps, q=12):
        cplx = np.iscomplexobj(u0) or any(np.iscomplexobj(a) for a in As)
        u0 = _f(u0, cplx)
        As = [_f(a, cplx) for a in As]
        o = np.zeros(u0.shape, order="F", dtype=u0.dtype)
        dv = C.c_long(0)
        f = self.fn("integrate_c128" if cplx else "integrate_f64")
        self._check(f(METHODS.get(method, method), _dp(u0), _ints(list(u0.shape)), u0.ndim,
                      _ptrs(As), C.byref(g), t0, t_final, C.c_long(n_steps), q, _dp(o),
                      C.byref(dv)))
        return o

    def fd_operator_1d(self, n, eps, alpha=0.0):
        o = np.zeros((n, n), order="F")
        self._check(self.fn("fd_operator_1d")(n, C.c_double(eps), C.c_double(alpha), _dp(o)))
        return o

    # ---- timing (reference arm only) ----
    def time_tucker(self, t, ms, reps=1):
        if self.kind != "reference":
            raise RuntimeError("time_tucker is a reference-harness helper")
        t = _f(t, False)
        ms = [_f(m, False) for m in ms]
        f = self.fn("time_tucker_f64")
        f.restype = C.c_double
        s = f(_dp(t), _ints(list(t.shape)), t.ndim, _ptrs(ms), reps)
        if s < 0:
            raise OracleError(2, self.fn("last_error")().decode())
        return s

    def time_tucker_mean(self, t, ms, warmup, steps):
        """Mean seconds per reference tucker() over `steps` calls (inputs
        converted once, outside the timed region)."""
        if self.kind != "reference":
            raise RuntimeError("time_tucker_mean is a reference-harness helper")
        t = _f(t, False)
        ms = [_f(m, False) for m in ms]
        f = self.fn("time_tucker_mean_f64")
        f.restype = C.c_double
        s = f(_dp(t), _ints(list(t.shape)), t.ndim, _ptrs(ms), int(warmup), int(steps))
        if s < 0:
            raise OracleError(2, self.fn("last_error")().decode())
        return s

    def time_integrate(self, method, u0, As, g, t0, t_final, n_steps, q=12):
        """The reference's integrate() loop time (IntegrateResult::loop_s)."""
        if self.kind != "reference":
            raise RuntimeError("time_integrate is a reference-harness helper")
        cplx = np.iscomplexobj(u0) or any(np.iscomplexobj(a) for a in As)
        u0 = _f(u0, cplx)
        As = [_f(a, cplx) for a in As]
        loop = C.c_double(0)
        f = self.fn("time_integrate_c128" if cplx else "time_integrate_f64")
        self._check(f(METHODS.get(method, method), _dp(u0), _ints(list(u0.shape)), u0.ndim,
                      _ptrs(As), C.byref(g), C.c_double(t0), C.c_double(t_final),
                      C.c_long(n_steps), q, C.byref(loop)))
        return loop.value

    def run_adr(self, n1, n2, n3, method, n_steps):
        """The reference's own ADR experiment (reference harness only):
        final state and rel. inf-norm error vs e^t u0 at T = 1."""
        if self.kind != "reference":
            raise RuntimeError("run_adr needs the reference harness")
        out = np.zeros((n1, n2, n3), order="F")
        err, sec = C.c_double(0), C.c_double(0)
        f = self.fn("run_adr")
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_long, C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self._check(f(n1, n2, n3, METHODS.get(method, method), n_steps, _dp(out), C.byref(err),
                      C.byref(sec)))
        return out, err.value, sec.value

    def run_riccati(self, n_hat, method, n_steps, t_final):
        """The reference's LQR Riccati experiment (build_riccati +
        to_problem_spec + integrate, reference harness only): final state."""
        if self.kind != "reference":
            raise RuntimeError("run_riccati needs the reference harness")
        n = n_hat * n_hat
        out = np.zeros((n, n), order="F")
        sec = C.c_double(0)
        f = self.fn("run_riccati")
        f.argtypes = [C.c_int, C.c_int, C.c_long, C.c_double, C.POINTER(C.c_double),
                      C.POINTER(C.c_double)]
        self._check(f(n_hat, METHODS.get(method, method), n_steps, t_final, _dp(out),
                      C.byref(sec)))
        return out, sec.value

    def num_threads(self):
        return self.fn("num_threads")() if self.kind == "reference" else 1


def periodic_laplacian_1d(n, h):
    """(1/h^2) circ(1,-2,1): the NLS config's periodic 1-D operator (new; the
    reference's fd_operator_1d is Dirichlet-only, src/problems.cpp:9-22)."""
    lib = C.CDLL(PORT_LIB)
    o = np.zeros((n, n), order="F")
    rc = lib.kpo_periodic_laplacian_1d(n, C.c_double(h), _dp(o))
    if rc:
        raise InvalidArgument(rc, "periodic_laplacian_1d")
    return o
