"""The reference's experiment harness on the device path: convergence sweeps
on its two benchmark problems (ADR, LQR Riccati), the Riccati steady-state
residual tracker, observed-order estimation, CSV/table output and the
invariant self-test battery (src/bench_runner.cpp, inc/bench_runner.hpp).

Same record layout, default step sweeps, error norms, CSV header and number
formatting (%.17g) as the reference, so its tables and CSV consumers work
unchanged; every integration runs through `integrators.integrate` (device
factors, CUDA-graph time loop).  Backend::DenseOracle (a validation backend)
is not provided.
"""
from __future__ import annotations

import math
import sys
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import integrators as _it
from . import problems as _pb
from ._lib import DivergenceError, InvalidArgument
from .integrators import Method, method_name


@dataclass
class RunRecord:
    """inc/bench_runner.hpp:17-26."""
    problem: str
    method: str
    n_steps: int = 0
    tau: float = 0.0
    error: float = 0.0
    observed_order: Optional[float] = None
    wallclock_s: float = 0.0
    loop_s: float = 0.0


def observed_order(errors: Sequence[float], taus: Sequence[float]) -> List[Optional[float]]:
    """p_k = log(e_{k-1}/e_k) / log(tau_{k-1}/tau_k); None where an error or
    step is not positive (src/bench_runner.cpp:17-33)."""
    if len(errors) != len(taus) or len(errors) < 2:
        raise InvalidArgument(1, "observed_order: need two matched sweeps")
    out = []
    for k in range(1, len(errors)):
        if errors[k - 1] <= 0 or errors[k] <= 0 or taus[k - 1] <= 0 or taus[k] <= 0:
            out.append(None)
        else:
            out.append(math.log(errors[k - 1] / errors[k]) / math.log(taus[k - 1] / taus[k]))
    return out


def fit_order(taus: Sequence[float], errors: Sequence[float]) -> float:
    """Least-squares slope of log(err) against log(tau) (src/bench_runner.cpp:35-49)."""
    if len(taus) != len(errors) or len(taus) < 2:
        raise InvalidArgument(1, "fit_order: need two matched sweeps")
    x = [math.log(t) for t in taus]
    y = [math.log(e) for e in errors]
    n = len(x)
    sx, sy = sum(x), sum(y)
    sxx = sum(v * v for v in x)
    sxy = sum(a * b for a, b in zip(x, y))
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)


def _g17(v: float) -> str:
    return "%.17g" % v


def write_csv(path: str, records: Sequence[RunRecord]) -> None:
    """src/bench_runner.cpp:61-71: header and %.17g fields; empty order cell
    for the first row of a sweep."""
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError("write_csv: cannot open " + path)
    with f:
        f.write("problem,method,steps,tau,error,order,wallclock_s\n")
        for r in records:
            order = _g17(r.observed_order) if r.observed_order is not None else ""
            f.write(f"{r.problem},{r.method},{r.n_steps},{_g17(r.tau)},{_g17(r.error)},"
                    f"{order},{_g17(r.wallclock_s)}\n")


def print_table(records: Sequence[RunRecord], out=None) -> None:
    """One block per (problem, method): steps / error / order / wallclock /
    loop rows (src/bench_runner.cpp:73-113)."""
    out = out or sys.stdout
    i = 0
    while i < len(records):
        j = i
        while (j < len(records) and records[j].method == records[i].method
               and records[j].problem == records[i].problem):
            j += 1
        out.write(f"{records[i].problem} / {records[i].method}\n")

        def row(name, fmt):
            out.write("  " + name.ljust(12) + "".join(fmt(r).rjust(12) for r in records[i:j])
                      + "\n")

        row("steps", lambda r: str(r.n_steps))
        row("error", lambda r: "%.3e" % r.error)
        row("order", lambda r: "--" if r.observed_order is None else "%.2f" % r.observed_order)
        row("wallclock_s", lambda r: "%.2f" % r.wallclock_s)
        row("loop_s", lambda r: "%.2f" % r.loop_s)
        i = j


def default_adr_steps(m, n1: int) -> List[int]:
    """src/bench_runner.cpp:115-131."""
    m = Method(m)
    if m == Method.LawsonEuler:
        return [800, 8800, 16800, 24800, 32800]
    if m in (Method.ExpEuler, Method.ExpEulerLinearSplit):
        return [50, 450, 850, 1250, 1650]
    if m == Method.Lawson2b:
        return [1500, 5500, 9500, 13500, 17500] if n1 < 60 else [3000, 4500, 6000, 7500, 9000]
    if m == Method.ETD2RK:
        return [40, 140, 240, 340, 440]
    raise InvalidArgument(1, "no default ADR sweep for this method")


def default_riccati_steps(m=None) -> List[int]:
    """src/bench_runner.cpp:133."""
    return [30, 65, 100, 135, 170]


def sweep(spec: _it.ProblemSpec, problem: str, m, steps: Sequence[int], error_of,
          log=None) -> List[RunRecord]:
    """Integrate once per step count, record errors and observed orders
    (src/bench_runner.cpp:137-177)."""
    log = log or sys.stdout
    m = Method(m)
    recs: List[RunRecord] = []
    for n in steps:
        try:
            res = _it.integrate(spec, _it.StepperConfig(m, int(n)))
        except DivergenceError as e:
            raise RuntimeError(f"{problem}/{method_name(m)} with {n} steps diverged: {e}")
        r = RunRecord(problem, method_name(m), int(n), (spec.t_final - spec.t0) / float(n),
                      float(error_of(res.final)), None, res.wallclock_s, res.loop_s)
        recs.append(r)
        log.write(f"  {problem}/{method_name(m)} steps={n} error={r.error:g} "
                  f"wallclock={res.wallclock_s:g}s\n")
    if len(recs) >= 2:
        orders = observed_order([r.error for r in recs], [r.tau for r in recs])
        for k, o in enumerate(orders):
            recs[k + 1].observed_order = o
    return recs


def _methods(names, default):
    if not names:
        return list(default)
    return [_it.parse_method(x) if isinstance(x, str) else Method(x) for x in names]


@dataclass
class AdrOptions:
    """inc/bench_runner.hpp:44-50 (backend: split only)."""
    n1: int = 40
    n2: int = 41
    n3: int = 42
    methods: list = field(default_factory=list)
    steps: list = field(default_factory=list)
    out_csv: str = ""


def run_adr(opt: AdrOptions, log=None) -> List[RunRecord]:
    """ADR sweeps, error = rel. inf-norm vs e^T u0 (src/bench_runner.cpp:181-203)."""
    log = log or sys.stdout
    c = _pb.adr(opt.n1, opt.n2, opt.n3)
    spec = _it.ProblemSpec(c.K, c.g, c.u0, 0.0, 1.0)
    exact = c.exact
    denom = float(np.abs(exact).max())
    pid = f"adr{opt.n1}"
    out: List[RunRecord] = []
    for m in _methods(opt.methods, [Method.LawsonEuler, Method.ExpEuler, Method.Lawson2b,
                                    Method.ETD2RK]):
        steps = opt.steps or default_adr_steps(m, opt.n1)
        out += sweep(spec, pid, m, steps,
                     lambda u: float(np.abs(np.asarray(u) - exact).max()) / denom, log)
    print_table(out, log)
    if opt.out_csv:
        write_csv(opt.out_csv, out)
    return out


@dataclass
class RiccatiOptions:
    """inc/bench_runner.hpp:54-61 (backend: split only)."""
    n_hat: int = 30
    methods: list = field(default_factory=list)
    steps: list = field(default_factory=list)
    ref_steps: int = 4096
    out_csv: str = ""


def run_riccati(opt: RiccatiOptions, log=None) -> List[RunRecord]:
    """Riccati sweeps, error = rel. Frobenius distance to an ETD2RK run with
    ref_steps steps (src/bench_runner.cpp:205-229)."""
    log = log or sys.stdout
    c = _pb.riccati(opt.n_hat)
    spec = _it.ProblemSpec(c.K, c.g, c.u0, 0.0, 0.025)
    log.write(f"riccati n_hat={opt.n_hat}: computing etd2rk reference with "
              f"{opt.ref_steps} steps\n")
    ref = np.asarray(_it.integrate(spec, _it.StepperConfig(Method.ETD2RK,
                                                           int(opt.ref_steps))).final)
    denom = float(np.linalg.norm(ref))
    pid = f"riccati{opt.n_hat}"
    out: List[RunRecord] = []
    for m in _methods(opt.methods, [Method.RosenbrockEuler, Method.ETD2RK]):
        steps = opt.steps or default_riccati_steps(m)
        out += sweep(spec, pid, m, steps,
                     lambda u: float(np.linalg.norm(np.asarray(u) - ref)) / denom, log)
    print_table(out, log)
    if opt.out_csv:
        write_csv(opt.out_csv, out)
    return out


@dataclass
class SteadyOptions:
    """inc/bench_runner.hpp:65-72."""
    n_hat: int = 20
    n_steps: int = 200
    sample_every: int = 10
    t_final: float = 0.2
    methods: list = field(default_factory=list)
    out_csv: str = ""


@dataclass
class SteadyRecord:
    method: str
    step: int = 0
    t: float = 0.0
    rel_residual: float = 0.0


def are_residual(u, c) -> float:
    """||A^T U + U A + C + U B U||_F on the device: the Kronecker-sum action
    of K = {A^T, A^T} plus the Riccati g (src/problems.cpp:279-281)."""
    from .api import kronsum_action, to_device, to_host, KroneckerSum
    ud = u if _it._is_torch(u) else to_device(np.asfortranarray(u))
    r = kronsum_action(ud, KroneckerSum([to_device(np.asfortranarray(f)) for f in c.K]))
    r += _it.eval_g(c.g, 0.0, ud)
    return float(np.linalg.norm(to_host(r)))


def run_steady(opt: SteadyOptions, log=None) -> List[SteadyRecord]:
    """Riccati steady state: relative ARE residual every sample_every steps
    (src/bench_runner.cpp:231-266).  The reference samples the trajectory
    inside one integrate(); here the run is split into segments of
    sample_every steps (the Riccati system is autonomous) with the same tau."""
    log = log or sys.stdout
    c = _pb.riccati(opt.n_hat)
    cnorm = float(np.linalg.norm(c.c_mat))
    tau = opt.t_final / opt.n_steps
    recs: List[SteadyRecord] = []
    for m in _methods(opt.methods, [Method.RosenbrockEuler, Method.ETD2RK]):
        u = _it.to_device(np.asfortranarray(c.u0))
        done = 0
        while done < opt.n_steps:
            k = min(opt.sample_every, opt.n_steps - done) if opt.sample_every > 0 else \
                opt.n_steps - done
            t0 = done * tau
            spec = _it.ProblemSpec(c.K, c.g, u, t0, t0 + k * tau)
            u = _it.integrate(spec, _it.StepperConfig(m, k)).final
            done += k
            if opt.sample_every > 0 and (done % opt.sample_every == 0 or done == opt.n_steps):
                recs.append(SteadyRecord(method_name(m), done, done * tau,
                                         are_residual(u, c) / cnorm))
        log.write(f"  steady/{method_name(m)}: final relative residual "
                  f"{recs[-1].rel_residual:g} at t={recs[-1].t:g}\n")
    if opt.out_csv:
        try:
            f = open(opt.out_csv, "w")
        except OSError:
            raise RuntimeError("run_steady: cannot open " + opt.out_csv)
        with f:
            f.write("problem,method,step,t,rel_residual\n")
            for r in recs:
                f.write(f"riccati{opt.n_hat},{r.method},{r.step},{_g17(r.t)},"
                        f"{_g17(r.rel_residual)}\n")
    return recs


# ------------------------------------------------------------------ selftest

def _taylor_phi_action(x: np.ndarray, ell: int, v: np.ndarray, terms: int = 60) -> np.ndarray:
    """phi_ell(X) v = sum_k X^k v / (k + ell)!, with scaling by repeated
    halving unnecessary for the small norms used below."""
    out = np.zeros_like(v)
    term = v.copy()
    for k in range(terms):
        out += term / math.factorial(k + ell)
        term = x @ term
    return out


def _taylor_phi(x: np.ndarray, ell: int) -> np.ndarray:
    """phi_ell(X) by Taylor series after scaling X/2^s and the phi doubling
    recurrence (validation oracle for the self-test)."""
    n = x.shape[0]
    s = max(0, int(math.ceil(math.log2(max(np.abs(x).sum(0).max(), 1e-300)))) + 1)
    y = x / 2.0 ** s
    phis = [_taylor_phi_action(y, l, np.eye(n)) for l in range(ell + 1)]
    for _ in range(s):
        p0 = phis[0]
        new = []
        for l in range(ell + 1):
            m = p0 @ phis[l]
            for k in range(1, l + 1):
                m = m + phis[k] / math.factorial(l - k)
            new.append(m / 2.0 ** l if l > 0 else m)
        phis = new
    return phis[ell]


def _kron_dense(ms):
    k = np.ones((1, 1))
    for m in ms:  # the left operand varies fastest
        k = np.kron(m, k)
    return k


def _kronsum_dense(fs):
    out = 0
    for mu, f in enumerate(fs):
        ms = [np.eye(g.shape[0]) for g in fs]
        ms[mu] = f
        out = out + _kron_dense(ms)
    return out


@dataclass
class SelftestOptions:
    """inc/bench_runner.hpp:82-87."""
    quad_nodes: int = _it.kDefaultQuadNodes
    inject_wrong_prefactor: bool = False


def selftest(opt: SelftestOptions = SelftestOptions(), out=None) -> bool:
    """The invariant battery of src/bench_runner.cpp:335-520 against the
    device path: GLL rule, expm/phiquad vs Taylor, phi recurrence, Tucker /
    Kronecker sum vs dense assembly, the GEMM core vs numpy, LU solve,
    splitting exact at l = 0 and second order for l = 1, 2 (d = 2, 3).  One
    [PASS]/[FAIL] line per check; returns True when all pass."""
    from . import api
    out = out or sys.stdout
    rng = np.random.default_rng(20230517)
    ok_all = [True]

    def check(name, ok, measured, bound):
        out.write(f"{'[PASS]' if ok else '[FAIL]'} {name} (measured {measured:g}, "
                  f"requires {bound})\n")
        ok_all[0] = ok_all[0] and bool(ok)

    def rmat(r, c, scale=1.0):
        return np.asfortranarray(rng.uniform(-scale, scale, (r, c)))

    def rstable(n, scale=1.0):
        m = rmat(n, n, scale)
        m -= np.abs(m).sum(0).max() * np.eye(n)
        return np.asfortranarray(m)

    q = opt.quad_nodes
    # quadrature rule
    worst_sum = worst_mono = 0.0
    for qq in range(2, 17):
        r = _it.gll_rule(qq)
        worst_sum = max(worst_sum, abs(r.weights.sum() - 1.0))
        for deg in range(0, 2 * qq - 2):
            worst_mono = max(worst_mono, abs(float(np.dot(r.weights, r.nodes ** deg))
                                             - 1.0 / (deg + 1)))
    check("gll weights sum to one (q=2..16)", worst_sum < 1e-14, worst_sum, "< 1e-14")
    check("gll exact on monomials up to degree 2q-3", worst_mono < 1e-13, worst_mono, "< 1e-13")
    # expm vs Taylor
    worst = 0.0
    for _ in range(3):
        x = rmat(8, 8)
        x *= 5.0 / np.abs(x).sum(0).max()
        want = _taylor_phi(x, 0)
        got = _it.expm(x)
        worst = max(worst, np.abs(got - want).sum(0).max() / np.abs(want).sum(0).max())
    check("expm matches Taylor oracle (8x8, norm 5)", worst < 1e-12, worst, "< 1e-12")
    # phiquad vs Taylor + recurrence
    worst = worst_rec = 0.0
    for nrm in (0.5, 3.0, 30.0):
        x = rmat(6, 6)
        x *= nrm / np.abs(x).sum(0).max()
        tab = _it.phiquad(x, 3, q)
        for ell in range(4):
            want = _taylor_phi(x, ell)
            worst = max(worst, np.abs(tab.phis[ell] - want).sum(0).max()
                        / np.abs(want).sum(0).max())
        for k in range(3):
            lhs = tab.phis[k]
            rhs = x @ tab.phis[k + 1] + np.eye(6) / math.factorial(k)
            worst_rec = max(worst_rec, np.abs(lhs - rhs).sum(0).max() / np.abs(lhs).sum(0).max())
    check("phiquad matches Taylor oracle (l <= 3, norm <= 30)", worst < 1e-11, worst, "< 1e-11")
    check("phi recurrence phi_k = X phi_{k+1} + I/k!", worst_rec < 1e-11, worst_rec, "< 1e-11")
    # tensor kernels vs dense assembly
    worst_t = worst_k = worst_g = 0.0
    for dims in ([3, 4], [2, 3, 4], [5, 2, 3]):
        v = np.asfortranarray(rng.uniform(-1, 1, dims))
        ms = [rmat(n, n) for n in dims]
        got = api.tucker(v, ms)
        want = (_kron_dense(ms) @ v.reshape(-1, order="F")).reshape(dims, order="F")
        worst_t = max(worst_t, np.linalg.norm(got - want) / np.linalg.norm(want))
        gotk = api.kronsum_action(v, api.KroneckerSum(ms))
        wantk = (_kronsum_dense(ms) @ v.reshape(-1, order="F")).reshape(dims, order="F")
        worst_k = max(worst_k, np.linalg.norm(gotk - wantk) / np.linalg.norm(wantk))
    for m_, n_, k_ in ((37, 41, 29), (130, 70, 300)):
        a = rmat(m_, k_)
        b = rmat(k_, n_)
        got = api.mode_product(np.asfortranarray(b), a, 0)  # a @ b on the DMMA GEMM
        want = a @ b
        worst_g = max(worst_g, np.abs(got - want).sum(0).max() / np.abs(want).sum(0).max())
    check("tucker matches dense Kronecker product", worst_t < 1e-13, worst_t, "< 1e-13")
    check("kronsum action matches dense assembly", worst_k < 1e-13, worst_k, "< 1e-13")
    check("blocked gemm matches naive reference", worst_g < 1e-13, worst_g, "< 1e-13")
    # LU
    worst = 0.0
    for _ in range(5):
        n = 20 + int(rng.integers(0, 180))
        a = rmat(n, n)
        x = rmat(n, 4)
        got = _it.solve(a, a @ x)
        worst = max(worst, np.abs(got - x).sum(0).max() / np.abs(x).sum(0).max())
    check("lu solve recovers random solutions", worst < 1e-10, worst, "< 1e-10")
    # splitting
    worst0 = 0.0
    for _ in range(5):
        fs = [rstable(4), rstable(5)]
        v = np.asfortranarray(rng.uniform(-1, 1, (4, 5)))
        sp = _it.build_split_phi(api.KroneckerSum(fs), 0.5, 0, q)
        got = _it.apply_split_phi(sp, v).reshape(-1, order="F")
        want = _taylor_phi(0.5 * _kronsum_dense(fs), 0) @ v.reshape(-1, order="F")
        worst0 = max(worst0, np.linalg.norm(got - want) / np.linalg.norm(want))
    check("splitting exact at l = 0", worst0 < 1e-12, worst0, "< 1e-12")
    for ell in (1, 2):
        for d in (2, 3):
            fs = [rstable(3 + mu) for mu in range(d)]
            dims = [3 + mu for mu in range(d)]
            v = np.asfortranarray(rng.uniform(-1, 1, dims))
            kd = _kronsum_dense(fs)
            taus, errs = [], []
            for e in range(3, 10):
                tau = 2.0 ** -e
                sp = _it.build_split_phi(api.KroneckerSum(fs), tau, ell, q)
                if opt.inject_wrong_prefactor:
                    sp.prefactor = float(math.factorial(ell) ** d)
                got = _it.apply_split_phi(sp, v).reshape(-1, order="F")
                want = _taylor_phi(tau * kd, ell) @ v.reshape(-1, order="F")
                taus.append(tau)
                errs.append(np.linalg.norm(got - want) / np.linalg.norm(want))
            slope = fit_order(taus, errs)
            check(f"splitting error order (l={ell}, d={d})", abs(slope - 2.0) <= 0.1, slope,
                  "2.0 +/- 0.1")
    out.write("selftest: all checks passed\n" if ok_all[0] else "selftest: FAILURES detected\n")
    return ok_all[0]
