"""Problem builders for the BASELINE configs (host numpy; column-major).

fd_operator_1d restates src/problems.cpp:9-22 (Dirichlet, h = 1/(n+1)).
The configs' PDEs are not in the reference; their
inputs follow SURVEY.md 8(d) with numpy-seeded synthetic data (seeds
1001-1005 for configs 1-5), fed identically to the oracle and the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .integrators import G, gfun, G_ALLEN_CAHN, G_BRUSSELATOR, G_NLS


def fd_operator_1d(n, eps, alpha=0.0):
    """eps*d2/dx2 + alpha*d/dx, 2nd-order central, n inner points of [0,1],
    homogeneous Dirichlet (src/problems.cpp:9-22)."""
    if n < 1:
        raise ValueError("fd_operator_1d: need n >= 1")
    h = 1.0 / (n + 1)
    lo = eps / (h * h) - alpha / (2.0 * h)
    di = -2.0 * eps / (h * h)
    hi = eps / (h * h) + alpha / (2.0 * h)
    a = np.zeros((n, n), order="F")
    i = np.arange(n)
    a[i, i] = di
    a[i[1:], i[:-1]] = lo
    a[i[:-1], i[1:]] = hi
    return a


def periodic_laplacian_1d(n, h):
    """(1/h^2) circ(1, -2, 1) (new: the reference is Dirichlet-only)."""
    c = 1.0 / (h * h)
    a = np.zeros((n, n), order="F")
    i = np.arange(n)
    a[i, i] = -2.0 * c
    a[i, (i + 1) % n] = c
    a[i, (i - 1) % n] = c
    return a


def grid(n):
    h = 1.0 / (n + 1)
    return (np.arange(n) + 1) * h


@dataclass
class Config:
    name: str
    method: str
    u0: np.ndarray
    K: List[np.ndarray]
    g: object
    tau: float
    n_steps: int
    t_end: Optional[float] = None  # exact T when tau = T / n_steps was given

    @property
    def t_final(self):
        return self.t_end if self.t_end is not None else self.tau * self.n_steps


def ac2d(n=128, n_steps=100, tau=1e-3, seed=1001):
    """configs[0]: 2-D Allen-Cahn u_t = 0.01 Lap u + u - u^3, exp-Euler."""
    r = np.random.default_rng(seed)
    x = grid(n)
    u0 = 0.4 * np.outer(np.sin(np.pi * x), np.sin(np.pi * x)) + 0.1 * r.uniform(-1, 1, (n, n))
    a = fd_operator_1d(n, 0.01)
    return Config("ac2d", "exp_euler", np.asfortranarray(u0), [a, a], G.allen_cahn(), tau,
                  n_steps)


def ac3d(n=128, n_steps=200, tau=5e-4, seed=1003):
    """configs[2]: 3-D Allen-Cahn, eps = 0.01 diffusion, ETD2RK."""
    r = np.random.default_rng(seed)
    x = np.sin(np.pi * grid(n))
    u0 = 0.4 * x[:, None, None] * x[None, :, None] * x[None, None, :] \
        + 0.1 * r.uniform(-1, 1, (n, n, n))
    a = fd_operator_1d(n, 0.01)
    return Config("ac3d", "etd2rk", np.asfortranarray(u0), [a, a, a], G.allen_cahn(), tau,
                  n_steps)


def _planes(n, planes):
    return range(n) if planes is None else range(planes[0], planes[1])


def brusselator(n=256, n_steps=100, tau=1e-3, method="etd2rk", seed=1004, a=1.0, b=3.0,
                diff=0.02, planes=None):
    """configs[3]: two species stacked as a 4th mode of size 2 (u first,
    v second) with a zero 2x2 factor -- the reference's own way to run it
    (SURVEY.md 8(c)); Dirichlet fd_operator_1d(n, 0.02) for both species.
    The noise of plane k (last spatial mode) comes from rng([seed, k]), so a
    slab `planes=(k0, k1)` is built without the rest (sharded runs)."""
    ks = _planes(n, planes)
    u0 = np.empty((n, n, len(ks), 2), order="F")
    for j, k in enumerate(ks):
        r = np.random.default_rng([seed, k])
        u0[:, :, j, 0] = a + 0.1 * r.uniform(-1, 1, (n, n))
        u0[:, :, j, 1] = b / a + 0.1 * r.uniform(-1, 1, (n, n))
    A = fd_operator_1d(n, diff)
    return Config("brusselator", method, u0, [A, A, A, np.zeros((2, 2), order="F")],
                  G.brusselator(a, b), tau, n_steps)


def nls(n=512, n_steps=50, tau=1e-3, method="etd2rk", seed=1005, k=(1.0, 0.5, 0.0),
        planes=None):
    """configs[4]: i u_t = -1/2 Lap u + |u|^2 u on [-8,8]^3 periodic, i.e.
    u' = (i/2) Lap u - i |u|^2 u; u0 = Gaussian wave packet (wave vector k)
    + 0.01 (N + iN) noise (plane k of the noise from rng([seed, k]))."""
    L = 16.0
    h = L / n
    x = -8.0 + h * np.arange(n)
    X, Y = np.meshgrid(x, x, indexing="ij")
    ks = _planes(n, planes)
    u0 = np.empty((n, n, len(ks)), dtype=np.complex128, order="F")
    for j, kk in enumerate(ks):
        z = x[kk]
        r = np.random.default_rng([seed, kk])
        u0[:, :, j] = np.exp(-(X * X + Y * Y + z * z) / 2.0) * \
            np.exp(1j * (k[0] * X + k[1] * Y + k[2] * z)) + \
            0.01 * (r.standard_normal((n, n)) + 1j * r.standard_normal((n, n)))
    A = 0.5j * periodic_laplacian_1d(n, h)
    return Config("nls", method, np.asfortranarray(u0), [A, A, A], G.nls(), tau, n_steps)


def adr(n1=40, n2=41, n3=42, n_steps=440, method="etd2rk", eps=0.75, alpha=0.1):
    """The reference's own benchmark problem (src/problems.cpp:45-128): 3-D
    advection-diffusion-reaction u_t = eps Lap u + alpha sum d_mu u + 1/(1+u^2)
    + Psi(t,x) on [0,1]^3 with the manufactured exact solution e^t u0,
    u0 = 64 x(1-x) y(1-y) z(1-z); T = 1 (tau = 1/n_steps).  Returns the
    Config plus the exact solution at T = 1."""
    p = lambda x: x * (1.0 - x)
    dp = lambda x: 1.0 - 2.0 * x
    gx = [grid(n) for n in (n1, n2, n3)]
    P = [p(x) for x in gx]
    D = [dp(x) for x in gx]
    p1, p2, p3 = P[0][:, None, None], P[1][None, :, None], P[2][None, None, :]
    d1, d2, d3 = D[0][:, None, None], D[1][None, :, None], D[2][None, None, :]
    u0 = 64.0 * p1 * p2 * p3
    lap = 64.0 * (-2.0) * (p2 * p3 + p1 * p3 + p1 * p2)
    adv = 64.0 * (d1 * p2 * p3 + d2 * p1 * p3 + d3 * p1 * p2)
    psi_a = np.asfortranarray(u0 - eps * lap - alpha * adv)
    u0 = np.asfortranarray(u0)
    K = [fd_operator_1d(n, eps, alpha) for n in (n1, n2, n3)]
    from .integrators import G
    g = G.adr(psi_a, np.asfortranarray(u0 * u0))
    cfg = Config("adr", method, u0, K, g, 1.0 / n_steps, n_steps)
    cfg.fields = (psi_a, np.asfortranarray(u0 * u0))
    cfg.exact = np.exp(1.0) * u0
    return cfg


def riccati(n_hat=30, n_steps=170, method="etd2rk", t_final=0.025, alpha=100.0):
    """The reference's LQR differential Riccati problem (src/problems.cpp:130-186,
    RiccatiProblem::to_problem_spec :252-283): U' = A^T U + U A + C + U B U on
    the n x n state, n = n_hat^2, with A = I (x) D1 + D2 (x) I (D1 = dxx - 10x dx,
    D2 = dyy - 100y dy, h = 1/(n_hat+1)), B = -b b^T, C = alpha c c^T (b, c
    indicators of x in (0.1,0.3] / (0.7,0.9]), U0 = 0, K = {A^T, A^T}.
    cfg.a_t = A^T; cfg.b, cfg.c_mat the g data."""
    if n_hat < 2:
        raise ValueError("build_riccati: need n_hat >= 2")
    h = 1.0 / (n_hat + 1)
    x = (np.arange(n_hat) + 1) * h
    a1, a2 = -10.0 * x, -100.0 * x
    d1 = np.zeros((n_hat, n_hat))
    d2 = np.zeros((n_hat, n_hat))
    i = np.arange(n_hat)
    d1[i, i] = -2.0 / (h * h)
    d2[i, i] = -2.0 / (h * h)
    d1[i[1:], i[1:] - 1] = 1.0 / (h * h) - a1[1:] / (2.0 * h)
    d2[i[1:], i[1:] - 1] = 1.0 / (h * h) - a2[1:] / (2.0 * h)
    d1[i[:-1], i[:-1] + 1] = 1.0 / (h * h) + a1[:-1] / (2.0 * h)
    d2[i[:-1], i[:-1] + 1] = 1.0 / (h * h) + a2[:-1] / (2.0 * h)
    eye = np.eye(n_hat)
    a = np.kron(eye, d1) + np.kron(d2, eye)  # rows i + j n_hat (x fastest)
    a_t = np.asfortranarray(a.T)
    b = np.tile(((x > 0.1) & (x <= 0.3)).astype(np.float64), n_hat)
    c = np.tile(((x > 0.7) & (x <= 0.9)).astype(np.float64), n_hat)
    c_mat = np.asfortranarray(np.outer(alpha * c, c))
    n = n_hat * n_hat
    from .integrators import G
    cfg = Config(f"riccati{n_hat}", method, np.zeros((n, n), order="F"), [a_t, a_t],
                 G.riccati(b, c_mat), t_final / n_steps, n_steps, t_final)
    cfg.a_t, cfg.b, cfg.c_mat = a_t, b, c_mat
    return cfg


def tucker_sweep(n, seed=1002, tau=1e-3):
    """configs[1]: V ~ N(0,1) and A = fd_operator_1d(n, 1.0) (L = phi_1(tau A))."""
    r = np.random.default_rng(seed)
    return np.asfortranarray(r.standard_normal((n, n, n))), fd_operator_1d(n, 1.0), tau
