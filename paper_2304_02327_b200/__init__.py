"""kronphi-b200: B200-native (sm_100a) direction-split phi-function action of
arXiv 2304.02327 -- the mu-mode/Tucker operator, the small-matrix phi_l
factors and the exponential Euler / ETD2RK / Lawson steppers, behind the C ABI
in include/kronphi_b200.h (libkronphi_b200.so, hand-written DMMA kernels).

The Python surface mirrors the reference C++ API (proj/include/kronphi/);
there is no CPU fallback -- a missing library or GPU raises.
"""
from ._lib import (DivergenceError, InvalidArgument, KronphiError, CudaError, Context,
                   default_context, LIB_PATH)
from .api import (KroneckerSum, fortran_empty, fortran_zeros, kronsum_action, mode_product,
                  mode_product_into, to_device, to_host, tucker)
from .integrators import (G, G_ADR, G_ALLEN_CAHN, G_BRUSSELATOR, G_CONST, G_NLS, G_RICCATI,
                          G_SQUARE, G_ZERO, eval_g, rosenbrock_euler_step, solve,
                          GLLRule, IntegrateResult, Method, PhiTable, ProblemSpec, SplitPhi,
                          StepperConfig, apply_split_phi, build_split_phi, etd2rk_step,
                          exp_euler_linear_split_step, exp_euler_step, expm, gfun, gll_rule,
                          integrate, integrate_config, kDefaultQuadNodes, lawson2b_step,
                          lawson_euler_step, method_name, parse_method, phiquad)

__all__ = [
    "DivergenceError", "InvalidArgument", "KronphiError", "CudaError", "Context",
    "default_context", "LIB_PATH", "KroneckerSum", "fortran_empty", "fortran_zeros",
    "kronsum_action", "mode_product", "mode_product_into", "to_device", "to_host", "tucker",
    "G", "G_ADR", "G_RICCATI", "eval_g", "rosenbrock_euler_step", "solve", "G_ALLEN_CAHN", "G_BRUSSELATOR", "G_CONST", "G_NLS", "G_SQUARE", "G_ZERO", "GLLRule",
    "IntegrateResult", "Method", "PhiTable", "ProblemSpec", "SplitPhi", "StepperConfig",
    "apply_split_phi", "build_split_phi", "etd2rk_step", "exp_euler_linear_split_step",
    "exp_euler_step", "expm", "gfun", "gll_rule", "integrate", "integrate_config",
    "kDefaultQuadNodes", "lawson2b_step", "lawson_euler_step", "method_name", "parse_method",
    "phiquad",
]
