// kp_g.cuh -- device evaluation of the closed set of nonlinearities g(t,u).
//
// Every operation is an explicitly rounded intrinsic (__dmul_rn, __dadd_rn,
// ...) so nvcc cannot contract it into an FMA: the values then match the CPU
// oracle's g (oracle/kp_oracle_impl.inc eval_g, compiled -ffp-contract=off)
// bit for bit.  The reference takes g as a host std::function
// (inc/integrators.hpp:60,112); the configs' g's are listed in SURVEY.md 8(a) a15.
#pragma once

#include "kronphi_b200.h"

namespace kp {

// Time of a g evaluation: absolute t, or (integrators) the device step
// counter's t0 + n tau plus the stage offset t.
__device__ __forceinline__ double g_time(const kp_gfun& g, double t) {
  return g.step_ctr ? g.t0 + double(*g.step_ctr) * g.tau + t : t;
}

// Real g at one entry.  x = u at this entry; partner = the other species'
// value at the same grid point (Brusselator only); second = whether this
// entry belongs to the second species (v); idx = the entry's linear index
// (auxiliary fields); t = time argument (see g_time).
__device__ __forceinline__ double g_real(const kp_gfun& g, double x, double partner, bool second,
                                         long long idx, double t) {
  switch (g.kind) {
    case KP_G_ADR: {  // src/problems.cpp:101-115 (FMA where g++ contracts a*b + c)
      const double et = exp(g_time(g, t));
      const double e2t = __dmul_rn(et, et);
      const double a = __ddiv_rn(1.0, __fma_rn(x, x, 1.0));
      const double b = __ddiv_rn(1.0, __fma_rn(e2t, g.aux[1][idx], 1.0));
      return __dsub_rn(__fma_rn(et, g.aux[0][idx], a), b);
    }
    case KP_G_SQUARE:
      return __dmul_rn(x, x);
    case KP_G_CONST:
      return g.p[0];
    case KP_G_ALLEN_CAHN:
      return __dsub_rn(x, __dmul_rn(__dmul_rn(x, x), x));
    case KP_G_BRUSSELATOR: {
      // u = first species, v = second; g = (a-(b+1)u+u^2 v, b u - u^2 v)
      const double u = second ? partner : x;
      const double v = second ? x : partner;
      const double uuv = __dmul_rn(__dmul_rn(u, u), v);
      if (!second) return __dadd_rn(__dsub_rn(g.p[0], __dmul_rn(__dadd_rn(g.p[1], 1.0), u)), uuv);
      return __dsub_rn(__dmul_rn(g.p[1], u), uuv);
    }
    default:  // KP_G_ZERO
      return 0.0;
  }
}

// Complex g at one entry (interleaved re/im).
__device__ __forceinline__ double2 g_cplx(const kp_gfun& g, double2 u) {
  switch (g.kind) {
    case KP_G_NLS: {  // -i |u|^2 u
      const double m = __dadd_rn(__dmul_rn(u.x, u.x), __dmul_rn(u.y, u.y));
      return make_double2(__dmul_rn(m, u.y), -__dmul_rn(m, u.x));
    }
    case KP_G_SQUARE:
      return make_double2(__dsub_rn(__dmul_rn(u.x, u.x), __dmul_rn(u.y, u.y)),
                          __dadd_rn(__dmul_rn(u.x, u.y), __dmul_rn(u.y, u.x)));
    case KP_G_CONST:
      return make_double2(g.p[0], 0.0);
    default:
      return make_double2(0.0, 0.0);
  }
}

}  // namespace kp
