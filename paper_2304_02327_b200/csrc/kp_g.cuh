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

// Real g at one entry.  x = u at this entry; partner = the other species'
// value at the same grid point (Brusselator only); second = whether this
// entry belongs to the second species (v).
__device__ __forceinline__ double g_real(const kp_gfun& g, double x, double partner,
                                         bool second) {
  switch (g.kind) {
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
