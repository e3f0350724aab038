// kp_epilogue.cuh -- the fused GEMM epilogues shared by the mode-product
// kernels (mode_product.cu: hand-written mainloop; gemm_cutlass.cu: CUTLASS
// mainloop).  See Epilogue in kp_internal.h.
#pragma once

#include "kp_g.cuh"
#include "kp_internal.h"

namespace kp {
namespace {

// Fused exchange (kp_scatter): destination of entry `elem` of the local output
// tensor (comps doubles per entry) in its owner's receive buffer.
//   dir 1: slab (A, B, C/P, S)  -> pencil of rank b / (B/P)
//   dir 2: pencil (A, B/P, C, S) -> slab of rank c / (C/P)
__device__ __forceinline__ double* scatter_ptr(const Epilogue& e, unsigned elem, int comps) {
  const unsigned A = e.sc_A, B = e.sc_B, C = e.sc_C, P = unsigned(e.sc_P), r = unsigned(e.sc_rank);
  const unsigned Bp = B / P, Cl = C / P;
  const unsigned t = elem / A, a = elem - t * A;
  unsigned s;
  unsigned long long idx;
  if (e.sc_dir == 1) {
    const unsigned t2 = t / B, b = t - t2 * B;
    const unsigned sp = t2 / Cl, cl = t2 - sp * Cl;
    s = b / Bp;
    idx = a + (unsigned long long)A * ((b - s * Bp) + (unsigned long long)Bp * (r * Cl + cl + (unsigned long long)C * sp));
  } else {
    const unsigned t2 = t / Bp, bl = t - t2 * Bp;
    const unsigned sp = t2 / C, c = t2 - sp * C;
    s = c / Cl;
    idx = a + (unsigned long long)A * ((r * Bp + bl) + (unsigned long long)B * ((c - s * Cl) + (unsigned long long)Cl * sp));
  }
  return e.sc_peers[s] + idx * comps;
}

// Store a real pair (entries elem, elem+1 of the local output; `two` = the
// second exists) either into C or, with a scatter, to the owners' buffers.
template <bool SCAT>
__device__ __forceinline__ void store_pair(const Epilogue& e, double* c, unsigned long long elem,
                                           double r0, double r1, bool two, int c_vec2) {
  if constexpr (SCAT) {
    double* p0 = scatter_ptr(e, unsigned(elem), 1);
    if (two) {
      // same destination run when elem is even and A is even (pairs never
      // straddle a row of A then); 16-byte aligned then too
      if ((e.sc_A % 2 == 0) && (elem % 2 == 0)) {
        *reinterpret_cast<double2*>(p0) = make_double2(r0, r1);
      } else {
        *p0 = r0;
        *scatter_ptr(e, unsigned(elem + 1), 1) = r1;
      }
    } else {
      *p0 = r0;
    }
    return;
  }
  if (two) {
    if (c_vec2) {
      *reinterpret_cast<double2*>(c) = make_double2(r0, r1);
    } else {
      c[0] = r0;
      c[1] = r1;
    }
  } else {
    c[0] = r0;
  }
}

// Epilogue on one output entry.  v = alpha*acc; idx = linear index into C
// (and X/D, which share C's layout).
__device__ __forceinline__ double epi_one(const Epilogue& e, double v, const double* C,
                                          long long idx, long long half, double* dval) {
  switch (e.kind) {
    case EPI_FMA_X:
      return __fma_rn(e.gamma, v, e.X[idx]);
    case EPI_ADD_G: {
      const double base = (e.beta != 0.0) ? __fma_rn(e.beta, C[idx], v) : v;
      const bool second = half > 0 && idx >= half;
      const double partner = half > 0 ? e.X[second ? idx - half : idx + half] : 0.0;
      return __dadd_rn(base, g_real(e.g, e.X[idx], partner, second, idx, e.t));
    }
    case EPI_ADD_X: {
      const double base = (e.beta != 0.0) ? __fma_rn(e.beta, C[idx], v) : v;
      return __dadd_rn(base, e.X[idx]);
    }
    case EPI_STAGE_D: {
      const double x = e.X[idx];
      const double s = __fma_rn(e.gamma, v, x);
      *dval = __dsub_rn(g_real(e.g, s, 0.0, false, idx, e.t2), g_real(e.g, x, 0.0, false, idx, e.t));
      return s;
    }
    default:
      return (e.beta != 0.0) ? __fma_rn(e.beta, C[idx], v) : v;
  }
}

// Complex epilogue on one (re, im) pair; idx = real index of the re part.
__device__ __forceinline__ double2 epi_pair_c(const Epilogue& e, double2 v, const double* C,
                                              long long idx, double2* dval) {
  switch (e.kind) {
    case EPI_FMA_X:
      return make_double2(__fma_rn(e.gamma, v.x, e.X[idx]), __fma_rn(e.gamma, v.y, e.X[idx + 1]));
    case EPI_ADD_G: {
      double2 b = v;
      if (e.beta != 0.0) b = make_double2(__fma_rn(e.beta, C[idx], v.x), __fma_rn(e.beta, C[idx + 1], v.y));
      const double2 gx = g_cplx(e.g, make_double2(e.X[idx], e.X[idx + 1]));
      return make_double2(__dadd_rn(b.x, gx.x), __dadd_rn(b.y, gx.y));
    }
    case EPI_ADD_X: {
      double2 b = v;
      if (e.beta != 0.0) b = make_double2(__fma_rn(e.beta, C[idx], v.x), __fma_rn(e.beta, C[idx + 1], v.y));
      return make_double2(__dadd_rn(b.x, e.X[idx]), __dadd_rn(b.y, e.X[idx + 1]));
    }
    case EPI_STAGE_D: {
      const double2 x = make_double2(e.X[idx], e.X[idx + 1]);
      const double2 st = make_double2(__fma_rn(e.gamma, v.x, x.x), __fma_rn(e.gamma, v.y, x.y));
      const double2 gs = g_cplx(e.g, st), gx = g_cplx(e.g, x);
      *dval = make_double2(__dsub_rn(gs.x, gx.x), __dsub_rn(gs.y, gx.y));
      return st;
    }
    default:
      if (e.beta != 0.0)
        return make_double2(__fma_rn(e.beta, C[idx], v.x), __fma_rn(e.beta, C[idx + 1], v.y));
      return v;
  }
}

}  // namespace
}  // namespace kp
