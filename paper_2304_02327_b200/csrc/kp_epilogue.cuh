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

// Finite test on the integer pipe (the FP64 datapath belongs to the DMMAs).
__device__ __forceinline__ bool fin(double x) {
  return (__double_as_longlong(x) & 0x7ff0000000000000LL) != 0x7ff0000000000000LL;
}

// Per-launch uniform facts of an Epilogue, evaluated once per thread instead
// of per entry (a per-entry `beta != 0` is a DSETP that waits behind the
// other warps' DMMAs on the shared FP64 datapath).
struct EpiU {
  bool beta;   // beta != 0: accumulate into C
  bool one;    // alpha == 1: v = acc exactly
  bool track;  // divergence tracking on
};
__device__ __forceinline__ EpiU epi_uniform(const Epilogue& e) {
  return EpiU{e.beta != 0.0, e.alpha == 1.0, e.bad_step != nullptr};
}

// The global inputs an epilogue kind reads for one output entry, loaded
// ahead of the arithmetic: the staged loops below issue the loads of several
// entries before the first use, so each thread has several HBM reads in
// flight instead of one dependent load per entry.
struct EpiIn {
  double c = 0.0, x = 0.0, p = 0.0;  // beta * C operand, X, species partner of X
};
__device__ __forceinline__ EpiIn epi_load(const Epilogue& e, const EpiU& u, const double* C,
                                          long long idx, long long half) {
  EpiIn in;
  switch (e.kind) {
    case EPI_FMA_X:
    case EPI_STAGE_D:
      in.x = e.X[idx];
      break;
    case EPI_ADD_G:
      if (u.beta) in.c = C[idx];
      in.x = e.X[idx];
      if (half > 0) in.p = e.X[idx >= half ? idx - half : idx + half];
      break;
    case EPI_ADD_X:
      if (u.beta) in.c = C[idx];
      in.x = e.X[idx];
      break;
    default:
      if (u.beta) in.c = C[idx];
  }
  return in;
}

// Epilogue arithmetic on one output entry.  v = alpha*acc; idx = linear
// index into C (and X/D, which share C's layout).
__device__ __forceinline__ double epi_apply(const Epilogue& e, const EpiU& u, double v,
                                            const EpiIn& in, long long idx, long long half,
                                            double* dval) {
  switch (e.kind) {
    case EPI_FMA_X:
      return __fma_rn(e.gamma, v, in.x);
    case EPI_ADD_G: {
      const double base = u.beta ? __fma_rn(e.beta, in.c, v) : v;
      const bool second = half > 0 && idx >= half;
      return __dadd_rn(base, g_real(e.g, in.x, in.p, second, idx, e.t));
    }
    case EPI_ADD_X: {
      const double base = u.beta ? __fma_rn(e.beta, in.c, v) : v;
      return __dadd_rn(base, in.x);
    }
    case EPI_STAGE_D: {
      const double s = __fma_rn(e.gamma, v, in.x);
      *dval = __dsub_rn(g_real(e.g, s, 0.0, false, idx, e.t2), g_real(e.g, in.x, 0.0, false, idx, e.t));
      return s;
    }
    default:
      return u.beta ? __fma_rn(e.beta, in.c, v) : v;
  }
}

// epi_load + epi_apply in one switch (the per-entry form of fused01.cu; the
// same operations in the same order, so the two forms agree bit for bit --
// one switch keeps that kernel's epilogue branch-light).
__device__ __forceinline__ double epi_one(const Epilogue& e, const EpiU& u, double v,
                                          const double* C, long long idx, long long half,
                                          double* dval) {
  switch (e.kind) {
    case EPI_FMA_X:
      return __fma_rn(e.gamma, v, e.X[idx]);
    case EPI_ADD_G: {
      const double base = u.beta ? __fma_rn(e.beta, C[idx], v) : v;
      const bool second = half > 0 && idx >= half;
      const double partner = half > 0 ? e.X[second ? idx - half : idx + half] : 0.0;
      return __dadd_rn(base, g_real(e.g, e.X[idx], partner, second, idx, e.t));
    }
    case EPI_ADD_X: {
      const double base = u.beta ? __fma_rn(e.beta, C[idx], v) : v;
      return __dadd_rn(base, e.X[idx]);
    }
    case EPI_STAGE_D: {
      const double x = e.X[idx];
      const double s = __fma_rn(e.gamma, v, x);
      *dval = __dsub_rn(g_real(e.g, s, 0.0, false, idx, e.t2), g_real(e.g, x, 0.0, false, idx, e.t));
      return s;
    }
    default:
      return u.beta ? __fma_rn(e.beta, C[idx], v) : v;
  }
}

// Complex entry (re, im at idx, idx + 1; idx even, so 16-byte loads).
struct EpiInC {
  double2 c = make_double2(0.0, 0.0), x = make_double2(0.0, 0.0);
};
__device__ __forceinline__ EpiInC epi_load_c(const Epilogue& e, const EpiU& u, const double* C,
                                             long long idx) {
  EpiInC in;
  if (e.kind != EPI_FMA_X && e.kind != EPI_STAGE_D && u.beta)
    in.c = *reinterpret_cast<const double2*>(C + idx);
  if (e.kind != EPI_STORE) in.x = *reinterpret_cast<const double2*>(e.X + idx);
  return in;
}
__device__ __forceinline__ double2 epi_apply_c(const Epilogue& e, const EpiU& u, double2 v,
                                               const EpiInC& in, double2* dval) {
  switch (e.kind) {
    case EPI_FMA_X:
      return make_double2(__fma_rn(e.gamma, v.x, in.x.x), __fma_rn(e.gamma, v.y, in.x.y));
    case EPI_ADD_G: {
      double2 b = v;
      if (u.beta) b = make_double2(__fma_rn(e.beta, in.c.x, v.x), __fma_rn(e.beta, in.c.y, v.y));
      const double2 gx = g_cplx(e.g, in.x);
      return make_double2(__dadd_rn(b.x, gx.x), __dadd_rn(b.y, gx.y));
    }
    case EPI_ADD_X: {
      double2 b = v;
      if (u.beta) b = make_double2(__fma_rn(e.beta, in.c.x, v.x), __fma_rn(e.beta, in.c.y, v.y));
      return make_double2(__dadd_rn(b.x, in.x.x), __dadd_rn(b.y, in.x.y));
    }
    case EPI_STAGE_D: {
      const double2 st = make_double2(__fma_rn(e.gamma, v.x, in.x.x), __fma_rn(e.gamma, v.y, in.x.y));
      const double2 gs = g_cplx(e.g, st), gx = g_cplx(e.g, in.x);
      *dval = make_double2(__dsub_rn(gs.x, gx.x), __dsub_rn(gs.y, gx.y));
      return st;
    }
    default:
      if (u.beta)
        return make_double2(__fma_rn(e.beta, in.c.x, v.x), __fma_rn(e.beta, in.c.y, v.y));
      return v;
  }
}

}  // namespace
}  // namespace kp

namespace kp {
namespace {

// The fused epilogue of one output tile of C staged in shared memory as a
// column-major TM x TN block (pitch LDS doubles; element (ml, nl) is
// alpha-less acc of C(m0 + ml, n0 + nl) of batch q).  NTH threads walk (m,
// m+1) pairs with consecutive threads on consecutive m: coalesced 16-byte
// stores and one copy of the epilogue code.  CPLX: 0 real; 1 rows are (re,
// im) pairs (complex mode 0); 2 rows 2p/2p+1 = re/im of the tensor, columns
// 2i/2i+1 = re/im of the factor, combined as (rr - ii, ri + ir) at complex
// offset p + i*P (complex modes >= 1).  Returns whether a non-finite value
// was written (the divergence flag).
//
// FLAT (real, no scatter): the tile's rows are rows of the stacked (batch x M)
// matrix -- rows ml < rb belong to batch q (row m0 + ml), rows ml >= rb to
// batch q + 1 (row ml - rb); rb is even, so (m, m+1) pairs never straddle.
template <int TM, int TN, int LDS, int NTH, int CPLX, bool SCAT, int EU = 4, bool FLAT = false>
__device__ __forceinline__ bool staged_epilogue(const GemmProblem& p, const Epilogue& e,
                                                const double* __restrict__ cs, int m0, int n0,
                                                long long q, int tid, int c_vec2,
                                                long long species_half, int rb = 0) {
  static_assert(!FLAT || (CPLX == 0 && !SCAT), "flat row blocks: real, unscattered tiles");
  double* __restrict__ Cb = p.C + q * p.sC;
  const long long cq = q * p.sC;
  const bool next_ok = q + 1 < p.batch;  // FLAT: the tile's second batch exists
  bool nonfinite = false;
  const EpiU u = epi_uniform(e);
  const double al = e.alpha;
  if constexpr (CPLX == 0 && !SCAT) {
    // plain store (a mode product of a Tucker operator): the decisions are
    // uniform, so no per-entry FP64 compare -- the FP64 datapath is the
    // DMMA's, and epilogue DSETP/DMUL stall behind the other warps' DMMAs
    if (e.kind == EPI_STORE && !u.beta && !u.track) {
      const bool one = u.one;
#pragma unroll 2
      for (int e2 = tid; e2 < TM * TN / 2; e2 += NTH) {
        const int ml = 2 * (e2 % (TM / 2)), nl = e2 / (TM / 2);
        int mrow = m0 + ml;
        const int ncol = n0 + nl;
        double* Cq = Cb;
        if constexpr (FLAT) {
          if (ml >= rb) {
            if (!next_ok) continue;
            mrow = ml - rb;
            Cq = Cb + p.sC;
          }
        }
        if (mrow >= p.M || ncol >= p.N) continue;
        double2 a2 = *reinterpret_cast<const double2*>(cs + ml + nl * LDS);
        if (!one) a2 = make_double2(al * a2.x, al * a2.y);
        double* dst = Cq + mrow + (long long)ncol * p.ldc;
        if (mrow + 1 < p.M) {
          if (c_vec2)
            *reinterpret_cast<double2*>(dst) = a2;
          else {
            dst[0] = a2.x;
            dst[1] = a2.y;
          }
        } else {
          dst[0] = a2.x;
        }
      }
      return false;
    }
  }
  // Batches of EU entries per thread: all global loads of a batch are issued
  // before its arithmetic and stores (program order keeps them ahead), so a
  // thread has EU x (1-3) reads in flight rather than one dependent read.
  // (EU is smaller where the DMMA accumulators leave few registers.)
  if constexpr (CPLX == 2) {
    constexpr int TOT = (TM / 2) * (TN / 2);
#pragma unroll 1
    for (int b0 = tid; b0 < TOT; b0 += EU * NTH) {
      EpiInC in[EU];
      long long off[EU];
      bool ok[EU];
#pragma unroll
      for (int j = 0; j < EU; ++j) {
        const int e2 = b0 + j * NTH;
        const int pl = e2 % (TM / 2), il = e2 / (TM / 2);
        const int mrow = m0 + 2 * pl, ncol = n0 + 2 * il;
        ok[j] = e2 < TOT && mrow < p.M && ncol < p.N;
        off[j] = mrow + (long long)(ncol >> 1) * p.ldc;
        if (ok[j]) in[j] = epi_load_c(e, u, p.C, cq + off[j]);
      }
#pragma unroll
      for (int j = 0; j < EU; ++j) {
        if (!ok[j]) continue;
        const int e2 = b0 + j * NTH;
        const int pl = e2 % (TM / 2), il = e2 / (TM / 2);
        const double* c0 = cs + 2 * pl + 2 * il * LDS;
        // 3M products staged by the mainloop (gemm_dmma.cu): P1 = re re at
        // (even, even), P2 = im im at (odd, odd), P3 = (re+im)(re+im) at (even, odd)
        const double c_rr = c0[0], c_p3 = c0[LDS], c_ii = c0[LDS + 1];
        double2 v = make_double2(__dsub_rn(c_rr, c_ii), __dsub_rn(__dsub_rn(c_p3, c_rr), c_ii));
        if (!u.one) v = make_double2(al * v.x, al * v.y);
        double2 dv = make_double2(0.0, 0.0);
        const double2 rr = epi_apply_c(e, u, v, in[j], &dv);
        double* dst = Cb + off[j];
        if constexpr (SCAT) dst = scatter_ptr(e, unsigned((cq + off[j]) >> 1), 2);
        *reinterpret_cast<double2*>(dst) = rr;
        if (u.track) nonfinite |= !fin(rr.x) || !fin(rr.y);
        if (e.kind == EPI_STAGE_D) *reinterpret_cast<double2*>(e.D + cq + off[j]) = dv;
      }
    }
    return nonfinite;
  }
  constexpr int TOT = TM * TN / 2;
#pragma unroll 1
  for (int b0 = tid; b0 < TOT; b0 += EU * NTH) {
    long long off[EU];
    bool ok[EU], two[EU];
    EpiIn in0[EU], in1[EU];
    EpiInC inc[EU];
#pragma unroll
    for (int j = 0; j < EU; ++j) {
      const int e2 = b0 + j * NTH;
      const int ml = 2 * (e2 % (TM / 2)), nl = e2 / (TM / 2);
      int mrow = m0 + ml;
      const int ncol = n0 + nl;
      bool qok = true;
      long long shift = 0;  // FLAT: rows of the next batch
      if constexpr (FLAT) {
        if (ml >= rb) {
          mrow = ml - rb;
          shift = p.sC;
          qok = next_ok;
        }
      }
      ok[j] = qok && e2 < TOT && mrow < p.M && ncol < p.N;
      two[j] = mrow + 1 < p.M;
      off[j] = shift + mrow + (long long)ncol * p.ldc;
      if (!ok[j]) continue;
      if constexpr (CPLX == 1) {
        inc[j] = epi_load_c(e, u, p.C, cq + off[j]);
      } else {
        in0[j] = epi_load(e, u, p.C, cq + off[j], species_half);
        if (two[j]) in1[j] = epi_load(e, u, p.C, cq + off[j] + 1, species_half);
      }
    }
#pragma unroll
    for (int j = 0; j < EU; ++j) {
      if (!ok[j]) continue;
      const int e2 = b0 + j * NTH;
      const int ml = 2 * (e2 % (TM / 2)), nl = e2 / (TM / 2);
      const long long o = cq + off[j];
      const double2 a2 = *reinterpret_cast<const double2*>(cs + ml + nl * LDS);
      const double v0 = u.one ? a2.x : al * a2.x, v1 = u.one ? a2.y : al * a2.y;
      if constexpr (CPLX == 1) {
        double2 dv = make_double2(0.0, 0.0);
        const double2 rr = epi_apply_c(e, u, make_double2(v0, v1), inc[j], &dv);
        double* dst = Cb + off[j];
        if constexpr (SCAT) dst = scatter_ptr(e, unsigned(o >> 1), 2);
        *reinterpret_cast<double2*>(dst) = rr;
        if (u.track) nonfinite |= !fin(rr.x) || !fin(rr.y);
        if (e.kind == EPI_STAGE_D) *reinterpret_cast<double2*>(e.D + o) = dv;
      } else {
        double d0 = 0.0, d1 = 0.0;
        const double r0 = epi_apply(e, u, v0, in0[j], o, species_half, &d0);
        double r1 = 0.0;
        if (two[j]) r1 = epi_apply(e, u, v1, in1[j], o + 1, species_half, &d1);
        if (u.track) nonfinite |= !fin(r0) || (two[j] && !fin(r1));
        store_pair<SCAT>(e, Cb + off[j], (unsigned long long)o, r0, r1, two[j], c_vec2);
        if (e.kind == EPI_STAGE_D) {
          if (two[j] && c_vec2) {
            *reinterpret_cast<double2*>(e.D + o) = make_double2(d0, d1);
          } else {
            e.D[o] = d0;
            if (two[j]) e.D[o + 1] = d1;
          }
        }
      }
    }
  }
  return nonfinite;
}

}  // namespace
}  // namespace kp
