// banded.cu -- the Kronecker-sum action for banded factors as one stencil pass.
//
// SURVEY.md 8(f) row 1.  In every BASELINE config the A_mu are tridiagonal
// (fd_operator_1d, src/problems.cpp:9-22) or periodic tridiagonal (NLS), yet
// kronsum_action (inc/mode_product.hpp:111-121) multiplies them densely: d
// GEMMs of 2 N n FLOP.  With at most three nonzeros per row the action is a
// (2d+1)-point stencil: one HBM-bound pass that reads u and writes r.
//
// Rounding follows the reference's dense CPU GEMM exactly: per output entry
// and mode the k loop is an FMA chain in increasing column order (the zero
// products of the dense loop add nothing), restarted at every KC = 256 slice
// boundary and folded into C like compute_tile (inc/kernels.hpp:241-263,
// :297); mode 0 stores, modes >= 1 accumulate (beta = 1, :65).  So for real
// data this pass reproduces the reference's kronsum_action bit for bit (the
// dense DMMA path agrees only to roundoff).  The optional g(t,u) of the
// ETD2RK / exp-Euler prologue is added last, as the reference's axpy does.
//
// Band detection (once per factor): a device scan collects, per row, up to
// three (column, value) pairs in increasing column order; more nonzeros =>
// not banded (dense path).
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "kp_g.cuh"
#include "kp_internal.h"
#include "kp_launch.cuh"

namespace kp {
namespace {

constexpr int KC = 256;  // inc/kernels.hpp:104

// rows of A (n x n, column-major; complex when comps == 2) -> 3 slots per row
// in increasing column order.  One warp per row: lanes test 32 columns at a
// time and the ballot hands the nonzeros out in order.  flags[0] |= 1 if a
// row has more than three nonzeros, flags[1] |= 1 if the factor has any.
__global__ void band_scan_kernel(const double* __restrict__ a, int n, int comps,
                                 int* __restrict__ cols, double* __restrict__ vals,
                                 int* __restrict__ flags) {
  const int i = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
  int cnt = 0;
  bool many = false;
  for (int j0 = 0; j0 < n && !many; j0 += 32) {
    const int j = j0 + lane;
    double re = 0.0, im = 0.0;
    if (j < n) {
      re = a[(size_t(i) + size_t(j) * n) * comps];
      if (comps == 2) im = a[(size_t(i) + size_t(j) * n) * comps + 1];
    }
    unsigned m = __ballot_sync(0xffffffffu, re != 0.0 || im != 0.0);
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      if (cnt == 3) {
        many = true;
        break;
      }
      if (lane == bit) {
        cols[i * 3 + cnt] = j;
        vals[(i * 3 + cnt) * 2] = re;
        vals[(i * 3 + cnt) * 2 + 1] = im;
      }
      ++cnt;
    }
  }
  if (lane == 0) {
    if (many) atomicOr(flags, 1);
    if (cnt > 0) atomicOr(flags + 1, 1);
    for (int c = cnt; c < 3 && !many; ++c) cols[i * 3 + c] = -1;
  }
}

struct BandArgs {
  int d;
  int n[4];               // output (interior) extents
  long long stride[4];    // input strides (the input may carry halo planes)
  const int* cols[4];
  const double* vals[4];  // (re, im) pairs
  int active[4];
  // slab sharding: mode `slab` holds global planes k0.. of n_glob with `halo`
  // extra planes on each side in the input; -1 = unsharded
  int slab, k0, n_glob, halo;
  int species;            // index of the 2-species mode for a coupled g, -1 none
};

// input offset (in elements of `stride[mu]`) of column j relative to row i
__device__ __forceinline__ long long col_off(const BandArgs& b, int mu, int i, int j) {
  if (mu != b.slab) return (long long)(j - i);
  const int lo = b.k0 - b.halo;
  int loc = (j - lo) % b.n_glob;
  if (loc < 0) loc += b.n_glob;
  return (long long)(loc - (i - lo));
}

// Adds one mode's term at entry idx into the running value c: the
// reference's FMA chain per KC slice, each slice folded as c = c + acc
// (mode 0's first slice stores: has_c == false).
__device__ __forceinline__ void term_real(const BandArgs& b, int mu, int imu, long long idx,
                                          const double* __restrict__ u, double& c, bool& has_c) {
  // imu: GLOBAL row of mode mu; idx: input index of the entry
  const int* cs = b.cols[mu] + imu * 3;
  const double* v = b.vals[mu] + imu * 6;
  double acc = 0.0;
  int slice = -1;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int j = cs[s];
    if (j < 0) break;
    const int sl = j / KC;
    if (sl != slice) {
      if (slice >= 0) {
        c = has_c ? __dadd_rn(c, acc) : acc;
        has_c = true;
      }
      slice = sl;
      acc = 0.0;
    }
    acc = __fma_rn(v[2 * s], u[idx + col_off(b, mu, imu, j) * b.stride[mu]], acc);
  }
  if (slice >= 0) {
    c = has_c ? __dadd_rn(c, acc) : acc;
    has_c = true;
  }
}

__device__ __forceinline__ double2 cmul_add(double2 a, double2 x, double2 acc) {
  // acc + a*x with the product formed first (generic complex micro-kernel)
  const double re = __dsub_rn(__dmul_rn(a.x, x.x), __dmul_rn(a.y, x.y));
  const double im = __dadd_rn(__dmul_rn(a.x, x.y), __dmul_rn(a.y, x.x));
  return make_double2(__dadd_rn(acc.x, re), __dadd_rn(acc.y, im));
}

__device__ __forceinline__ void term_cplx(const BandArgs& b, int mu, int imu, long long idx,
                                          const double2* __restrict__ u, double2& c,
                                          bool& has_c) {
  const int* cs = b.cols[mu] + imu * 3;
  const double* v = b.vals[mu] + imu * 6;
  double2 acc = make_double2(0.0, 0.0);
  int slice = -1;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int j = cs[s];
    if (j < 0) break;
    const int sl = j / KC;
    if (sl != slice) {
      if (slice >= 0) {
        c = has_c ? make_double2(__dadd_rn(c.x, acc.x), __dadd_rn(c.y, acc.y)) : acc;
        has_c = true;
      }
      slice = sl;
      acc = make_double2(0.0, 0.0);
    }
    acc = cmul_add(make_double2(v[2 * s], v[2 * s + 1]),
                   u[idx + col_off(b, mu, imu, j) * b.stride[mu]], acc);
  }
  if (slice >= 0) {
    c = has_c ? make_double2(__dadd_rn(c.x, acc.x), __dadd_rn(c.y, acc.y)) : acc;
    has_c = true;
  }
}

// r = sum_mu u x_mu A_mu (+ g(t,u) when with_g), one output entry per thread
template <bool CPLX>
__global__ void kronsum_band_kernel(BandArgs b, long long total, const double* __restrict__ u,
                                    double* __restrict__ r, bool with_g, kp_gfun g, double t) {
  // entries < 2^32 (checked by the launcher): 32-bit index arithmetic
  for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < (unsigned)total;
       idx += gridDim.x * blockDim.x) {
    unsigned rem = idx;
    long long in = 0;
    int ii[4];
#pragma unroll
    for (int mu = 0; mu < 4; ++mu) {
      if (mu < b.d) {
        const unsigned q = rem / unsigned(b.n[mu]);
        ii[mu] = int(rem - q * unsigned(b.n[mu]));
        rem = q;
        in += (long long)(ii[mu] + (mu == b.slab ? b.halo : 0)) * b.stride[mu];
        if (mu == b.slab) ii[mu] += b.k0;  // global row for the factor lookup
      }
    }
    if constexpr (!CPLX) {
      double acc = 0.0;
      bool has = false;
#pragma unroll
      for (int mu = 0; mu < 4; ++mu) {
        if (mu >= b.d || !b.active[mu]) continue;
        term_real(b, mu, ii[mu], in, u, acc, has);
      }
      if (with_g) {
        int isp = 0;
#pragma unroll
        for (int mu = 0; mu < 4; ++mu)
          if (mu == b.species) isp = ii[mu];
        const bool second = b.species >= 0 && isp == 1;
        const double partner =
            b.species >= 0 ? u[second ? in - b.stride[b.species] : in + b.stride[b.species]] : 0.0;
        acc = __dadd_rn(acc, g_real(g, u[in], partner, second, idx, t));
      }
      r[idx] = acc;
    } else {
      const double2* uc = reinterpret_cast<const double2*>(u);
      double2 acc = make_double2(0.0, 0.0);
      bool has = false;
#pragma unroll
      for (int mu = 0; mu < 4; ++mu) {
        if (mu >= b.d || !b.active[mu]) continue;
        term_cplx(b, mu, ii[mu], in, uc, acc, has);
      }
      if (with_g) {
        const double2 gg = g_cplx(g, uc[in]);
        acc = make_double2(__dadd_rn(acc.x, gg.x), __dadd_rn(acc.y, gg.y));
      }
      reinterpret_cast<double2*>(r)[idx] = acc;
    }
  }
}


// ---- v2: the same arithmetic, laid out for the memory system ----
// One thread per (i0, i1) line, marching over a chunk of the slower modes
// (z = i2 + n2 * i3): the mode-0 / mode-1 row structures (offsets already
// multiplied by the strides, values, KC slice breaks) live in registers for
// the whole march, the mode-2 / mode-3 rows are block-uniform loads, warps
// read 32 consecutive entries (coalesced) and the neighbour planes come from
// L1/L2.  No integer divisions per entry, 32-bit output index arithmetic.
// With a 2-species g (Brusselator) each thread computes BOTH species of a
// grid point, so the partner value is the other centre (no extra HBM read).
template <bool CPLX>
struct BandRow {
  int off[3];  // (column - row) * stride, < 2^31 (checked by the launcher)
  typename std::conditional<CPLX, double2, double>::type v[3];
  int n;
  unsigned brk;  // bit s: entry s starts a new KC slice
};

template <bool CPLX>
__device__ __forceinline__ void load_row(const BandArgs& b, int mu, int i, BandRow<CPLX>& rw) {
  const int ig = (mu == b.slab) ? i + b.k0 : i;  // global row
  const int* cs = b.cols[mu] + ig * 3;
  const double* v = b.vals[mu] + ig * 6;
  rw.n = 0;
  rw.brk = 0;
  int prev = -1;
  // entries past n are padded with (offset 0, value 0): see row_combine
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    rw.off[s] = 0;
    if constexpr (CPLX)
      rw.v[s] = make_double2(0.0, 0.0);
    else
      rw.v[s] = 0.0;
  }
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int j = __ldg(cs + s);
    if (j < 0) break;
    const int sl = j / KC;
    if (s > 0 && sl != prev) rw.brk |= 1u << s;
    prev = sl;
    rw.off[s] = int(col_off(b, mu, ig, j) * b.stride[mu]);
    if constexpr (CPLX)
      rw.v[s] = make_double2(__ldg(v + 2 * s), __ldg(v + 2 * s + 1));
    else
      rw.v[s] = __ldg(v + 2 * s);
    rw.n = s + 1;
  }
}

// Gather the three u values of one row term (padded entries read the
// centre: offset 0) and fold them into c with the reference's rounding.
//
// Fast path (no KC break in the row): c + fma(v2, x2, fma(v1, x1, fma(v0,
// x0, 0))).  This equals term_real's chain exactly for finite data: the
// chain's accumulator is never -0 (it starts from +0, and an exact
// cancellation rounds to +0), so a padded fma(0, x, acc) = acc + (+-0)
// returns acc, an empty row adds +0 to a c that is never -0, and the first
// mode's 0 + acc is acc.  (A non-finite centre turns the padded products
// into NaN: only diverged states, which the step's finite check rejects
// either way.)  Rows that straddle a KC = 256 slice boundary take the
// general chain (uniform per warp for modes >= 1).
template <bool CPLX, typename T>
__device__ __forceinline__ void row_gather(const BandRow<CPLX>& rw, const T* __restrict__ u,
                                           unsigned in, T* x) {
#pragma unroll
  for (int s = 0; s < 3; ++s) x[s] = u[in + unsigned(rw.off[s])];
}

template <bool IMAG = false>
__device__ __forceinline__ void row_combine(const BandRow<false>& rw, const double* x, double& c) {
  if (rw.brk == 0) {
    const double acc = __fma_rn(rw.v[2], x[2], __fma_rn(rw.v[1], x[1], __fma_rn(rw.v[0], x[0], 0.0)));
    c = __dadd_rn(c, acc);
    return;
  }
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    if (s >= rw.n) break;
    if ((rw.brk >> s) & 1u) {
      c = __dadd_rn(c, acc);
      acc = 0.0;
    }
    acc = __fma_rn(rw.v[s], x[s], acc);
  }
  c = __dadd_rn(c, acc);
}

// IMAG: every value of the row is purely imaginary (a.x == +-0; the NLS
// factors i/2 * Laplacian).  a * x is then (-(a.y x.y), a.y x.x): the generic
// micro-kernel's two products with a.x are signed zeros, and adding a signed
// zero changes no value, so half of the FP64 work (4 of 8 operations per
// term, and the first term's add to the +0 accumulator) is dropped.  Every
// entry keeps its VALUE (== holds; only the sign of an exact zero can differ).
// The complex stencil is otherwise FP64-bound: ~80 DMUL/DADD per entry is 0.64
// ms of the FP64 pipe at 512^3, the HBM floor is 0.66 ms.
template <bool IMAG = false>
__device__ __forceinline__ void row_combine(const BandRow<true>& rw, const double2* x, double2& c) {
  double2 acc = make_double2(0.0, 0.0);
  if constexpr (IMAG) {
    if (rw.brk == 0) {
      double2 t = make_double2(-__dmul_rn(rw.v[0].y, x[0].y), __dmul_rn(rw.v[0].y, x[0].x));
#pragma unroll
      for (int s = 1; s < 3; ++s)
        t = make_double2(__dsub_rn(t.x, __dmul_rn(rw.v[s].y, x[s].y)),
                         __dadd_rn(t.y, __dmul_rn(rw.v[s].y, x[s].x)));
      c = make_double2(__dadd_rn(c.x, t.x), __dadd_rn(c.y, t.y));
      return;
    }
  }
  if (rw.brk == 0) {
    acc = cmul_add(rw.v[2], x[2], cmul_add(rw.v[1], x[1], cmul_add(rw.v[0], x[0], acc)));
    c = make_double2(__dadd_rn(c.x, acc.x), __dadd_rn(c.y, acc.y));
    return;
  }
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    if (s >= rw.n) break;
    if ((rw.brk >> s) & 1u) {
      c = make_double2(__dadd_rn(c.x, acc.x), __dadd_rn(c.y, acc.y));
      acc = make_double2(0.0, 0.0);
    }
    acc = cmul_add(rw.v[s], x[s], acc);
  }
  c = make_double2(__dadd_rn(c.x, acc.x), __dadd_rn(c.y, acc.y));
}

template <bool CPLX>
__device__ __forceinline__ bool row_imag(const BandRow<CPLX>& rw) {
  if constexpr (CPLX)
    return rw.v[0].x == 0.0 && rw.v[1].x == 0.0 && rw.v[2].x == 0.0;
  else
    return false;
}

// b.n / b.stride / b.active are padded to 4 modes (extent 1, inactive).
// PAIR: the species mode (3, extent 2) is iterated inside the thread (nz =
// n2 then).  M3: mode 3 has an active factor.  A block's mode-2 rows
// (z-chunk <= ZMAX) are decoded once into shared memory.
constexpr int ZMAX = 32;

// SMR (v5, KP_BAND=v5): the block's mode-0 / mode-1 rows in shared memory
// instead of registers (fewer registers per thread, more resident warps)
template <bool CPLX, bool PAIR, bool M3, bool SMR = false>
__global__ void __launch_bounds__(256, SMR ? ((CPLX || PAIR) ? 4 : 6) : ((CPLX || PAIR) ? 3 : 4))
    kronsum_band2_kernel(BandArgs b, int nz, int zchunk, const double* __restrict__ u,
                         double* __restrict__ r, bool with_g, kp_gfun g, double t) {
  pdl_wait();
  using T = typename std::conditional<CPLX, double2, double>::type;
  __shared__ BandRow<CPLX> rows2[ZMAX];
  const T* __restrict__ ut = reinterpret_cast<const T*>(u);
  T* __restrict__ rt = reinterpret_cast<T*>(r);
  const int z0 = blockIdx.z * zchunk;
  const int z1 = min(nz, z0 + zchunk);
  const int tid = threadIdx.x + 32 * threadIdx.y;
  if (b.active[2] && tid < z1 - z0) {
    const int z = z0 + tid;
    load_row(b, 2, PAIR ? z : z % b.n[2], rows2[tid]);
  }
  const int i0 = blockIdx.x * 32 + threadIdx.x;
  const int i1 = blockIdx.y * 8 + threadIdx.y;
  __shared__ BandRow<CPLX> rows0s[SMR ? 32 : 1], rows1s[SMR ? 8 : 1];
  if constexpr (SMR) {
    if (threadIdx.y == 0 && b.active[0] && i0 < b.n[0]) load_row(b, 0, i0, rows0s[threadIdx.x]);
    if (threadIdx.x == 0 && b.active[1] && i1 < b.n[1]) load_row(b, 1, i1, rows1s[threadIdx.y]);
  }
  __syncthreads();
  if (i0 >= b.n[0] || i1 >= b.n[1]) return;
  BandRow<CPLX> r0l, r1l;
  if (!SMR && b.active[0]) load_row(b, 0, i0, r0l);
  if (!SMR && b.active[1]) load_row(b, 1, i1, r1l);
  const BandRow<CPLX>& r0 = SMR ? rows0s[threadIdx.x] : r0l;
  const BandRow<CPLX>& r1 = SMR ? rows1s[threadIdx.y] : r1l;
  const int h2 = b.slab == 2 ? b.halo : 0, h3 = b.slab == 3 ? b.halo : 0;
  const unsigned in01 = unsigned(i0 + (b.slab == 0 ? b.halo : 0)) * unsigned(b.stride[0]) +
                        unsigned(i1 + (b.slab == 1 ? b.halo : 0)) * unsigned(b.stride[1]);
  const unsigned plane = unsigned(b.n[0]) * unsigned(b.n[1]);
  const unsigned out01 = unsigned(i0) + unsigned(i1) * unsigned(b.n[0]);
  const unsigned st2 = unsigned(b.stride[2]), st3 = unsigned(b.stride[3]);
  const unsigned n2 = unsigned(b.n[2]);
  const bool a0 = b.active[0], a1 = b.active[1], a2 = b.active[2];
  BandRow<CPLX> r3a, r3b;
  if (M3) {
    if (PAIR) {
      load_row(b, 3, 0, r3a);
      load_row(b, 3, 1, r3b);
    }
  }
  // one entry: the Kronecker-sum value (without g) at input index `in`
  auto entry = [&](unsigned in, const BandRow<CPLX>& q2, const BandRow<CPLX>& q3) -> T {
    T x0[3], x1[3], x2[3], x3[3];
    if (a0) row_gather(r0, ut, in, x0);
    if (a1) row_gather(r1, ut, in, x1);
    if (a2) row_gather(q2, ut, in, x2);
    if (M3) row_gather(q3, ut, in, x3);
    T c;
    if constexpr (CPLX)
      c = make_double2(0.0, 0.0);
    else
      c = 0.0;
    if (a0) row_combine(r0, x0, c);
    if (a1) row_combine(r1, x1, c);
    if (a2) row_combine(q2, x2, c);
    if (M3) row_combine(q3, x3, c);
    return c;
  };
  // L1 prefetch PD planes ahead: the march is otherwise one dependent HBM
  // round trip per plane (latency-bound at the occupancy the rows allow)
  constexpr int PD = 3;
  const int zlim = min(z1 + 1, PAIR ? nz + h2 : nz);  // last plane the march reads (+1 neighbour)
  auto prefetch = [&](int z) {
    if (z >= zlim) return;
    unsigned in;
    if constexpr (PAIR) {
      in = in01 + (unsigned(z) + h2) * st2 + unsigned(h3) * st3;
    } else {
      const unsigned i3 = unsigned(z) / n2, i2 = unsigned(z) - i3 * n2;
      in = in01 + (i2 + h2) * st2 + (i3 + h3) * st3;
    }
    asm volatile("prefetch.global.L1 [%0];" ::"l"(ut + in));
    if constexpr (PAIR) asm volatile("prefetch.global.L1 [%0];" ::"l"(ut + in + st3));
  };
#pragma unroll
  for (int k = 1; k <= PD; ++k) prefetch(z0 + k);
  for (int z = z0; z < z1; ++z) {
    prefetch(z + PD + 1);
    const BandRow<CPLX>& q2 = rows2[z - z0];
    if constexpr (PAIR) {
      const unsigned iz = unsigned(z);
      const unsigned in0 = in01 + (iz + h2) * st2 + unsigned(h3) * st3;
      const unsigned in1 = in0 + st3;
      const unsigned idx0 = out01 + iz * plane;
      const unsigned idx1 = idx0 + n2 * plane;
      const T c0 = entry(in0, q2, r3a);
      const T c1 = entry(in1, q2, r3b);
      if (with_g) {
        const double u0 = ut[in0], u1 = ut[in1];
        rt[idx0] = __dadd_rn(c0, g_real(g, u0, u1, false, idx0, t));
        rt[idx1] = __dadd_rn(c1, g_real(g, u1, u0, true, idx1, t));
      } else {
        rt[idx0] = c0;
        rt[idx1] = c1;
      }
    } else {
      const unsigned i3 = unsigned(z) / n2, i2 = unsigned(z) - i3 * n2;
      const unsigned in = in01 + (i2 + h2) * st2 + (i3 + h3) * st3;
      const unsigned idx = out01 + (i2 + i3 * n2) * plane;
      BandRow<CPLX> q3;
      if (M3) load_row(b, 3, int(i3), q3);
      const T c = entry(in, q2, q3);
      if (!with_g) {
        rt[idx] = c;
      } else if constexpr (CPLX) {
        const double2 gg = g_cplx(g, ut[in]);
        rt[idx] = make_double2(__dadd_rn(c.x, gg.x), __dadd_rn(c.y, gg.y));
      } else {
        rt[idx] = __dadd_rn(c, g_real(g, ut[in], 0.0, false, idx, t));
      }
    }
  }
}


// ---- v3: TMA plane ring (d = 3 + optional species; the configs' shapes) ----
// A block owns a 32 x 8 tile of (i0, i1) lines and marches a chunk of planes
// z.  The (32+2) x (8+2) input tile of every plane it needs (the +-1 halo in
// i0 and i1 included, zero-filled outside the tensor) arrives by TMA
// (cp.async.bulk.tensor) into a ring of D3 plane slots, each with its own
// mbarrier: D3 - 3 planes stay in flight ahead of the one being computed, so
// the march is no longer one dependent HBM round trip per plane.  Each
// entry's neighbours are read from shared memory (row deltas of -1 / 0 / +1;
// a periodic wrap-around column falls back to a global load), then the same
// row_combine as v2 -- bit-identical results.
constexpr int D3 = 8, TX = 32, TY = 8, PY = TY + 2;
// tile width and the centre's x offset: a TMA box must start on a 16-byte
// boundary, so a real tile starts 2 entries left of the block (t0 - 2, even)
// and is TX + 4 wide; a complex entry is 16 bytes, so t0 - 1 works
template <bool CPLX>
constexpr int tile_px() { return CPLX ? TX + 2 : TX + 4; }
template <bool CPLX>
constexpr int tile_xo() { return CPLX ? 1 : 2; }

template <bool CPLX>
struct BandRow3 : BandRow<CPLX> {
  int dl[3];  // column - row (mode units); |dl| > 1: a wrap-around, read from global
};

template <bool CPLX>
__device__ __forceinline__ void load_row3(const BandArgs& b, int mu, int i, BandRow3<CPLX>& rw) {
  load_row(b, mu, i, static_cast<BandRow<CPLX>&>(rw));
  const int ig = (mu == b.slab) ? i + b.k0 : i;
  const int* cs = b.cols[mu] + ig * 3;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    rw.dl[s] = 0;
    if (s < rw.n) rw.dl[s] = int(col_off(b, mu, ig, __ldg(cs + s)));
  }
}

__device__ __forceinline__ unsigned s3_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void s3_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(s3_u32(bar)),
      "r"(parity)
      : "memory");
}

template <bool CPLX, bool PAIR>
__global__ void __launch_bounds__(256)
    kronsum_band3_kernel(const __grid_constant__ CUtensorMap map, BandArgs b, int nz,
                         int zchunk, const double* __restrict__ u, double* __restrict__ r,
                         bool with_g, kp_gfun g, double t) {
  pdl_wait();
  using T = typename std::conditional<CPLX, double2, double>::type;
  constexpr int NSP = PAIR ? 2 : 1;
  constexpr int PX = tile_px<CPLX>(), XO = tile_xo<CPLX>();
  constexpr unsigned TILE_B = PX * PY * sizeof(T);  // bytes of one plane tile (a TMA box)
  // tiles start on 128-byte boundaries (the TMA destination alignment)
  constexpr unsigned TILE = ((TILE_B + 127) / 128 * 128) / sizeof(T);  // padded, in elements
  constexpr unsigned SLOT_BYTES = TILE_B * NSP;  // bytes landing per slot
  constexpr unsigned SLOT_PAD = TILE * sizeof(T) * NSP;
  extern __shared__ __align__(128) unsigned char s3raw[];
  T* ring = reinterpret_cast<T*>(s3raw);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(s3raw + D3 * SLOT_PAD);
  __shared__ BandRow3<CPLX> rows2[ZMAX];
  const T* __restrict__ ut = reinterpret_cast<const T*>(u);
  T* __restrict__ rt = reinterpret_cast<T*>(r);

  const int z0 = blockIdx.z * zchunk;
  const int z1 = min(nz, z0 + zchunk);
  const int tid = threadIdx.x + 32 * threadIdx.y;
  const int t0 = blockIdx.x * TX, t1 = blockIdx.y * TY;
  const int h2 = b.slab == 2 ? b.halo : 0;
  // input planes z0-1 .. z1 (with the slab halo offset h2); plane j of the
  // march (j = p - (z0 - 1)) lives in slot j % D3, phase (j / D3) & 1
  const int jmax = z1 - z0 + 1;
  auto issue = [&](int j) {
    const int slot = j % D3;
    const int zin = z0 - 1 + j + h2;
    unsigned long long* bar = &full[slot];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s3_u32(bar)),
                 "r"(SLOT_BYTES)
                 : "memory");
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) {
      T* dst = ring + (size_t(slot) * NSP + sp) * TILE;
      const int c0 = CPLX ? 2 * (t0 - XO) : t0 - XO;
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(s3_u32(dst)),
          "l"(reinterpret_cast<unsigned long long>(&map)), "r"(c0), "r"(t1 - 1), "r"(zin),
          "r"(sp), "r"(s3_u32(bar))
          : "memory");
    }
  };
  if (tid == 0) {
    for (int s = 0; s < D3; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s3_u32(&full[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (b.active[2] && tid < z1 - z0) load_row3(b, 2, PAIR ? z0 + tid : (z0 + tid) % b.n[2], rows2[tid]);
  __syncthreads();
  if (tid == 0)
    for (int j = 0; j < min(D3, jmax + 1); ++j) issue(j);

  const int lx = threadIdx.x, ly = threadIdx.y;
  const int i0 = t0 + lx, i1 = t1 + ly;
  const bool live = i0 < b.n[0] && i1 < b.n[1];
  BandRow3<CPLX> r0, r1;
  if (live && b.active[0]) load_row3(b, 0, i0, r0);
  if (live && b.active[1]) load_row3(b, 1, i1, r1);
  const unsigned in01 = unsigned(i0) * unsigned(b.stride[0]) + unsigned(i1) * unsigned(b.stride[1]);
  const unsigned plane = unsigned(b.n[0]) * unsigned(b.n[1]);
  const unsigned out01 = unsigned(i0) + unsigned(i1) * unsigned(b.n[0]);
  const unsigned st2 = unsigned(b.stride[2]), st3 = unsigned(b.stride[3]);
  const unsigned n2 = unsigned(b.n[2]);
  const bool a0 = b.active[0], a1 = b.active[1], a2 = b.active[2];
  const int cen = (ly + 1) * PX + (lx + XO);  // the entry's offset in a plane tile

  for (int z = z0; z < z1; ++z) {
    const int jc = z - z0 + 1;  // the centre plane's march index
#pragma unroll
    for (int k = -1; k <= 1; ++k) {
      const int j = jc + k;
      s3_wait(&full[j % D3], unsigned((j / D3) & 1));
    }
    if (live) {
      const BandRow3<CPLX>& q2 = rows2[z - z0];
      const T* tc[NSP];
#pragma unroll
      for (int sp = 0; sp < NSP; ++sp) tc[sp] = ring + (size_t(jc % D3) * NSP + sp) * TILE;
      const unsigned iz = unsigned(z);
      unsigned in_base;
      if constexpr (PAIR) {
        in_base = in01 + (iz + h2) * st2;
      } else {
        const unsigned i3 = iz / n2, i2 = iz - i3 * n2;
        in_base = in01 + (i2 + h2) * st2 + i3 * st3;
      }
#pragma unroll
      for (int sp = 0; sp < NSP; ++sp) {
        const T* tp = tc[sp];
        const unsigned in = in_base + unsigned(sp) * st3;
        T x0[3], x1[3], x2[3];
        if (a0) {
#pragma unroll
          for (int s = 0; s < 3; ++s)
            x0[s] = (r0.dl[s] >= -1 && r0.dl[s] <= 1) ? tp[cen + r0.dl[s]]
                                                      : ut[in + unsigned(r0.off[s])];
        }
        if (a1) {
#pragma unroll
          for (int s = 0; s < 3; ++s)
            x1[s] = (r1.dl[s] >= -1 && r1.dl[s] <= 1) ? tp[cen + r1.dl[s] * PX]
                                                      : ut[in + unsigned(r1.off[s])];
        }
        if (a2) {
#pragma unroll
          for (int s = 0; s < 3; ++s) {
            const int dz = q2.dl[s];
            x2[s] = (dz >= -1 && dz <= 1)
                        ? ring[(size_t((jc + dz) % D3) * NSP + sp) * TILE + cen]
                        : ut[in + unsigned(q2.off[s])];
          }
        }
        T c;
        if constexpr (CPLX)
          c = make_double2(0.0, 0.0);
        else
          c = 0.0;
        if (a0) row_combine(static_cast<const BandRow<CPLX>&>(r0), x0, c);
        if (a1) row_combine(static_cast<const BandRow<CPLX>&>(r1), x1, c);
        if (a2) row_combine(static_cast<const BandRow<CPLX>&>(q2), x2, c);
        const unsigned idx = out01 + (PAIR ? iz + unsigned(sp) * n2 : iz) * plane;
        if (!with_g) {
          rt[idx] = c;
        } else if constexpr (CPLX) {
          const double2 gg = g_cplx(g, tp[cen]);
          rt[idx] = make_double2(__dadd_rn(c.x, gg.x), __dadd_rn(c.y, gg.y));
        } else if constexpr (PAIR) {
          const double uc = tp[cen], upart = tc[1 - sp][cen];
          rt[idx] = __dadd_rn(c, g_real(g, uc, upart, sp == 1, idx, t));
        } else {
          rt[idx] = __dadd_rn(c, g_real(g, tp[cen], 0.0, false, idx, t));
        }
      }
    }
    __syncthreads();  // every thread is done with plane z-1's slot
    if (tid == 0 && jc - 1 + D3 <= jmax) issue(jc - 1 + D3);
  }
}


// ---- v4: v2 with the z line in registers (opt-in, KP_BAND=v4) ----
// Each thread keeps u at planes z-1, z, z+1 of its (i0, i1) line in
// registers while it marches, so per plane it loads the next plane's centre
// and the four in-plane neighbours (i0 +- 1, i1 +- 1) instead of nine
// values; a row entry with a zero delta reads the centre register, a
// wrap-around entry (periodic rows) falls back to a load.  Same values into
// the same row_combine as v2: bit-identical.  Measured no faster than v2
// (NLS 512^3 2.00 vs 1.71 ms, AC3D / Brusselator equal): v2's neighbour
// loads already hit L1, and the march is latency-bound, not load-count-bound.
template <bool CPLX, bool PAIR>
__global__ void __launch_bounds__(256, (CPLX || PAIR) ? 2 : 3)
    kronsum_band4_kernel(BandArgs b, int nz, int zchunk, const double* __restrict__ u,
                         double* __restrict__ r, bool with_g, kp_gfun g, double t) {
  pdl_wait();
  using T = typename std::conditional<CPLX, double2, double>::type;
  constexpr int NSP = PAIR ? 2 : 1;
  __shared__ BandRow3<CPLX> rows2[ZMAX];
  const T* __restrict__ ut = reinterpret_cast<const T*>(u);
  T* __restrict__ rt = reinterpret_cast<T*>(r);
  const int z0 = blockIdx.z * zchunk;
  const int z1 = min(nz, z0 + zchunk);
  const int tid = threadIdx.x + 32 * threadIdx.y;
  if (b.active[2] && tid < z1 - z0) load_row3(b, 2, z0 + tid, rows2[tid]);
  __syncthreads();
  const int i0 = blockIdx.x * 32 + threadIdx.x;
  const int i1 = blockIdx.y * 8 + threadIdx.y;
  if (i0 >= b.n[0] || i1 >= b.n[1]) return;
  BandRow3<CPLX> r0, r1;
  if (b.active[0]) load_row3(b, 0, i0, r0);
  if (b.active[1]) load_row3(b, 1, i1, r1);
  const int h2 = b.slab == 2 ? b.halo : 0;
  const unsigned in01 = unsigned(i0) * unsigned(b.stride[0]) + unsigned(i1) * unsigned(b.stride[1]);
  const unsigned plane = unsigned(b.n[0]) * unsigned(b.n[1]);
  const unsigned out01 = unsigned(i0) + unsigned(i1) * unsigned(b.n[0]);
  const unsigned st2 = unsigned(b.stride[2]), st3 = unsigned(b.stride[3]);
  const unsigned n2 = unsigned(b.n[2]);
  const int zin_max = int(n2) + 2 * h2;  // input planes (with the slab halo)
  const bool a0 = b.active[0], a1 = b.active[1], a2 = b.active[2];
  auto in_of = [&](int z, int sp) { return in01 + unsigned(z + h2) * st2 + unsigned(sp) * st3; };
  auto load_plane = [&](int z, int sp) -> T {
    const int zi = z + h2;
    if (zi < 0 || zi >= zin_max) {
      if constexpr (CPLX)
        return make_double2(0.0, 0.0);
      else
        return 0.0;
    }
    return ut[in_of(z, sp)];
  };
  T xm[NSP], xc[NSP], xp[NSP];
#pragma unroll
  for (int sp = 0; sp < NSP; ++sp) {
    xm[sp] = load_plane(z0 - 1, sp);
    xc[sp] = load_plane(z0, sp);
    xp[sp] = load_plane(z0 + 1, sp);
  }
  for (int z = z0; z < z1; ++z) {
    T xn[NSP];
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) xn[sp] = load_plane(z + 2, sp);  // in flight during z
    const BandRow3<CPLX>& q2 = rows2[z - z0];
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) {
      const unsigned in = in_of(z, sp);
      T x0[3], x1[3], x2[3];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        if (a0) x0[s] = r0.dl[s] == 0 ? xc[sp] : ut[in + unsigned(r0.off[s])];
        if (a1) x1[s] = r1.dl[s] == 0 ? xc[sp] : ut[in + unsigned(r1.off[s])];
        if (a2) {
          const int dz = q2.dl[s];
          x2[s] = dz == 0 ? xc[sp]
                          : (dz == -1 ? xm[sp] : (dz == 1 ? xp[sp] : ut[in + unsigned(q2.off[s])]));
        }
      }
      T c;
      if constexpr (CPLX)
        c = make_double2(0.0, 0.0);
      else
        c = 0.0;
      if (a0) row_combine(static_cast<const BandRow<CPLX>&>(r0), x0, c);
      if (a1) row_combine(static_cast<const BandRow<CPLX>&>(r1), x1, c);
      if (a2) row_combine(static_cast<const BandRow<CPLX>&>(q2), x2, c);
      const unsigned idx = out01 + (PAIR ? unsigned(z) + unsigned(sp) * n2 : unsigned(z)) * plane;
      if (!with_g) {
        rt[idx] = c;
      } else if constexpr (CPLX) {
        const double2 gg = g_cplx(g, xc[sp]);
        rt[idx] = make_double2(__dadd_rn(c.x, gg.x), __dadd_rn(c.y, gg.y));
      } else if constexpr (PAIR) {
        rt[idx] = __dadd_rn(c, g_real(g, xc[sp], xc[1 - sp], sp == 1, idx, t));
      } else {
        rt[idx] = __dadd_rn(c, g_real(g, xc[sp], 0.0, false, idx, t));
      }
    }
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) {
      xm[sp] = xc[sp];
      xc[sp] = xp[sp];
      xp[sp] = xn[sp];
    }
  }
}

#ifndef KP_B6_PAIR_BLOCKS
#define KP_B6_PAIR_BLOCKS 3  // measured: 2 -> NLS 1.85 ms, 3 -> 1.60 ms (v2 1.63)
#endif
// ---- v6: v2's march with a lean per-plane loop (the default) ----
// v2's traversal and arithmetic exactly (bit-identical), restricted to the
// configs' shapes -- z runs over mode 2 only (order <= 3, or the 2-species
// pair in slot 3 with no factor on it) -- so the per-plane loop carries no
// index division, no mode-3 row, and its rows by value (v2's conditional
// row references cost local-memory round trips and shared-memory address
// rebuilds every plane: 116 SASS instructions per entry on AC3D, ncu
// source page).  Two planes per iteration keep both planes' loads in flight.
template <bool CPLX, bool PAIR>
__global__ void __launch_bounds__(256, (CPLX || PAIR) ? KP_B6_PAIR_BLOCKS : 4)
    kronsum_band6_kernel(BandArgs b, int nz, int zchunk, const double* __restrict__ u,
                         double* __restrict__ r, bool with_g, kp_gfun g, double t) {
  pdl_wait();
  using T = typename std::conditional<CPLX, double2, double>::type;
  __shared__ BandRow<CPLX> rows2[ZMAX];
  const T* __restrict__ ut = reinterpret_cast<const T*>(u);
  T* __restrict__ rt = reinterpret_cast<T*>(r);
  const int z0 = blockIdx.z * zchunk;
  const int z1 = min(nz, z0 + zchunk);
  const int tid = threadIdx.x + 32 * threadIdx.y;
  const bool a0 = b.active[0], a1 = b.active[1], a2 = b.active[2];
  if (a2 && tid < z1 - z0) load_row(b, 2, z0 + tid, rows2[tid]);
  __syncthreads();
  const int i0 = blockIdx.x * 32 + threadIdx.x;
  const int i1 = blockIdx.y * 8 + threadIdx.y;
  if (i0 >= b.n[0] || i1 >= b.n[1]) return;
  BandRow<CPLX> r0, r1;
  if (a0) load_row(b, 0, i0, r0);
  if (a1) load_row(b, 1, i1, r1);
  const int h2 = b.slab == 2 ? b.halo : 0, h3 = b.slab == 3 ? b.halo : 0;
  const unsigned st2 = unsigned(b.stride[2]), st3 = unsigned(b.stride[3]);
  const unsigned in01 = unsigned(i0 + (b.slab == 0 ? b.halo : 0)) * unsigned(b.stride[0]) +
                        unsigned(i1 + (b.slab == 1 ? b.halo : 0)) * unsigned(b.stride[1]) +
                        unsigned(h2) * st2 + unsigned(h3) * st3;
  const unsigned plane = unsigned(b.n[0]) * unsigned(b.n[1]);
  const unsigned out01 = unsigned(i0) + unsigned(i1) * unsigned(b.n[0]);
  const unsigned sp_out = unsigned(b.n[2]) * plane;  // species 1 output offset (PAIR)
  auto entry = [&](unsigned in, const BandRow<CPLX>& q2) -> T {
    T x0[3], x1[3], x2[3];
    if (a0) row_gather(r0, ut, in, x0);
    if (a1) row_gather(r1, ut, in, x1);
    if (a2) row_gather(q2, ut, in, x2);
    T c;
    if constexpr (CPLX)
      c = make_double2(0.0, 0.0);
    else
      c = 0.0;
    if (a0) row_combine(r0, x0, c);
    if (a1) row_combine(r1, x1, c);
    if (a2) row_combine(q2, x2, c);
    return c;
  };
#pragma unroll 1
  for (int z = z0; z < z1; ++z) {
    const BandRow<CPLX> q2 = rows2[z - z0];
    const unsigned in0 = in01 + unsigned(z) * st2;
    const unsigned idx0 = out01 + unsigned(z) * plane;
    if constexpr (PAIR) {
      const unsigned in1 = in0 + st3, idx1 = idx0 + sp_out;
      const T c0 = entry(in0, q2);
      const T c1 = entry(in1, q2);
      if (with_g) {
        const double u0 = ut[in0], u1 = ut[in1];
        rt[idx0] = __dadd_rn(c0, g_real(g, u0, u1, false, idx0, t));
        rt[idx1] = __dadd_rn(c1, g_real(g, u1, u0, true, idx1, t));
      } else {
        rt[idx0] = c0;
        rt[idx1] = c1;
      }
    } else {
      const T c = entry(in0, q2);
      if (!with_g) {
        rt[idx0] = c;
      } else if constexpr (CPLX) {
        const double2 gg = g_cplx(g, ut[in0]);
        rt[idx0] = make_double2(__dadd_rn(c.x, gg.x), __dadd_rn(c.y, gg.y));
      } else {
        rt[idx0] = __dadd_rn(c, g_real(g, ut[in0], 0.0, false, idx0, t));
      }
    }
  }
}

// ---- v8: v6 with the thread's z line in registers, one plane AHEAD ----
// v6's only HBM miss per plane is the first touch of plane z + 1 (its mode-2
// "+1" neighbour); every other value was touched an iteration earlier.  v8
// loads that value one iteration early: at plane z the centres of planes
// z - 1, z, z + 1 are registers and the load of plane z + 2's centre is
// issued before plane z is computed, so the miss has a whole iteration of
// the SM's other warps to land.  Interior mode-2 rows (columns z-1, z, z+1,
// no KC break) read the z line; other rows gather through their offsets.
// Same chains in the same order as v6: bit-identical.
constexpr int ZMAX8 = 64;
template <bool CPLX>
__device__ __forceinline__ bool interior_row8(const BandRow<CPLX>& rw, int st) {
  return rw.n == 3 && rw.brk == 0 && rw.off[0] == -st && rw.off[1] == 0 && rw.off[2] == st;
}

// YH (opt-in, KP_B8_YH=1): the thread's mode-1 neighbours (rows i1 - 1, i1 + 1)
// of the NEXT plane are loaded one iteration early as well (the warps of a
// tile march unsynchronised, so a warp that is ahead takes its neighbour
// rows' first touch itself; L1 hit rate 63 %).  Measured slower: the extra
// registers cost more than the exposed misses.
template <bool CPLX, bool PAIR, int MB, bool YH>
__global__ void __launch_bounds__(256, MB)
    kronsum_band8_kernel(BandArgs b, int nz, int zchunk, int pf2, int hpf,
                         const double* __restrict__ u,
                         double* __restrict__ r, bool with_g, kp_gfun g, double t) {
  pdl_wait();
  using T = typename std::conditional<CPLX, double2, double>::type;
  constexpr int NSP = PAIR ? 2 : 1;
  __shared__ BandRow<CPLX> rows2[ZMAX8];
  __shared__ unsigned char pat2[ZMAX8];
  const T* __restrict__ ut = reinterpret_cast<const T*>(u);
  T* __restrict__ rt = reinterpret_cast<T*>(r);
  const int z0 = blockIdx.z * zchunk;
  const int z1 = min(nz, z0 + zchunk);
  const int tid = threadIdx.x + 32 * threadIdx.y;
  const bool a0 = b.active[0], a1 = b.active[1], a2 = b.active[2];
  const unsigned st2 = unsigned(b.stride[2]), st3 = unsigned(b.stride[3]);
  bool im = CPLX;  // all of this thread's rows purely imaginary (row_combine<IMAG>)
  if (a2 && tid < z1 - z0) {
    load_row(b, 2, z0 + tid, rows2[tid]);
    pat2[tid] = interior_row8(rows2[tid], int(st2));
    im = im && row_imag(rows2[tid]);
  }
  const int i0 = blockIdx.x * 32 + threadIdx.x;
  const int i1 = blockIdx.y * 8 + threadIdx.y;
  const bool inb = i0 < b.n[0] && i1 < b.n[1];
  BandRow<CPLX> r0, r1;
  if (inb && a0) {
    load_row(b, 0, i0, r0);
    im = im && row_imag(r0);
  }
  if (inb && a1) {
    load_row(b, 1, i1, r1);
    im = im && row_imag(r1);
  }
  const bool imag = __syncthreads_and(im) != 0;
  if (!inb) return;
  const int h2 = b.slab == 2 ? b.halo : 0, h3 = b.slab == 3 ? b.halo : 0;
  const unsigned in01 = unsigned(i0 + (b.slab == 0 ? b.halo : 0)) * unsigned(b.stride[0]) +
                        unsigned(i1 + (b.slab == 1 ? b.halo : 0)) * unsigned(b.stride[1]) +
                        unsigned(h2) * st2 + unsigned(h3) * st3;
  const unsigned plane = unsigned(b.n[0]) * unsigned(b.n[1]);
  const unsigned out01 = unsigned(i0) + unsigned(i1) * unsigned(b.n[0]);
  const unsigned sp_out = unsigned(b.n[2]) * plane;  // species 1 output offset (PAIR)
  const int plo = -h2, phi = nz + h2;                 // planes plo .. phi - 1 exist
  // rim prefetch (see the loop): lanes 0 / 31 take the mode-0 neighbour beyond
  // the warp, the tile's first / last warp its mode-1 neighbour row
  int halo_off = 0;
  if (b.slab != 0 && b.slab != 1 && b.stride[0] == 1) {
    if (threadIdx.y == 0 && i1 > 0)
      halo_off = -int(b.stride[1]);
    else if (threadIdx.y == 7 && i1 + 1 < b.n[1])
      halo_off = int(b.stride[1]);
    else if (threadIdx.x == 0 && i0 > 0)
      halo_off = -1;
    else if (threadIdx.x == 31 && i0 + 1 < b.n[0])
      halo_off = 1;
  }
  const bool halo_pf = halo_off != 0 && hpf != 0;
  auto centre = [&](int p, int sp) -> T {
    if (p >= plo && p < phi) return ut[in01 + unsigned(p) * st2 + unsigned(sp) * st3];
    if constexpr (CPLX)
      return make_double2(0.0, 0.0);
    else
      return 0.0;
  };
  T zm[NSP], zc[NSP], zp[NSP];
#pragma unroll
  for (int sp = 0; sp < NSP; ++sp) {
    zm[sp] = centre(z0 - 1, sp);
    zc[sp] = centre(z0, sp);
    zp[sp] = centre(z0 + 1, sp);
  }
  // mode-1 neighbours of the current plane (valid when the row has the
  // columns i1 - 1, i1, i1 + 1 in this order; KC breaks stay with row_combine)
  const bool y_int = YH && a1 && r1.n == 3 && r1.off[0] == -int(b.stride[1]) && r1.off[1] == 0 &&
                     r1.off[2] == int(b.stride[1]);
  T ym[NSP], yp[NSP];
#pragma unroll
  for (int sp = 0; sp < NSP; ++sp) {
    if (y_int) {
      const unsigned in = in01 + unsigned(z0) * st2 + unsigned(sp) * st3;
      ym[sp] = ut[in - unsigned(b.stride[1])];
      yp[sp] = ut[in + unsigned(b.stride[1])];
    } else {
      ym[sp] = zc[sp];
      yp[sp] = zc[sp];
    }
  }
  auto march = [&](auto imag_tag) {
  constexpr bool IM = decltype(imag_tag)::value;
  unsigned rim[NSP] = {};
#pragma unroll 1
  for (int z = z0; z < z1; ++z) {
    T zn[NSP], ymn[NSP], ypn[NSP];
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) zn[sp] = centre(z + 2, sp);
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) {
      ymn[sp] = ym[sp];
      ypn[sp] = yp[sp];
      if (y_int && z + 1 < phi) {
        const unsigned in = in01 + unsigned(z + 1) * st2 + unsigned(sp) * st3;
        ymn[sp] = ut[in - unsigned(b.stride[1])];
        ypn[sp] = ut[in + unsigned(b.stride[1])];
      }
    }
    if (pf2 > 0 && z + pf2 < phi) {
#pragma unroll
      for (int sp = 0; sp < NSP; ++sp)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(ut + in01 + unsigned(z + pf2) * st2 +
                                                        unsigned(sp) * st3));
    }
    // the tile's rim of the NEXT plane belongs to other blocks' lines: bring
    // it into L1 now, or every warp waits an L2 round trip on its two edge
    // lanes (and the tile's first / last row) once per plane.  A plain load
    // whose result is only "used" (an empty asm) an iteration later:
    // prefetch.global.L1 measured 8x SLOWER for the whole kernel (NLS 1.5 ->
    // 13 ms) on this B200.
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) asm volatile("" ::"r"(rim[sp]));
    if (halo_pf && z + 1 < phi) {
#pragma unroll
      for (int sp = 0; sp < NSP; ++sp)
        asm volatile("ld.global.u32 %0, [%1];"
                     : "=r"(rim[sp])
                     : "l"(ut + in01 + unsigned(z + 1) * st2 + unsigned(sp) * st3 +
                           unsigned(halo_off)));
    }
    const BandRow<CPLX> q2 = rows2[z - z0];
    const bool int2 = pat2[z - z0];
    const unsigned in0 = in01 + unsigned(z) * st2;
    const unsigned idx0 = out01 + unsigned(z) * plane;
    T res[NSP];
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) {
      const unsigned in = in0 + unsigned(sp) * st3;
      T x0[3], x1[3], x2[3];
      if (a0) row_gather(r0, ut, in, x0);
      if (a1) {
        if (y_int) {
          x1[0] = ym[sp];
          x1[1] = zc[sp];
          x1[2] = yp[sp];
        } else {
          row_gather(r1, ut, in, x1);
        }
      }
      if (a2) {
        if (int2) {
          x2[0] = zm[sp];
          x2[1] = zc[sp];
          x2[2] = zp[sp];
        } else {
          row_gather(q2, ut, in, x2);
        }
      }
      T c;
      if constexpr (CPLX)
        c = make_double2(0.0, 0.0);
      else
        c = 0.0;
      if (a0) row_combine<IM>(r0, x0, c);
      if (a1) row_combine<IM>(r1, x1, c);
      if (a2) row_combine<IM>(q2, x2, c);
      res[sp] = c;
    }
    if constexpr (PAIR) {
      const unsigned idx1 = idx0 + sp_out;
      if (with_g) {
        const double u0 = zc[0], u1 = zc[1];
        rt[idx0] = __dadd_rn(res[0], g_real(g, u0, u1, false, idx0, t));
        rt[idx1] = __dadd_rn(res[1], g_real(g, u1, u0, true, idx1, t));
      } else {
        rt[idx0] = res[0];
        rt[idx1] = res[1];
      }
    } else if (!with_g) {
      rt[idx0] = res[0];
    } else if constexpr (CPLX) {
      const double2 gg = g_cplx(g, zc[0]);
      rt[idx0] = make_double2(__dadd_rn(res[0].x, gg.x), __dadd_rn(res[0].y, gg.y));
    } else {
      rt[idx0] = __dadd_rn(res[0], g_real(g, zc[0], 0.0, false, idx0, t));
    }
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) {
      zm[sp] = zc[sp];
      zc[sp] = zp[sp];
      zp[sp] = zn[sp];
      ym[sp] = ymn[sp];
      yp[sp] = ypn[sp];
    }
  }
  };
  if constexpr (CPLX) {
    if (imag)
      march(std::true_type{});
    else
      march(std::false_type{});
  } else {
    march(std::false_type{});
  }
}

// v8 launcher; false = not applicable
bool launch_band8(kp_ctx* ctx, const BandArgs& b2, bool cplx, bool pair, int nz, const double* u,
                  double* r, bool with_g, const kp_gfun& g, double t) {
  static const int mode = [] {
    const char* v = getenv("KP_BAND");
    if (!v || !*v) return 1;
    return std::string(v) == "v8" ? 2 : 0;
  }();
  if (mode == 0 || b2.active[3] || (!pair && b2.n[3] != 1)) return false;
  // default for complex tensors (NLS 512^3: 1.48 vs v6's 1.68 ms; 2 blocks of
  // 124 registers) and species pairs (Brusselator 2 x 256^3: 256 vs v2's 305
  // us; 3 blocks per SM, shorter z chunks); for single real tensors v6
  // measured faster (AC3D 17 vs 21 us): KP_BAND=v8 runs it for every form
  if (mode == 1 && !cplx && !pair) return false;
  static const int pf2 = [] {
    const char* v = getenv("KP_B8_PF");
    return v && *v ? atoi(v) : 4;
  }();
  static const int hpf = [] {
    const char* v = getenv("KP_B8_HPF");
    return v && *v ? atoi(v) : 1;
  }();
  static const long long per_sm_env = [] {
    const char* v = getenv("KP_B8_BLOCKS");
    return v && *v ? std::max(1LL, atoll(v)) : 0LL;
  }();
  const long long per_sm = per_sm_env ? per_sm_env : (pair ? 8LL : 4LL);
  const long long bxy = (long long)((b2.n[0] + 31) / 32) * ((b2.n[1] + 7) / 8);
  const long long want = ctx->num_sms * per_sm;
  const int zchunk =
      int(std::min<long long>(ZMAX8, std::max<long long>(1, (nz * bxy + want - 1) / want)));
  if ((nz + zchunk - 1) / zchunk > 65535 || (b2.n[1] + 7) / 8 > 65535) return false;
  dim3 grid(unsigned((b2.n[0] + 31) / 32), unsigned((b2.n[1] + 7) / 8),
            unsigned((nz + zchunk - 1) / zchunk));
  auto go = [&](auto kern) {
    launch_pdl(ctx, kern, grid, dim3(32, 8), 0, b2, nz, zchunk, pf2, hpf, u, r, with_g, g, t);
    ctx->launches--;  // counted once by the caller
  };
  static const int mb_env = [] {  // resident blocks per SM the kernel is compiled for
    const char* v = getenv("KP_B8_MINB");
    return v && *v ? atoi(v) : 0;
  }();
  const int mb = mb_env ? mb_env : (pair ? 3 : 0);
  static const bool yh = [] {  // opt-in: measured slower (NLS 1.60 vs 1.49 ms)
    const char* v = getenv("KP_B8_YH");
    return v && std::string(v) == "1";
  }();
  auto pick = [&](auto cp, auto pr, auto m) {
    constexpr bool C = decltype(cp)::value, P = decltype(pr)::value;
    constexpr int M = decltype(m)::value;
    yh ? go(kronsum_band8_kernel<C, P, M, true>) : go(kronsum_band8_kernel<C, P, M, false>);
  };
  using std::integral_constant;
  const std::true_type T1{};
  const std::false_type F0{};
  if (cplx)
    mb == 3 ? pick(T1, F0, integral_constant<int, 3>{}) : pick(T1, F0, integral_constant<int, 2>{});
  else if (pair)
    mb == 3 ? pick(F0, T1, integral_constant<int, 3>{}) : pick(F0, T1, integral_constant<int, 2>{});
  else
    mb == 3 ? pick(F0, F0, integral_constant<int, 3>{}) : pick(F0, F0, integral_constant<int, 4>{});
  return true;
}

// ---- v7: register-tiled march, nothing but registers on the critical path ----
// ncu on v6 (NLS 512^3): the L1 data pipe is the limiter (LSU wavefronts 73 %
// of peak: nine 16-byte gathers per entry, each 4-5 wavefronts per warp, plus
// spills), with the FP64 pipe at 40 % (a complex entry is ~80 DMUL/DADD) and
// one exposed HBM miss per plane.  v7 takes every neighbour from registers:
//   * a thread owns a strip of RY consecutive mode-1 rows of one mode-0
//     column and marches mode 2; the strip of plane z (+ one halo row each
//     side) is loaded TWO iterations early, so (RY + 2) x 2 loads per thread
//     are always in flight and no load result is awaited in the iteration
//     that issued it;
//   * mode-1 neighbours are the strip's registers, mode-2 neighbours the
//     strips of planes z - 1 / z + 1, mode-0 neighbours come by warp shuffle
//     (lanes 0 / 31 load the one value beyond the warp, one iteration early);
//   * (RY + 2) / RY aligned loads per entry instead of nine.
// Rows are canonicalised once (canon_row): a row whose columns lie in
// {i-1, i, i+1} becomes the three slots (i-1, i, i+1) with zero values in
// the missing ones -- a leading fma(0, x, +0) is +0 and a trailing fma(0, x,
// acc) is acc (the chain's accumulator is never -0, see row_gather), so the
// chain's value is unchanged bit for bit; KC = 256 slice breaks keep their
// slot.  Rows that reach elsewhere (the periodic wrap) gather through their
// offsets as in v6 (lane-divergent for mode 0, warp-uniform otherwise).
// Same chains in the same mode order: bit-identical to v6.
// NSP = 2: both species of a grid point per thread (species stride st3).
constexpr int ZMAX7 = 128;

// true: rw rewritten as slots (-st, 0, +st); false: left alone
template <bool CPLX>
__device__ __forceinline__ bool canon_row(BandRow<CPLX>& rw, int st) {
  int slot[3] = {0, 0, 0};
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    if (s >= rw.n) break;
    const int o = rw.off[s];
    if (o == -st)
      slot[s] = 0;
    else if (o == 0)
      slot[s] = 1;
    else if (o == st)
      slot[s] = 2;
    else
      return false;
    // the chain runs in column order: the slots must come in that order too
    // (a slab's wrap row has its -st neighbour last)
    if (s > 0 && slot[s] <= slot[s - 1]) return false;
  }
  BandRow<CPLX> c;
  c.n = 3;
  c.brk = 0;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    c.off[s] = (s - 1) * st;
    if constexpr (CPLX)
      c.v[s] = make_double2(0.0, 0.0);
    else
      c.v[s] = 0.0;
  }
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    if (s >= rw.n) break;
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (slot[s] == q) {
        c.v[q] = rw.v[s];
        if ((rw.brk >> s) & 1u) c.brk |= 1u << q;
      }
  }
  rw = c;
  return true;
}

// The rare rows (periodic wrap): gather through the row's own offsets and fold
// it into c.  Out of line on purpose -- inlined, the compiler predicates these
// gathers into the march and every plane issues their (masked) address
// arithmetic and loads: 300 instructions per entry instead of 150 (ncu).
template <bool CPLX>
__device__ __noinline__ typename std::conditional<CPLX, double2, double>::type slow_term(
    const BandRow<CPLX>* rw, const typename std::conditional<CPLX, double2, double>::type* ut,
    unsigned in, typename std::conditional<CPLX, double2, double>::type c) {
  using T = typename std::conditional<CPLX, double2, double>::type;
  const BandRow<CPLX> q = *rw;
  T x[3];
  row_gather(q, ut, in, x);
  row_combine(q, x, c);
  return c;
}

template <bool CPLX, int NSP, int RY, int WY, int MB>
__global__ void __launch_bounds__(32 * WY, MB)
    kronsum_band7_kernel(BandArgs b, int zchunk, int pf2, const double* __restrict__ u,
                         double* __restrict__ r, bool with_g, kp_gfun g, double t) {
  pdl_wait();
  using T = typename std::conditional<CPLX, double2, double>::type;
  constexpr int NROW = WY * RY;
  __shared__ BandRow<CPLX> rows1[NROW];
  __shared__ BandRow<CPLX> rows2[ZMAX7];
  __shared__ BandRow<CPLX> rows0[32];  // the non-canonical mode-0 rows (slow_term)
  __shared__ unsigned char pat1[NROW], pat2[ZMAX7];
  const T* __restrict__ ut = reinterpret_cast<const T*>(u);
  T* __restrict__ rt = reinterpret_cast<T*>(r);
  const int n0 = b.n[0], n1 = b.n[1], n2 = b.n[2];
  const int z0 = blockIdx.z * zchunk;
  const int z1 = min(n2, z0 + zchunk);
  const int lane = threadIdx.x;
  const int tid = threadIdx.x + 32 * threadIdx.y;
  const bool a0 = b.active[0], a1 = b.active[1], a2 = b.active[2];
  const int st1 = int(b.stride[1]), st2 = int(b.stride[2]), st3 = int(b.stride[3]);
  const int yb = blockIdx.y * NROW;
  bool im = CPLX;  // all of this thread's rows purely imaginary (row_combine<IMAG>)
  if (a1 && tid < NROW && yb + tid < n1) {
    load_row(b, 1, yb + tid, rows1[tid]);
    im = im && row_imag(rows1[tid]);
    pat1[tid] = canon_row(rows1[tid], st1);
  }
  if (a2)
    for (int i = tid; i < z1 - z0; i += 32 * WY) {
      load_row(b, 2, z0 + i, rows2[i]);
      im = im && row_imag(rows2[i]);
      pat2[i] = canon_row(rows2[i], st2);
    }
  const int i0 = blockIdx.x * 32 + lane;
  const int y0 = yb + threadIdx.y * RY;
  const bool xv = i0 < n0;
  BandRow<CPLX> r0;
  bool pat0 = true;
  r0.n = 0;
  r0.brk = 0;
  if (a0 && xv) {
    load_row(b, 0, i0, r0);
    im = im && row_imag(r0);
    if (threadIdx.y == 0) rows0[lane] = r0;
    pat0 = canon_row(r0, 1);
  }
  const bool imag = __syncthreads_and(im) != 0;
  if (y0 >= n1) return;  // whole warps only: the shuffles need all 32 lanes
  const int h2 = b.slab == 2 ? b.halo : 0;
  // input index of (i0, y0, plane 0); planes -h2 .. n2 + h2 - 1 exist
  const unsigned in01 = unsigned(i0) + unsigned(y0) * unsigned(st1) + unsigned(h2) * unsigned(st2);
  const unsigned plane = unsigned(n0) * unsigned(n1);
  const unsigned out01 = unsigned(i0) + unsigned(y0) * unsigned(n0);
  const unsigned sp_out = unsigned(n2) * plane;  // species 1 output offset
  bool yv[RY + 2];  // strip rows -1 .. RY inside the tensor
#pragma unroll
  for (int k = 0; k < RY + 2; ++k) yv[k] = (y0 + k - 1 >= 0) && (y0 + k - 1 < n1);
  // lanes 0 / 31 fetch the mode-0 neighbour beyond the warp (when it exists)
  const bool edge_l = lane == 0 && i0 - 1 >= 0 && xv;
  const bool edge_r = lane == 31 && i0 + 1 < n0;
  const int edge_off = edge_l ? -1 : 1;
  T zm[NSP][RY], cur[NSP][RY + 2], nxt[NSP][RY + 2], pre[NSP][RY + 2];
  T xe[NSP][RY], xen[NSP][RY];  // edge values of the current / next plane
  auto zero = [](T& x) {
    if constexpr (CPLX)
      x = make_double2(0.0, 0.0);
    else
      x = 0.0;
  };
  auto load_strip = [&](int p, T(*s)[RY + 2]) {
    const bool pv = xv && p >= -h2 && p < n2 + h2;
    const unsigned base = in01 + unsigned(p) * unsigned(st2) - unsigned(st1);
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp)
#pragma unroll
      for (int k = 0; k < RY + 2; ++k) {
        if (pv && yv[k])
          s[sp][k] = ut[base + unsigned(k) * unsigned(st1) + unsigned(sp) * unsigned(st3)];
        else
          zero(s[sp][k]);
      }
  };
  auto load_edge = [&](int p, T(*e)[RY]) {
    const bool pv = (edge_l || edge_r) && p >= -h2 && p < n2 + h2;
    const unsigned base = in01 + unsigned(p) * unsigned(st2) + unsigned(edge_off);
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp)
#pragma unroll
      for (int k = 0; k < RY; ++k) {
        if (pv && yv[k + 1])
          e[sp][k] = ut[base + unsigned(k) * unsigned(st1) + unsigned(sp) * unsigned(st3)];
        else
          zero(e[sp][k]);
      }
  };
  auto shfl = [&](const T& v, bool up) -> T {
    if constexpr (CPLX) {
      return up ? make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1))
                : make_double2(__shfl_down_sync(0xffffffffu, v.x, 1),
                               __shfl_down_sync(0xffffffffu, v.y, 1));
    } else {
      return up ? __shfl_up_sync(0xffffffffu, v, 1) : __shfl_down_sync(0xffffffffu, v, 1);
    }
  };
  {
    T tmp[NSP][RY + 2];
    load_strip(z0 - 1, tmp);
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp)
#pragma unroll
      for (int k = 0; k < RY; ++k) zm[sp][k] = tmp[sp][k + 1];
  }
  load_strip(z0, cur);
  load_edge(z0, xe);
  load_strip(z0 + 1, nxt);
  auto march = [&](auto imag_tag) {
  constexpr bool IM = decltype(imag_tag)::value;
#pragma unroll 1
  for (int z = z0; z < z1; ++z) {
    load_strip(z + 2, pre);
    load_edge(z + 1, xen);
    if (pf2 > 0 && xv && z + pf2 < n2 + h2) {
      const unsigned base = in01 + unsigned(z + pf2) * unsigned(st2);
#pragma unroll
      for (int sp = 0; sp < NSP; ++sp)
#pragma unroll
        for (int k = 0; k < RY; ++k)
          if (yv[k + 1])
            asm volatile("prefetch.global.L2 [%0];" ::"l"(
                ut + base + unsigned(k) * unsigned(st1) + unsigned(sp) * unsigned(st3)));
    }
    const BandRow<CPLX> q2 = rows2[z - z0];
    const bool int2 = pat2[z - z0];
    const unsigned inz = in01 + unsigned(z) * unsigned(st2);
    const unsigned idz = out01 + unsigned(z) * plane;
    T res[NSP][RY];
#pragma unroll
    for (int k = 0; k < RY; ++k) {
#pragma unroll
      for (int sp = 0; sp < NSP; ++sp) {
        const unsigned in = inz + unsigned(k) * unsigned(st1) + unsigned(sp) * unsigned(st3);
        const T ctr = cur[sp][k + 1];
        T c;
        zero(c);
        if (a0) {
          // all 32 lanes shuffle (rows past the tensor hold zeros)
          T xl = shfl(ctr, true), xr = shfl(ctr, false);
          if (lane == 0) xl = xe[sp][k];
          if (lane == 31) xr = xe[sp][k];
          const T x[3] = {xl, ctr, xr};
          if (xv && yv[k + 1]) {
            if (pat0)
              row_combine<IM>(r0, x, c);
            else
              c = slow_term<CPLX>(&rows0[lane], ut, in, c);
          }
        }
        if (!xv || !yv[k + 1]) continue;
        if (a1) {
          if (pat1[threadIdx.y * RY + k]) {
            const BandRow<CPLX> q1 = rows1[threadIdx.y * RY + k];
            const T x[3] = {cur[sp][k], ctr, cur[sp][k + 2]};
            row_combine<IM>(q1, x, c);
          } else {
            c = slow_term<CPLX>(&rows1[threadIdx.y * RY + k], ut, in, c);
          }
        }
        if (a2) {
          if (int2) {
            const T x[3] = {zm[sp][k], ctr, nxt[sp][k + 1]};
            row_combine<IM>(q2, x, c);
          } else {
            c = slow_term<CPLX>(&rows2[z - z0], ut, in, c);
          }
        }
        res[sp][k] = c;
      }
    }
#pragma unroll
    for (int k = 0; k < RY; ++k) {
      if (!xv || !yv[k + 1]) continue;
      const unsigned idx = idz + unsigned(k) * unsigned(n0);
      if constexpr (NSP == 2) {
        if (with_g) {
          const double u0 = cur[0][k + 1], u1 = cur[1][k + 1];
          rt[idx] = __dadd_rn(res[0][k], g_real(g, u0, u1, false, idx, t));
          rt[idx + sp_out] = __dadd_rn(res[1][k], g_real(g, u1, u0, true, idx + sp_out, t));
        } else {
          rt[idx] = res[0][k];
          rt[idx + sp_out] = res[1][k];
        }
      } else if (!with_g) {
        rt[idx] = res[0][k];
      } else if constexpr (CPLX) {
        const double2 gg = g_cplx(g, cur[0][k + 1]);
        rt[idx] = make_double2(__dadd_rn(res[0][k].x, gg.x), __dadd_rn(res[0][k].y, gg.y));
      } else {
        rt[idx] = __dadd_rn(res[0][k], g_real(g, cur[0][k + 1], 0.0, false, idx, t));
      }
    }
#pragma unroll
    for (int sp = 0; sp < NSP; ++sp) {
#pragma unroll
      for (int k = 0; k < RY; ++k) {
        zm[sp][k] = cur[sp][k + 1];
        xe[sp][k] = xen[sp][k];
      }
#pragma unroll
      for (int k = 0; k < RY + 2; ++k) {
        cur[sp][k] = nxt[sp][k];
        nxt[sp][k] = pre[sp][k];
      }
    }
  }
  };
  if constexpr (CPLX) {
    if (imag)
      march(std::true_type{});
    else
      march(std::false_type{});
  } else {
    march(std::false_type{});
  }
}

// v7 launcher; false = not applicable
bool launch_band7(kp_ctx* ctx, const BandArgs& b2, bool cplx, bool pair, int nz, const double* u,
                  double* r, bool with_g, const kp_gfun& g, double t) {
  static const int mode = [] {  // opt-in (KP_BAND=v7): measured slower than v6
    const char* v = getenv("KP_BAND");
    return v && std::string(v) == "v7" ? 2 : 0;
  }();
  if (mode == 0 || b2.active[3] || b2.d < 3 || (!pair && b2.n[3] != 1)) return false;
  if ((b2.slab >= 0 && b2.slab != 2) || b2.stride[0] != 1) return false;
  static const int ry_env = [] {
    const char* v = getenv("KP_B7_RY");
    return v && *v ? atoi(v) : 0;
  }();
  static const int pf2 = [] {
    const char* v = getenv("KP_B7_PF");
    return v && *v ? atoi(v) : 6;
  }();
  static const long long per_sm = [] {
    const char* v = getenv("KP_B7_BLOCKS");
    return v && *v ? std::max(1LL, atoll(v)) : 12LL;
  }();
  const int ry = ry_env ? ry_env : ((cplx || pair) ? 2 : 4);
  if (ry != 2 && ry != 4) return false;
  if ((cplx || pair) && ry != 2) return false;
  constexpr int B7_WY = 4;
  const long long bxy = (long long)((b2.n[0] + 31) / 32) * ((b2.n[1] + B7_WY * ry - 1) / (B7_WY * ry));
  // enough blocks for a few waves; chunks as long as that allows (each chunk
  // start re-reads two planes)
  const long long want = ctx->num_sms * per_sm;
  long long chunks = std::max<long long>(1, (want + bxy - 1) / bxy);
  int zchunk = int(std::max<long long>(4, (nz + chunks - 1) / chunks));
  zchunk = std::min(zchunk, ZMAX7);
  const long long gz = (nz + zchunk - 1) / zchunk;
  const long long gy = (b2.n[1] + B7_WY * ry - 1) / (B7_WY * ry);
  if (gz > 65535 || gy > 65535) return false;
  dim3 grid(unsigned((b2.n[0] + 31) / 32), unsigned(gy), unsigned(gz));
  auto go = [&](auto kern) {
    launch_pdl(ctx, kern, grid, dim3(32, B7_WY), 0, b2, zchunk, pf2, u, r, with_g, g, t);
    ctx->launches--;  // counted once by the caller
  };
  if (cplx)
    go(kronsum_band7_kernel<true, 1, 2, B7_WY, 3>);
  else if (pair)
    go(kronsum_band7_kernel<false, 2, 2, B7_WY, 3>);
  else if (ry == 2)
    go(kronsum_band7_kernel<false, 1, 2, B7_WY, 4>);
  else
    go(kronsum_band7_kernel<false, 1, 4, B7_WY, 4>);
  return true;
}

// v6 launcher; false = not applicable (KP_BAND=v2 forces the v2 kernel)
bool launch_band6(kp_ctx* ctx, const BandArgs& b2, bool cplx, bool pair, int nz, int zchunk,
                  dim3 grid, const double* u, double* r, bool with_g, const kp_gfun& g,
                  double t) {
  // default for single-species tensors (AC3D 14.3 vs v2 20.2 us; NLS 512^3
  // 1.60 vs 1.63 ms); the species-pair form is opt-in (KP_BAND=v6): it
  // measured no faster than v2 on the Brusselator
  static const int mode = [] {
    const char* v = getenv("KP_BAND");
    if (!v || !*v) return 1;
    return std::string(v) == "v6" ? 2 : 0;
  }();
  if (mode == 0 || b2.active[3] || (!pair && b2.n[3] != 1)) return false;
  if (mode == 1 && pair) return false;
  auto go = [&](auto kern) {
    launch_pdl(ctx, kern, grid, dim3(32, 8), 0, b2, nz, zchunk, u, r, with_g, g, t);
    ctx->launches--;  // counted once by the caller
  };
  if (cplx)
    go(kronsum_band6_kernel<true, false>);
  else if (pair)
    go(kronsum_band6_kernel<false, true>);
  else
    go(kronsum_band6_kernel<false, false>);
  return true;
}

bool launch_band4(kp_ctx* ctx, const BandArgs& b2, bool cplx, bool pair, int nz, int zchunk,
                  dim3 grid, const double* u, double* r, bool with_g, const kp_gfun& g,
                  double t) {
  static const bool off = [] {
    const char* v = getenv("KP_BAND");
    return !(v && std::string(v) == "v4");
  }();
  if (off || b2.active[3] || b2.d < 3 || (!pair && b2.n[3] != 1)) return false;
  if (b2.slab >= 0 && b2.slab != 2) return false;
  auto go = [&](auto kern) {
    launch_pdl(ctx, kern, grid, dim3(32, 8), 0, b2, nz, zchunk, u, r, with_g, g, t);
    ctx->launches--;  // counted once by the caller
  };
  if (cplx)
    go(kronsum_band4_kernel<true, false>);
  else if (pair)
    go(kronsum_band4_kernel<false, true>);
  else
    go(kronsum_band4_kernel<false, false>);
  return true;
}

// v3 launcher; false = not applicable (the v2 kernel runs)
bool launch_band3(kp_ctx* ctx, const BandArgs& b2, bool cplx, bool pair, int nz,
                  const double* u, double* r, bool with_g, const kp_gfun& g, double t) {
  // opt-in (KP_BAND=v3): measured slower than v2 on the configs (AC3D 29.6
  // vs 27.9 us, NLS 512^3 2.14 vs 1.71 ms): the per-plane block barrier and
  // the single issuing thread cost more than the latency the ring hides
  static const bool off = [] {
    const char* v = getenv("KP_BAND");
    return !(v && std::string(v) == "v3");
  }();
  if (off || b2.active[3] || b2.d < 3 || (!pair && b2.n[3] != 1)) return false;
  if (b2.slab >= 0 && b2.slab != 2) return false;
  if (b2.stride[0] != 1 || b2.stride[1] != b2.n[0] ||
      b2.stride[2] != (long long)b2.n[0] * b2.n[1])
    return false;
  const int esz = cplx ? 16 : 8;
  if ((long long)b2.n[0] * esz % 16 || (reinterpret_cast<uintptr_t>(u) % 16)) return false;
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  if (!enc) return false;
  const long long h2 = b2.slab == 2 ? b2.halo : 0;
  const long long planes = pair ? b2.n[2] + 2 * h2 : (long long)b2.n[2] * b2.n[3] + 2 * h2;
  const long long nsp = pair ? 2 : 1;
  const int ce = cplx ? 2 : 1;  // doubles per element
  cuuint64_t dims[4] = {cuuint64_t(b2.n[0]) * ce, cuuint64_t(b2.n[1]), cuuint64_t(planes),
                        cuuint64_t(nsp)};
  const long long sp_stride = pair ? b2.stride[3] : planes * b2.n[0] * b2.n[1];
  cuuint64_t strides[3] = {cuuint64_t(b2.n[0]) * esz, cuuint64_t(b2.n[0]) * b2.n[1] * esz,
                           cuuint64_t(sp_stride) * esz};
  const int px = cplx ? tile_px<true>() : tile_px<false>();
  cuuint32_t box[4] = {cuuint32_t(px * ce), cuuint32_t(PY), 1u, 1u};
  cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  CUtensorMap map;
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(u), dims, strides, box,
          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  const long long bxy = (long long)((b2.n[0] + TX - 1) / TX) * ((b2.n[1] + TY - 1) / TY);
  const long long want = ctx->num_sms * 6LL;  // resident blocks per wave (smem-bound)
  const int zchunk = int(std::min<long long>(ZMAX, std::max<long long>(4, (nz * bxy + want - 1) / want)));
  if ((nz + zchunk - 1) / zchunk > 65535) return false;
  dim3 grid(unsigned((b2.n[0] + TX - 1) / TX), unsigned((b2.n[1] + TY - 1) / TY),
            unsigned((nz + zchunk - 1) / zchunk));
  const size_t tile_pad = (size_t(px) * PY * esz + 127) / 128 * 128;
  const size_t smem = size_t(D3) * tile_pad * nsp + D3 * 8;
  auto go = [&](auto kern) {
    ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), int(smem));
    launch_pdl(ctx, kern, grid, dim3(32, 8), smem, map, b2, nz, zchunk, u, r, with_g, g, t);
    ctx->launches--;  // counted once by the caller
  };
  if (cplx)
    go(kronsum_band3_kernel<true, false>);
  else if (pair)
    go(kronsum_band3_kernel<false, true>);
  else
    go(kronsum_band3_kernel<false, false>);
  return true;
}


// ---- the whole exp-Euler time loop of a small 2-D state in ONE launch ----
// (AC2D, configs[0]: 128 x 128, 100 steps; the regular loop is launch-bound
// at ~14 us per step for three ~2 us kernels.)  A cluster of SJ = 16 CTAs
// (distributed shared memory) holds the whole problem on chip: the phi_1
// factor L (128 x 128, 128 KiB) in every CTA's shared memory, the state in
// column blocks (CTA j owns columns [8j, 8j+8)).  Per step:
//   1  r = K u + g(u) on the column block (the banded row chains of v2; the
//      mode-1 neighbours of the block's edge columns are read from the
//      neighbour CTAs' shared memory);
//   2  y = L r (mode 0): each column block is independent (DMMA);
//   3  gather the row block [8j, 8j+8) of y and of u from all 16 CTAs;
//   4  u' = fma(tau, y L^T, u) (mode 1 + the exp-Euler update) on the rows;
//   5  scatter u' back into column blocks.
// Cluster barriers separate the phases; the loop never leaves the SMs.  The
// arithmetic is the regular path's (same row chains, same DMMA k order, the
// same FMA epilogue), so results are bit-identical to it.
constexpr int SN = 128, SJ = 16, SB = SN / SJ;
constexpr int SNT = 256, SW = SNT / 32, WR = SN / SW, MT = WR / 8;  // 8 warps, 16 rows each
constexpr int LP = SN + 8, RP = SN + 4;  // smem pitches of L and r (bank-conflict free)

__device__ __forceinline__ void sdmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(SNT, 1)
    small2d_expeuler_kernel(BandArgs b, const double* __restrict__ L, kp_gfun g, double tau,
                            long n_steps, double* __restrict__ u, int* bad) {
  namespace cgx = cooperative_groups;
  cgx::cluster_group cluster = cgx::this_cluster();
  const int j = int(cluster.block_rank());
  constexpr int HB = SB + 2;           // column block with a halo column each side
  extern __shared__ __align__(16) double sm[];
  // pitches chosen so the DMMA fragment loads are bank-conflict free:
  // L(row, k) at row + LP k (LP = 8 mod 32), r(k, c) at k + RP c (RP = 4 mod 32)
  double* Ls = sm;                     // L, column-major 128 x 128, pitch LP
  double* ub = Ls + LP * SN;           // u(:, 8j-1 .. 8j+8)   128 x 10 (halo columns 0, 9)
  double* rb = ub + SN * HB;           // r(:, block)          128 x 8, pitch RP
  double* yr = rb + RP * SB;           // y(rows 8j.., :)      8 x 128 (p fastest)
  double* ur = yr + SB * SN;           // u(rows 8j.., :)      8 x 128
  BandRow<false>* rows = reinterpret_cast<BandRow<false>*>(ur + SB * SN);  // [2][128]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
  for (int i = tid; i < SN * SN; i += SNT) Ls[(i % SN) + LP * (i / SN)] = L[i];
  for (int i = tid; i < SN * HB; i += SNT) {
    const int i0 = i % SN, h = i / SN;
    const int c = (j * SB + h - 1 + SN) % SN;  // halo columns wrap (periodic rows read them)
    ub[i] = u[i0 + (long long)SN * c];
  }
  for (int i = tid; i < 2 * SN; i += SNT) load_row(b, i / SN, i % SN, rows[i]);
  cluster.sync();
  // push targets: the row owner of row i is CTA i / 8; the column owner of
  // column c is CTA c / 8, which also holds c as a halo column of its neighbours
  bool nonfinite = false;
  int first_bad = 0;
  for (long step = 0; step < n_steps; ++step) {
    // ---- 1: r = K u + g(u) on the column block (local: the halo columns)
#pragma unroll
    for (int it = 0; it < SN * SB / SNT; ++it) {
      const int e = tid + SNT * it;
      const int i0 = e % SN, cl = e / SN, c = j * SB + cl;
      const BandRow<false>& r0 = rows[i0];
      const BandRow<false>& r1 = rows[SN + c];
      double x0[3], x1[3];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        x0[s] = ub[i0 + r0.off[s] + SN * (cl + 1)];
        int dc = r1.off[s] / SN;  // column delta, -1 / 0 / +1 modulo n (checked)
        if (dc > 1) dc -= SN;
        if (dc < -1) dc += SN;
        x1[s] = ub[i0 + SN * (cl + 1 + dc)];
      }
      double acc = 0.0;
      row_combine(r0, x0, acc);
      row_combine(r1, x1, acc);
      rb[i0 + RP * cl] =
          __dadd_rn(acc, g_real(g, ub[i0 + SN * (cl + 1)], 0.0, false, i0 + SN * c, 0.0));
    }
    __syncthreads();
    // ---- 2: y = L r (M = 128: warp w rows WR w.., N = 8, K = 128); push y
    // and u into the row owners' yr / ur
    {
      double acc[MT][2];
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) acc[mi][0] = acc[mi][1] = 0.0;
#pragma unroll 8
      for (int ks = 0; ks < SN / 4; ++ks) {
        const int k = 4 * ks + tq;
        const double bv = rb[k + RP * gq];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
          sdmma(acc[mi][0], acc[mi][1], Ls[(WR * warp + 8 * mi + gq) + LP * k], bv);
      }
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) {
        const int row = WR * warp + 8 * mi + gq, owner = row / SB, p = row - owner * SB;
        double* dy = cluster.map_shared_rank(yr, owner);
        double* du = cluster.map_shared_rank(ur, owner);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = j * SB + 2 * tq + h;
          dy[p + SB * c] = acc[mi][h];
          du[p + SB * c] = ub[row + SN * (2 * tq + h + 1)];
        }
      }
    }
    cluster.sync();
    // ---- 3: u' = fma(tau, y L^T, u) on the rows (M = 8, N = 128: warp w cols
    // WR w.., K = 128); push u' into the column owners' blocks and halos
    {
      double acc[MT][2];
#pragma unroll
      for (int ni = 0; ni < MT; ++ni) acc[ni][0] = acc[ni][1] = 0.0;
#pragma unroll 8
      for (int ks = 0; ks < SN / 4; ++ks) {
        const int k = 4 * ks + tq;
        const double av = yr[gq + SB * k];
#pragma unroll
        for (int ni = 0; ni < MT; ++ni)
          sdmma(acc[ni][0], acc[ni][1], av, Ls[(WR * warp + 8 * ni + gq) + LP * k]);
      }
#pragma unroll
      for (int ni = 0; ni < MT; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = WR * warp + 8 * ni + 2 * tq + h, row = j * SB + gq;
          const double v = __fma_rn(tau, acc[ni][h], ur[gq + SB * col]);
          if (!isfinite(v) && !nonfinite) {
            nonfinite = true;
            first_bad = int(step) + 1;
          }
          const int owner = col / SB, cl = col - owner * SB;
          cluster.map_shared_rank(ub, owner)[row + SN * (cl + 1)] = v;
          if (cl == 0)  // right halo of the left neighbour (wrapping)
            cluster.map_shared_rank(ub, (owner + SJ - 1) % SJ)[row + SN * (SB + 1)] = v;
          if (cl == SB - 1)  // left halo of the right neighbour
            cluster.map_shared_rank(ub, (owner + 1) % SJ)[row] = v;
        }
    }
    cluster.sync();
  }
  for (int i = tid; i < SN * SB; i += SNT)
    u[(i % SN) + (long long)SN * (j * SB + i / SN)] = ub[(i % SN) + SN * (i / SN + 1)];
  if (nonfinite) atomicMin(bad, first_bad);
}

}  // namespace

// forward (defined below)
void kronsum_banded(kp_ctx* ctx, bool cplx, const double* u, const std::vector<int>& dims,
                    const std::vector<const int*>& cols, const std::vector<const double*>& vals,
                    const std::vector<char>& active, double* r, bool with_g, const kp_gfun& g,
                    long long half, int slab, int k0, int n_glob, int halo, double t);

// Scan a factor into caller-provided device arrays (3n ints, 6n doubles),
// flags into slot `slot` (< 8) of the context's scratch, no sync;
// band_flags() then reads every slot back with ONE sync.
void band_scan_async(kp_ctx* ctx, const double* a, int n, bool cplx, int* dc, double* dv,
                     int slot) {
  int* flags = reinterpret_cast<int*>(ctx->d_flag) + 16 + 2 * slot;
  KP_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), ctx->stream));
  band_scan_kernel<<<(n + 7) / 8, 256, 0, ctx->stream>>>(a, n, cplx ? 2 : 1, dc, dv, flags);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
}
// (too_many, any_nonzero) of slots 0..nslots-1
std::vector<std::pair<bool, bool>> band_flags(kp_ctx* ctx, int nslots) {
  KP_CUDA(cudaMemcpyAsync(ctx->h_flag + 16, reinterpret_cast<int*>(ctx->d_flag) + 16,
                          2 * nslots * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  KP_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<std::pair<bool, bool>> f(nslots);
  for (int k = 0; k < nslots; ++k) f[k] = {ctx->h_flag[16 + 2 * k] != 0, ctx->h_flag[17 + 2 * k] != 0};
  return f;
}
bool band_scan(kp_ctx* ctx, const double* a, int n, bool cplx, int* dc, double* dv) {
  band_scan_async(ctx, a, n, cplx, dc, dv, 0);
  return !band_flags(ctx, 1)[0].first;
}

// Scan a factor into fresh allocations (owned by the caller).
bool band_of(kp_ctx* ctx, const double* a, int n, bool cplx, int** cols, double** vals) {
  int* dc = nullptr;
  double* dv = nullptr;
  KP_CUDA(cudaMalloc(&dc, sizeof(int) * 3 * size_t(n)));
  KP_CUDA(cudaMalloc(&dv, sizeof(double) * 6 * size_t(n)));
  if (!band_scan(ctx, a, n, cplx, dc, dv)) {
    cudaFree(dc);
    cudaFree(dv);
    return false;
  }
  *cols = dc;
  *vals = dv;
  return true;
}

// The whole exp-Euler loop of a 128 x 128 real state in one cluster launch
// (small2d_expeuler_kernel); false = not applicable.  u: device, in/out;
// L: the phi_1 factor of both modes (prefactor and fold 1); cols/vals: the
// band rows of A_0 and A_1; *bad: the first non-finite step (atomicMin).
bool small2d_expeuler(kp_ctx* ctx, const std::vector<int>& dims,
                      const std::vector<const int*>& cols, const std::vector<const double*>& vals,
                      const double* L, const kp_gfun& g, double tau, long n_steps, double* u,
                      int* bad) {
  static const bool off = getenv("KP_SMALL_LOOP") && std::string(getenv("KP_SMALL_LOOP")) == "0";
  if (off || dims.size() != 2 || dims[0] != SN || dims[1] != SN) return false;
  if (!(g.kind == KP_G_ZERO || g.kind == KP_G_SQUARE || g.kind == KP_G_CONST ||
        g.kind == KP_G_ALLEN_CAHN))
    return false;
  BandArgs b{};
  b.d = 2;
  for (int mu = 0; mu < 4; ++mu) {
    b.n[mu] = mu < 2 ? SN : 1;
    b.stride[mu] = mu == 0 ? 1 : (mu == 1 ? SN : 0);
    b.cols[mu] = mu < 2 ? cols[mu] : nullptr;
    b.vals[mu] = mu < 2 ? vals[mu] : nullptr;
    b.active[mu] = mu < 2 ? 1 : 0;
  }
  b.slab = -1;
  b.species = -1;
  auto kern = small2d_expeuler_kernel;
  // mode-1 rows must reach only the neighbour columns (mod n): the halo
  std::vector<int> hc(3 * SN);
  KP_CUDA(cudaMemcpyAsync(hc.data(), cols[1], hc.size() * sizeof(int), cudaMemcpyDeviceToHost,
                          ctx->stream));
  KP_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < SN; ++i)
    for (int s = 0; s < 3; ++s) {
      const int c = hc[3 * i + s];
      if (c < 0) continue;
      const int dlt = ((c - i) % SN + SN) % SN;
      if (!(dlt == 0 || dlt == 1 || dlt == SN - 1)) return false;
    }
  const size_t smem = sizeof(double) * (size_t(LP) * SN + size_t(SN) * (SB + 2) +
                                        size_t(RP) * SB + 2ull * SB * SN) +
                      2 * SN * sizeof(BandRow<false>);
  ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), int(smem));  // per device
  KP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(SJ);
  cfg.blockDim = dim3(SNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = SJ;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    return false;
  }
  KP_CUDA(cudaLaunchKernelEx(&cfg, kern, b, L, g, tau, n_steps, u, bad));
  ctx->launches++;
  return true;
}

// kronsum_action through the stencil when every factor is banded (workspace
// slots 30..37 hold the row structures); false = caller takes the dense path.
bool kronsum_try_banded(kp_ctx* ctx, bool cplx, const double* t, const std::vector<int>& dims,
                        const double* const* as, double* out) {
  const int d = int(dims.size());
  if (!banded_kronsum_enabled() || d > 4) return false;
  std::vector<const int*> cols(d);
  std::vector<const double*> vals(d);
  std::vector<char> active(d, 1);
  for (int mu = 0; mu < d; ++mu) {
    int* c = static_cast<int*>(ctx->ws.get(30 + mu, sizeof(int) * 3 * size_t(dims[mu])));
    double* v = static_cast<double*>(ctx->ws.get(34 + mu, sizeof(double) * 6 * size_t(dims[mu])));
    band_scan_async(ctx, as[mu], dims[mu], cplx, c, v, mu);
    cols[mu] = c;
    vals[mu] = v;
  }
  for (const auto& f : band_flags(ctx, d))
    if (f.first) return false;
  kronsum_banded(ctx, cplx, t, dims, cols, vals, active, out, false, kp_gfun{}, 0, -1, 0, 0, 0,
                 0.0);
  return true;
}

// KP_KRONSUM=dense selects the reference's dense form (read per call, so a
// process can compare both)
bool banded_kronsum_enabled() {
  const char* v = getenv("KP_KRONSUM");
  return !(v && std::string(v) == "dense");
}

// r = sum_mu u x_mu A_mu (+ g) with banded factors.  dims: up to 4 modes;
// inactive modes (zero factors) are skipped; cols/vals from band_of.
void kronsum_banded(kp_ctx* ctx, bool cplx, const double* u, const std::vector<int>& dims,
                    const std::vector<const int*>& cols, const std::vector<const double*>& vals,
                    const std::vector<char>& active, double* r, bool with_g, const kp_gfun& g,
                    long long half, int slab, int k0, int n_glob, int halo, double t) {
  const int d = int(dims.size());
  if (d > 4) throw invalid_argument("kronsum (banded): order > 4 unsupported");
  BandArgs b{};
  b.d = d;
  b.slab = slab;
  b.k0 = k0;
  b.n_glob = n_glob;
  b.halo = (slab >= 0) ? halo : 0;
  b.species = -1;
  if (half > 0) {
    if (dims.back() != 2) throw invalid_argument("brusselator g: slowest mode must hold 2 species");
    b.species = d - 1;
  }
  long long st = 1, total = 1;
  for (int mu = 0; mu < d; ++mu) {
    b.n[mu] = dims[mu];
    b.stride[mu] = st;
    st *= dims[mu] + (mu == slab ? 2 * b.halo : 0);
    total *= dims[mu];
    b.cols[mu] = cols[mu];
    b.vals[mu] = vals[mu];
    b.active[mu] = active[mu];
  }
  if (total > 0xffffffffLL) throw invalid_argument("kronsum: tensor too large for the stencil path");
  static const bool v1 = [] {  // KP_BAND=v1: the one-entry-per-thread kernel (A/B)
    const char* v = getenv("KP_BAND");
    return v && std::string(v) == "v1";
  }();
  if (v1) {
    const unsigned grid = unsigned(
        std::max<long long>(1, std::min<long long>((total + 255) / 256, ctx->num_sms * 16LL)));
    if (cplx)
      kronsum_band_kernel<true><<<grid, 256, 0, ctx->stream>>>(b, total, u, r, with_g, g, t);
    else
      kronsum_band_kernel<false><<<grid, 256, 0, ctx->stream>>>(b, total, u, r, with_g, g, t);
  } else {
    // pad to 4 modes; the 2-species mode (always the last, extent 2) is
    // moved to slot 3 so a thread can own both species of a grid point
    BandArgs b2 = b;
    for (int mu = d; mu < 4; ++mu) {
      b2.n[mu] = 1;
      b2.stride[mu] = 0;
      b2.cols[mu] = nullptr;
      b2.vals[mu] = nullptr;
      b2.active[mu] = 0;
    }
    bool pair = false;
    if (b.species >= 0 && !cplx) {
      const int sp = b.species;  // = d - 1
      if (sp != 3) {
        std::swap(b2.n[sp], b2.n[3]);
        std::swap(b2.stride[sp], b2.stride[3]);
        std::swap(b2.cols[sp], b2.cols[3]);
        std::swap(b2.vals[sp], b2.vals[3]);
        std::swap(b2.active[sp], b2.active[3]);
        if (b2.slab == sp) b2.slab = 3;
        else if (b2.slab == 3) b2.slab = sp;
      }
      b2.species = 3;
      pair = true;
    }
    const int nz = pair ? b2.n[2] : b2.n[2] * b2.n[3];
    const long long bxy = (long long)((b2.n[0] + 31) / 32) * ((b2.n[1] + 7) / 8);
    static const long long per_sm = [] {
      const char* v = getenv("KP_BAND_BLOCKS");
      return v && *v ? std::max(1LL, atoll(v)) : 4LL;
    }();
    // z chunks long enough to amortise a thread's row set-up (AC3D: 13 planes;
    // measured best at 4 blocks per SM, KP_BAND_BLOCKS overrides)
    const long long want = ctx->num_sms * per_sm;
    int zchunk = int(std::min<long long>(ZMAX, std::max<long long>(1, (nz * bxy + want - 1) / want)));
    if ((nz + zchunk - 1) / zchunk > 65535)
      throw invalid_argument("kronsum: modes 2-3 too large for the stencil path");
    dim3 grid(unsigned((b2.n[0] + 31) / 32), unsigned((b2.n[1] + 7) / 8),
              unsigned((nz + zchunk - 1) / zchunk));
    if (grid.y > 65535) throw invalid_argument("kronsum: mode 1 too large for the stencil path");
    long long ext = 1;  // input extent incl. halo planes: 32-bit offsets
    for (int mu = 0; mu < d; ++mu) ext *= dims[mu] + (mu == slab ? 2 * b.halo : 0);
    if (ext > 0x7fffffffLL) throw invalid_argument("kronsum: tensor too large for the stencil path");
    const bool m3 = b2.active[3] != 0;
    if (launch_band3(ctx, b2, cplx, pair, nz, u, r, with_g, g, t)) {
      ctx->launches++;
      KP_CUDA(cudaGetLastError());
      return;
    }
    if (!m3 && launch_band4(ctx, b2, cplx, pair, nz, zchunk, grid, u, r, with_g, g, t)) {
      ctx->launches++;
      KP_CUDA(cudaGetLastError());
      return;
    }
    if (launch_band8(ctx, b2, cplx, pair, nz, u, r, with_g, g, t) ||
        launch_band7(ctx, b2, cplx, pair, nz, u, r, with_g, g, t)) {
      ctx->launches++;
      KP_CUDA(cudaGetLastError());
      return;
    }
    if (launch_band6(ctx, b2, cplx, pair, nz, zchunk, grid, u, r, with_g, g, t)) {
      ctx->launches++;
      KP_CUDA(cudaGetLastError());
      return;
    }
    auto go = [&](auto kern) {
      launch_pdl(ctx, kern, grid, dim3(32, 8), 0, b2, nz, zchunk, u, r, with_g, g, t);
      ctx->launches--;  // counted once below
    };
    static const bool v5 = [] {
      const char* v = getenv("KP_BAND");
      return v && std::string(v) == "v5";
    }();
    if (v5 && !m3) {
      if (cplx)
        go(kronsum_band2_kernel<true, false, false, true>);
      else if (pair)
        go(kronsum_band2_kernel<false, true, false, true>);
      else
        go(kronsum_band2_kernel<false, false, false, true>);
    } else if (cplx) {
      m3 ? go(kronsum_band2_kernel<true, false, true>) : go(kronsum_band2_kernel<true, false, false>);
    } else if (pair) {
      m3 ? go(kronsum_band2_kernel<false, true, true>) : go(kronsum_band2_kernel<false, true, false>);
    } else {
      m3 ? go(kronsum_band2_kernel<false, false, true>) : go(kronsum_band2_kernel<false, false, false>);
    }
  }
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
}

}  // namespace kp

// ---- C ABI: the banded action on a slab with halo planes (sharded runs) ----
using namespace kp;

extern "C" int kp_kronsum_slab_f64(kp_ctx* ctx, const double* u_ext, const int* dims, int d,
                                   const double* const* as, int slab_mode, int k0, int n_glob,
                                   const kp_gfun* g, double* r);
extern "C" int kp_kronsum_slab_c128(kp_ctx* ctx, const double* u_ext, const int* dims, int d,
                                    const double* const* as, int slab_mode, int k0, int n_glob,
                                    const kp_gfun* g, double* r);

namespace {
int slab_impl(kp_ctx* ctx, bool cplx, const double* u_ext, const int* dims, int d,
              const double* const* as, int slab_mode, int k0, int n_glob, const kp_gfun* g,
              double* r) {
  try {
    if (!ctx) throw invalid_argument("kronphi_b200: null context");
    KP_CUDA(cudaSetDevice(ctx->device));
    if (d <= 0 || d > 4 || !dims || !as)
      throw invalid_argument("kronsum_slab: order must be 1..4");
    std::vector<int> dv(dims, dims + d);
    if (slab_mode < 0 || slab_mode >= d) throw invalid_argument("kronsum_slab: bad slab mode");
    std::vector<const int*> cols(d);
    std::vector<const double*> vals(d);
    std::vector<char> active(d, 1);
    for (int mu = 0; mu < d; ++mu) {
      const int n = (mu == slab_mode) ? n_glob : dv[mu];
      int* c = static_cast<int*>(ctx->ws.get(30 + mu, sizeof(int) * 3 * size_t(n)));
      double* v = static_cast<double*>(ctx->ws.get(34 + mu, sizeof(double) * 6 * size_t(n)));
      band_scan_async(ctx, as[mu], n, cplx, c, v, mu);
      cols[mu] = c;
      vals[mu] = v;
    }
    const auto flags = band_flags(ctx, d);  // one sync for every factor
    for (int mu = 0; mu < d; ++mu) {
      if (flags[mu].first)
        throw invalid_argument("kronsum_slab: factor " + std::to_string(mu) +
                               " has more than three nonzeros in a row");
      // an all-zero factor (the stacked species mode) contributes nothing
      const int n = (mu == slab_mode) ? n_glob : dv[mu];
      if (n <= 2) active[mu] = flags[mu].second;
    }
    long long half = 0;
    if (g && g->kind == KP_G_BRUSSELATOR) half = 1;  // species = last mode
    kronsum_banded(ctx, cplx, u_ext, dv, cols, vals, active, r, g != nullptr,
                   g ? *g : kp_gfun{}, half, slab_mode, k0, n_glob, 1, 0.0);
    return KP_OK;
  } catch (const std::invalid_argument& e) {
    kp_set_last_error(e.what());
    return KP_EINVAL;
  } catch (const kp::cuda_error& e) {
    kp_set_last_error(e.what());
    return KP_ECUDA;
  } catch (const std::exception& e) {
    kp_set_last_error(e.what());
    return KP_ERUNTIME;
  }
}
}  // namespace

extern "C" int kp_kronsum_slab_f64(kp_ctx* ctx, const double* u_ext, const int* dims, int d,
                                   const double* const* as, int slab_mode, int k0, int n_glob,
                                   const kp_gfun* g, double* r) {
  return slab_impl(ctx, false, u_ext, dims, d, as, slab_mode, k0, n_glob, g, r);
}
extern "C" int kp_kronsum_slab_c128(kp_ctx* ctx, const double* u_ext, const int* dims, int d,
                                    const double* const* as, int slab_mode, int k0, int n_glob,
                                    const kp_gfun* g, double* r) {
  return slab_impl(ctx, true, u_ext, dims, d, as, slab_mode, k0, n_glob, g, r);
}

// ---- pre-scanned band structures: the slab action without a per-call scan ----
// kp_kronsum_slab_* scans its factors on every call (one host sync); a
// host loop that applies the same factors every step (the sharded
// integrators) scans once with kp_band_create and calls the _banded form,
// which never synchronizes -- the CPU keeps running ahead of the GPU.
struct kp_band {
  int n = 0;
  bool cplx = false, any = false;
  int* cols = nullptr;
  double* vals = nullptr;
};

extern "C" int kp_band_create(kp_ctx* ctx, const double* a, int n, int cplx, kp_band** out) {
  try {
    if (!ctx || !a || !out || n <= 0) throw invalid_argument("band_create: bad arguments");
    KP_CUDA(cudaSetDevice(ctx->device));
    auto* b = new kp_band;
    b->n = n;
    b->cplx = cplx != 0;
    try {
      KP_CUDA(cudaMalloc(&b->cols, sizeof(int) * 3 * size_t(n)));
      KP_CUDA(cudaMalloc(&b->vals, sizeof(double) * 6 * size_t(n)));
      band_scan_async(ctx, a, n, b->cplx, b->cols, b->vals, 0);
      const auto f = band_flags(ctx, 1)[0];
      if (f.first) throw invalid_argument("band_create: more than three nonzeros in a row");
      b->any = f.second;
    } catch (...) {
      cudaFree(b->cols);
      cudaFree(b->vals);
      delete b;
      throw;
    }
    *out = b;
    return KP_OK;
  } catch (const std::invalid_argument& e) {
    kp_set_last_error(e.what());
    return KP_EINVAL;
  } catch (const kp::cuda_error& e) {
    kp_set_last_error(e.what());
    return KP_ECUDA;
  } catch (const std::exception& e) {
    kp_set_last_error(e.what());
    return KP_ERUNTIME;
  }
}

extern "C" int kp_band_destroy(kp_band* b) {
  if (!b) return KP_OK;
  cudaFree(b->cols);
  cudaFree(b->vals);
  delete b;
  return KP_OK;
}

namespace {
int slab_banded_impl(kp_ctx* ctx, bool cplx, const double* u_ext, const int* dims, int d,
                     const kp_band* const* bands, int slab_mode, int k0, int n_glob,
                     const kp_gfun* g, double* r) {
  try {
    if (!ctx) throw invalid_argument("kronphi_b200: null context");
    KP_CUDA(cudaSetDevice(ctx->device));
    if (d <= 0 || d > 4 || !dims || !bands)
      throw invalid_argument("kronsum_slab: order must be 1..4");
    std::vector<int> dv(dims, dims + d);
    if (slab_mode < 0 || slab_mode >= d) throw invalid_argument("kronsum_slab: bad slab mode");
    std::vector<const int*> cols(d);
    std::vector<const double*> vals(d);
    std::vector<char> active(d, 1);
    for (int mu = 0; mu < d; ++mu) {
      const kp_band* b = bands[mu];
      const int n = (mu == slab_mode) ? n_glob : dv[mu];
      if (!b || b->n != n || b->cplx != cplx)
        throw invalid_argument("kronsum_slab: band " + std::to_string(mu) +
                               " does not match the mode size / type");
      cols[mu] = b->cols;
      vals[mu] = b->vals;
      if (n <= 2) active[mu] = b->any;  // the stacked species mode contributes nothing
    }
    long long half = 0;
    if (g && g->kind == KP_G_BRUSSELATOR) half = 1;
    kronsum_banded(ctx, cplx, u_ext, dv, cols, vals, active, r, g != nullptr,
                   g ? *g : kp_gfun{}, half, slab_mode, k0, n_glob, 1, 0.0);
    return KP_OK;
  } catch (const std::invalid_argument& e) {
    kp_set_last_error(e.what());
    return KP_EINVAL;
  } catch (const kp::cuda_error& e) {
    kp_set_last_error(e.what());
    return KP_ECUDA;
  } catch (const std::exception& e) {
    kp_set_last_error(e.what());
    return KP_ERUNTIME;
  }
}
}  // namespace

extern "C" int kp_kronsum_slab_banded_f64(kp_ctx* ctx, const double* u_ext, const int* dims,
                                          int d, const kp_band* const* bands, int slab_mode,
                                          int k0, int n_glob, const kp_gfun* g, double* r) {
  return slab_banded_impl(ctx, false, u_ext, dims, d, bands, slab_mode, k0, n_glob, g, r);
}
extern "C" int kp_kronsum_slab_banded_c128(kp_ctx* ctx, const double* u_ext, const int* dims,
                                           int d, const kp_band* const* bands, int slab_mode,
                                           int k0, int n_glob, const kp_gfun* g, double* r) {
  return slab_banded_impl(ctx, true, u_ext, dims, d, bands, slab_mode, k0, n_glob, g, r);
}
