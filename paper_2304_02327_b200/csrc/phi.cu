// phi.cu -- the small-matrix phi_l(tau A_mu) factors on the device, batched.
//
// Restates the reference's matrix-function layer with the same algorithms and
// thresholds, every O(n^3) step on the DMMA GEMM (launch_gemm):
//   expm          inc/matrix_functions.hpp:76-95  (Pade 3/5/7/9/13, theta table :20-22)
//   pade_low/13   inc/matrix_functions.hpp:37-72  (elementwise sums in the same
//                 order, each product/sum separately rounded like the
//                 reference's temporaries)
//   lu_factor     inc/linsolve.hpp:125-146 (64-wide panels, partial pivoting
//                 over the full column, trailing update = GEMM)
//   lu_solve      inc/linsolve.hpp:149-176
//   phiquad       inc/matrix_functions.hpp:146-199 (GLL nodes on the host,
//                 src/gll_rule.cpp:35-72; q-1 expms batched in one pass)
//   phi_square_step inc/matrix_functions.hpp:121-138 (all orders from
//                 same-scale values; phi0*phi_j as one batched GEMM)
// Matrices of one call are processed as a batch (stride n*n) so the 11 GLL
// nodes (and several factors) share every launch.  The data-dependent
// branches of the reference (scaling exponent, Pade degree, singularity) read
// small device results back to the host: a handful of 8-byte syncs per build.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <string>
#include <vector>

#include <cooperative_groups.h>

#include "kp_internal.h"

namespace cg = cooperative_groups;

namespace kp {
namespace {

constexpr int LU_NB = 64;  // inc/linsolve.hpp:22

const double kPadeTheta[5] = {1.495585217958292e-2, 2.539398330063230e-1,
                              9.504178996162932e-1, 2.097847961257068e0, 5.371920351148152e0};
const std::vector<std::vector<double>>& pade_coeffs() {  // inc/matrix_functions.hpp:24-35
  static const std::vector<std::vector<double>> b = {
      {120., 60., 12., 1.},
      {30240., 15120., 3360., 420., 30., 1.},
      {17297280., 8648640., 1995840., 277200., 25200., 1512., 56., 1.},
      {17643225600., 8821612800., 2075673600., 302702400., 30270240., 2162160., 110880.,
       3960., 90., 1.},
      {64764752532480000., 32382376266240000., 7771770303897600., 1187353796428800.,
       129060195264000., 10559470521600., 670442572800., 33522128640., 1323241920.,
       40840800., 960960., 16380., 182., 1.}};
  return b;
}

double factorial(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f *= i;
  return f;
}

unsigned grid1(kp_ctx* ctx, long long n, int threads = 256) {
  return unsigned(std::max<long long>(1, std::min<long long>((n + threads - 1) / threads,
                                                              ctx->num_sms * 16LL)));
}

// ---------------------------------------------------------------- kernels

// out[b] = max_j sum_i |x_b(i,j)|, sums in increasing i (inc/matrix.hpp norm1).
// One warp per 32 columns: 32 x 32 tiles staged through shared memory so the
// loads are coalesced along the column while each lane keeps its column's
// sequential sum; the per-warp maxima meet in an atomicMax on the bit pattern
// (non-negative doubles order like their int64 bits).  out must be zeroed.
__global__ void norm1_kernel(const double* __restrict__ x, int n, long long stride,
                             double* __restrict__ out) {
  __shared__ double tile[32][33];
  const double* xb = x + blockIdx.y * stride;
  const int lane = threadIdx.x, c0 = blockIdx.x * 32;
  double s = 0.0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    double v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c)  // 32 independent loads in flight
      v[c] = (i < n && c0 + c < n) ? xb[i + (long long)(c0 + c) * n] : 0.0;
#pragma unroll
    for (int c = 0; c < 32; ++c) tile[c][lane] = fabs(v[c]);
    __syncwarp();
    const int m = min(32, n - i0);
    for (int r = 0; r < m; ++r) s = __dadd_rn(s, tile[lane][r]);
    __syncwarp();
  }
  double best = (c0 + lane < n) ? s : 0.0;
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(out + blockIdx.y),
              static_cast<unsigned long long>(__double_as_longlong(best)));
}

// y_b = x * scale_b  (per-batch scalar; x shared when xstride == 0)
__global__ void scale_batch_kernel(const double* __restrict__ x, long long xstride,
                                   const double* __restrict__ scale, long long nn, int batch,
                                   double* __restrict__ y) {
  const long long total = nn * batch;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long b = t / nn, e = t - b * nn;
    y[t] = __dmul_rn(x[b * xstride + e], scale[b]);
  }
}

// Pade numerator/denominator sums of pade_low (inc/matrix_functions.hpp:45-50):
// u = b1 I, v = b0 I, then for p: u += b[2p+3] pow_p, v += b[2p+2] pow_p.
__global__ void pade_uv_kernel(const double* __restrict__ pw, int npow, long long nn, int n,
                               int batch, double b0, double b1, const double* __restrict__ bu,
                               const double* __restrict__ bv, double* __restrict__ u,
                               double* __restrict__ v) {
  const long long total = nn * batch;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long b = t / nn, e = t - b * nn;
    const bool diag = (e % (n + 1)) == 0;
    double uu = diag ? b1 : 0.0, vv = diag ? b0 : 0.0;
    for (int p = 0; p < npow; ++p) {
      const double x = pw[(long long)p * nn * batch + t];
      uu = __dadd_rn(uu, __dmul_rn(bu[p], x));
      vv = __dadd_rn(vv, __dmul_rn(bv[p], x));
    }
    u[t] = uu;
    v[t] = vv;
    (void)b;
  }
}

// pade13 sums (inc/matrix_functions.hpp:63-69):
//   w1 = c0*a6 + c1*a4 + c2*a2                    (then multiplied by a6)
//   w2 = d0*a6 + d1*a4 + d2*a2 + d3*I             (added after the product)
__global__ void pade13_w_kernel(const double* __restrict__ a2, const double* __restrict__ a4,
                                const double* __restrict__ a6, long long total, int n,
                                long long nn, double c0, double c1, double c2,
                                double* __restrict__ w) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    w[t] = __dadd_rn(__dadd_rn(__dmul_rn(c0, a6[t]), __dmul_rn(c1, a4[t])),
                     __dmul_rn(c2, a2[t]));
  }
  (void)n;
  (void)nn;
}
__global__ void pade13_add_kernel(const double* __restrict__ a2, const double* __restrict__ a4,
                                  const double* __restrict__ a6, long long total, int n,
                                  long long nn, double d0, double d1, double d2, double d3,
                                  double* __restrict__ w) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long e = t % nn;
    const double eye = (e % (n + 1)) == 0 ? 1.0 : 0.0;
    const double rhs = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(d0, a6[t]), __dmul_rn(d1, a4[t])),
                                           __dmul_rn(d2, a2[t])),
                                 __dmul_rn(d3, eye));
    w[t] = __dadd_rn(w[t], rhs);
  }
}

// lhs = v - u, rhs = v + u
__global__ void pm_kernel(const double* __restrict__ u, const double* __restrict__ v,
                          long long total, double* __restrict__ lhs, double* __restrict__ rhs) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const double uu = u[t], vv = v[t];
    lhs[t] = __dsub_rn(vv, uu);
    rhs[t] = __dadd_rn(vv, uu);
  }
}

// ---- LU (inc/linsolve.hpp) ----

// Panel factorization of a_b(j0:n, j0:j0+nb) (lu_panel, :56-81): one CTA per
// matrix.  Pivot = first row of maximal |a| (strict >, increasing i).
__global__ void lu_panel_kernel(double* __restrict__ a, int n, long long stride, int j0, int nb,
                                int* __restrict__ piv, int* __restrict__ singular) {
  double* ab = a + blockIdx.x * stride;
  int* pb = piv + (long long)blockIdx.x * n;
  __shared__ double sval[32];
  __shared__ int sidx[32];
  __shared__ int s_p;
  __shared__ double s_inv;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int j = j0; j < j0 + nb; ++j) {
    double* colj = ab + (long long)j * n;
    // argmax |a(i, j)|, i >= j; ties -> smallest i
    double best = -1.0;
    int bi = n;
    for (int i = j + tid; i < n; i += nt) {
      const double v = fabs(colj[i]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if ((tid & 31) == 0) {
      sval[tid >> 5] = best;
      sidx[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid < 32) {
      best = tid < (nt >> 5) ? sval[tid] : -1.0;
      bi = tid < (nt >> 5) ? sidx[tid] : n;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (tid == 0) {
        if (!(best > 0.0)) {
          *singular = 1;
          bi = j;
        }
        s_p = bi;
        pb[j] = bi;
      }
    }
    __syncthreads();
    const int p = s_p;
    if (p != j) {
      for (int c = j0 + tid; c < j0 + nb; c += nt) {
        const double t = ab[j + (long long)c * n];
        ab[j + (long long)c * n] = ab[p + (long long)c * n];
        ab[p + (long long)c * n] = t;
      }
    }
    __syncthreads();
    if (tid == 0) s_inv = 1.0 / colj[j];
    __syncthreads();
    const double inv = s_inv;
    for (int i = j + 1 + tid; i < n; i += nt) colj[i] = __dmul_rn(colj[i], inv);
    __syncthreads();
    for (int c = j + 1; c < j0 + nb; ++c) {
      double* colc = ab + (long long)c * n;
      const double ajc = colc[j];
      if (ajc == 0.0) continue;
      for (int i = j + 1 + tid; i < n; i += nt) colc[i] = __fma_rn(-colj[i], ajc, colc[i]);
    }
    __syncthreads();
  }
}

// The same panel factorization with the panel spread over a thread-block
// cluster: one cluster per matrix, the panel rows j0..n-1 split into
// contiguous chunks of rows_per (<= 256) rows, one chunk per CTA.  Each row
// lives in registers: warps 0-7 hold its columns 0..31, warps 8-15 its
// columns 32..63 (so the live column range is warp-uniform).
// Per column there is no cluster-wide barrier: every CTA PUSHES its local
// pivot candidate (|a|, row, and the row's 64 values) into a slot of every
// CTA's shared memory with st.async, which completes bytes on the receiver's
// mbarrier; the owner of row j pushes row j the same way.  Each CTA then
// waits on its own mbarrier, reduces the candidates locally (same tie rule as
// lu_panel_kernel: largest |a|, then smallest row), takes the pivot row from
// the winner's slot, the owners of rows j and p swap their registers, the
// multipliers l_i are formed by the half holding column j and passed through
// shared memory, and every thread rank-1 updates its live columns.  Slots
// and mbarriers are double-buffered by column parity: a CTA can run at most
// one column ahead of any other (it needs their next candidates), so a slot
// is never overwritten while its previous contents are still in use.
// The arithmetic is exactly lu_panel_kernel's (x * (1/pivot),
// fma(-l_i, u_c, a_ic), u_c == 0 skipped): the factors are bitwise identical.
constexpr int LUC_THREADS = 512;
constexpr int LUC_HALF = LU_NB / 2;
constexpr int LUC_ROWS = LUC_THREADS / 2;  // rows per CTA (max)
constexpr int LUC_MAXCL = 16;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_addr(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
// 16 bytes into another CTA's shared memory, completing on its mbarrier
__device__ __forceinline__ void push16(uint32_t raddr, double x, double y, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
          raddr),
      "d"(x), "d"(y), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nKP_WAIT%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra KP_WAIT%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// Cluster-wide barrier with release/acquire at cluster scope (setup/teardown).
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Dynamic index into a thread's register row: a switch on a warp-uniform
// index compiles to one indirect branch instead of a 32-way select chain.
#define KP_CASE32(M) M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) \
  M(13) M(14) M(15) M(16) M(17) M(18) M(19) M(20) M(21) M(22) M(23) M(24) M(25) M(26) M(27) \
  M(28) M(29) M(30) M(31)
__device__ __forceinline__ double reg_get(const double (&r)[LUC_HALF], int k) {
  double v = 0.0;
  switch (k) {
#define KP_GET(K) \
  case K:         \
    v = r[K];     \
    break;
    KP_CASE32(KP_GET)
#undef KP_GET
  }
  return v;
}
__device__ __forceinline__ void reg_set(double (&r)[LUC_HALF], int k, double v) {
  switch (k) {
#define KP_SET(K) \
  case K:         \
    r[K] = v;     \
    break;
    KP_CASE32(KP_SET)
#undef KP_SET
  }
}
// r[k] -= l * u[k] for k >= k0 (u[k] == 0 skipped): Duff's device on a
// warp-uniform start, so only the live columns are visited.
__device__ __forceinline__ void row_update_from(double (&r)[LUC_HALF], int k0, double l,
                                                const double* __restrict__ u) {
  switch (k0) {
#define KP_UPD(K)                                   \
  case K: {                                         \
    const double ajc = u[K];                        \
    if (ajc != 0.0) r[K] = __fma_rn(-l, ajc, r[K]); \
  }                                                 \
    [[fallthrough]];
    KP_CASE32(KP_UPD)
#undef KP_UPD
    default:
      break;
  }
}

__device__ __forceinline__ void argmax_merge(double& best, int& bi, double ov, int oi) {
  if (ov > best || (ov == best && oi < bi)) {
    best = ov;
    bi = oi;
  }
}

__device__ __forceinline__ void warp_argmax(double& best, int& bi) {
  for (int o = 16; o > 0; o >>= 1)
    argmax_merge(best, bi, __shfl_xor_sync(0xffffffffu, best, o),
                 __shfl_xor_sync(0xffffffffu, bi, o));
}

__global__ void __launch_bounds__(LUC_THREADS, 1)
    lu_panel_cluster_kernel(double* __restrict__ a, int n, long long stride, int j0, int nb,
                            int rows_per, int* __restrict__ piv, int* __restrict__ singular) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = int(cl.block_rank());
  const int ncta = int(cl.num_blocks());
  __shared__ __align__(16) double in_row[2][LUC_MAXCL][LU_NB];  // candidates' rows
  __shared__ __align__(16) double in_hdr[2][LUC_MAXCL][2];      // (|a|, row) per rank
  __shared__ __align__(16) double in_jrow[2][LU_NB];            // row j
  __shared__ __align__(16) double out_row[LU_NB];   // this CTA's candidate row
  __shared__ __align__(16) double out_jrow[LU_NB];  // row j (its owner only)
  __shared__ __align__(8) unsigned long long mbar[2];
  __shared__ double lmul[LUC_ROWS];  // multipliers of the current column
  __shared__ double wv[8];
  __shared__ int wi[8];
  __shared__ int s_piv[LU_NB];  // pivots, flushed at the end
  __shared__ int s_sing;
  double* ab = a + blockIdx.y * stride;
  int* pb = piv + (long long)blockIdx.y * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = warp >> 3;                // column half of this thread
  const int lr = (warp & 7) * 32 + lane;  // local row
  const int r0 = j0 + rank * rows_per;
  const int rows = max(0, min(n, r0 + rows_per) - r0);
  const bool has_row = lr < rows;
  const int row = r0 + lr;
  const uint32_t bytes_per_col = uint32_t(ncta) * (LU_NB + 2) * 8 + LU_NB * 8;
  if (tid == 0) {
    s_sing = 0;
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mbar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double r[LUC_HALF];
#pragma unroll
  for (int k = 0; k < LUC_HALF; ++k) {
    const int c = h * LUC_HALF + k;
    r[k] = (has_row && c < nb) ? ab[row + (long long)(j0 + c) * n] : 0.0;
  }
  cluster_barrier();  // every CTA's mbarriers are initialised before any push
  // push lanes: thread t sends 16 bytes (chunk t % 32) to rank t / 32
  const int dst = tid >> 5, chunk = lane;
  const bool pusher = dst < ncta;
#pragma unroll 1
  for (int jj = 0; jj < nb; ++jj) {
    const int j = j0 + jj, buf = jj & 1;
    const int hj = jj / LUC_HALF, kj = jj % LUC_HALF;
    const int oj = jj / rows_per;
    // 1. local argmax over the rows >= j (the warps holding column jj)
    if (h == hj) {
      double best = -1.0;
      int bi = n;
      if (has_row && row >= j) {
        best = fabs(reg_get(r, kj));
        bi = row;
      }
      warp_argmax(best, bi);
      if (lane == 0) {
        wv[warp & 7] = best;
        wi[warp & 7] = bi;
      }
    }
    __syncthreads();
    double lbest = lane < 8 ? wv[lane] : -1.0;
    int lbi = lane < 8 ? wi[lane] : n;
    warp_argmax(lbest, lbi);
    if (has_row && row == lbi) {
#pragma unroll
      for (int k = 0; k < LUC_HALF; ++k) out_row[h * LUC_HALF + k] = r[k];
    }
    if (has_row && row == j) {
#pragma unroll
      for (int k = 0; k < LUC_HALF; ++k) out_jrow[h * LUC_HALF + k] = r[k];
    }
    __syncthreads();
    // 2. push the candidate (and row j) to every rank; expect this column's bytes
    if (tid == 0) mbar_expect(smem_addr(&mbar[buf]), bytes_per_col);
    if (pusher) {
      const uint32_t rbar = cluster_addr(smem_addr(&mbar[buf]), dst);
      const double2 v = reinterpret_cast<const double2*>(out_row)[chunk];
      push16(cluster_addr(smem_addr(&in_row[buf][rank][2 * chunk]), dst), v.x, v.y, rbar);
      if (chunk == 0)
        push16(cluster_addr(smem_addr(&in_hdr[buf][rank][0]), dst), lbest, double(lbi), rbar);
      if (rank == oj) {
        const double2 w = reinterpret_cast<const double2*>(out_jrow)[chunk];
        push16(cluster_addr(smem_addr(&in_jrow[buf][2 * chunk]), dst), w.x, w.y, rbar);
      }
    }
    mbar_wait(smem_addr(&mbar[buf]), uint32_t((jj >> 1) & 1));
    // 3. global pivot (every warp, from local copies)
    double best = -1.0;
    int bi = n;
    if (lane < ncta) {
      best = in_hdr[buf][lane][0];
      bi = int(in_hdr[buf][lane][1]);
    }
    warp_argmax(best, bi);
    const bool sing = !(best > 0.0);
    const int p = sing ? j : bi;  // singular column: no swap, pivot row = row j
    if (tid == 0) {
      if (sing) s_sing = 1;
      s_piv[jj] = p;
    }
    const int op = (p - j0) / rows_per;
    const double* prow = (p == j) ? in_jrow[buf] : in_row[buf][op];
    // 4. swap rows j and p, multipliers of column jj
    if (p != j && has_row) {
      if (row == j) {
#pragma unroll
        for (int k = 0; k < LUC_HALF; ++k) r[k] = prow[h * LUC_HALF + k];
      } else if (row == p) {
#pragma unroll
        for (int k = 0; k < LUC_HALF; ++k) r[k] = in_jrow[buf][h * LUC_HALF + k];
      }
    }
    const bool below = has_row && row > j;
    if (h == hj && below) {
      const double l = __dmul_rn(reg_get(r, kj), 1.0 / prow[jj]);
      reg_set(r, kj, l);
      lmul[lr] = l;
    }
    __syncthreads();
    // 5. rank-1 update of the columns > jj
    const int k0 = jj + 1 - h * LUC_HALF;  // first live column of this half
    if (below && k0 < LUC_HALF) row_update_from(r, max(k0, 0), lmul[lr], prow + h * LUC_HALF);
  }
  cluster_barrier();  // all pushes into every CTA have landed and been consumed
  if (rank == 0) {
    if (tid < nb) pb[j0 + tid] = s_piv[tid];
    if (tid == 0 && s_sing) *singular = 1;
  }
#pragma unroll
  for (int k = 0; k < LUC_HALF; ++k) {
    const int c = h * LUC_HALF + k;
    if (has_row && c < nb) ab[row + (long long)(j0 + c) * n] = r[k];
  }
}

// Row swaps j0..j0+nb-1 applied to columns [c0, c1) (lu_apply_swaps, :85-92)
// of a matrix with leading dimension ld (ld rows); one thread per column.
__global__ void swaps_kernel(double* __restrict__ a, int ld, long long stride,
                             const int* __restrict__ piv, int n, int j0, int nb, int c0, int c1) {
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  double* col = a + blockIdx.y * stride + (long long)c * ld;
  const int* pb = piv + (long long)blockIdx.y * n;
  for (int j = j0; j < j0 + nb; ++j) {
    const int p = pb[j];
    if (p != j) {
      const double t = col[j];
      col[j] = col[p];
      col[p] = t;
    }
  }
}

// Inverses of the diagonal nb x nb blocks of a factored LU (blockIdx.z = 0:
// unit lower L, 1: upper U) for the blocks blk0 .. blk0 + gridDim.x - 1:
// inv[(b * nblk + blk) * 2 + z] is LU_NB x LU_NB column-major (rows/cols
// beyond nb zero).  Thread t solves for column t of the inverse by
// substitution in shared memory.
__global__ void __launch_bounds__(LU_NB) tri_inv_kernel(const double* __restrict__ lu, int n,
                                                         long long stride, int blk0, int nblk,
                                                         double* __restrict__ inv) {
  __shared__ double T[LU_NB][LU_NB + 1];
  const int blk = blk0 + blockIdx.x, b = blockIdx.y, upper = blockIdx.z;
  const int j0 = blk * LU_NB, nb = min(LU_NB, n - j0);
  const double* src = lu + b * stride + j0 + (long long)j0 * n;
  const int t = threadIdx.x;
  // the block, padded with the identity beyond nb
  for (int i = 0; i < LU_NB; ++i)
    T[i][t] = (i < nb && t < nb) ? src[i + (long long)t * n] : (i == t ? 1.0 : 0.0);
  __syncthreads();
  // column t of the inverse: x = e_t, column-oriented substitution with the
  // whole column in registers (all indices static after unrolling)
  double x[LU_NB];
#pragma unroll
  for (int i = 0; i < LU_NB; ++i) x[i] = (i == t) ? 1.0 : 0.0;
  if (!upper) {
#pragma unroll
    for (int r = 0; r < LU_NB; ++r)
#pragma unroll
      for (int i = r + 1; i < LU_NB; ++i) x[i] = __fma_rn(-T[i][r], x[r], x[i]);
  } else {
#pragma unroll
    for (int r = LU_NB - 1; r >= 0; --r) {
      x[r] = x[r] / T[r][r];
#pragma unroll
      for (int i = 0; i < r; ++i) x[i] = __fma_rn(-T[i][r], x[r], x[i]);
    }
  }
  double* dst = inv + ((long long)(b * nblk + blk) * 2 + upper) * LU_NB * LU_NB + t * LU_NB;
#pragma unroll
  for (int i = 0; i < LU_NB; ++i) dst[i] = (i < nb && t < nb) ? x[i] : 0.0;
}

// dst_b(0:rows, 0:cols) = src_b(0:rows, 0:cols), column-major blocks
__global__ void copy_block_kernel(const double* __restrict__ src, long long lds, long long ss,
                                  double* __restrict__ dst, long long ldd, long long ds, int rows,
                                  int cols) {
  const long long total = (long long)rows * cols;
  const double* s = src + blockIdx.y * ss;
  double* d = dst + blockIdx.y * ds;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long c = e / rows, r = e - c * rows;
    d[r + c * ldd] = s[r + c * lds];
  }
}

// phi_j = sum_i coeff[i] exps[i] + endpoint * I (phiquad, :179-194): each
// term separately rounded then added, in increasing i.
__global__ void quad_combine_kernel(const double* __restrict__ exps, int nexp, long long nn,
                                    int n, int batch, const double* __restrict__ coeff,
                                    double endpoint, double* __restrict__ out,
                                    long long out_stride) {
  const long long total = nn * batch;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long b = t / nn, e = t - b * nn;
    double m = 0.0;  // skipped terms (theta = 0, j > 1) carry c = 0: m + 0*x == m
    for (int i = 0; i < nexp; ++i)
      m = __dadd_rn(m, __dmul_rn(coeff[i], exps[((long long)i * batch + b) * nn + e]));
    if ((e % (n + 1)) == 0) m = __dadd_rn(m, endpoint);
    out[b * out_stride + e] = m;
  }
}

// One phi_square_step combine for order l (:130-136):
// m = P0*P_l (given); for k=1..l: m += (1/(l-k)!) P_k; m *= 2^-l
__global__ void square_combine_kernel(const double* __restrict__ prod, const double* __restrict__ phis,
                                      long long nn, int batch, int ell_max, int ell,
                                      double* __restrict__ out) {
  const long long total = nn * batch;
  const double sc = ldexp(1.0, -ell);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long b = t / nn, e = t - b * nn;
    const long long base = b * (long long)(ell_max + 1) * nn + e;
    double m = prod[base + (long long)ell * nn];
    if (ell > 0) {
      for (int k = 1; k <= ell; ++k) {
        double f = 1.0;
        for (int i = 2; i <= ell - k; ++i) f *= i;
        m = __dadd_rn(m, __dmul_rn(1.0 / f, phis[base + (long long)k * nn]));
      }
      m = __dmul_rn(m, sc);
    }
    out[base + (long long)ell * nn] = m;
  }
}

__global__ void all_finite_batch_kernel(const double* __restrict__ x, long long total,
                                        int* __restrict__ flag) {
  bool ok = true;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x)
    ok &= isfinite(x[t]);
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) *flag = 0;
}

// ------------------------------------------------------------- host side

// Batched square matmul C_b = A_b B_b (A/B shared when the stride is 0).
void matmul_batch(kp_ctx* ctx, int n, int batch, const double* A, long long sA, const double* B,
                  long long sB, double* C, long long sC, double alpha = 1.0, double beta = 0.0) {
  GemmProblem p;
  p.M = n;
  p.N = n;
  p.K = n;
  p.batch = batch;
  p.A = A;
  p.lda = n;
  p.sA = sA;
  p.B = B;
  p.sBk = 1;
  p.sBn = n;
  p.sB = sB;
  p.C = C;
  p.ldc = n;
  p.sC = sC;
  Epilogue e;
  e.alpha = alpha;
  e.beta = beta;
  launch_gemm(ctx, p, e);
}

template <typename T>
T* slot(kp_ctx* ctx, int s, size_t count) {
  return static_cast<T*>(ctx->ws.get(s, count * sizeof(T)));
}

// Workspace slots used by this file (others: 0..1 Tucker ping-pong,
// 2..7 steppers, 8..12 host staging / complex factor).
enum : int {
  S_NORMS = 20, S_PIV, S_LHS, S_POW, S_U, S_V, S_AU, S_ARG, S_EXPS, S_TAB, S_PROD, S_COEF,
  S_T1, S_T2, S_A2, S_A4, S_A6, S_SING,
  S_TINV = 56, S_X2 = 57, S_U12 = 58
};

std::vector<double> norms1(kp_ctx* ctx, const double* x, int n, int batch) {
  double* d = slot<double>(ctx, S_NORMS, std::max(batch, 1));
  KP_CUDA(cudaMemsetAsync(d, 0, batch * sizeof(double), ctx->stream));
  norm1_kernel<<<dim3((n + 31) / 32, batch), 32, 0, ctx->stream>>>(x, n, (long long)n * n, d);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
  std::vector<double> h(batch);
  KP_CUDA(cudaMemcpyAsync(h.data(), d, batch * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  KP_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

void check_finite(kp_ctx* ctx, const double* x, long long total, const char* who) {
  int* flag = slot<int>(ctx, S_SING, 4);
  const int one = 1;
  KP_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  all_finite_batch_kernel<<<grid1(ctx, total), 256, 0, ctx->stream>>>(x, total, flag);
  ctx->launches++;
  int h = 1;
  KP_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  KP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (!h) throw invalid_argument(std::string(who) + ": non-finite entries");
}

// Launch the cluster panel kernel when the panel rows fit a cluster
// (<= 16 CTAs of 256 rows); false -> caller uses the one-CTA kernel.  KP_LU_PANEL=simple forces the one-CTA kernel (read per call).
bool lu_panel_cluster(kp_ctx* ctx, double* a, int n, long long nn, int j0, int nb, int batch,
                      int* piv, int* sing) {
  constexpr int kMaxRows = LUC_ROWS;
  static int max_cluster = 0;  // 0 = not probed yet, -1 = unavailable
  const char* env = std::getenv("KP_LU_PANEL");
  if (env && std::string(env) == "simple") return false;
  if (max_cluster == 0) {  // probe once: 16-CTA clusters are opt-in (non-portable)
    max_cluster = 8;
    if (cudaFuncSetAttribute(lu_panel_cluster_kernel,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16, 1);
      cfg.blockDim = dim3(LUC_THREADS);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, lu_panel_cluster_kernel, &cfg) ==
              cudaSuccess &&
          nclusters > 0)
        max_cluster = 16;
    }
    (void)cudaGetLastError();
  }
  if (max_cluster < 0) return false;
  const int rows_total = n - j0;
  int ncta = std::max(1, (rows_total + kMaxRows - 1) / kMaxRows);
  if (ncta > max_cluster) return false;
  const int rows_per = (rows_total + ncta - 1) / ncta;
  ncta = (rows_total + rows_per - 1) / rows_per;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncta, batch);
  cfg.blockDim = dim3(LUC_THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KP_CUDA(cudaLaunchKernelEx(&cfg, lu_panel_cluster_kernel, a, n, nn, j0, nb, rows_per, piv,
                             sing));
  return true;
}

// lu_factor + lu_solve(lhs, rhs) for a batch; rhs overwritten with the solution.
// One batched GEMM C_b (+)= alpha * A_b * B_b with A M-contiguous and B
// K-contiguous (all operands column-major sub-blocks with the given lds).
void gemm_kb(kp_ctx* ctx, int M, int N, int K, int batch, const double* A, long long lda,
             long long sA, const double* B, long long ldb, long long sB, double* C, long long ldc,
             long long sC, double alpha, double beta) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  GemmProblem p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.batch = batch;
  p.A = A;
  p.lda = lda;
  p.sA = sA;
  p.B = B;
  p.sBk = 1;
  p.sBn = ldb;
  p.sB = sB;
  p.C = C;
  p.ldc = ldc;
  p.sC = sC;
  Epilogue e;
  e.alpha = alpha;
  e.beta = beta;
  launch_gemm(ctx, p, e);
}

// lu_factor + lu_solve(lhs, rhs) for a batch; rhs overwritten with the solution.
// Factorization as the reference's (inc/linsolve.hpp:95-117: 64-wide panels
// with partial pivoting, GEMM trailing updates); the triangular solves --
// U12 = L11^{-1} A12 of each panel and the forward/backward substitutions of
// lu_solve (:119-146) -- multiply by the inverted nb x nb diagonal blocks on
// the DMMA GEMM, and the substitutions are left-looking (one long-K GEMM per
// block row instead of a K = 64 update of every remaining row).  Same
// algorithm to rounding (~1e-16 per operation); tolerance-tested.
// lu_factor phase: lhs factored in place, pivots in piv (n per matrix), the
// inverted diagonal blocks in the S_TINV slot for the solve phase.
void lu_factor_phase(kp_ctx* ctx, int n, int batch, double* lhs, int* piv) {
  const long long nn = (long long)n * n;
  const int nblk = (n + LU_NB - 1) / LU_NB;
  const long long bsz = (long long)LU_NB * LU_NB;
  int* sing = slot<int>(ctx, S_SING, 4);
  double* tinv = slot<double>(ctx, S_TINV, size_t(batch) * nblk * 2 * bsz);
  const long long tstride = (long long)nblk * 2 * bsz;  // per matrix
  KP_CUDA(cudaMemsetAsync(sing, 0, sizeof(int), ctx->stream));
  const int nt = 256;
  for (int j0 = 0; j0 < n; j0 += LU_NB) {  // lu_factor (:95-117)
    const int nb = std::min(LU_NB, n - j0);
    if (!lu_panel_cluster(ctx, lhs, n, nn, j0, nb, batch, piv, sing))
      lu_panel_kernel<<<batch, 512, 0, ctx->stream>>>(lhs, n, nn, j0, nb, piv, sing);
    ctx->launches++;
    if (j0 > 0) {
      swaps_kernel<<<dim3((j0 + nt - 1) / nt, batch), nt, 0, ctx->stream>>>(lhs, n, nn, piv, n, j0,
                                                                          nb, 0, j0);
      ctx->launches++;
    }
    // L11^{-1} and U11^{-1} of this (final) diagonal block
    tri_inv_kernel<<<dim3(1, batch, 2), LU_NB, 0, ctx->stream>>>(lhs, n, nn, j0 / LU_NB, nblk,
                                                                  tinv);
    ctx->launches++;
    const int rest = n - j0 - nb;
    if (rest > 0) {
      swaps_kernel<<<dim3((rest + nt - 1) / nt, batch), nt, 0, ctx->stream>>>(
          lhs, n, nn, piv, n, j0, nb, j0 + nb, n);
      ctx->launches++;
      // U12 = L11^{-1} A12 (GEMM into scratch, copied back)
      double* u12 = slot<double>(ctx, S_U12, size_t(batch) * LU_NB * rest);
      const double* linv = tinv + (long long)(j0 / LU_NB) * 2 * bsz;
      double* a12 = lhs + j0 + (long long)(j0 + nb) * n;
      gemm_kb(ctx, nb, rest, nb, batch, linv, LU_NB, tstride, a12, n, nn, u12, LU_NB,
              (long long)LU_NB * rest, 1.0, 0.0);
      const long long tot = (long long)nb * rest;
      copy_block_kernel<<<dim3(unsigned(std::min<long long>((tot + 255) / 256, 4096)), batch), 256,
                          0, ctx->stream>>>(u12, LU_NB, (long long)LU_NB * rest, a12, n, nn, nb,
                                            rest);
      ctx->launches++;
      // A22 -= L21 * U12
      gemm_kb(ctx, rest, rest, nb, batch, lhs + (j0 + nb) + (long long)j0 * n, n, nn, a12, n, nn,
              lhs + (j0 + nb) + (long long)(j0 + nb) * n, n, nn, -1.0, 1.0);
    }
    KP_CUDA(cudaGetLastError());
  }
  int hs = 0;
  KP_CUDA(cudaMemcpyAsync(&hs, sing, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  KP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hs) throw runtime_error("lu_factor: matrix is singular");
}

// lu_solve phase on factors from lu_factor_phase (tinv: the S_TINV slot it
// left, or recomputed by the caller); rhs_b: n x nrhs, column-major.
void lu_solve_phase(kp_ctx* ctx, int n, int batch, const double* lhs, const int* piv,
                    const double* tinv, double* rhs, int nrhs) {
  const long long rs = (long long)n * nrhs;
  const long long nn = (long long)n * n;
  const int nblk = (n + LU_NB - 1) / LU_NB;
  const long long bsz = (long long)LU_NB * LU_NB;
  const long long tstride = (long long)nblk * 2 * bsz;
  const int nt = 256;
  // lu_solve (:119-146): P b, then L y = b (rhs -> x2), then U x = y (x2 -> rhs)
  swaps_kernel<<<dim3((nrhs + nt - 1) / nt, batch), nt, 0, ctx->stream>>>(rhs, n, rs, piv, n, 0,
                                                                          n, 0, nrhs);
  ctx->launches++;
  double* x2 = slot<double>(ctx, S_X2, size_t(batch) * rs);
  for (int i = 0; i < nblk; ++i) {
    const int j0 = i * LU_NB, nb = std::min(LU_NB, n - j0);
    // b_i -= L(i, 0:i) y(0:i)
    gemm_kb(ctx, nb, nrhs, j0, batch, lhs + j0, n, nn, x2, n, rs, rhs + j0, n, rs, -1.0, 1.0);
    // y_i = L_ii^{-1} b_i
    gemm_kb(ctx, nb, nrhs, nb, batch, tinv + (long long)i * 2 * bsz, LU_NB, tstride, rhs + j0, n,
            rs, x2 + j0, n, rs, 1.0, 0.0);
  }
  for (int i = nblk - 1; i >= 0; --i) {
    const int j0 = i * LU_NB, nb = std::min(LU_NB, n - j0), j1 = j0 + nb;
    // y_i -= U(i, i+1:) x(i+1:)
    gemm_kb(ctx, nb, nrhs, n - j1, batch, lhs + j0 + (long long)j1 * n, n, nn, rhs + j1, n, rs,
            x2 + j0, n, rs, -1.0, 1.0);
    // x_i = U_ii^{-1} y_i
    gemm_kb(ctx, nb, nrhs, nb, batch, tinv + ((long long)i * 2 + 1) * bsz, LU_NB, tstride,
            x2 + j0, n, rs, rhs + j0, n, rs, 1.0, 0.0);
  }
  KP_CUDA(cudaGetLastError());
}


void lu_solve_batch(kp_ctx* ctx, int n, int batch, double* lhs, double* rhs, int nrhs = -1) {
  if (nrhs < 0) nrhs = n;
  int* piv = slot<int>(ctx, S_PIV, size_t(n) * batch);
  lu_factor_phase(ctx, n, batch, lhs, piv);
  const int nblk = (n + LU_NB - 1) / LU_NB;
  const double* tinv = slot<double>(ctx, S_TINV, size_t(batch) * nblk * 2 * LU_NB * LU_NB);
  lu_solve_phase(ctx, n, batch, lhs, piv, tinv, rhs, nrhs);
}

// pade_low for a batch of matrices sharing one degree (inc/matrix_functions.hpp:37-54):
// the linear system (v - u) r = v + u, solved by the caller (one LU for all
// degrees of an expm batch).
void pade_low_batch(kp_ctx* ctx, const double* a, int n, int batch, int idx, double* lhs_out,
                    double* rhs_out) {
  const auto& b = pade_coeffs()[idx];
  const int npow = (int(b.size()) - 2) / 2;
  const long long nn = (long long)n * n, tot = nn * batch;
  double* pw = slot<double>(ctx, S_POW, size_t(tot) * npow);
  matmul_batch(ctx, n, batch, a, nn, a, nn, pw, nn);  // A^2
  for (int p = 1; p < npow; ++p)
    matmul_batch(ctx, n, batch, pw + (p - 1) * tot, nn, pw, nn, pw + p * tot, nn);
  double* u = slot<double>(ctx, S_U, tot);
  double* v = slot<double>(ctx, S_V, tot);
  double* cf = slot<double>(ctx, S_COEF, 256);
  std::vector<double> hc(16, 0.0);
  for (int p = 0; p < npow; ++p) {
    hc[p] = b[2 * p + 3];
    hc[8 + p] = b[2 * p + 2];
  }
  KP_CUDA(cudaMemcpyAsync(cf, hc.data(), 16 * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
  pade_uv_kernel<<<grid1(ctx, tot), 256, 0, ctx->stream>>>(pw, npow, nn, n, batch, b[0], b[1], cf,
                                                           cf + 8, u, v);
  ctx->launches++;
  double* au = slot<double>(ctx, S_AU, tot);
  matmul_batch(ctx, n, batch, a, nn, u, nn, au, nn);  // u = a*u
  pm_kernel<<<grid1(ctx, tot), 256, 0, ctx->stream>>>(au, v, tot, lhs_out, rhs_out);  // v-u | v+u
  ctx->launches++;
}

// pade13 (inc/matrix_functions.hpp:57-72) for a batch: the system as above
void pade13_batch(kp_ctx* ctx, const double* a, int n, int batch, double* lhs_out,
                  double* rhs_out) {
  const auto& b = pade_coeffs()[4];
  const long long nn = (long long)n * n, tot = nn * batch;
  double* a2 = slot<double>(ctx, S_A2, tot);
  double* a4 = slot<double>(ctx, S_A4, tot);
  double* a6 = slot<double>(ctx, S_A6, tot);
  matmul_batch(ctx, n, batch, a, nn, a, nn, a2, nn);
  matmul_batch(ctx, n, batch, a2, nn, a2, nn, a4, nn);
  matmul_batch(ctx, n, batch, a4, nn, a2, nn, a6, nn);
  double* w = slot<double>(ctx, S_T1, tot);
  double* t = slot<double>(ctx, S_T2, tot);
  const unsigned g = grid1(ctx, tot);
  pade13_w_kernel<<<g, 256, 0, ctx->stream>>>(a2, a4, a6, tot, n, nn, b[13], b[11], b[9], w);
  matmul_batch(ctx, n, batch, a6, nn, w, nn, t, nn);
  pade13_add_kernel<<<g, 256, 0, ctx->stream>>>(a2, a4, a6, tot, n, nn, b[7], b[5], b[3], b[1], t);
  double* u = slot<double>(ctx, S_U, tot);
  matmul_batch(ctx, n, batch, a, nn, t, nn, u, nn);
  pade13_w_kernel<<<g, 256, 0, ctx->stream>>>(a2, a4, a6, tot, n, nn, b[12], b[10], b[8], w);
  double* z = slot<double>(ctx, S_V, tot);
  matmul_batch(ctx, n, batch, a6, nn, w, nn, z, nn);
  pade13_add_kernel<<<g, 256, 0, ctx->stream>>>(a2, a4, a6, tot, n, nn, b[6], b[4], b[2], b[0], z);
  pm_kernel<<<g, 256, 0, ctx->stream>>>(u, z, tot, lhs_out, rhs_out);
  ctx->launches += 5;
  KP_CUDA(cudaGetLastError());
}

}  // namespace

// expm of a batch of matrices x_b (inc/matrix_functions.hpp:76-95).  Degree
// and scaling per matrix from its own 1-norm; the Pade systems of all
// matrices are assembled group by group (same degree and scaling) in one
// group-ordered buffer, solved by ONE batched LU, and each group squared.
void expm_batch(kp_ctx* ctx, const double* x, int n, int batch, double* out) {
  const long long nn = (long long)n * n;
  const std::vector<double> nrm = norms1(ctx, x, n, batch);
  std::vector<int> branch(batch), sc(batch, 0);
  for (int b = 0; b < batch; ++b) {
    int br = 4;
    for (int idx = 0; idx < 4; ++idx)
      if (nrm[b] <= kPadeTheta[idx]) {
        br = idx;
        break;
      }
    branch[b] = br;
    if (br == 4) {
      double v = nrm[b];
      while (v > kPadeTheta[4]) {
        v *= 0.5;
        ++sc[b];
      }
    }
  }
  // Order: every degree-13 matrix first, by decreasing scaling exponent,
  // then one group per low degree.  The degree-13 block then runs as ONE
  // batch (each matrix scaled by its own 2^-s, one pade13 pass, and the
  // squarings over the prefix still needing one), so a few large matrices of
  // different scalings share every GEMM launch instead of each filling a
  // fraction of a wave on its own.  Per-matrix arithmetic is unchanged.
  std::vector<int> order;
  for (int b = 0; b < batch; ++b)
    if (branch[b] == 4) order.push_back(b);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sc[a] > sc[b]; });
  const int n13 = int(order.size());
  std::vector<std::pair<int, int>> low;  // (first position, size) per low degree
  for (int br = 0; br < 4; ++br) {
    const int first = int(order.size());
    for (int b = 0; b < batch; ++b)
      if (branch[b] == br) order.push_back(b);
    if (int(order.size()) > first) low.emplace_back(first, int(order.size()) - first);
  }
  double* gin = slot<double>(ctx, S_ARG, size_t(nn) * batch);
  double* lhs = slot<double>(ctx, S_LHS, size_t(nn) * batch);
  double* rhs = slot<double>(ctx, S_TAB, size_t(nn) * batch);
  for (int i = 0; i < batch; ++i)
    KP_CUDA(cudaMemcpyAsync(gin + i * nn, x + order[i] * nn, nn * sizeof(double),
                            cudaMemcpyDeviceToDevice, ctx->stream));
  if (n13 > 0) {
    if (n13 > 256) throw invalid_argument("expm: at most 256 matrices per batch");
    double* scale = slot<double>(ctx, S_COEF, 256);
    std::vector<double> hs(n13);
    for (int i = 0; i < n13; ++i) hs[i] = std::ldexp(1.0, -sc[order[i]]);
    KP_CUDA(cudaMemcpyAsync(scale, hs.data(), n13 * sizeof(double), cudaMemcpyHostToDevice,
                            ctx->stream));
    scale_batch_kernel<<<grid1(ctx, nn * n13), 256, 0, ctx->stream>>>(gin, nn, scale, nn, n13,
                                                                       gin);
    ctx->launches++;
    pade13_batch(ctx, gin, n, n13, lhs, rhs);
    KP_CUDA(cudaStreamSynchronize(ctx->stream));  // S_COEF is reused by pade_low_batch
  }
  for (const auto& gr : low)
    pade_low_batch(ctx, gin + gr.first * nn, n, gr.second, branch[order[gr.first]],
                   lhs + gr.first * nn, rhs + gr.first * nn);
  lu_solve_batch(ctx, n, batch, lhs, rhs);
  // squarings: matrix i of the degree-13 block needs sc[order[i]] of them;
  // sorted by decreasing s, the ones still needing a squaring are a prefix
  const int smax = n13 > 0 ? sc[order[0]] : 0;
  for (int it = 0; it < smax; ++it) {
    int g = 0;
    while (g < n13 && sc[order[g]] > it) ++g;
    double* tmp = slot<double>(ctx, S_T1, size_t(nn) * g);
    matmul_batch(ctx, n, g, rhs, nn, rhs, nn, tmp, nn);  // f = f*f
    KP_CUDA(cudaMemcpyAsync(rhs, tmp, nn * g * sizeof(double), cudaMemcpyDeviceToDevice,
                            ctx->stream));
  }
  for (int i = 0; i < batch; ++i)
    KP_CUDA(cudaMemcpyAsync(out + order[i] * nn, rhs + i * nn, nn * sizeof(double),
                            cudaMemcpyDeviceToDevice, ctx->stream));
}

// lu_factor (inc/linsolve.hpp:95-117) of one n x n matrix in place; piv: n
// device ints (the row swapped into position j at step j).
void lu_factor_dev(kp_ctx* ctx, double* a, int n, int* piv) { lu_factor_phase(ctx, n, 1, a, piv); }

// lu_solve (inc/linsolve.hpp:119-146) with factors from lu_factor_dev: b
// (n x nrhs) overwritten with the solution.
void lu_solve_dev(kp_ctx* ctx, const double* lu, const int* piv, int n, double* b, int nrhs) {
  const int nblk = (n + LU_NB - 1) / LU_NB;
  const long long bsz = (long long)LU_NB * LU_NB;
  double* tinv = slot<double>(ctx, S_TINV, size_t(nblk) * 2 * bsz);
  tri_inv_kernel<<<dim3(nblk, 1, 2), LU_NB, 0, ctx->stream>>>(lu, n, (long long)n * n, 0, nblk,
                                                              tinv);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
  lu_solve_phase(ctx, n, 1, lu, piv, tinv, b, nrhs);
}

void solve_dev(kp_ctx* ctx, const double* a, int n, const double* b, int nrhs, double* x) {
  const long long nn = (long long)n * n;
  double* lu = slot<double>(ctx, S_LHS, size_t(nn));
  KP_CUDA(cudaMemcpyAsync(lu, a, nn * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  if (x != b)
    KP_CUDA(cudaMemcpyAsync(x, b, (long long)n * nrhs * sizeof(double), cudaMemcpyDeviceToDevice,
                            ctx->stream));
  lu_solve_batch(ctx, n, 1, lu, x, nrhs);
}

// phiquad (inc/matrix_functions.hpp:146-199) for one matrix x (device):
// writes phis[0..ell_max] (each n x n, consecutive) and returns s.
int phiquad_dev(kp_ctx* ctx, const double* x, int n, int ell_max, int q, int forced,
                double* phis) {
  if (ell_max < 0) throw invalid_argument("phiquad: negative ell_max");
  const long long nn = (long long)n * n;
  check_finite(ctx, x, nn, "phiquad");
  const double d = norms1(ctx, x, n, 1)[0];
  int s = 0;
  for (double v = d; v >= 1.0; v *= 0.5) ++s;
  if (forced >= 0) {
    if (forced < s) throw invalid_argument("phiquad: forced scaling below minimum");
    s = forced;
  }
  std::vector<double> nodes(q), weights(q);
  gll_rule_host(q, nodes.data(), weights.data());
  // args_i = (x * 2^-s) * (1 - theta_i), i < q-1 (two roundings, as :162-174)
  double* y = slot<double>(ctx, S_T2, nn);
  double* sc = slot<double>(ctx, S_COEF, 256);
  std::vector<double> hs(q + 1);
  hs[0] = std::ldexp(1.0, -s);
  for (int i = 0; i < q - 1; ++i) hs[1 + i] = 1.0 - nodes[i];
  KP_CUDA(cudaMemcpyAsync(sc, hs.data(), (q + 1) * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
  scale_batch_kernel<<<grid1(ctx, nn), 256, 0, ctx->stream>>>(x, 0, sc, nn, 1, y);
  double* args = slot<double>(ctx, S_EXPS, size_t(nn) * (q - 1) * 2);
  double* exps = args + nn * (q - 1);
  scale_batch_kernel<<<grid1(ctx, nn * (q - 1)), 256, 0, ctx->stream>>>(y, 0, sc + 1, nn, q - 1,
                                                                       args);
  ctx->launches += 2;
  expm_batch(ctx, args, n, q - 1, exps);
  // phi_0 = exps[0]; phi_j = sum_i w_i theta_i^{j-1}/(j-1)! exps[i] + w_{q-1}/(j-1)! I
  KP_CUDA(cudaMemcpyAsync(phis, exps, nn * sizeof(double), cudaMemcpyDeviceToDevice,
                          ctx->stream));
  for (int j = 1; j <= ell_max; ++j) {
    const double jm1 = factorial(j - 1);
    std::vector<double> c(q, 0.0);
    for (int i = 0; i < q - 1; ++i) {
      const double th = nodes[i];
      if (j > 1 && th == 0.0) {
        c[i] = 0.0;  // skipped term: adding +0.0 leaves m unchanged
        continue;
      }
      c[i] = weights[i] * std::pow(th, double(j - 1)) / jm1;
    }
    double* cd = slot<double>(ctx, S_COEF, 256);
    KP_CUDA(cudaMemcpyAsync(cd, c.data(), q * sizeof(double), cudaMemcpyHostToDevice,
                            ctx->stream));
    quad_combine_kernel<<<grid1(ctx, nn), 256, 0, ctx->stream>>>(
        exps, q - 1, nn, n, 1, cd, weights[q - 1] / jm1, phis + j * nn, nn);
    ctx->launches++;
    KP_CUDA(cudaStreamSynchronize(ctx->stream));  // cd is reused by the next order
  }
  // s doubling steps (phi_square_step)
  double* prod = slot<double>(ctx, S_PROD, size_t(nn) * (ell_max + 1));
  double* nxt = slot<double>(ctx, S_TAB, size_t(nn) * (ell_max + 1));
  for (int step = 0; step < s; ++step) {
    matmul_batch(ctx, n, ell_max + 1, phis, 0, phis, nn, prod, nn);  // P0 * P_l
    for (int l = 0; l <= ell_max; ++l) {
      square_combine_kernel<<<grid1(ctx, nn), 256, 0, ctx->stream>>>(prod, phis, nn, 1, ell_max, l,
                                                                     nxt);
      ctx->launches++;
    }
    KP_CUDA(cudaMemcpyAsync(phis, nxt, nn * (ell_max + 1) * sizeof(double),
                            cudaMemcpyDeviceToDevice, ctx->stream));
  }
  KP_CUDA(cudaGetLastError());
  return s;
}

namespace {
// R(X) = [[Xr, -Xi], [Xi, Xr]] (2n x 2n real) for complex X (n x n interleaved)
__global__ void embed_kernel(const double2* __restrict__ x, int n, double* __restrict__ r) {
  const long long nn = (long long)n * n, ld = 2LL * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = int(t % n), j = int(t / n);
    const double2 v = x[t];
    r[i + j * ld] = v.x;
    r[(i + n) + j * ld] = v.y;
    r[i + (j + n) * ld] = -v.y;
    r[(i + n) + (j + n) * ld] = v.x;
  }
}
// X = R[0:n, 0:n] + i R[n:2n, 0:n]
__global__ void extract_kernel(const double* __restrict__ r, int n, double2* __restrict__ x) {
  const long long nn = (long long)n * n, ld = 2LL * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = int(t % n), j = int(t / n);
    x[t] = make_double2(r[i + j * ld], r[(i + n) + j * ld]);
  }
}
constexpr int S_EMB = 45, S_EMB2 = 46;
}  // namespace

// Complex matrix functions through the real representation R(X): R is an
// algebra homomorphism, so R(exp X) = exp R(X) and likewise for phi_l and
// the Pade/LU steps.  For the purely imaginary NLS factors (i/2)Delta the
// 1-norms, hence the scaling exponent and Pade degrees, equal the reference's
// complex ones; agreement with the reference's complex arithmetic is at
// roundoff level (tests/test_phi_gpu.py).
void expm_batch_c128(kp_ctx* ctx, const double* x, int n, int batch, double* out) {
  const long long nn = (long long)n * n, rr = 4 * nn;
  double* r = static_cast<double*>(ctx->ws.get(S_EMB, size_t(rr) * batch * sizeof(double)));
  double* e = static_cast<double*>(ctx->ws.get(S_EMB2, size_t(rr) * batch * sizeof(double)));
  for (int b = 0; b < batch; ++b) {
    embed_kernel<<<grid1(ctx, nn), 256, 0, ctx->stream>>>(
        reinterpret_cast<const double2*>(x) + b * nn, n, r + b * rr);
    ctx->launches++;
  }
  expm_batch(ctx, r, 2 * n, batch, e);
  for (int b = 0; b < batch; ++b) {
    extract_kernel<<<grid1(ctx, nn), 256, 0, ctx->stream>>>(e + b * rr, n,
                                                            reinterpret_cast<double2*>(out) + b * nn);
    ctx->launches++;
  }
  KP_CUDA(cudaGetLastError());
}

int phiquad_dev_c128(kp_ctx* ctx, const double* x, int n, int ell_max, int q, int forced,
                     double* phis) {
  const long long nn = (long long)n * n, rr = 4 * nn;
  double* r = static_cast<double*>(ctx->ws.get(S_EMB, size_t(rr) * sizeof(double)));
  double* tab = static_cast<double*>(ctx->ws.get(S_EMB2, size_t(rr) * (ell_max + 1) * sizeof(double)));
  embed_kernel<<<grid1(ctx, nn), 256, 0, ctx->stream>>>(reinterpret_cast<const double2*>(x), n, r);
  ctx->launches++;
  const int s = phiquad_dev(ctx, r, 2 * n, ell_max, q, forced, tab);
  for (int j = 0; j <= ell_max; ++j) {
    extract_kernel<<<grid1(ctx, nn), 256, 0, ctx->stream>>>(tab + j * rr, n,
                                                            reinterpret_cast<double2*>(phis) + j * nn);
    ctx->launches++;
  }
  KP_CUDA(cudaGetLastError());
  return s;
}

}  // namespace kp
