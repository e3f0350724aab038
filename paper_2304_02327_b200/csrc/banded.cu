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
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "kp_g.cuh"
#include "kp_internal.h"

namespace kp {
namespace {

constexpr int KC = 256;  // inc/kernels.hpp:104

// rows of A (n x n, column-major; complex when comps == 2) -> 3 slots per row
__global__ void band_scan_kernel(const double* __restrict__ a, int n, int comps,
                                 int* __restrict__ cols, double* __restrict__ vals,
                                 int* __restrict__ too_many) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int cnt = 0;
  for (int j = 0; j < n; ++j) {
    const double re = a[(size_t(i) + size_t(j) * n) * comps];
    const double im = comps == 2 ? a[(size_t(i) + size_t(j) * n) * comps + 1] : 0.0;
    if (re != 0.0 || im != 0.0) {
      if (cnt == 3) {
        *too_many = 1;
        return;
      }
      cols[i * 3 + cnt] = j;
      vals[(i * 3 + cnt) * 2] = re;
      vals[(i * 3 + cnt) * 2 + 1] = im;
      ++cnt;
    }
  }
  for (; cnt < 3; ++cnt) cols[i * 3 + cnt] = -1;
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

}  // namespace

// forward (defined below)
void kronsum_banded(kp_ctx* ctx, bool cplx, const double* u, const std::vector<int>& dims,
                    const std::vector<const int*>& cols, const std::vector<const double*>& vals,
                    const std::vector<char>& active, double* r, bool with_g, const kp_gfun& g,
                    long long half, int slab, int k0, int n_glob, int halo, double t);

// Scan a factor into caller-provided device arrays (3n ints, 6n doubles);
// false if some row has more than three nonzeros.
bool band_scan(kp_ctx* ctx, const double* a, int n, bool cplx, int* dc, double* dv) {
  int* flag = reinterpret_cast<int*>(ctx->d_flag) + 8;
  KP_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  band_scan_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(a, n, cplx ? 2 : 1, dc, dv, flag);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
  KP_CUDA(cudaMemcpyAsync(ctx->h_flag + 8, flag, sizeof(int), cudaMemcpyDeviceToHost,
                          ctx->stream));
  KP_CUDA(cudaStreamSynchronize(ctx->stream));
  return ctx->h_flag[8] == 0;
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
    if (!band_scan(ctx, as[mu], dims[mu], cplx, c, v)) return false;
    cols[mu] = c;
    vals[mu] = v;
  }
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
  const unsigned grid =
      unsigned(std::max<long long>(1, std::min<long long>((total + 255) / 256, ctx->num_sms * 16LL)));
  if (cplx)
    kronsum_band_kernel<true><<<grid, 256, 0, ctx->stream>>>(b, total, u, r, with_g, g, t);
  else
    kronsum_band_kernel<false><<<grid, 256, 0, ctx->stream>>>(b, total, u, r, with_g, g, t);
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
      if (!band_scan(ctx, as[mu], n, cplx, c, v))
        throw invalid_argument("kronsum_slab: factor " + std::to_string(mu) +
                               " has more than three nonzeros in a row");
      cols[mu] = c;
      vals[mu] = v;
      // an all-zero factor (the stacked species mode) contributes nothing
      if (n <= 2) {
        std::vector<int> hc(3 * size_t(n));
        KP_CUDA(cudaMemcpy(hc.data(), c, hc.size() * sizeof(int), cudaMemcpyDeviceToHost));
        bool any = false;
        for (int x : hc) any |= (x >= 0);
        active[mu] = any;
      }
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
