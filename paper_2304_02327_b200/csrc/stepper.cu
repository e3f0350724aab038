// stepper.cu -- exponential integrators on device-resident state.
//
// Replaces the reference's time loop (inc/integrators.hpp):
//   lawson_euler_step :116-122   lawson2b_step :124-132   exp_euler_step :134-141
//   exp_euler_linear_split_step :143-151   etd2rk_step :153-164
//   integrate :219-373 (Split backend: factors built once, per-step finite check)
// Every elementwise update of a step is fused into the epilogue of the GEMM
// that produces its input, so a step streams the state through HBM once per
// mode product (3 d launches for ETD2RK, 2 d for exponential Euler):
//   r     = K u + g(t,u)                     kronsum, last term EPI_ADD_G
//   stage = u + tau*SP1(r); D = g(stage)-g(u)  Tucker(phi1), last mode EPI_STAGE_D
//   u'    = stage + tau*SP2(D)               Tucker(phi2), last mode EPI_FMA_X
// (a coupled g -- the Brusselator's two species -- cannot form D inside one
// tile, so it gets one elementwise pass instead).  The rounding of every fused
// update equals the reference's (axpy/add_scaled contract to FMAs there).
//
// Modes whose phi factor is exactly a scalar multiple of I (the zero species
// mode of the stacked Brusselator, phi_l(0) = c I) are folded into the alpha
// of the last real mode -- the same single rounding as the reference's extra
// mode product -- and zero Kronecker-sum terms are skipped (they add +0).
//
// The loop runs as a CUDA graph of two steps (ping-pong buffers), replayed;
// divergence is detected on the device (epilogue atomicMin of the step
// counter) and reported with the reference's message and step index.
#include <climits>
#include <map>
#include <memory>
#include <tuple>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kp_g.cuh"
#include "kp_internal.h"
#include "kp_launch.cuh"

namespace kp {

namespace {

using ModeFn = void (*)(kp_ctx*, const double*, const std::vector<int>&, int, const double*, int,
                        const Epilogue&, double*);

unsigned grid_ew(kp_ctx* ctx, long long n) {
  return unsigned(std::max<long long>(1, std::min<long long>((n + 255) / 256, ctx->num_sms * 8LL)));
}

template <bool CPLX>
struct Elt;
template <>
struct Elt<false> {
  using T = double;
  static __device__ __forceinline__ T g(const kp_gfun& gf, const T* u, long long i, long long half,
                                        double t) {
    const bool second = half > 0 && i >= half;
    const double partner = half > 0 ? u[second ? i - half : i + half] : 0.0;
    return g_real(gf, u[i], partner, second, i, t);
  }
  static __device__ __forceinline__ T fma(double a, T x, T y) { return __fma_rn(a, x, y); }
  static __device__ __forceinline__ T sub(T a, T b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ bool finite(T x) { return isfinite(x); }
};
template <>
struct Elt<true> {
  using T = double2;
  static __device__ __forceinline__ T g(const kp_gfun& gf, const T* u, long long i, long long,
                                        double) {
    return g_cplx(gf, u[i]);
  }
  static __device__ __forceinline__ T fma(double a, T x, T y) {
    return make_double2(__fma_rn(a, x.x, y.x), __fma_rn(a, x.y, y.y));
  }
  static __device__ __forceinline__ T sub(T a, T b) {
    return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
  }
  static __device__ __forceinline__ bool finite(T x) { return isfinite(x.x) && isfinite(x.y); }
};

// w0 = u + tau*g(u); if two: w1 = u + (tau/2)*g(u)   (Lawson prologues, :118, :127-129)
template <bool CPLX>
__global__ void lawson_pre_kernel(kp_gfun g, double t, long long n, long long half, double tau,
                                  bool two,
                                  const typename Elt<CPLX>::T* __restrict__ u,
                                  typename Elt<CPLX>::T* __restrict__ w) {
  pdl_wait();
  using E = Elt<CPLX>;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const auto gn = E::g(g, u, i, half, t);
    w[i] = E::fma(tau, gn, u[i]);
    if (two) w[n + i] = E::fma(0.5 * tau, gn, u[i]);
  }
}

// out = y1 + (tau/2) g(stage), y = [stage; y1]   (lawson2b :130-131)
template <bool CPLX>
__global__ void lawson2b_post_kernel(kp_gfun g, double t2, long long n, long long half, double tau,
                                     const typename Elt<CPLX>::T* __restrict__ y,
                                     typename Elt<CPLX>::T* __restrict__ out, int* bad,
                                     const int* ctr, int* next) {
  pdl_wait();
  using E = Elt<CPLX>;
  bool nf = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const auto r = E::fma(0.5 * tau, E::g(g, y, i, half, t2), y[n + i]);
    out[i] = r;
    nf |= !E::finite(r);
  }
  if (nf) atomicMin(bad, *ctr + 1);
  if (next && blockIdx.x == 0 && threadIdx.x == 0) *next = *ctr + 1;
}

// d = g(stage) - g(u)   (etd2rk :161-162, unfused form for coupled g)
template <bool CPLX>
__global__ void gdiff_kernel(kp_gfun g, double t, double t2, long long n, long long half,
                             const typename Elt<CPLX>::T* __restrict__ s,
                             const typename Elt<CPLX>::T* __restrict__ u,
                             typename Elt<CPLX>::T* __restrict__ d) {
  pdl_wait();
  using E = Elt<CPLX>;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = E::sub(E::g(g, s, i, half, t2), E::g(g, u, i, half, t));
}

// Two-species (Brusselator) forms of the three kernels above: one thread
// owns both species of a grid point (i, i + half), so each value is read
// once (the unpaired kernels re-read the partner from HBM).  Same
// arithmetic per entry.
__global__ void lawson_pre_pair_kernel(kp_gfun g, double t, long long half, double tau, bool two,
                                       const double* __restrict__ u, double* __restrict__ w) {
  pdl_wait();
  const long long n = 2 * half;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < half;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = u[i], b = u[i + half];
    const double ga = g_real(g, a, b, false, i, t), gb = g_real(g, b, a, true, i + half, t);
    w[i] = __fma_rn(tau, ga, a);
    w[i + half] = __fma_rn(tau, gb, b);
    if (two) {
      w[n + i] = __fma_rn(0.5 * tau, ga, a);
      w[n + i + half] = __fma_rn(0.5 * tau, gb, b);
    }
  }
}

__global__ void lawson2b_post_pair_kernel(kp_gfun g, double t2, long long half, double tau,
                                          const double* __restrict__ y, double* __restrict__ out,
                                          int* bad, const int* ctr, int* next) {
  pdl_wait();
  const long long n = 2 * half;
  bool nf = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < half;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = y[i], b = y[i + half];
    const double ra = __fma_rn(0.5 * tau, g_real(g, a, b, false, i, t2), y[n + i]);
    const double rb = __fma_rn(0.5 * tau, g_real(g, b, a, true, i + half, t2), y[n + i + half]);
    out[i] = ra;
    out[i + half] = rb;
    nf |= !isfinite(ra) || !isfinite(rb);
  }
  if (nf) atomicMin(bad, *ctr + 1);
  if (next && blockIdx.x == 0 && threadIdx.x == 0) *next = *ctr + 1;
}

__global__ void gdiff_pair_kernel(kp_gfun g, double t, double t2, long long half,
                                  const double* __restrict__ s, const double* __restrict__ u,
                                  double* __restrict__ d) {
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < half;
       i += (long long)gridDim.x * blockDim.x) {
    const double sa = s[i], sb = s[i + half], ua = u[i], ub = u[i + half];
    d[i] = __dsub_rn(g_real(g, sa, sb, false, i, t2), g_real(g, ua, ub, false, i, t));
    d[i + half] = __dsub_rn(g_real(g, sb, sa, true, i + half, t2), g_real(g, ub, ua, true, i + half, t));
  }
}

__global__ void tick_kernel(const int* ctr, int* next) {
  pdl_wait();
  *next = *ctr + 1;
}

__global__ void scale_matrix_kernel(const double* __restrict__ a, long long n, double s,
                                    double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = __dmul_rn(a[i], s);
}

// Workspace slots of the stepper (tucker ping-pong uses 0/1 inside).
enum : int {
  S_R = 2, S_S = 3, S_D = 4, S_W = 5, S_Y = 6, S_U2 = 7, S_CTR = 40,
  S_G = 49, S_WZ = 50, S_J1 = 51, S_J2 = 52, S_J3 = 53, S_PHI1 = 54, S_PHI2 = 55
};

}  // namespace

// d = g(t + tau, s) - g(t, u) over n entries (the ETD2RK difference as its own
// pass, for g's the GEMM epilogue cannot evaluate: the coupled Brusselator).
void gdiff_dev(kp_ctx* ctx, const kp_gfun& g, double t, double tau, const double* s,
               const double* u, long long n, long long half, bool cplx, double* dd) {
  if (n <= 0) return;
  if (!cplx && half > 0) {
    launch_pdl(ctx, gdiff_pair_kernel, dim3(grid_ew(ctx, half)), dim3(256), 0, g, t, t + tau,
               half, s, u, dd);
  } else if (cplx) {
    launch_pdl(ctx, gdiff_kernel<true>, dim3(grid_ew(ctx, n)), dim3(256), 0, g, t, t + tau, n,
               half, reinterpret_cast<const double2*>(s), reinterpret_cast<const double2*>(u),
               reinterpret_cast<double2*>(dd));
  } else {
    launch_pdl(ctx, gdiff_kernel<false>, dim3(grid_ew(ctx, n)), dim3(256), 0, g, t, t + tau, n,
               half, s, u, dd);
  }
  KP_CUDA(cudaGetLastError());
}

// Per-mode factor list with the scalar-identity folding described above.
struct FactorSet {
  std::vector<const double*> f;
  std::vector<char> active;
  double fold = 1.0;
  double pref = 1.0;
};

class Integrator {
 public:
  kp_ctx* ctx;
  int method;
  bool cplx;
  std::vector<int> dims;
  int d;
  kp_gfun g;
  double tau;
  long long n_entries;  // entries of u (complex counts once)
  long long half = 0;   // Brusselator species offset
  ModeFn mp;
  int comps;
  std::vector<const double*> A;
  std::vector<char> a_active;
  FactorSet f1, f2, fj;  // fj: Rosenbrock's per-step factors
  int q_nodes = 12;
  bool given_jacobians = false;  // kp_step: J factors supplied by the caller
  std::vector<double*> owned;
  long diverged_at = 0;  // first non-finite step of the last run() (0 = none)
  bool nonlocal = false;  // g needs more than the entry itself (Riccati): own buffers
  // banded Kronecker sum (banded.cu): per-mode 3-slot row structure
  bool banded = false;
  std::vector<const int*> band_cols;
  std::vector<const double*> band_vals;

  Integrator(kp_ctx* c, int m, bool cp, const std::vector<int>& dv, const double* const* as,
             const kp_gfun& gf, double tau_)
      : ctx(c), method(m), cplx(cp), dims(dv), d(int(dv.size())), g(gf), tau(tau_) {
    n_entries = 1;
    for (int x : dims) n_entries *= x;
    mp = cplx ? mode_product_c128 : mode_product_f64;
    comps = cplx ? 2 : 1;
    A.assign(as, as + d);
    if (g.kind == KP_G_BRUSSELATOR) {
      if (cplx || dims.back() != 2)
        throw invalid_argument("brusselator g: slowest mode must hold 2 species");
      half = n_entries / 2;
    }
    if (g.kind == KP_G_NLS && !cplx) throw invalid_argument("g: NLS needs a complex tensor");
    nonlocal = (g.kind == KP_G_RICCATI);
    if (nonlocal && (cplx || d != 2 || dims[0] != dims[1] || !g.aux[0] || !g.aux[1]))
      throw invalid_argument("riccati g: needs a real n x n state and aux = {b, C}");

    if (cplx && (g.kind == KP_G_ALLEN_CAHN || g.kind == KP_G_BRUSSELATOR))
      throw invalid_argument("g: unsupported nonlinearity kind for complex");
    a_active.assign(d, 1);
    int nact = 0;
    for (int mu = 0; mu < d; ++mu) {
      a_active[mu] = !is_zero(A[mu], dims[mu]);
      nact += a_active[mu];
    }
    if (nact == 0) a_active[d - 1] = 1;
    if (banded_kronsum_enabled() && !nonlocal && d <= 4 &&
        (method == KP_EXP_EULER || method == KP_ETD2RK || method == KP_ROSENBROCK_EULER)) {
      banded = true;
      band_cols.assign(d, nullptr);
      band_vals.assign(d, nullptr);
      for (int mu = 0; mu < d && banded; ++mu) {
        if (!a_active[mu]) continue;
        int same = -1;
        for (int m2 = 0; m2 < mu; ++m2)
          if (a_active[m2] && A[m2] == A[mu] && dims[m2] == dims[mu]) same = m2;
        if (same >= 0) {
          band_cols[mu] = band_cols[same];
          band_vals[mu] = band_vals[same];
          continue;
        }
        int* c = nullptr;
        double* v = nullptr;
        if (band_of(ctx, A[mu], dims[mu], cplx, &c, &v)) {
          band_cols[mu] = c;
          band_vals[mu] = v;
          owned_i.push_back(c);
          owned.push_back(v);
        } else {
          banded = false;
        }
      }
    }
  }
  std::vector<int*> owned_i;
  ~Integrator() {
    for (double* p : owned) cudaFree(p);
    for (int* p : owned_i) cudaFree(p);
  }

  // exact zero matrix? (only small factors are checked; big ones never are)
  bool is_zero(const double* m, int n) {
    if (n > 64) return false;
    std::vector<double> h(size_t(n) * n * comps);
    KP_CUDA(cudaMemcpyAsync(h.data(), m, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
    for (double x : h)
      if (x != 0.0) return false;
    return true;
  }
  // exactly c*I (real c)?  (small factors only)
  bool scalar_identity(const double* m, int n, double* c) {
    if (n > 64) return false;
    std::vector<double> h(size_t(n) * n * comps);
    KP_CUDA(cudaMemcpyAsync(h.data(), m, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
    const double c0 = h[0];
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < comps; ++k) {
          const double v = h[(size_t(i) + size_t(j) * n) * comps + k];
          const double want = (i == j && k == 0) ? c0 : 0.0;
          if (v != want) return false;
        }
    *c = c0;
    return true;
  }

  double* alloc(size_t doubles) {
    double* p = nullptr;
    KP_CUDA(cudaMalloc(&p, std::max<size_t>(doubles, 2) * sizeof(double)));
    owned.push_back(p);
    return p;
  }

  // build_split_phi (inc/split_phi.hpp:25-43) for orders ell_lo..ell_hi from
  // ONE table per distinct factor (phi_j depends only on phi_{<=j}, so the
  // table of ell_max = 2 gives bit-identical phi_1 to the reference's separate
  // ell = 1 build, inc/integrators.hpp:277-278).  ell = 0 uses expm.
  void build(int ell_lo, int ell_hi, int q, FactorSet* out_lo, FactorSet* out_hi) {
    // distinct factors: same device pointer and size => same matrix (the
    // Python/C++ layers upload equal host factors once)
    std::vector<const double*> distinct;
    std::vector<int> which(d);
    for (int mu = 0; mu < d; ++mu) {
      which[mu] = -1;
      for (int m2 = 0; m2 < mu; ++m2)
        if (A[m2] == A[mu] && dims[m2] == dims[mu]) {
          which[mu] = which[m2];
          break;
        }
      if (which[mu] < 0) {
        which[mu] = int(distinct.size());
        distinct.push_back(A[mu]);
      }
    }
    std::vector<double*> lo(distinct.size()), hi(distinct.size());
    for (size_t j = 0; j < distinct.size(); ++j) {
      int mu = 0;
      while (which[mu] != int(j)) ++mu;
      const int n = dims[mu];
      const long long nn = (long long)n * n;
      double* scaled = alloc(nn * comps);
      scale_matrix_kernel<<<grid_ew(ctx, nn * comps), 256, 0, ctx->stream>>>(distinct[j],
                                                                            nn * comps, tau, scaled);
      ctx->launches++;
      KP_CUDA(cudaGetLastError());
      if (ell_hi == 0) {
        double* e = alloc(nn * comps);
        if (cplx)
          expm_batch_c128(ctx, scaled, n, 1, e);
        else
          expm_batch(ctx, scaled, n, 1, e);
        lo[j] = hi[j] = e;
      } else {
        double* tab = alloc(nn * comps * (ell_hi + 1));
        if (cplx)
          phiquad_dev_c128(ctx, scaled, n, ell_hi, q, -1, tab);
        else
          phiquad_dev(ctx, scaled, n, ell_hi, q, -1, tab);
        lo[j] = tab + nn * comps * ell_lo;
        hi[j] = tab + nn * comps * ell_hi;
      }
    }
    auto fill = [&](FactorSet* fs, const std::vector<double*>& src, int ell) {
      if (!fs) return;
      fs->f.resize(d);
      fs->active.assign(d, 1);
      fs->fold = 1.0;
      double fact = 1.0;
      for (int i = 2; i <= ell; ++i) fact *= i;
      fs->pref = std::pow(fact, double(d - 1));
      int nact = d;
      for (int mu = 0; mu < d; ++mu) {
        fs->f[mu] = src[which[mu]];
        double c = 0.0;
        if (nact > 1 && scalar_identity(fs->f[mu], dims[mu], &c)) {
          fs->active[mu] = 0;
          fs->fold *= c;
          --nact;
        }
      }
    };
    fill(out_lo, lo, ell_lo);
    fill(out_hi, hi, ell_hi);
  }

  // Tucker over the active modes; the skipped scalars multiply the last one.
  void tucker(const FactorSet& fs, const double* in, const std::vector<int>& tdims, double* out,
              const Epilogue* last) {
    std::vector<int> act;
    for (int mu = 0; mu < d; ++mu)
      if (fs.active[mu]) act.push_back(mu);
    const double* cur = in;
    size_t k0 = 0;
    if (!cplx && act.size() >= 3 && act[0] == 0 && act[1] == 1) {
      // modes 0 and 1 in one pass over small slices (fused01.cu); slot 1 =
      // the buffer the unfused loop would leave mode 1's result in
      double* dst = static_cast<double*>(
          ctx->ws.get(1, size_t(n_total(tdims)) * comps * sizeof(double)));
      if (fused01_f64(ctx, in, tdims, fs.f[0], tdims[0], fs.f[1], tdims[1], fs.pref, Epilogue{},
                      dst)) {
        cur = dst;
        k0 = 2;
      }
    }
    for (size_t k = k0; k < act.size(); ++k) {
      const int mu = act[k];
      const bool first = (k == 0), fin = (k + 1 == act.size());
      double* dst = fin ? out
                        : static_cast<double*>(ctx->ws.get(int(k & 1), size_t(n_total(tdims)) *
                                                                        comps * sizeof(double)));
      Epilogue e;
      if (fin && last) e = *last;
      e.alpha = (first ? fs.pref : 1.0) * (fin ? fs.fold : 1.0);
      mp(ctx, cur, tdims, mu, fs.f[mu], tdims[mu], e, dst);
      cur = dst;
    }
  }
  static long long n_total(const std::vector<int>& v) {
    long long n = 1;
    for (int x : v) n *= x;
    return n;
  }

  void kronsum(const double* u, double* r, const Epilogue& last) {
    if (banded) {  // one stencil pass, the reference's per-entry rounding (banded.cu)
      kronsum_banded(ctx, cplx, u, dims, band_cols, band_vals, a_active, r,
                     last.kind == EPI_ADD_G, last.g, half, -1, 0, 0, 0, last.t);
      return;
    }
    std::vector<int> act;
    for (int mu = 0; mu < d; ++mu)
      if (a_active[mu]) act.push_back(mu);
    for (size_t k = 0; k < act.size(); ++k) {
      Epilogue e;
      if (k + 1 == act.size()) e = last;
      e.alpha = 1.0;
      e.beta = k > 0 ? 1.0 : 0.0;
      mp(ctx, u, dims, act[k], A[act[k]], dims[act[k]], e, r);
    }
  }

  double* buf(int slot, long long entries) {
    return static_cast<double*>(ctx->ws.get(slot, size_t(entries) * comps * sizeof(double)));
  }

  template <bool C>
  void launch_pre(const double* u, double* w, bool two, double t) {
    using T = typename Elt<C>::T;
    if (!C && half > 0) {
      launch_pdl(ctx, lawson_pre_pair_kernel, dim3(grid_ew(ctx, half)), dim3(256), 0, g, t, half,
                 tau, two, u, w);
      return;
    }
    launch_pdl(ctx, lawson_pre_kernel<C>, dim3(grid_ew(ctx, n_entries)), dim3(256), 0, g, t,
               n_entries, half, tau, two, reinterpret_cast<const T*>(u), reinterpret_cast<T*>(w));
  }
  template <bool C>
  void launch_post(const double* y, double* out, int* bad, const int* ctr, double t2,
                   int* next) {
    using T = typename Elt<C>::T;
    if (!C && half > 0) {
      launch_pdl(ctx, lawson2b_post_pair_kernel, dim3(grid_ew(ctx, half)), dim3(256), 0, g, t2,
                 half, tau, y, out, bad, ctr, next);
      return;
    }
    launch_pdl(ctx, lawson2b_post_kernel<C>, dim3(grid_ew(ctx, n_entries)), dim3(256), 0, g, t2,
               n_entries, half, tau, reinterpret_cast<const T*>(y), reinterpret_cast<T*>(out), bad,
               ctr, next);
  }
  template <bool C>
  void launch_gdiff(const double* s, const double* u, double* dd, double t) {
    using T = typename Elt<C>::T;
    if (!C && half > 0) {
      launch_pdl(ctx, gdiff_pair_kernel, dim3(grid_ew(ctx, half)), dim3(256), 0, g, t, t + tau,
                 half, s, u, dd);
      return;
    }
    launch_pdl(ctx, gdiff_kernel<C>, dim3(grid_ew(ctx, n_entries)), dim3(256), 0, g, t, t + tau,
               n_entries, half, reinterpret_cast<const T*>(s), reinterpret_cast<const T*>(u),
               reinterpret_cast<T*>(dd));
  }

  // One step u -> out (out != u).  bad/ctr: divergence tracking (may be null).
  // One step; returns whether its last kernel already wrote *next =
  // *ctr + 1 (else the caller advances the counter).
  bool step(const double* u, double* out, double t, int* bad, const int* ctr,
            int* next = nullptr) {
    if (g.step_ctr) g.step_ctr = ctr;  // time-dependent g: this step's counter
    Epilogue fin;
    fin.bad_step = bad;
    fin.step_ctr = ctr;
    if (method == KP_ROSENBROCK_EULER && !given_jacobians) rosenbrock_factors(u);
    if (nonlocal) {
      step_nonlocal(u, out, t, fin);
      KP_CUDA(cudaGetLastError());
      return false;
    }
    fin.step_next = ctr ? next : nullptr;
    switch (method) {
      case KP_LAWSON_EULER: {  // :116-122
        double* w = buf(S_W, n_entries);
        cplx ? launch_pre<true>(u, w, false, t) : launch_pre<false>(u, w, false, t);
        tucker(f1, w, dims, out, &fin);
        break;
      }
      case KP_LAWSON2B: {  // :124-132, both Tuckers as one over [w0; w1]
        double* w = buf(S_W, 2 * n_entries);
        double* y = buf(S_Y, 2 * n_entries);
        cplx ? launch_pre<true>(u, w, true, t) : launch_pre<false>(u, w, true, t);
        std::vector<int> sd = dims;
        sd.push_back(2);
        FactorSet fs = f1;
        fs.f.push_back(nullptr);
        fs.active.push_back(0);
        const int d_save = d;
        d = d + 1;  // the stacking mode is never active
        tucker(fs, w, sd, y, nullptr);
        d = d_save;
        if (bad) {
          cplx ? launch_post<true>(y, out, bad, ctr, t + tau, fin.step_next)
               : launch_post<false>(y, out, bad, ctr, t + tau, fin.step_next);
        } else {
          int* dummy = static_cast<int*>(ctx->ws.get(S_CTR + 1, 16));
          cplx ? launch_post<true>(y, out, dummy, dummy, t + tau, nullptr)
               : launch_post<false>(y, out, dummy, dummy, t + tau, nullptr);
        }
        break;
      }
      case KP_EXP_EULER:          // :134-141
      case KP_ROSENBROCK_EULER: {  // :166-194 (factors rebuilt above)
        double* r = buf(S_R, n_entries);
        Epilogue eg;
        eg.kind = EPI_ADD_G;
        eg.X = u;
        eg.g = g;
        eg.t = t;
        kronsum(u, r, eg);
        fin.kind = EPI_FMA_X;
        fin.X = u;
        fin.gamma = tau;
        tucker(method == KP_ROSENBROCK_EULER ? fj : f1, r, dims, out, &fin);
        break;
      }
      case KP_EXP_EULER_LS: {  // :143-151  (f1 = exp factors, f2 = phi1)
        double* y = buf(S_Y, n_entries);
        double* gn = buf(S_D, n_entries);
        tucker(f1, u, dims, y, nullptr);
        Epilogue none;
        eval_g(u, gn, t);
        fin.kind = EPI_FMA_X;
        fin.X = y;
        fin.gamma = tau;
        tucker(f2, gn, dims, out, &fin);
        (void)none;
        break;
      }
      case KP_ETD2RK: {  // :153-164
        double* r = buf(S_R, n_entries);
        double* s = buf(S_S, n_entries);
        double* dd = buf(S_D, n_entries);
        Epilogue eg;
        eg.kind = EPI_ADD_G;
        eg.X = u;
        eg.g = g;
        eg.t = t;
        kronsum(u, r, eg);
        Epilogue es;
        es.X = u;
        es.gamma = tau;
        es.g = g;
        es.t = t;
        es.t2 = t + tau;
        if (half == 0) {
          es.kind = EPI_STAGE_D;
          es.D = dd;
          tucker(f1, r, dims, s, &es);
        } else {
          es.kind = EPI_FMA_X;
          tucker(f1, r, dims, s, &es);
          cplx ? launch_gdiff<true>(s, u, dd, t) : launch_gdiff<false>(s, u, dd, t);
        }
        fin.kind = EPI_FMA_X;
        fin.X = s;
        fin.gamma = tau;
        tucker(f2, dd, dims, out, &fin);
        break;
      }
      default:
        throw invalid_argument("step: unknown method " + std::to_string(method));
    }
    KP_CUDA(cudaGetLastError());
    return fin.step_next != nullptr;
  }

  void eval_g(const double* u, double* out, double t) {
    if (nonlocal) {
      riccati_g(ctx, g, u, dims[0], buf(S_WZ, 2LL * dims[0]), out);
      return;
    }
    launch_eval_g(ctx, g, t, u, size_t(n_entries), size_t(half), cplx, out);
  }

  // nonlocal-g step: g values come from eval_g into buffers, the GEMM
  // epilogues only add them (same operations, unfused)
  void step_nonlocal(const double* u, double* out, double t, Epilogue fin) {
    double* gn = buf(S_G, n_entries);
    eval_g(u, gn, t);
    switch (method) {
      case KP_LAWSON_EULER:
      case KP_LAWSON2B: {
        double* w = buf(S_W, 2 * n_entries);
        launch_fma(ctx, size_t(n_entries), tau, gn, u, w);  // u + tau g
        if (method == KP_LAWSON_EULER) {
          tucker(f1, w, dims, out, &fin);
          return;
        }
        launch_fma(ctx, size_t(n_entries), 0.5 * tau, gn, u, w + n_entries);
        double* stage = buf(S_S, n_entries);
        double* y = buf(S_Y, n_entries);
        tucker(f1, w, dims, stage, nullptr);
        tucker(f1, w + n_entries, dims, y, nullptr);
        double* gs = buf(S_D, n_entries);
        eval_g(stage, gs, t + tau);
        Epilogue none;
        (void)none;
        launch_fma(ctx, size_t(n_entries), 0.5 * tau, gs, y, out);  // y + tau/2 g(stage)
        check_finite_into(out, fin);
        return;
      }
      case KP_EXP_EULER:
      case KP_ROSENBROCK_EULER: {
        double* r = buf(S_R, n_entries);
        Epilogue ex;
        ex.kind = EPI_ADD_X;
        ex.X = gn;
        kronsum(u, r, ex);
        fin.kind = EPI_FMA_X;
        fin.X = u;
        fin.gamma = tau;
        tucker(method == KP_ROSENBROCK_EULER ? fj : f1, r, dims, out, &fin);
        return;
      }
      case KP_EXP_EULER_LS: {
        double* y = buf(S_Y, n_entries);
        tucker(f1, u, dims, y, nullptr);
        fin.kind = EPI_FMA_X;
        fin.X = y;
        fin.gamma = tau;
        tucker(f2, gn, dims, out, &fin);
        return;
      }
      case KP_ETD2RK: {
        double* r = buf(S_R, n_entries);
        double* s = buf(S_S, n_entries);
        double* dd = buf(S_D, n_entries);
        Epilogue ex;
        ex.kind = EPI_ADD_X;
        ex.X = gn;
        kronsum(u, r, ex);
        Epilogue es;
        es.kind = EPI_FMA_X;
        es.X = u;
        es.gamma = tau;
        tucker(f1, r, dims, s, &es);
        eval_g(s, dd, t + tau);
        launch_fma(ctx, size_t(n_entries), -1.0, gn, dd, dd);  // g(stage) - g(u)
        fin.kind = EPI_FMA_X;
        fin.X = s;
        fin.gamma = tau;
        tucker(f2, dd, dims, out, &fin);
        return;
      }
      default:
        throw invalid_argument("step: unknown method " + std::to_string(method));
    }
  }

  // non-finite check of an elementwise result (the GEMM epilogues do it inline)
  void check_finite_into(const double* x, const Epilogue& fin) {
    if (fin.bad_step) finite_flag(ctx, size_t(n_entries) * comps, x, fin.bad_step, fin.step_ctr);
  }

  // Rosenbrock-Euler (inc/integrators.hpp:166-194): phi_1 of the current
  // Jacobian factors, rebuilt every step (one build when they coincide)
  void rosenbrock_factors(const double* u) {
    const int n = dims[0];
    const long long nn = (long long)n * n;
    double* j1 = buf(S_J1, nn);
    double* j2 = buf(S_J2, nn);
    const int nf = riccati_jacobians(ctx, g, u, A[0], n, buf(S_WZ, 2LL * n), j1, j2);
    double* scaled = buf(S_J3, nn);
    fj.f.assign(2, nullptr);
    fj.active.assign(2, 1);
    fj.fold = 1.0;
    fj.pref = 1.0;
    for (int k = 0; k < nf; ++k) {
      scale_matrix_kernel<<<grid_ew(ctx, nn), 256, 0, ctx->stream>>>(k == 0 ? j1 : j2, nn, tau,
                                                                      scaled);
      ctx->launches++;
      double* tab = k == 0 ? buf(S_PHI1, 2 * nn) : buf(S_PHI2, 2 * nn);
      phiquad_dev(ctx, scaled, n, 1, q_nodes, -1, tab);
      fj.f[k] = tab + nn;
    }
    if (nf == 1) fj.f[1] = fj.f[0];
  }

  void setup(int q) {
    switch (method) {  // inc/integrators.hpp:263-283
      case KP_LAWSON_EULER:
      case KP_LAWSON2B:
        build(0, 0, q, &f1, nullptr);
        break;
      case KP_EXP_EULER:
        build(1, 1, q, nullptr, &f1);
        break;
      case KP_EXP_EULER_LS:
        build(0, 0, q, &f1, nullptr);
        build(1, 1, q, nullptr, &f2);
        break;
      case KP_ETD2RK:
        build(1, 2, q, &f1, &f2);
        break;
      case KP_ROSENBROCK_EULER:  // :224-226
        if (!nonlocal)
          throw invalid_argument("integrate: Rosenbrock-Euler requires jacobian_factors");
        q_nodes = q;  // factors are built per step from the Jacobian
        break;
      default:
        throw invalid_argument("integrate: unknown method " + std::to_string(method));
    }
  }

  // integrate loop (:290-367) on u (device, in/out).  Returns loop seconds.
  // sample_every > 0: after every sample_every steps the state is copied to
  // the host and handed to fn (the reference's trajectory, :365-366); the
  // loop then runs eagerly (same kernels as the graph replay).
  double run(double* u, double t0, long n_steps, bool use_graph, int sample_every = 0,
             kp_sample_fn sample_fn = nullptr, void* sample_user = nullptr) {
    // step counter in two alternating slots (step k reads slot k&1 and its
    // last kernel writes slot (k+1)&1), divergence flag in between
    int* cbuf = static_cast<int*>(ctx->ws.get(S_CTR, 16));
    int* slot[2] = {cbuf, cbuf + 2};
    int* bad = cbuf + 1;
    const int init[4] = {0, INT_MAX, 0, 0};
    KP_CUDA(cudaMemcpyAsync(cbuf, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
    int* ctr = slot[0];
    double* ub[2] = {u, buf(S_U2, n_entries)};
    // a 128 x 128 real exp-Euler state: the whole loop in one cluster launch
    // (banded.cu small2d_expeuler_kernel; same arithmetic, bit-identical)
    if (method == KP_EXP_EULER && d == 2 && !cplx && banded && !nonlocal && half == 0 &&
        !(sample_every > 0 && sample_fn) && a_active[0] && a_active[1] && f1.active[0] &&
        f1.active[1] && f1.f[0] == f1.f[1] && f1.pref == 1.0 && f1.fold == 1.0) {
      cudaEvent_t e0, e1;
      KP_CUDA(cudaEventCreate(&e0));
      KP_CUDA(cudaEventCreate(&e1));
      KP_CUDA(cudaEventRecord(e0, ctx->stream));
      const bool done = small2d_expeuler(ctx, dims, band_cols, band_vals, f1.f[0], g, tau,
                                         n_steps, u, bad);
      KP_CUDA(cudaEventRecord(e1, ctx->stream));
      if (done) {
        int hb[2];
        KP_CUDA(cudaMemcpyAsync(hb, cbuf, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
        KP_CUDA(cudaStreamSynchronize(ctx->stream));
        float ms = 0.f;
        KP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        diverged_at = (hb[1] != INT_MAX) ? long(hb[1]) : 0;
        return ms * 1e-3;
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    // device time of the loop = [e0,e1] (first, eager step) + [e2,e3] (graph
    // replays + tail); the host-side capture/instantiation between e1 and e2
    // is set-up, not stepping, and is excluded
    cudaEvent_t ev[4];
    for (auto& e : ev) KP_CUDA(cudaEventCreate(&e));
    long n = 0;
    // time-dependent g's read t = t0 + (*ctr) tau on the device (graph-safe)
    g.step_ctr = ctr;
    g.t0 = t0;
    g.tau = tau;
    auto one = [&](long k) {
      int *c = slot[k & 1], *c2 = slot[(k + 1) & 1];
      if (!step(ub[k & 1], ub[(k + 1) & 1], 0.0, bad, c, c2))
        launch_pdl(ctx, tick_kernel, dim3(1), dim3(1), 0, (const int*)c, c2);
    };
    // first step eagerly: sizes every workspace slot before any capture
    KP_CUDA(cudaEventRecord(ev[0], ctx->stream));
    one(n++);
    KP_CUDA(cudaEventRecord(ev[1], ctx->stream));
    cudaGraphExec_t exec = nullptr;
    unsigned long long per = 0;
    // steps per graph: an even number (ping-pong buffers and counter slots
    // return to their start); 8 for small states, whose steps are a few
    // microseconds each and would otherwise pay a graph launch every 2
    const long span = (n_entries <= (1L << 17) && n_steps - n >= 10) ? 8 : 2;
    const bool sampling = sample_every > 0 && sample_fn;
    double* hs = nullptr;
    if (sampling) {
      hs = static_cast<double*>(ctx->pin_out.get(size_t(n_entries) * comps * sizeof(double)));
      if (1 % sample_every == 0) {  // the eager first step completes a sample
        KP_CUDA(cudaMemcpyAsync(hs, ub[1], size_t(n_entries) * comps * sizeof(double),
                                cudaMemcpyDeviceToHost, ctx->stream));
        KP_CUDA(cudaStreamSynchronize(ctx->stream));
        sample_fn(sample_user, 1, hs);
      }
    }
    if (use_graph && !sampling && method != KP_ROSENBROCK_EULER && n_steps - n >= 4) {
      cudaGraph_t graph;
      const unsigned long long l0 = ctx->launches;
      KP_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      // `span` steps starting at an odd one (n is odd here): ub1 -> ub0 ->
      // ... -> ub1; t is unused by the closed set of g's (time-dependent
      // ones read the device counter), so replays stay exact
      for (long j = 1; j <= span; ++j) one(j);
      KP_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
      per = ctx->launches - l0;
      ctx->launches = l0;
      KP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
    }
    KP_CUDA(cudaEventRecord(ev[2], ctx->stream));
    if (exec) {
      while (n_steps - n >= span) {
        KP_CUDA(cudaGraphLaunch(exec, ctx->stream));
        ctx->launches += per;
        n += span;
      }
    }
    while (n < n_steps) {
      one(n++);
      if (sampling && n % sample_every == 0) {
        KP_CUDA(cudaMemcpyAsync(hs, ub[n & 1], size_t(n_entries) * comps * sizeof(double),
                                cudaMemcpyDeviceToHost, ctx->stream));
        KP_CUDA(cudaStreamSynchronize(ctx->stream));
        sample_fn(sample_user, n, hs);
      }
    }
    KP_CUDA(cudaEventRecord(ev[3], ctx->stream));
    if (exec) cudaGraphExecDestroy(exec);
    if (n_steps & 1)
      KP_CUDA(cudaMemcpyAsync(u, ub[1], size_t(n_entries) * comps * sizeof(double),
                              cudaMemcpyDeviceToDevice, ctx->stream));
    int hb[2];
    KP_CUDA(cudaMemcpyAsync(hb, cbuf, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
    float ms1 = 0.f, ms2 = 0.f;
    KP_CUDA(cudaEventElapsedTime(&ms1, ev[0], ev[1]));
    KP_CUDA(cudaEventElapsedTime(&ms2, ev[2], ev[3]));
    for (auto& e : ev) cudaEventDestroy(e);
    const float ms = ms1 + ms2;
    diverged_at = (hb[1] != INT_MAX) ? long(hb[1]) : 0;
    return ms * 1e-3;
  }
};


// ======================================================================
// Slab-sharded integrate; replaces parallel.py's
// ShardedIntegrator behind the C ABI (kp_integrate_sharded_*).
//
// Global layout: spatial modes n_1..n_ds, species S (2 for the stacked
// Brusselator: the slowest mode), viewed column-major as (A, B, C, S) with
// A = n_1..n_{ds-2}, B = n_{ds-1}, C = n_ds.  Rank r owns the slab of planes
// [r C/P, (r+1) C/P) of the last spatial mode; the pencil layout splits B
// instead (modes < ds-1 and g are slab-local, mode ds is pencil-local).
//
// Mode ds (the exchange step), two ways:
//   A: all-to-all pencil transpose (comm.cu pack -> grouped send/recv ->
//      unpack), mode ds on the pencil, the step's last update fused into its
//      epilogue, transposed back.  Every entry is computed from the same
//      inputs in the same k order as on one GPU: bitwise equal to the
//      single-GPU integrate.
//   B: every rank multiplies its slab by its column block of the factor
//      (a full-size partial product), the partials are reduce-scattered into
//      slabs (ncclReduceScatter), the epilogue runs as an elementwise pass.
//      P x the bytes of one transpose but no transpose back and no pencil
//      copy of u; sums the k range in a different order (tolerance-level).
//   mode_d = 0 picks by measurement: one step of each, device time (max over
//   ranks), the faster wins.
// The Kronecker sum of banded factors (every config) is the stencil of
// banded.cu on the slab with a one-plane halo exchange.
//
// Exchanges are stream-ordered (NCCL on the context's stream): no host sync
// or barrier inside a step, and the step is captured into a CUDA graph.
// The same code drives all P ranks inside one process (comm == NULL,
// "emulated": the exchanges become device copies between the ranks'
// buffers) -- how the data movement is tested bitwise on one GPU.
// ======================================================================

__global__ void add_into_kernel(long long n, const double* __restrict__ x, double* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = __dadd_rn(y[i], x[i]);
}

class ShardExchange {
 public:
  int P = 1;
  kp_comm* comm = nullptr;      // NCCL, one local rank
  std::vector<int> ranks;       // ranks this process drives
  std::vector<double*> send, recv;  // per local rank scratch (repartition)
  long long cap = 0;

  int nlocal() const { return int(ranks.size()); }

  // send/recv scratch of local rank i: grow-only workspace slots 80+i / 96+i
  // (no cudaMalloc / cudaFree per call)
  kp_ctx* wctx = nullptr;
  void scratch(long long doubles) {
    send.resize(ranks.size());
    recv.resize(ranks.size());
    for (size_t i = 0; i < ranks.size(); ++i) {
      if (i >= 16) throw invalid_argument("sharded: at most 16 emulated ranks");
      send[i] = static_cast<double*>(wctx->ws.get(80 + int(i), size_t(doubles) * 8));
      recv[i] = static_cast<double*>(wctx->ws.get(96 + int(i), size_t(doubles) * 8));
    }
  }

  // y[i] = x[i] re-partitioned (dir 1: slab -> pencil, 2: back)
  void repartition(kp_ctx* ctx, int dir, long long A, long long B, long long C, long long S,
                   int comps, const std::vector<const double*>& x, const std::vector<double*>& y) {
    const long long n = A * B * C * S / P * comps;  // doubles per rank
    if (P == 1) {
      if (x[0] != y[0])
        KP_CUDA(cudaMemcpyAsync(y[0], x[0], size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice,
                                ctx->stream));
      return;
    }
    wctx = ctx;
    scratch(n);
    if (comm) {
      comm_repartition(ctx, comm, dir, A, B, C, S, comps, x[0], y[0], send[0], recv[0]);
      return;
    }
    const long long blk = n / P;
    for (int r = 0; r < P; ++r)
      repartition_pack(ctx, dir, P, r, A, B, C, S, comps, x[r], send[r], true);
    for (int r = 0; r < P; ++r)
      for (int s = 0; s < P; ++s)
        KP_CUDA(cudaMemcpyAsync(recv[s] + r * blk, send[r] + s * blk, size_t(blk) * sizeof(double),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    for (int r = 0; r < P; ++r)
      repartition_pack(ctx, dir, P, r, A, B, C, S, comps, recv[r], y[r], false);
  }

  // ext[i] = (plane doubles) x (Cl + 2) x S: fill planes 0 and Cl+1 of every
  // species from the neighbours' last / first interior planes (periodic in
  // the rank index; a Dirichlet factor never reads the wrapped plane)
  void halo(kp_ctx* ctx, long long plane, long long Cl, long long S,
            const std::vector<double*>& ext) {
    auto at = [&](double* e, long long sp, long long k) { return e + (sp * (Cl + 2) + k) * plane; };
    if (comm && P > 1) {
      const int r = ranks[0], up = (r + 1) % P, down = (r + P - 1) % P;
      std::vector<const double*> sends;
      std::vector<int> to, from;
      std::vector<double*> recvs;
      for (long long sp = 0; sp < S; ++sp) {  // same order as kp_comm_halo_f64
        sends.push_back(at(ext[0], sp, Cl));  // last interior -> up (its left halo)
        to.push_back(up);
        sends.push_back(at(ext[0], sp, 1));   // first interior -> down (its right halo)
        to.push_back(down);
        recvs.push_back(at(ext[0], sp, 0));   // left halo <- down's last
        from.push_back(down);
        recvs.push_back(at(ext[0], sp, Cl + 1));  // right halo <- up's first
        from.push_back(up);
      }
      comm_sendrecv(ctx, comm, sends, to, recvs, from, size_t(plane));
      return;
    }
    const int n = nlocal();  // emulated (or P == 1): device copies
    for (int i = 0; i < n; ++i) {
      const int dn = (i + n - 1) % n, upi = (i + 1) % n;
      for (long long sp = 0; sp < S; ++sp) {
        KP_CUDA(cudaMemcpyAsync(at(ext[i], sp, 0), at(ext[dn], sp, Cl), size_t(plane) * 8,
                                cudaMemcpyDeviceToDevice, ctx->stream));
        KP_CUDA(cudaMemcpyAsync(at(ext[i], sp, Cl + 1), at(ext[upi], sp, 1), size_t(plane) * 8,
                                cudaMemcpyDeviceToDevice, ctx->stream));
      }
    }
  }

  // y[i] = sum over ranks of the ranks[i]-th C/P-plane block (per species) of
  // the full-size partials part[*]  (plane doubles per plane)
  void reduce_scatter(kp_ctx* ctx, long long plane, long long C, long long S,
                      const std::vector<double*>& part, const std::vector<double*>& y) {
    const long long Cl = C / P, cnt = plane * Cl;
    if (comm) {
      for (long long sp = 0; sp < S; ++sp)
        comm_reduce_scatter(ctx, comm, part[0] + sp * plane * C, y[0] + sp * cnt, size_t(cnt));
      return;
    }
    for (int s = 0; s < P; ++s)
      for (long long sp = 0; sp < S; ++sp) {
        double* dst = y[s] + sp * cnt;
        KP_CUDA(cudaMemcpyAsync(dst, part[0] + sp * plane * C + s * cnt, size_t(cnt) * 8,
                                cudaMemcpyDeviceToDevice, ctx->stream));
        for (int r = 1; r < P; ++r) {
          add_into_kernel<<<grid_ew(ctx, cnt), 256, 0, ctx->stream>>>(
              cnt, part[r] + sp * plane * C + s * cnt, dst);
          ctx->launches++;
        }
      }
  }

  // Peer mappings for the fused exchange (mode_d 3): all[r] = rank r's copy
  // of a per-rank buffer as seen from this process.  Emulated: the local
  // buffers themselves; NCCL: CUDA IPC handles all-gathered over the
  // communicator and opened (NVLink P2P).  false = not mappable.
  std::vector<void*> opened;
  bool map(kp_ctx* ctx, const std::vector<double*>& local, std::vector<double*>& all,
           void* dev_scratch) {
    all.assign(P, nullptr);
    if (!comm) {
      for (int i = 0; i < nlocal(); ++i) all[ranks[i]] = local[i];
      return true;
    }
    if (P == 1) {
      all[0] = local[0];
      return true;
    }
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, local[0]) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    const size_t hb = sizeof(h);
    unsigned char* d = static_cast<unsigned char*>(dev_scratch);
    KP_CUDA(cudaMemcpyAsync(d, &h, hb, cudaMemcpyHostToDevice, ctx->stream));
    comm_allgather_bytes(ctx, comm, d, d + hb, hb);
    std::vector<unsigned char> hs(hb * P);
    KP_CUDA(cudaMemcpyAsync(hs.data(), d + hb, hb * P, cudaMemcpyDeviceToHost, ctx->stream));
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
    bool ok = true;
    for (int r = 0; r < P; ++r) {
      if (r == ranks[0]) {
        all[r] = local[0];
        continue;
      }
      cudaIpcMemHandle_t hr;
      std::memcpy(&hr, hs.data() + hb * r, hb);
      void* ptr = nullptr;
      if (cudaIpcOpenMemHandle(&ptr, hr, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = false;
        continue;
      }
      opened.push_back(ptr);
      all[r] = static_cast<double*>(ptr);
    }
    // every rank must have mapped every peer (a max over ranks of "failed")
    double bad = ok ? 0.0 : 1.0;
    bad = max_over_ranks(ctx, bad, static_cast<double*>(dev_scratch));
    return bad == 0.0;
  }
  // after peer stores: every rank's stores have landed before anyone reads
  // (a one-double NCCL all-reduce, stream-ordered: no host sync)
  void fence(kp_ctx* ctx, double* scratch) {
    if (comm && P > 1) comm_allreduce(ctx, comm, scratch, 1, 1);
  }
  ~ShardExchange() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
  }

  // max over all ranks of a host value (NCCL all-reduce through the device)
  double max_over_ranks(kp_ctx* ctx, double v, double* dev_scratch) {
    if (!comm || P == 1) return v;
    KP_CUDA(cudaMemcpyAsync(dev_scratch, &v, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    comm_allreduce(ctx, comm, dev_scratch, 1, 1);
    KP_CUDA(cudaMemcpyAsync(&v, dev_scratch, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
    return v;
  }
};

class ShardedIntegrator {
 public:
  kp_ctx* ctx;
  ShardExchange& X;
  Integrator G;  // global set-up: factor sets, band structures, g checks
  int method, P, ds, comps, mode_d = 1;
  bool cplx;
  long long A, B, C, S, Cl, Bp, nloc;
  std::vector<int> dl, dp;  // local slab / pencil dims (incl. species)
  struct Rank {
    int r;
    double *u, *ub, *ext, *rr, *rp, *up, *sp, *dq, *dd, *t0, *t1, *w, *y, *part, *out, *tr;
    // fused exchange (mode_d 3): state ping-pong, receive buffers per site
    // and step parity, and the device arrays of the P ranks' copies
    double* S[2] = {nullptr, nullptr};
    double* pen[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    double* upb[2] = {nullptr, nullptr};
    double* ddb[2] = {nullptr, nullptr};
    double* const* pS[2] = {nullptr, nullptr};
    double* const* ppen[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    double* const* pupb[2] = {nullptr, nullptr};
    double* const* pddb[2] = {nullptr, nullptr};
    double* const* part_arr = nullptr;  // staging for setup_fused
    int* cnt;  // [ctr slot 0, bad, ctr slot 1]
  };
  std::vector<Rank> R;
  std::vector<double*> owned;
  double* scratch = nullptr;

  ShardedIntegrator(kp_ctx* c, ShardExchange& x, int m, bool cp, const std::vector<int>& gdims,
                    const double* const* as, const kp_gfun& g, double tau)
      : ctx(c), X(x), G(c, m, cp, gdims, as, g, tau), method(m), P(x.P), comps(cp ? 2 : 1),
        cplx(cp) {
    if (g.kind == KP_G_ADR || g.kind == KP_G_RICCATI || g.step_ctr)
      throw invalid_argument("sharded integrate: the ADR and Riccati g's are not supported "
                             "(time-dependent / nonlocal)");
    if (method == KP_ROSENBROCK_EULER || method == KP_EXP_EULER_LS)
      throw invalid_argument("sharded integrate: lawson_euler, lawson2b, exp_euler, etd2rk");
    S = (g.kind == KP_G_BRUSSELATOR) ? 2 : 1;
    ds = int(gdims.size()) - (S == 2 ? 1 : 0);
    if (ds < 2) throw invalid_argument("sharded integrate: needs >= 2 spatial modes");
    A = 1;
    for (int mu = 0; mu < ds - 2; ++mu) A *= gdims[mu];
    B = gdims[ds - 2];
    C = gdims[ds - 1];
    if (B % P || C % P)
      throw invalid_argument("sharded integrate: n_(d-1) and n_d must be divisible by P");
    Cl = C / P;
    Bp = B / P;
    dl = gdims;
    dl[ds - 1] = int(Cl);
    dp = gdims;
    dp[ds - 2] = int(Bp);
    nloc = A * B * Cl * S;
    KP_CUDA(cudaMalloc(&scratch, 64));
    owned.push_back(scratch);
  }
  ~ShardedIntegrator() {
    for (double* p : owned) cudaFree(p);
  }
  double* alloc(long long entries) {
    double* p = nullptr;
    KP_CUDA(cudaMalloc(&p, size_t(std::max<long long>(entries, 1)) * comps * sizeof(double)));
    owned.push_back(p);
    return p;
  }
  bool fused_ready = false;
  // allocate and map the fused exchange's buffers (all ranks must succeed)
  bool setup_fused() {
    if (fused_ready) return true;
    // the Kronecker sum's last mode runs as the halo stencil (no pencil term)
    if ((method == KP_EXP_EULER || method == KP_ETD2RK) && !G.banded) return false;
    double* scratch2 = nullptr;
    KP_CUDA(cudaMalloc(&scratch2, 4096));
    owned.push_back(scratch2);
    auto site = [&](double* Rank::*one, double* const* Rank::*arr) -> bool {
      std::vector<double*> loc;
      for (auto& k : R) loc.push_back(k.*one);
      std::vector<double*> all;
      if (!X.map(ctx, loc, all, scratch2)) return false;
      double** dev = nullptr;
      KP_CUDA(cudaMalloc(&dev, sizeof(double*) * all.size()));
      owned.push_back(reinterpret_cast<double*>(dev));
      KP_CUDA(cudaMemcpyAsync(dev, all.data(), sizeof(double*) * all.size(),
                              cudaMemcpyHostToDevice, ctx->stream));
      for (auto& k : R) k.*arr = dev;
      return true;
    };
    // member pointers cannot name array elements: map through staging members
    bool ok = true;
    for (int a = 0; a < 2 && ok; ++a) {
      each([&](Rank& k) { k.S[a] = alloc(nloc); });
      each([&](Rank& k) { k.tr = k.S[a]; });
      ok = site(&Rank::tr, &Rank::part_arr);
      each([&](Rank& k) { k.pS[a] = k.part_arr; });
      for (int t = 0; t < 2 && ok; ++t) {
        each([&](Rank& k) { k.pen[t][a] = alloc(nloc); k.tr = k.pen[t][a]; });
        ok = site(&Rank::tr, &Rank::part_arr);
        each([&](Rank& k) { k.ppen[t][a] = k.part_arr; });
      }
      if (!ok) break;
      each([&](Rank& k) { k.upb[a] = alloc(nloc); k.tr = k.upb[a]; });
      ok = site(&Rank::tr, &Rank::part_arr);
      each([&](Rank& k) { k.pupb[a] = k.part_arr; });
      if (!ok) break;
      each([&](Rank& k) { k.ddb[a] = alloc(nloc); k.tr = k.ddb[a]; });
      ok = site(&Rank::tr, &Rank::part_arr);
      each([&](Rank& k) { k.pddb[a] = k.part_arr; });
    }
    each([&](Rank& k) { k.tr = alloc(nloc); });
    fused_ready = ok;
    return ok;
  }

  void setup(int q, int md, const std::vector<double*>& user_u) {
    G.setup(q);
    for (const FactorSet* fs : {&G.f1, &G.f2}) {
      if (fs->f.empty()) continue;
      for (int mu = 0; mu < ds; ++mu)
        if (!fs->active[mu])
          throw invalid_argument("sharded integrate: a spatial phi factor is a multiple of I");
    }
    const long long plane = A * B;
    R.resize(X.nlocal());
    for (int i = 0; i < X.nlocal(); ++i) {
      Rank& k = R[i];
      k.r = X.ranks[i];
      k.u = user_u[i];
      k.ub = alloc(nloc);
      k.ext = alloc(plane * (Cl + 2) * S);
      k.rr = alloc(nloc);
      k.rp = alloc(nloc);
      k.up = alloc(nloc);
      k.sp = alloc(2 * nloc);  // [stage; y1] for Lawson2b
      k.dq = alloc(nloc);
      k.dd = alloc(nloc);
      k.t0 = alloc(nloc);
      k.t1 = alloc(nloc);
      k.w = alloc(2 * nloc);
      k.y = alloc(nloc);
      k.out = alloc(nloc);
      k.tr = alloc(nloc);
      k.part = md == 1 ? nullptr : alloc(A * B * C * S);
      int* cb = nullptr;
      KP_CUDA(cudaMalloc(&cb, 16));
      owned.push_back(reinterpret_cast<double*>(cb));
      const int init[4] = {0, INT_MAX, 0, 0};
      KP_CUDA(cudaMemcpyAsync(cb, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
      k.cnt = cb;
    }
  }

  template <typename F>
  void each(F&& f) {
    for (auto& k : R) f(k);
  }
  std::vector<const double*> cv(double* Rank::*m, long long off = 0) {
    std::vector<const double*> v;
    for (auto& k : R) v.push_back(k.*m + off);
    return v;
  }
  std::vector<double*> mv(double* Rank::*m, long long off = 0) {
    std::vector<double*> v;
    for (auto& k : R) v.push_back(k.*m + off);
    return v;
  }
  void to_pencil(const std::vector<const double*>& x, const std::vector<double*>& y) {
    X.repartition(ctx, 1, A, B, C, S, comps, x, y);
  }
  void to_slab(const std::vector<const double*>& x, const std::vector<double*>& y) {
    X.repartition(ctx, 2, A, B, C, S, comps, x, y);
  }

  // modes 0 .. ds-2 of a Tucker on the slab: returns the buffer holding the result
  const double* tucker_slab(const FactorSet& fs, const double* x, Rank& k) {
    const double* cur = x;
    for (int mu = 0; mu < ds - 1; ++mu) {
      double* dst = (mu & 1) ? k.t1 : k.t0;
      Epilogue e;
      e.alpha = (mu == 0) ? fs.pref : 1.0;
      G.mp(ctx, cur, dl, mu, fs.f[mu], dl[mu], e, dst);
      cur = dst;
    }
    return cur;
  }
  // Tucker with the last spatial mode on the pencil (option A): in (slab) ->
  // out (pencil), `last(k)` = the epilogue of the last mode
  template <typename L>
  void tucker_A(const FactorSet& fs, const std::vector<const double*>& in,
                const std::vector<double*>& out, L&& last) {
    std::vector<const double*> mid;
    for (size_t i = 0; i < R.size(); ++i) mid.push_back(tucker_slab(fs, in[i], R[i]));
    std::vector<const double*> pen = mid;  // P = 1: the pencil is the slab
    if (P > 1) {
      std::vector<double*> pb;
      for (size_t i = 0; i < R.size(); ++i) pb.push_back(mid[i] == R[i].t0 ? R[i].t1 : R[i].t0);
      to_pencil(mid, pb);
      pen.assign(pb.begin(), pb.end());
    }
    for (size_t i = 0; i < R.size(); ++i) {
      Epilogue e = last(R[i]);
      e.alpha = fs.fold * (ds == 1 ? fs.pref : 1.0);
      G.mp(ctx, pen[i], dp, ds - 1, fs.f[ds - 1], dp[ds - 1], e, out[i]);
    }
  }
  // Tucker with the last spatial mode as partial products + reduce-scatter
  // (option B): in (slab) -> out (slab), no epilogue
  void tucker_B(const FactorSet& fs, const std::vector<const double*>& in,
                const std::vector<double*>& out) {
    std::vector<int> fd = dl;
    fd[ds - 1] = int(C);
    std::vector<double*> parts;
    for (size_t i = 0; i < R.size(); ++i) {
      Rank& k = R[i];
      const double* mid = tucker_slab(fs, in[i], k);
      Epilogue e;
      e.alpha = fs.fold * (ds == 1 ? fs.pref : 1.0);
      // columns [r Cl, (r+1) Cl) of the C x C factor: a C x Cl matrix, ld C
      const double* blk = fs.f[ds - 1] + (long long)k.r * Cl * C * comps;
      G.mp(ctx, mid, dl, ds - 1, blk, int(C), e, k.part);
      parts.push_back(k.part);
    }
    X.reduce_scatter(ctx, A * B * comps, C, S, parts, out);
  }

  // r = K u + g(u) in slab layout (u: slab)
  void kronsum_g(const std::vector<const double*>& u, const std::vector<double*>& r, double t) {
    if (G.banded && P == 1) {  // one rank: the plain stencil on u, no halo planes
      each([&](Rank& k) {
        kronsum_banded(ctx, cplx, u[&k - R.data()], dl, G.band_cols, G.band_vals, G.a_active,
                       r[&k - R.data()], true, G.g, S == 2 ? 1 : 0, -1, 0, 0, 0, t);
      });
      return;
    }
    if (G.banded) {
      const long long plane = A * B * comps;
      // interior planes of every species into ext, then the halo planes
      each([&](Rank& k) {
        const long long i = &k - R.data();
        KP_CUDA(cudaMemcpy2DAsync(k.ext + plane, size_t(plane * (Cl + 2)) * 8, u[i],
                                  size_t(plane * Cl) * 8, size_t(plane * Cl) * 8, size_t(S),
                                  cudaMemcpyDeviceToDevice, ctx->stream));
      });
      X.halo(ctx, plane, Cl, S, mv(&Rank::ext));
      each([&](Rank& k) {
        const long long i = &k - R.data();
        kronsum_banded(ctx, cplx, k.ext, dl, G.band_cols, G.band_vals, G.a_active, r[i], true,
                       G.g, S == 2 ? 1 : 0, ds - 1, int(k.r * Cl), int(C), 1, t);
      });
      return;
    }
    // dense: terms 0..ds-2 on the slab, the last on the pencil, back to the slab
    each([&](Rank& k) {
      const long long i = &k - R.data();
      bool first = true;
      for (int mu = 0; mu < ds - 1; ++mu) {
        if (!G.a_active[mu]) continue;
        Epilogue e;
        e.beta = first ? 0.0 : 1.0;
        G.mp(ctx, u[i], dl, mu, G.A[mu], dl[mu], e, k.rr);
        first = false;
      }
      if (first) KP_CUDA(cudaMemsetAsync(k.rr, 0, size_t(nloc) * comps * 8, ctx->stream));
    });
    to_pencil(cv(&Rank::rr), mv(&Rank::rp));
    each([&](Rank& k) {
      Epilogue e;
      e.kind = EPI_ADD_G;
      e.beta = 1.0;
      e.X = k.up;
      e.g = G.g;
      e.t = t;
      G.mp(ctx, k.up, dp, ds - 1, G.A[ds - 1], dp[ds - 1], e, k.rp);
    });
    to_slab(cv(&Rank::rp), r);
  }

  void pre(const double* u, double* w, bool two, double t) {
    const long long half = S == 2 ? nloc / 2 : 0;
    if (!cplx && half > 0) {
      launch_pdl(ctx, lawson_pre_pair_kernel, dim3(grid_ew(ctx, half)), dim3(256), 0, G.g, t,
                 half, G.tau, two, u, w);
    } else if (cplx) {
      launch_pdl(ctx, lawson_pre_kernel<true>, dim3(grid_ew(ctx, nloc)), dim3(256), 0, G.g, t,
                 nloc, half, G.tau, two, reinterpret_cast<const double2*>(u),
                 reinterpret_cast<double2*>(w));
    } else {
      launch_pdl(ctx, lawson_pre_kernel<false>, dim3(grid_ew(ctx, nloc)), dim3(256), 0, G.g, t,
                 nloc, half, G.tau, two, u, w);
    }
  }
  void post(const double* y, double* out, int* bad, const int* ctr, double t2, int* next) {
    const long long half = S == 2 ? nloc / 2 : 0;
    if (!cplx && half > 0) {
      launch_pdl(ctx, lawson2b_post_pair_kernel, dim3(grid_ew(ctx, half)), dim3(256), 0, G.g, t2,
                 half, G.tau, y, out, bad, ctr, next);
    } else if (cplx) {
      launch_pdl(ctx, lawson2b_post_kernel<true>, dim3(grid_ew(ctx, nloc)), dim3(256), 0, G.g,
                 t2, nloc, half, G.tau, reinterpret_cast<const double2*>(y),
                 reinterpret_cast<double2*>(out), bad, ctr, next);
    } else {
      launch_pdl(ctx, lawson2b_post_kernel<false>, dim3(grid_ew(ctx, nloc)), dim3(256), 0, G.g,
                 t2, nloc, half, G.tau, y, out, bad, ctr, next);
    }
  }
  void gdiff(const double* s, const double* u, double* dd, double t) {
    gdiff_dev(ctx, G.g, t, G.tau, s, u, nloc, S == 2 ? nloc / 2 : 0, cplx, dd);
  }
  void fma(double b, const double* y, const double* x, double* z) {
    launch_fma(ctx, size_t(nloc) * comps, b, y, x, z);
  }

  // ---- fused exchange (mode_d 3): the GEMM epilogues store every entry
  // straight into its owner's buffer (peer memory over NVLink), so the
  // re-partition overlaps the mode product tile by tile; plain re-partitions
  // are a scatter kernel; a one-double NCCL all-reduce fences each exchange
  // (emulated ranks: stream order).  Receive buffers alternate by step parity,
  // so one fence per exchange also orders the next step's stores after this
  // step's reads.
  Epilogue scat(const Rank& k, int dir, double* const* peers) const {
    Epilogue e;
    e.sc_dir = dir;
    e.sc_P = P;
    e.sc_rank = k.r;
    e.sc_A = unsigned(A);
    e.sc_B = unsigned(B);
    e.sc_C = unsigned(C);
    e.sc_peers = peers;
    return e;
  }
  void fence() { X.fence(ctx, scratch); }
  // modes 0..ds-2 of a Tucker, the last of them scattering into the ranks'
  // pencil buffers pen[t][par]
  void tucker_to_pencil(const FactorSet& fs, int t, int par, const std::vector<const double*>& in) {
    each([&](Rank& k) {
      const double* cur = in[&k - R.data()];
      for (int mu = 0; mu < ds - 1; ++mu) {
        const bool last = (mu == ds - 2);
        double* dst = (mu & 1) ? k.t1 : k.t0;
        Epilogue e = last ? scat(k, 1, k.ppen[t][par]) : Epilogue{};
        e.alpha = (mu == 0) ? fs.pref : 1.0;
        G.mp(ctx, cur, dl, mu, fs.f[mu], dl[mu], e, dst);
        cur = dst;
      }
    });
    fence();
  }
  void step_fused(const std::vector<const double*>& u, int slot) {
    const double tau = G.tau, t = 0.0;
    const int par = slot, nxt = 1 - slot;
    auto fin_of = [&](Rank& k) {
      Epilogue f;
      f.bad_step = k.cnt + 1;
      f.step_ctr = k.cnt + (slot ? 2 : 0);
      f.step_next = k.cnt + (slot ? 0 : 2);
      return f;
    };
    auto last_mode = [&](const FactorSet& fs, int tk, Rank& k, Epilogue e, double* out) {
      e.alpha = fs.fold * (ds == 1 ? fs.pref : 1.0);
      G.mp(ctx, k.pen[tk][par], dp, ds - 1, fs.f[ds - 1], dp[ds - 1], e, out);
    };
    auto with_scat = [&](Epilogue e, Rank& k) {
      const Epilogue sc = scat(k, 2, k.pS[nxt]);
      e.sc_dir = sc.sc_dir;
      e.sc_P = sc.sc_P;
      e.sc_rank = sc.sc_rank;
      e.sc_A = sc.sc_A;
      e.sc_B = sc.sc_B;
      e.sc_C = sc.sc_C;
      e.sc_peers = sc.sc_peers;
      return e;
    };
    switch (method) {
      case KP_EXP_EULER:
      case KP_ETD2RK: {
        kronsum_g(u, mv(&Rank::rr), t);
        each([&](Rank& k) {
          scatter_copy(ctx, u[&k - R.data()], nloc, comps, scat(k, 1, k.pupb[par]));
        });
        tucker_to_pencil(G.f1, 0, par, cv(&Rank::rr));  // (fences the u scatter too)
        if (method == KP_EXP_EULER) {
          each([&](Rank& k) {
            Epilogue f = fin_of(k);
            f.kind = EPI_FMA_X;
            f.X = k.upb[par];
            f.gamma = tau;
            last_mode(G.f1, 0, k, with_scat(f, k), k.out);
          });
          fence();
          return;
        }
        const bool paired = S == 2;
        each([&](Rank& k) {
          Epilogue e;
          e.X = k.upb[par];
          e.gamma = tau;
          e.g = G.g;
          e.t = t;
          e.t2 = t + tau;
          if (paired) {
            e.kind = EPI_FMA_X;
          } else {
            e.kind = EPI_STAGE_D;
            e.D = k.dq;
          }
          last_mode(G.f1, 0, k, e, k.sp);
          if (paired) gdiff(k.sp, k.upb[par], k.dq, t);
          scatter_copy(ctx, k.dq, nloc, comps, scat(k, 2, k.pddb[par]));
        });
        fence();
        std::vector<const double*> dd;
        for (auto& k : R) dd.push_back(k.ddb[par]);
        tucker_to_pencil(G.f2, 1, par, dd);
        each([&](Rank& k) {
          Epilogue f = fin_of(k);
          f.kind = EPI_FMA_X;
          f.X = k.sp;
          f.gamma = tau;
          last_mode(G.f2, 1, k, with_scat(f, k), k.out);
        });
        fence();
        return;
      }
      case KP_LAWSON_EULER:
      case KP_LAWSON2B: {
        const bool two = method == KP_LAWSON2B;
        each([&](Rank& k) { pre(u[&k - R.data()], k.w, two, t); });
        if (!two) {
          tucker_to_pencil(G.f1, 0, par, cv(&Rank::w));
          each([&](Rank& k) { last_mode(G.f1, 0, k, with_scat(fin_of(k), k), k.out); });
          fence();
          return;
        }
        tucker_to_pencil(G.f1, 0, par, cv(&Rank::w));
        tucker_to_pencil(G.f1, 1, par, cv(&Rank::w, nloc * comps));
        each([&](Rank& k) {
          last_mode(G.f1, 0, k, Epilogue{}, k.sp);
          last_mode(G.f1, 1, k, Epilogue{}, k.sp + nloc * comps);
          post(k.sp, k.out, k.cnt + 1, k.cnt + (slot ? 2 : 0), t + tau, k.cnt + (slot ? 0 : 2));
          scatter_copy(ctx, k.out, nloc, comps, scat(k, 2, k.pS[nxt]));
        });
        fence();
        return;
      }
      default:
        throw invalid_argument("sharded integrate: unsupported method");
    }
  }

  // one step: u[i] -> o[i] (slab).  slot = counter slot of this step.
  void step(const std::vector<const double*>& u, const std::vector<double*>& o, int slot) {
    if (mode_d == 3) {  // the output lands in the ranks' S[1 - slot] (o is S[1 - slot])
      step_fused(u, slot);
      return;
    }
    const double tau = G.tau, t = 0.0;
    auto fin_of = [&](Rank& k) {
      Epilogue f;
      f.bad_step = k.cnt + 1;
      f.step_ctr = k.cnt + (slot ? 2 : 0);
      f.step_next = k.cnt + (slot ? 0 : 2);
      return f;
    };
    const bool B_ = (mode_d == 2);
    switch (method) {
      case KP_EXP_EULER:
      case KP_ETD2RK: {
        // u on the pencil: the fused last-mode epilogues read it (A), the
        // dense Kronecker sum's last term needs it (both)
        if (!B_ || !G.banded) {
          if (P == 1)
            each([&](Rank& k) { k.up = const_cast<double*>(u[&k - R.data()]); });
          else
            to_pencil(u, mv(&Rank::up));
        }
        kronsum_g(u, mv(&Rank::rr), t);
        if (B_) {
          tucker_B(G.f1, cv(&Rank::rr), mv(&Rank::y));
          if (method == KP_EXP_EULER) {
            each([&](Rank& k) {
              const long long i = &k - R.data();
              fma(tau, k.y, u[i], o[i]);
              finite_flag(ctx, size_t(nloc) * comps, o[i], k.cnt + 1, k.cnt + (slot ? 2 : 0));
              tick(k, slot);
            });
            return;
          }
          each([&](Rank& k) {
            const long long i = &k - R.data();
            fma(tau, k.y, u[i], k.sp);  // stage
            gdiff(k.sp, u[i], k.dd, t);
          });
          tucker_B(G.f2, cv(&Rank::dd), mv(&Rank::y));
          each([&](Rank& k) {
            const long long i = &k - R.data();
            fma(tau, k.y, k.sp, o[i]);
            finite_flag(ctx, size_t(nloc) * comps, o[i], k.cnt + 1, k.cnt + (slot ? 2 : 0));
            tick(k, slot);
          });
          return;
        }
        if (method == KP_EXP_EULER) {
          tucker_A(G.f1, cv(&Rank::rr), outs(o), [&](Rank& k) {
            Epilogue f = fin_of(k);
            f.kind = EPI_FMA_X;
            f.X = k.up;
            f.gamma = tau;
            return f;
          });
          back(o);
          return;
        }
        const bool paired = S == 2;  // the coupled g: its own pass (as on one GPU)
        tucker_A(G.f1, cv(&Rank::rr), mv(&Rank::sp), [&](Rank& k) {
          Epilogue e;
          e.X = k.up;
          e.gamma = tau;
          e.g = G.g;
          e.t = t;
          e.t2 = t + tau;
          if (paired) {
            e.kind = EPI_FMA_X;
          } else {
            e.kind = EPI_STAGE_D;
            e.D = k.dq;
          }
          return e;
        });
        if (paired) each([&](Rank& k) { gdiff(k.sp, k.up, k.dq, t); });
        if (P > 1) to_slab(cv(&Rank::dq), mv(&Rank::dd));
        tucker_A(G.f2, P > 1 ? cv(&Rank::dd) : cv(&Rank::dq), outs(o), [&](Rank& k) {
          Epilogue f = fin_of(k);
          f.kind = EPI_FMA_X;
          f.X = k.sp;
          f.gamma = tau;
          return f;
        });
        back(o);
        return;
      }
      case KP_LAWSON_EULER:
      case KP_LAWSON2B: {
        const bool two = method == KP_LAWSON2B;
        each([&](Rank& k) { pre(u[&k - R.data()], k.w, two, t); });
        if (!two) {
          if (B_) {
            tucker_B(G.f1, cv(&Rank::w), o);
            each([&](Rank& k) {
              finite_flag(ctx, size_t(nloc) * comps, o[&k - R.data()], k.cnt + 1,
                          k.cnt + (slot ? 2 : 0));
              tick(k, slot);
            });
            return;
          }
          tucker_A(G.f1, cv(&Rank::w), outs(o), [&](Rank& k) { return fin_of(k); });
          back(o);
          return;
        }
        // [stage; y1] in one buffer (the post kernel's layout)
        if (B_) {
          tucker_B(G.f1, cv(&Rank::w), mv(&Rank::sp));
          tucker_B(G.f1, cv(&Rank::w, nloc * comps), mv(&Rank::sp, nloc * comps));
          each([&](Rank& k) {
            post(k.sp, o[&k - R.data()], k.cnt + 1, k.cnt + (slot ? 2 : 0), t + tau,
                 k.cnt + (slot ? 0 : 2));
          });
          return;
        }
        tucker_A(G.f1, cv(&Rank::w), mv(&Rank::sp), [&](Rank&) { return Epilogue{}; });
        tucker_A(G.f1, cv(&Rank::w, nloc * comps), mv(&Rank::sp, nloc * comps),
                 [&](Rank&) { return Epilogue{}; });
        {
          const auto ov = outs(o);
          each([&](Rank& k) {
            post(k.sp, ov[&k - R.data()], k.cnt + 1, k.cnt + (slot ? 2 : 0), t + tau,
                 k.cnt + (slot ? 0 : 2));
          });
        }
        back(o);
        return;
      }
      default:
        throw invalid_argument("sharded integrate: unsupported method");
    }
  }
  // where the last (pencil) result of a step goes: straight into o at P = 1
  std::vector<double*> outs(const std::vector<double*>& o) {
    return P == 1 ? o : mv(&Rank::out);
  }
  void back(const std::vector<double*>& o) {
    if (P > 1) to_slab(cv(&Rank::out), o);
  }
  void tick(Rank& k, int slot) {
    launch_pdl(ctx, tick_kernel, dim3(1), dim3(1), 0, (const int*)(k.cnt + (slot ? 2 : 0)),
               k.cnt + (slot ? 0 : 2));
  }

  // n_steps steps on the ranks' u (in/out); returns the loop's device time
  // (this process; the caller takes the max over ranks)
  double run(long n_steps, bool use_graph) {
    std::vector<const double*> cu[2] = {cv(&Rank::u), cv(&Rank::ub)};
    std::vector<double*> mu_[2] = {mv(&Rank::u), mv(&Rank::ub)};
    if (mode_d == 3) {  // the state lives in the peer-mapped S buffers
      each([&](Rank& k) {
        KP_CUDA(cudaMemcpyAsync(k.S[0], k.u, size_t(nloc) * comps * 8, cudaMemcpyDeviceToDevice,
                                ctx->stream));
      });
      fence();
      for (int a = 0; a < 2; ++a) {
        cu[a].clear();
        mu_[a].clear();
        for (auto& k : R) {
          cu[a].push_back(k.S[a]);
          mu_[a].push_back(k.S[a]);
        }
      }
    }
    cudaEvent_t ev[4];
    for (auto& e : ev) KP_CUDA(cudaEventCreate(&e));
    long n = 0;
    KP_CUDA(cudaEventRecord(ev[0], ctx->stream));
    step(cu[0], mu_[1], 0);
    ++n;
    KP_CUDA(cudaEventRecord(ev[1], ctx->stream));
    cudaGraphExec_t exec = nullptr;
    unsigned long long per = 0;
    if (use_graph && n_steps - n >= 4) {
      // two steps (ping-pong) as one graph; if capturing the exchanges fails
      // (a transport that cannot be captured), the loop runs eagerly
      cudaGraph_t graph = nullptr;
      const unsigned long long l0 = ctx->launches;
      try {
        KP_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        step(cu[1], mu_[0], 1);
        step(cu[0], mu_[1], 0);
        KP_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
        KP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        per = ctx->launches - l0;
      } catch (const std::exception&) {
        cudaStreamCaptureStatus st;
        if (cudaStreamIsCapturing(ctx->stream, &st) == cudaSuccess &&
            st != cudaStreamCaptureStatusNone) {
          cudaGraph_t g2 = nullptr;
          cudaStreamEndCapture(ctx->stream, &g2);
          if (g2) cudaGraphDestroy(g2);
        }
        cudaGetLastError();
        exec = nullptr;
      }
      ctx->launches = l0;
      if (graph) cudaGraphDestroy(graph);
    }
    KP_CUDA(cudaEventRecord(ev[2], ctx->stream));
    if (exec)
      while (n_steps - n >= 2) {
        KP_CUDA(cudaGraphLaunch(exec, ctx->stream));
        ctx->launches += per;
        n += 2;
      }
    while (n < n_steps) {
      step(cu[n & 1], mu_[(n + 1) & 1], int(n & 1));
      ++n;
    }
    KP_CUDA(cudaEventRecord(ev[3], ctx->stream));
    if (exec) cudaGraphExecDestroy(exec);
    if (mode_d == 3)
      each([&](Rank& k) {
        KP_CUDA(cudaMemcpyAsync(k.u, k.S[n_steps & 1], size_t(nloc) * comps * 8,
                                cudaMemcpyDeviceToDevice, ctx->stream));
      });
    else if (n_steps & 1)
      each([&](Rank& k) {
        KP_CUDA(cudaMemcpyAsync(k.u, k.ub, size_t(nloc) * comps * 8, cudaMemcpyDeviceToDevice,
                                ctx->stream));
      });
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
    float ms1 = 0.f, ms2 = 0.f;
    KP_CUDA(cudaEventElapsedTime(&ms1, ev[0], ev[1]));
    KP_CUDA(cudaEventElapsedTime(&ms2, ev[2], ev[3]));
    for (auto& e : ev) cudaEventDestroy(e);
    return double(ms1 + ms2) * 1e-3;
  }
  void reset_counters() {
    each([&](Rank& k) {
      const int init[4] = {0, INT_MAX, 0, 0};
      KP_CUDA(cudaMemcpyAsync(k.cnt, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
    });
  }
  // first non-finite step over all ranks (0 = none)
  long first_bad() {
    double worst = double(INT_MAX);
    each([&](Rank& k) {
      int hb[2];
      KP_CUDA(cudaMemcpyAsync(hb, k.cnt, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
      KP_CUDA(cudaStreamSynchronize(ctx->stream));
      worst = std::min(worst, double(hb[1]));
    });
    if (X.comm && P > 1) worst = -X.max_over_ranks(ctx, -worst, scratch);
    return worst >= double(INT_MAX) ? 0 : long(worst);
  }
  // mode_d = 0: one step of each kind on scratch copies of the state, the
  // faster (device time, max over ranks) is used for the run
  void choose_mode_d(int requested) {
    if (requested == 3 && !setup_fused())
      throw invalid_argument("sharded integrate: the fused exchange needs peer-mappable "
                             "buffers and banded factors");
    if (requested == 1 || requested == 2 || requested == 3 || P == 1) {
      mode_d = (P == 1 && requested != 3) ? 1 : requested;
      if (requested == 0) mode_d = 1;
      return;
    }
    double best = 1e300;
    int pick = 1;
    std::vector<int> cand = {1, 2};
    if (setup_fused()) cand.push_back(3);
    for (int md : cand) {
      mode_d = md;
      if (md == 2)
        each([&](Rank& k) {
          if (!k.part) k.part = alloc(A * B * C * S);
        });
      for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms up (workspace, kernels)
        cudaEvent_t e0, e1;
        KP_CUDA(cudaEventCreate(&e0));
        KP_CUDA(cudaEventCreate(&e1));
        // the trial writes a scratch copy (out -> y buffer), u is untouched
        KP_CUDA(cudaEventRecord(e0, ctx->stream));
        step(cv(&Rank::u), mv(&Rank::tr), 0);
        KP_CUDA(cudaEventRecord(e1, ctx->stream));
        KP_CUDA(cudaStreamSynchronize(ctx->stream));
        float ms = 0.f;
        KP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const double sec = X.max_over_ranks(ctx, double(ms) * 1e-3, scratch);
        if (rep == 1 && sec < best) {
          best = sec;
          pick = md;
        }
      }
    }
    mode_d = pick;
    reset_counters();
  }
};

}  // namespace kp

// ============================================================== C ABI
namespace kp {
namespace {

std::vector<int> dims_of(const int* dims, int d, const char* who) {
  if (d <= 0 || !dims) throw invalid_argument(std::string(who) + ": Tensor: empty dims");
  std::vector<int> v(dims, dims + d);
  for (int x : v)
    if (x <= 0) throw invalid_argument(std::string(who) + ": Tensor: nonpositive dim");
  return v;
}

// RAII: run on a capturable stream (the context's own one when the caller's
// stream is the legacy default stream), ordered after the caller's work.
struct StreamScope {
  kp_ctx* ctx;
  cudaStream_t saved;
  explicit StreamScope(kp_ctx* c) : ctx(c), saved(c->stream) {
    if (saved == nullptr) {
      KP_CUDA(cudaStreamSynchronize(nullptr));
      ctx->stream = ctx->own_stream;
    }
  }
  ~StreamScope() {
    if (saved == nullptr) {
      cudaStreamSynchronize(ctx->own_stream);
      ctx->stream = saved;
    }
  }
};

void build_split(kp_ctx* ctx, bool cplx, const double* const* as, const int* dims, int d,
                 double tau, int ell, int q, double* const* factors, double* prefactor) {
  const auto dv = dims_of(dims, d, "build_split_phi");
  if (ell < 0) throw invalid_argument("build_split_phi: negative ell");
  const int comps = cplx ? 2 : 1;
  for (int mu = 0; mu < d; ++mu) {
    int same = -1;
    for (int m2 = 0; m2 < mu; ++m2)
      if (as[m2] == as[mu] && dv[m2] == dv[mu]) same = m2;
    const long long nn = (long long)dv[mu] * dv[mu] * comps;
    if (same >= 0) {
      KP_CUDA(cudaMemcpyAsync(factors[mu], factors[same], nn * sizeof(double),
                              cudaMemcpyDeviceToDevice, ctx->stream));
      continue;
    }
    double* scaled = static_cast<double*>(ctx->ws.get(47, nn * sizeof(double)));
    scale_matrix_kernel<<<grid_ew(ctx, nn), 256, 0, ctx->stream>>>(as[mu], nn, tau, scaled);
    ctx->launches++;
    if (ell == 0) {
      cplx ? expm_batch_c128(ctx, scaled, dv[mu], 1, factors[mu])
           : expm_batch(ctx, scaled, dv[mu], 1, factors[mu]);
    } else {
      double* tab = static_cast<double*>(ctx->ws.get(48, nn * (ell + 1) * sizeof(double)));
      cplx ? phiquad_dev_c128(ctx, scaled, dv[mu], ell, q, -1, tab)
           : phiquad_dev(ctx, scaled, dv[mu], ell, q, -1, tab);
      KP_CUDA(cudaMemcpyAsync(factors[mu], tab + nn * ell, nn * sizeof(double),
                              cudaMemcpyDeviceToDevice, ctx->stream));
    }
  }
  double f = 1.0;
  for (int i = 2; i <= ell; ++i) f *= i;
  *prefactor = std::pow(f, double(d - 1));
}

FactorSet given_factors(Integrator& it, const double* const* f, double pref) {
  FactorSet fs;
  fs.f.assign(f, f + it.d);
  fs.active.assign(it.d, 1);
  fs.pref = pref;
  int nact = it.d;
  for (int mu = 0; mu < it.d; ++mu) {
    double c = 0.0;
    if (nact > 1 && it.scalar_identity(fs.f[mu], it.dims[mu], &c)) {
      fs.active[mu] = 0;
      fs.fold *= c;
      --nact;
    }
  }
  return fs;
}

}  // namespace
}  // namespace kp

using namespace kp;

namespace {
template <typename F>
int guard_c(F&& f, long* step_out = nullptr) {
  try {
    f();
    return KP_OK;
  } catch (const kp::divergence_error& e) {
    kp_set_last_error(e.what());
    if (step_out) *step_out = e.step;
    return KP_EDIVERGE;
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

void ctx_ok(kp_ctx* ctx) {
  if (!ctx) throw invalid_argument("kronphi_b200: null context");
  KP_CUDA(cudaSetDevice(ctx->device));
}

int integrate_impl(kp_ctx* ctx, bool cplx, int method, double* u, const int* dims, int d,
                   const double* const* as, const kp_gfun* g, double t0, double t_final,
                   long n_steps, int q, long* diverged_step, double* loop_seconds,
                   int sample_every = 0, kp_sample_fn sample_fn = nullptr,
                   void* sample_user = nullptr) {
  if (diverged_step) *diverged_step = 0;
  return guard_c(
      [&] {
        ctx_ok(ctx);
        const auto dv = dims_of(dims, d, "integrate");
        if (n_steps <= 0) throw invalid_argument("integrate: n_steps must be positive");
        if (!(t_final > t0)) throw invalid_argument("integrate: empty time interval");
        if (!as || !g) throw invalid_argument("integrate: null factors or g");
        StreamScope scope(ctx);
        const double tau = (t_final - t0) / double(n_steps);
        Integrator it(ctx, method, cplx, dv, as, *g, tau);
        it.setup(q);
        static const bool no_graph = getenv("KP_NO_GRAPH") != nullptr;  // debugging aid
        if (sample_every < 0) throw invalid_argument("integrate: negative sample_every");
        const double sec = it.run(u, t0, n_steps, !no_graph, sample_every, sample_fn, sample_user);
        if (loop_seconds) *loop_seconds = sec;
        if (it.diverged_at) {  // DivergenceError(n+1, t+tau), inc/integrators.hpp:86-97,364
          const long k = it.diverged_at;
          // t + tau with t = t0 + (k-1) tau, as the reference computes it
          const double tk = (t0 + double(k - 1) * tau) + tau;
          throw divergence_error("state became non-finite at step " + std::to_string(k) +
                                     " (t = " + std::to_string(tk) + ")",
                                 k);
        }
      },
      diverged_step);
}

int host_integrate_impl(kp_ctx* ctx, bool cplx, int method, const double* u0, const int* dims,
                        int d, const double* const* as, const kp_gfun* g, double t0,
                        double t_final, long n_steps, int q, double* u_final, long* diverged_step,
                        double* loop_seconds) {
  if (diverged_step) *diverged_step = 0;
  double* du = nullptr;
  std::vector<double*> da;
  int rc = guard_c([&] {
    ctx_ok(ctx);
    const auto dv = dims_of(dims, d, "integrate");
    const int comps = cplx ? 2 : 1;
    size_t n = comps;
    for (int x : dv) n *= size_t(x);
    KP_CUDA(cudaMalloc(&du, n * sizeof(double)));
    // uploads on the context's stream + a sync: a plain cudaMemcpy from
    // pageable memory may return before its DMA lands, and the integration
    // runs on the context's NON-blocking stream (it then read stale memory
    // now and then -- a second integrate() in one process saw the previous
    // run's state)
    KP_CUDA(cudaMemcpyAsync(du, u0, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    // equal host factors are uploaded once (the device build dedupes by pointer)
    std::vector<const double*> dptr(d);
    for (int mu = 0; mu < d; ++mu) {
      const size_t nn = size_t(dv[mu]) * dv[mu] * comps;
      int same = -1;
      for (int m2 = 0; m2 < mu; ++m2)
        if (dv[m2] == dv[mu] &&
            (as[m2] == as[mu] || std::memcmp(as[m2], as[mu], nn * sizeof(double)) == 0))
          same = m2;
      if (same >= 0) {
        dptr[mu] = dptr[same];
        continue;
      }
      double* p = nullptr;
      KP_CUDA(cudaMalloc(&p, nn * sizeof(double)));
      da.push_back(p);
      KP_CUDA(cudaMemcpyAsync(p, as[mu], nn * sizeof(double), cudaMemcpyHostToDevice,
                              ctx->stream));
      dptr[mu] = p;
    }
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
    int r2 = integrate_impl(ctx, cplx, method, du, dims, d, dptr.data(), g, t0, t_final, n_steps,
                            q, diverged_step, loop_seconds);
    if (r2 == KP_EDIVERGE) throw divergence_error(kp_last_error(), diverged_step ? *diverged_step : 0);
    if (r2 != KP_OK) {
      const std::string m = kp_last_error();
      if (r2 == KP_EINVAL) throw invalid_argument(m);
      if (r2 == KP_ECUDA) throw cuda_error(m);
      throw runtime_error(m);
    }
    KP_CUDA(cudaMemcpyAsync(u_final, du, n * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
  }, diverged_step);
  if (du) cudaFree(du);
  for (double* p : da) cudaFree(p);
  return rc;
}

int step_impl(kp_ctx* ctx, bool cplx, int method, const double* u, const int* dims, int d,
              double t, double tau, const double* const* as, const double* const* f1,
              double pref1, const double* const* f2, double pref2, const kp_gfun* g,
              double* out) {
  return guard_c([&] {
    ctx_ok(ctx);
    const auto dv = dims_of(dims, d, "step");
    if (!g || !f1) throw invalid_argument("step: null factors or g");
    if (out == u) throw invalid_argument("step: out must not alias u");
    std::vector<const double*> zeros;
    if (!as) {  // Lawson methods need no K
      zeros.assign(d, f1[0]);
      as = zeros.data();
    }
    Integrator it(ctx, method, cplx, dv, as, *g, tau);
    if (method == KP_ROSENBROCK_EULER) {
      // rosenbrock_euler_step(u, t, tau, k, g, jac_factors, rule): f1 = J_mu;
      // phi_1(tau J_mu) per call, identical factors share one build (:176-186)
      it.given_jacobians = true;
      it.fj.f.assign(d, nullptr);
      it.fj.active.assign(d, 1);
      for (int mu = 0; mu < d; ++mu) {
        int same = -1;
        for (int m2 = 0; m2 < mu; ++m2)
          if (f1[m2] == f1[mu] && dv[m2] == dv[mu]) same = m2;
        if (same >= 0) {
          it.fj.f[mu] = it.fj.f[same];
          continue;
        }
        const long long nn = (long long)dv[mu] * dv[mu] * (cplx ? 2 : 1);
        double* scaled = it.alloc(nn);
        scale_matrix_kernel<<<grid_ew(ctx, nn), 256, 0, ctx->stream>>>(f1[mu], nn, tau, scaled);
        ctx->launches++;
        double* tab = it.alloc(2 * nn);
        cplx ? phiquad_dev_c128(ctx, scaled, dv[mu], 1, 12, -1, tab)
             : phiquad_dev(ctx, scaled, dv[mu], 1, 12, -1, tab);
        it.fj.f[mu] = tab + nn;
      }
    } else {
      it.f1 = given_factors(it, f1, pref1);
      if (f2) it.f2 = given_factors(it, f2, pref2);
    }
    it.step(u, out, t, nullptr, nullptr);
  });
}

}  // namespace

extern "C" {

int kp_gll_rule(int q, double* nodes, double* weights) {
  return guard_c([&] { gll_rule_host(q, nodes, weights); });
}

int kp_solve_f64(kp_ctx* ctx, const double* a, int n, const double* b, int nrhs, double* x) {
  return guard_c([&] {
    ctx_ok(ctx);
    if (n <= 0 || nrhs < 0) throw invalid_argument("solve: size mismatch");
    if (!a || !b || !x) throw invalid_argument("solve: null pointer");
    if (nrhs > 0) solve_dev(ctx, a, n, b, nrhs, x);
  });
}
int kp_expm_f64(kp_ctx* ctx, const double* x, int n, double* out) {
  return guard_c([&] {
    ctx_ok(ctx);
    if (n <= 0) throw invalid_argument("expm: matrix not square");
    expm_batch(ctx, x, n, 1, out);
  });
}
int kp_expm_c128(kp_ctx* ctx, const double* x, int n, double* out) {
  return guard_c([&] {
    ctx_ok(ctx);
    if (n <= 0) throw invalid_argument("expm: matrix not square");
    expm_batch_c128(ctx, x, n, 1, out);
  });
}
int kp_phiquad_f64(kp_ctx* ctx, const double* x, int n, int ell_max, int q, int forced,
                   double* phis, int* s) {
  return guard_c([&] {
    ctx_ok(ctx);
    const int r = phiquad_dev(ctx, x, n, ell_max, q, forced, phis);
    if (s) *s = r;
  });
}
int kp_phiquad_c128(kp_ctx* ctx, const double* x, int n, int ell_max, int q, int forced,
                    double* phis, int* s) {
  return guard_c([&] {
    ctx_ok(ctx);
    const int r = phiquad_dev_c128(ctx, x, n, ell_max, q, forced, phis);
    if (s) *s = r;
  });
}
int kp_build_split_phi_f64(kp_ctx* ctx, const double* const* as, const int* dims, int d,
                           double tau, int ell, int q, double* const* factors, double* pref) {
  return guard_c([&] {
    ctx_ok(ctx);
    build_split(ctx, false, as, dims, d, tau, ell, q, factors, pref);
  });
}
int kp_build_split_phi_c128(kp_ctx* ctx, const double* const* as, const int* dims, int d,
                            double tau, int ell, int q, double* const* factors, double* pref) {
  return guard_c([&] {
    ctx_ok(ctx);
    build_split(ctx, true, as, dims, d, tau, ell, q, factors, pref);
  });
}
int kp_step_f64(kp_ctx* ctx, int method, const double* u, const int* dims, int d, double t,
                double tau, const double* const* as, const double* const* f1, double pref1,
                const double* const* f2, double pref2, const kp_gfun* g, double* out) {
  return step_impl(ctx, false, method, u, dims, d, t, tau, as, f1, pref1, f2, pref2, g, out);
}
int kp_step_c128(kp_ctx* ctx, int method, const double* u, const int* dims, int d, double t,
                 double tau, const double* const* as, const double* const* f1, double pref1,
                 const double* const* f2, double pref2, const kp_gfun* g, double* out) {
  return step_impl(ctx, true, method, u, dims, d, t, tau, as, f1, pref1, f2, pref2, g, out);
}
int kp_integrate_f64(kp_ctx* ctx, int method, double* u, const int* dims, int d,
                     const double* const* as, const kp_gfun* g, double t0, double t_final,
                     long n_steps, int q, long* diverged_step, double* loop_seconds) {
  return integrate_impl(ctx, false, method, u, dims, d, as, g, t0, t_final, n_steps, q,
                        diverged_step, loop_seconds);
}
int kp_integrate_c128(kp_ctx* ctx, int method, double* u, const int* dims, int d,
                      const double* const* as, const kp_gfun* g, double t0, double t_final,
                      long n_steps, int q, long* diverged_step, double* loop_seconds) {
  return integrate_impl(ctx, true, method, u, dims, d, as, g, t0, t_final, n_steps, q,
                        diverged_step, loop_seconds);
}
}  // extern "C"

namespace {
int sharded_impl(kp_ctx* ctx, kp_comm* comm, int P_local, bool cplx, int method,
                 double* const* u, const int* dims, int d, const double* const* as,
                 const kp_gfun* g, double t0, double t_final, long n_steps, int q, int mode_d,
                 int* mode_used, long* diverged_step, double* loop_seconds) {
  if (diverged_step) *diverged_step = 0;
  return guard_c(
      [&] {
        ctx_ok(ctx);
        auto dl = dims_of(dims, d, "integrate_sharded");
        if (n_steps <= 0) throw invalid_argument("integrate: n_steps must be positive");
        if (!(t_final > t0)) throw invalid_argument("integrate: empty time interval");
        if (!as || !g || !u) throw invalid_argument("integrate_sharded: null argument");
        if (mode_d < 0 || mode_d > 3) throw invalid_argument("integrate_sharded: mode_d 0..3");
        StreamScope scope(ctx);
        ShardExchange X;
        if (comm) {
          X.comm = comm;
          X.P = comm_size(comm);
          X.ranks = {comm_rank(comm)};
        } else {
          if (P_local < 1) throw invalid_argument("integrate_sharded: P must be >= 1");
          X.P = P_local;
          for (int r = 0; r < P_local; ++r) X.ranks.push_back(r);
        }
        const int S = (g->kind == KP_G_BRUSSELATOR) ? 2 : 1;
        const int ds = d - (S == 2 ? 1 : 0);
        if (ds < 2) throw invalid_argument("sharded integrate: needs >= 2 spatial modes");
        std::vector<int> gd = dl;
        gd[ds - 1] *= X.P;
        const double tau = (t_final - t0) / double(n_steps);
        kp_gfun gg = *g;
        ShardedIntegrator it(ctx, X, method, cplx, gd, as, gg, tau);
        std::vector<double*> us(u, u + X.nlocal());
        it.setup(q, mode_d == 1 ? 1 : 2, us);
        it.choose_mode_d(mode_d);
        if (mode_used) *mode_used = it.mode_d;
        static const bool no_graph = getenv("KP_NO_GRAPH") != nullptr;
        const double sec = it.run(n_steps, !no_graph);
        if (loop_seconds) *loop_seconds = it.X.max_over_ranks(ctx, sec, it.scratch);
        const long k = it.first_bad();
        if (k) {
          const double tk = (t0 + double(k - 1) * tau) + tau;
          throw divergence_error("state became non-finite at step " + std::to_string(k) +
                                     " (t = " + std::to_string(tk) + ")",
                                 k);
        }
      },
      diverged_step);
}
}  // namespace

extern "C" {

int kp_integrate_sharded_f64(kp_ctx* ctx, kp_comm* comm, int method, double* u_local,
                             const int* dims_local, int d, const double* const* as,
                             const kp_gfun* g, double t0, double t_final, long n_steps, int q,
                             int mode_d, int* mode_used, long* diverged_step,
                             double* loop_seconds) {
  if (!comm) {
    kp_set_last_error("integrate_sharded: null communicator");
    return KP_EINVAL;
  }
  return sharded_impl(ctx, comm, 1, false, method, &u_local, dims_local, d, as, g, t0, t_final,
                      n_steps, q, mode_d, mode_used, diverged_step, loop_seconds);
}
int kp_integrate_sharded_c128(kp_ctx* ctx, kp_comm* comm, int method, double* u_local,
                              const int* dims_local, int d, const double* const* as,
                              const kp_gfun* g, double t0, double t_final, long n_steps, int q,
                              int mode_d, int* mode_used, long* diverged_step,
                              double* loop_seconds) {
  if (!comm) {
    kp_set_last_error("integrate_sharded: null communicator");
    return KP_EINVAL;
  }
  return sharded_impl(ctx, comm, 1, true, method, &u_local, dims_local, d, as, g, t0, t_final,
                      n_steps, q, mode_d, mode_used, diverged_step, loop_seconds);
}
int kp_integrate_sharded_local_f64(kp_ctx* ctx, int P, int method, double* const* u_slabs,
                                   const int* dims_local, int d, const double* const* as,
                                   const kp_gfun* g, double t0, double t_final, long n_steps,
                                   int q, int mode_d, int* mode_used, long* diverged_step,
                                   double* loop_seconds) {
  return sharded_impl(ctx, nullptr, P, false, method, u_slabs, dims_local, d, as, g, t0, t_final,
                      n_steps, q, mode_d, mode_used, diverged_step, loop_seconds);
}
int kp_integrate_sharded_local_c128(kp_ctx* ctx, int P, int method, double* const* u_slabs,
                                    const int* dims_local, int d, const double* const* as,
                                    const kp_gfun* g, double t0, double t_final, long n_steps,
                                    int q, int mode_d, int* mode_used, long* diverged_step,
                                    double* loop_seconds) {
  return sharded_impl(ctx, nullptr, P, true, method, u_slabs, dims_local, d, as, g, t0, t_final,
                      n_steps, q, mode_d, mode_used, diverged_step, loop_seconds);
}

}  // extern "C"

namespace {
// mode-d-sharded Tucker operator (the headline op of bench.py at N > 1)
int tucker_sharded_impl(kp_ctx* ctx, kp_comm* comm, int P_local, const double* const* t,
                        const int* dims, int d, const double* const* ms, double pref, int mode_d,
                        double* const* out) {
  return guard_c([&] {
    ctx_ok(ctx);
    auto dl = dims_of(dims, d, "tucker_sharded");
    if (d < 2) throw invalid_argument("tucker_sharded: needs order >= 2");
    if (!t || !ms || !out) throw invalid_argument("tucker_sharded: null argument");
    if (mode_d < 1 || mode_d > 3) throw invalid_argument("tucker_sharded: mode_d 1, 2 or 3");
    ShardExchange X;
    X.wctx = ctx;
    if (comm) {
      X.comm = comm;
      X.P = comm_size(comm);
      X.ranks = {comm_rank(comm)};
    } else {
      if (P_local < 1 || P_local > 16) throw invalid_argument("tucker_sharded: P in 1..16");
      X.P = P_local;
      for (int r = 0; r < P_local; ++r) X.ranks.push_back(r);
    }
    const int P = X.P;
    long long A = 1;
    for (int mu = 0; mu < d - 2; ++mu) A *= dl[mu];
    const long long B = dl[d - 2], Cl = dl[d - 1], C = Cl * P;
    if (B % P) throw invalid_argument("tucker_sharded: n_(d-1) must be divisible by P");
    const long long n = A * B * Cl;
    std::vector<int> dp = dl;
    dp[d - 2] = int(B / P);
    dp[d - 1] = int(C);
    // mode_d 3 (fused): mode d-1's epilogue stores every entry straight into
    // its owner's pencil buffer (peer memory); the mappings are cached per
    // (context, communicator, buffer)
    double* const* peers = nullptr;
    std::vector<double*> pbuf;
    if (mode_d == 3) {
      for (int i = 0; i < X.nlocal(); ++i)
        pbuf.push_back(static_cast<double*>(ctx->ws.get(144 + i, size_t(n) * 8)));
      struct Key {
        kp_ctx* c;
        kp_comm* m;
        double* p;
        size_t n;
        bool operator<(const Key& o) const {
          return std::tie(c, m, p, n) < std::tie(o.c, o.m, o.p, o.n);
        }
      };
      static std::map<Key, std::pair<double**, std::shared_ptr<ShardExchange>>> cache;
      const Key key{ctx, comm, pbuf[0], size_t(n)};
      auto it = cache.find(key);
      if (it == cache.end()) {
        auto keep = std::make_shared<ShardExchange>();
        keep->P = X.P;
        keep->comm = X.comm;
        keep->ranks = X.ranks;
        double* scr = static_cast<double*>(ctx->ws.get(176, 4096));
        std::vector<double*> all;
        if (!keep->map(ctx, pbuf, all, scr))
          throw invalid_argument("tucker_sharded: peer buffers cannot be mapped");
        double** dev = nullptr;
        KP_CUDA(cudaMalloc(&dev, sizeof(double*) * all.size()));
        KP_CUDA(cudaMemcpyAsync(dev, all.data(), sizeof(double*) * all.size(),
                                cudaMemcpyHostToDevice, ctx->stream));
        it = cache.emplace(key, std::make_pair(dev, keep)).first;
      }
      peers = it->second.first;
    }
    std::vector<const double*> mid;
    for (int i = 0; i < X.nlocal(); ++i) {
      const double* cur = t[i];
      for (int mu = 0; mu < d - 1; ++mu) {
        double* dst = static_cast<double*>(ctx->ws.get(112 + 2 * i + (mu & 1), size_t(n) * 8));
        Epilogue e;
        if (mode_d == 3 && mu == d - 2) {
          e.sc_dir = 1;
          e.sc_P = P;
          e.sc_rank = X.ranks[i];
          e.sc_A = unsigned(A);
          e.sc_B = unsigned(B);
          e.sc_C = unsigned(C);
          e.sc_peers = peers;
        }
        e.alpha = (mu == 0) ? pref : 1.0;
        mode_product_f64(ctx, cur, dl, mu, ms[mu], dl[mu], e, dst);
        cur = dst;
      }
      mid.push_back(cur);
    }
    if (mode_d == 3) {
      double* scr = static_cast<double*>(ctx->ws.get(177, 64));
      X.fence(ctx, scr);
      for (int i = 0; i < X.nlocal(); ++i) {
        Epilogue e;
        mode_product_f64(ctx, pbuf[i], P > 1 ? dp : dl, d - 1, ms[d - 1], int(C), e, out[i]);
      }
      return;
    }
    if (mode_d == 1) {
      std::vector<const double*> pen = mid;
      if (P > 1) {
        std::vector<double*> pb;
        for (int i = 0; i < X.nlocal(); ++i)
          pb.push_back(static_cast<double*>(ctx->ws.get(144 + i, size_t(n) * 8)));
        X.repartition(ctx, 1, A, B, C, 1, 1, mid, pb);
        pen.assign(pb.begin(), pb.end());
      }
      for (int i = 0; i < X.nlocal(); ++i) {
        Epilogue e;
        mode_product_f64(ctx, pen[i], P > 1 ? dp : dl, d - 1, ms[d - 1], int(C), e, out[i]);
      }
      return;
    }
    std::vector<int> fd = dl;
    fd[d - 1] = int(C);
    std::vector<double*> parts;
    for (int i = 0; i < X.nlocal(); ++i) {
      double* part = static_cast<double*>(ctx->ws.get(160 + i, size_t(n) * P * 8));
      Epilogue e;
      mode_product_f64(ctx, mid[i], dl, d - 1, ms[d - 1] + (long long)X.ranks[i] * Cl * C,
                       int(C), e, part);
      parts.push_back(part);
    }
    std::vector<double*> ov(out, out + X.nlocal());
    X.reduce_scatter(ctx, A * B, C, 1, parts, ov);
  });
}
}  // namespace

extern "C" {

int kp_tucker_sharded_f64(kp_ctx* ctx, kp_comm* comm, const double* t_slab,
                          const int* dims_local, int d, const double* const* ms,
                          double prefactor, int mode_d, double* out) {
  if (!comm) {
    kp_set_last_error("tucker_sharded: null communicator");
    return KP_EINVAL;
  }
  return tucker_sharded_impl(ctx, comm, 1, &t_slab, dims_local, d, ms, prefactor, mode_d, &out);
}
int kp_tucker_sharded_local_f64(kp_ctx* ctx, int P, const double* const* t_slabs,
                                const int* dims_local, int d, const double* const* ms,
                                double prefactor, int mode_d, double* const* outs) {
  return tucker_sharded_impl(ctx, nullptr, P, t_slabs, dims_local, d, ms, prefactor, mode_d,
                             outs);
}

int kp_integrate_sampled_f64(kp_ctx* ctx, int method, double* u, const int* dims, int d,
                             const double* const* as, const kp_gfun* g, double t0,
                             double t_final, long n_steps, int q, int sample_every,
                             kp_sample_fn fn, void* user, long* diverged_step,
                             double* loop_seconds) {
  return integrate_impl(ctx, false, method, u, dims, d, as, g, t0, t_final, n_steps, q,
                        diverged_step, loop_seconds, sample_every, fn, user);
}
int kp_integrate_sampled_c128(kp_ctx* ctx, int method, double* u, const int* dims, int d,
                              const double* const* as, const kp_gfun* g, double t0,
                              double t_final, long n_steps, int q, int sample_every,
                              kp_sample_fn fn, void* user, long* diverged_step,
                              double* loop_seconds) {
  return integrate_impl(ctx, true, method, u, dims, d, as, g, t0, t_final, n_steps, q,
                        diverged_step, loop_seconds, sample_every, fn, user);
}
int kp_host_integrate_f64(kp_ctx* ctx, int method, const double* u0, const int* dims, int d,
                          const double* const* as, const kp_gfun* g, double t0, double t_final,
                          long n_steps, int q, double* u_final, long* diverged_step,
                          double* loop_seconds) {
  return host_integrate_impl(ctx, false, method, u0, dims, d, as, g, t0, t_final, n_steps, q,
                             u_final, diverged_step, loop_seconds);
}
int kp_host_integrate_c128(kp_ctx* ctx, int method, const double* u0, const int* dims, int d,
                           const double* const* as, const kp_gfun* g, double t0, double t_final,
                           long n_steps, int q, double* u_final, long* diverged_step,
                           double* loop_seconds) {
  return host_integrate_impl(ctx, true, method, u0, dims, d, as, g, t0, t_final, n_steps, q,
                             u_final, diverged_step, loop_seconds);
}

}  // extern "C"
