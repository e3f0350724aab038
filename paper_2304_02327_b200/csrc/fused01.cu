// fused01.cu -- modes 0 and 1 of a Tucker operator in ONE kernel for small
// square slices (n0 = n1 = N in {64, 128}, order >= 3).
//
// The reference applies V x_1 M_1 x_2 M_2 as two mode products
// (tucker, inc/mode_product.hpp:101-108 -> mode_product_into :61-87), each a
// full pass over the tensor.  For a slice V_q (N x N, q = the slower
// indices) both products stay inside the slice:
//     W_q = M_2 (M_1 V_q)^T^T  i.e.  W_q(i, k) = sum_c (sum_j M_1(i,j) V_q(j,c)) M_2(k,c)
// so one CTA owns a slice: V_q streams into shared memory k-slice by k-slice
// together with M_1's columns (cp.async ring), T = alpha * M_1 V_q
// overwrites V_q in shared memory, M_2's columns stream through the same
// ring, and W_q leaves through the coalesced epilogue.  The intermediate
// never touches HBM and one launch replaces two; at N = 128 the slice is
// 128 KiB of the SM's 227 KiB.
//
// Arithmetic is that of the two-launch path (gemm_dmma.cu): DMMA m8n8k4
// with every accumulator summed over k in increasing groups of four, T
// rounded to double after the alpha multiply, W through epi_one -- so the
// fused and unfused Tuckers agree bit for bit (test_fused01_bitwise).
#include <cstdlib>
#include <string>

#include "kp_epilogue.cuh"
#include "kp_launch.cuh"

namespace kp {
namespace {

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(double* s, const double* g) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int K>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K));
}

template <int N>
struct F01 {
  static constexpr int WARPS_M = (N == 128) ? 4 : 2, WARPS_N = 2;
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int WM = N / WARPS_M, WN = N / WARPS_N;  // 32 x 64 / 32 x 32 warp tiles
  static constexpr int MI = WM / 8, NI = WN / 8;
  static constexpr int LD = N + 4;  // = 4 (mod 16) doubles: fragment loads conflict-free
  static constexpr int BK = 16, STAGES = 3, KS = N / BK;
  static constexpr int F_STAGE = BK * LD;
  static constexpr size_t SMEM = (size_t(N) * LD + size_t(STAGES) * F_STAGE) * sizeof(double);
};

// smem: Ts = the slice (column-major, pitch LD), then STAGES factor slices
// (row kk of a slice = column 16 s + kk of the factor, pitch LD).
template <int N>
__global__ void __launch_bounds__(F01<N>::NT, 1)
    fused01_kernel(const double* __restrict__ V, const double* __restrict__ M1,
                   const double* __restrict__ M2, double alpha0, Epilogue e,
                   double* __restrict__ out) {
  pdl_wait();
  using C = F01<N>;
  extern __shared__ __align__(16) double smem[];
  double* Ts = smem;
  double* Fs = smem + N * C::LD;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tig = lane & 3;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const long long q = blockIdx.x;
  const double* Vq = V + q * N * N;

  // global k-slice x: x < KS -> M1 columns + V_q rows of slice x; else M2 columns
  auto issue = [&](int x) {
    const double* F = x < C::KS ? M1 : M2;
    const int s = x < C::KS ? x : x - C::KS;
    double* dst = Fs + (x % C::STAGES) * C::F_STAGE;
#pragma unroll
    for (int c = tid; c < C::BK * N / 2; c += C::NT) {
      const int kk = c / (N / 2), i = (c % (N / 2)) * 2;
      cp16(dst + kk * C::LD + i, F + i + (long long)(s * C::BK + kk) * N);
    }
    if (x < C::KS) {
#pragma unroll
      for (int c = tid; c < N * C::BK / 2; c += C::NT) {
        const int col = c / (C::BK / 2), j = s * C::BK + (c % (C::BK / 2)) * 2;
        cp16(Ts + j + col * C::LD, Vq + j + (long long)col * N);
      }
    }
  };

  double acc[C::MI][C::NI][2];
#pragma unroll
  for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < C::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    issue(s);
    cp_commit();
  }
#pragma unroll 1
  for (int gs = 0; gs < 2 * C::KS; ++gs) {
    cp_wait<C::STAGES - 2>();
    __syncthreads();
    if (gs + C::STAGES - 1 < 2 * C::KS) issue(gs + C::STAGES - 1);
    cp_commit();
    const double* F = Fs + (gs % C::STAGES) * C::F_STAGE;
    if (gs < C::KS) {
      // mode 0: T(i, c) += M1(i, j) V_q(j, c); A = M1 slice, B = V_q in Ts
#pragma unroll
      for (int kg = 0; kg < C::BK / 4; ++kg) {
        const int kl = kg * 4 + tig, kglob = gs * C::BK + kl;
        double a[C::MI], b[C::NI];
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi) a[mi] = F[kl * C::LD + wm * C::WM + mi * 8 + g];
#pragma unroll
        for (int ni = 0; ni < C::NI; ++ni) b[ni] = Ts[kglob + (wn * C::WN + ni * 8 + g) * C::LD];
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < C::NI; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
      if (gs == C::KS - 1) {
        __syncthreads();  // every read of V_q is done: T overwrites it
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < C::NI; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int m = wm * C::WM + mi * 8 + g, n = wn * C::WN + ni * 8 + 2 * tig + h;
              Ts[m + n * C::LD] = alpha0 * acc[mi][ni][h];
              acc[mi][ni][h] = 0.0;
            }
        // the next iteration's barrier orders these stores before mode 1 reads
      }
    } else {
      // mode 1: W(i, k) += T(i, c) M2(k, c); A = T in Ts, B = M2 slice
#pragma unroll
      for (int kg = 0; kg < C::BK / 4; ++kg) {
        const int kl = kg * 4 + tig, kglob = (gs - C::KS) * C::BK + kl;
        double a[C::MI], b[C::NI];
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi) a[mi] = Ts[(wm * C::WM + mi * 8 + g) + kglob * C::LD];
#pragma unroll
        for (int ni = 0; ni < C::NI; ++ni) b[ni] = F[kl * C::LD + wn * C::WN + ni * 8 + g];
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < C::NI; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
    }
  }
  cp_wait<0>();
  __syncthreads();  // mode-1 reads of Ts done: stage W there
#pragma unroll
  for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < C::NI; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = wm * C::WM + mi * 8 + g, n = wn * C::WN + ni * 8 + 2 * tig + h;
        Ts[m + n * C::LD] = acc[mi][ni][h];
      }
  __syncthreads();
  // coalesced (m, m+1) pairs, the same epilogue code as the GEMM kernels
  const long long cq = q * N * N;
  const EpiU u = epi_uniform(e);
#pragma unroll 1
  for (int e2 = tid; e2 < N * N / 2; e2 += C::NT) {
    const int ml = 2 * (e2 % (N / 2)), nl = e2 / (N / 2);
    const double2 a2 = *reinterpret_cast<const double2*>(Ts + ml + nl * C::LD);
    const long long off = cq + ml + (long long)nl * N;
    double d0 = 0.0, d1 = 0.0;
    const double r0 = epi_one(e, u, e.alpha * a2.x, out, off, 0, &d0);
    const double r1 = epi_one(e, u, e.alpha * a2.y, out, off + 1, 0, &d1);
    *reinterpret_cast<double2*>(out + off) = make_double2(r0, r1);
  }
}

// Row-split form (N = 128): CTA (q, r) owns rows [r MR, r MR + MR) of T
// and of W -- W's rows depend only on the same rows of T, so the R CTAs of
// a slice never talk.  V_q is no longer stored: its k-rows stream through
// the ring (8-byte copies, k-major so both operands' fragment loads are
// conflict-free) next to the M1 rows of the CTA's block, and only the T
// block stays resident (MR x N).  At MR = 64 a CTA needs 105 KiB, so two
// CTAs share an SM (the other one's mainloop covers each barrier) and the
// 2Q CTAs fill the 148 SMs where Q = 128 slices could not.  BK = 8: two DMMA
// k-groups per stage, k still in increasing order.
template <int N, int MR>
struct F01R {
  static constexpr int R = N / MR;
  static constexpr int WARPS_M = MR / 32, WARPS_N = 2;
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int WM = 32, WN = N / WARPS_N;
  static constexpr int MI = WM / 8, NI = WN / 8;
  static constexpr int LDT = MR + 4, LDA = MR + 4, LDB = N + 4;  // = 4 (mod 16)
  static constexpr int BK = 8, STAGES = 3, KS = N / BK;
  static constexpr int STAGE = BK * LDA + BK * LDB;
  static constexpr size_t SMEM = (size_t(N) * LDT + size_t(STAGES) * STAGE) * sizeof(double);
};

__device__ __forceinline__ void cp8(double* s, const double* g) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g));
}

template <int N, int MR>
__global__ void __launch_bounds__(F01R<N, MR>::NT, 2)
    fused01r_kernel(const double* __restrict__ V, const double* __restrict__ M1,
                    const double* __restrict__ M2, double alpha0, Epilogue e,
                    double* __restrict__ out) {
  pdl_wait();
  using C = F01R<N, MR>;
  extern __shared__ __align__(16) double smem[];
  double* Th = smem;                 // T block: T(i, c) at i + c * LDT, i < MR
  double* Ss = smem + N * C::LDT;    // stages: A (BK x LDA) then B (BK x LDB)
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tig = lane & 3;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const long long q = blockIdx.x / C::R;
  const int r0 = (blockIdx.x % C::R) * MR;
  const double* Vq = V + q * N * N;

  auto issue = [&](int x) {
    double* As = Ss + (x % C::STAGES) * C::STAGE;
    double* Bs = As + C::BK * C::LDA;
    if (x < C::KS) {
      const int k0 = x * C::BK;
      // A: M1(r0 + i, k0 + kk) -> As[kk][i]
#pragma unroll
      for (int c = tid; c < C::BK * MR / 2; c += C::NT) {
        const int kk = c / (MR / 2), i = (c % (MR / 2)) * 2;
        cp16(As + kk * C::LDA + i, M1 + r0 + i + (long long)(k0 + kk) * N);
      }
      // B: V_q(k0 + kk, col) -> Bs[kk][col]
#pragma unroll
      for (int c = tid; c < C::BK * N; c += C::NT) {
        const int col = c / C::BK, kk = c % C::BK;
        cp8(Bs + kk * C::LDB + col, Vq + k0 + kk + (long long)col * N);
      }
    } else {
      const int k0 = (x - C::KS) * C::BK;
      // B: M2(i, k0 + kk) -> Bs[kk][i]
#pragma unroll
      for (int c = tid; c < C::BK * N / 2; c += C::NT) {
        const int kk = c / (N / 2), i = (c % (N / 2)) * 2;
        cp16(Bs + kk * C::LDB + i, M2 + i + (long long)(k0 + kk) * N);
      }
    }
  };

  double acc[C::MI][C::NI][2];
#pragma unroll
  for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < C::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    issue(s);
    cp_commit();
  }
#pragma unroll 1
  for (int gs = 0; gs < 2 * C::KS; ++gs) {
    cp_wait<C::STAGES - 2>();
    __syncthreads();
    if (gs + C::STAGES - 1 < 2 * C::KS) issue(gs + C::STAGES - 1);
    cp_commit();
    const double* As = Ss + (gs % C::STAGES) * C::STAGE;
    const double* Bs = As + C::BK * C::LDA;
    if (gs < C::KS) {
      // mode 0: T(i, c) += M1(r0 + i, j) V_q(j, c)
#pragma unroll
      for (int kg = 0; kg < C::BK / 4; ++kg) {
        const int kl = kg * 4 + tig;
        double a[C::MI], b[C::NI];
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi) a[mi] = As[kl * C::LDA + wm * C::WM + mi * 8 + g];
#pragma unroll
        for (int ni = 0; ni < C::NI; ++ni) b[ni] = Bs[kl * C::LDB + wn * C::WN + ni * 8 + g];
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < C::NI; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
      if (gs == C::KS - 1) {
        // T block -> Th (nothing reads Th during mode 0); the next
        // iteration's barrier orders these stores before mode 1 reads
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < C::NI; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int m = wm * C::WM + mi * 8 + g, n = wn * C::WN + ni * 8 + 2 * tig + h;
              Th[m + n * C::LDT] = alpha0 * acc[mi][ni][h];
              acc[mi][ni][h] = 0.0;
            }
      }
    } else {
      // mode 1: W(i, k) += T(i, c) M2(k, c)
#pragma unroll
      for (int kg = 0; kg < C::BK / 4; ++kg) {
        const int kl = kg * 4 + tig, kglob = (gs - C::KS) * C::BK + kl;
        double a[C::MI], b[C::NI];
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi) a[mi] = Th[(wm * C::WM + mi * 8 + g) + kglob * C::LDT];
#pragma unroll
        for (int ni = 0; ni < C::NI; ++ni) b[ni] = Bs[kl * C::LDB + wn * C::WN + ni * 8 + g];
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < C::NI; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
    }
  }
  pdl_trigger();  // the next kernel may start its prologue during our epilogue
  cp_wait<0>();
  __syncthreads();  // mode-1 reads of Th done: stage the W block there
#pragma unroll
  for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < C::NI; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = wm * C::WM + mi * 8 + g, n = wn * C::WN + ni * 8 + 2 * tig + h;
        Th[m + n * C::LDT] = acc[mi][ni][h];
      }
  __syncthreads();
  const long long cq = q * N * N + r0;
  const EpiU u = epi_uniform(e);
#pragma unroll 1
  for (int e2 = tid; e2 < MR * N / 2; e2 += C::NT) {
    const int ml = 2 * (e2 % (MR / 2)), nl = e2 / (MR / 2);
    const double2 a2 = *reinterpret_cast<const double2*>(Th + ml + nl * C::LDT);
    const long long off = cq + ml + (long long)nl * N;
    double d0 = 0.0, d1 = 0.0;
    const double v0 = epi_one(e, u, e.alpha * a2.x, out, off, 0, &d0);
    const double v1 = epi_one(e, u, e.alpha * a2.y, out, off + 1, 0, &d1);
    *reinterpret_cast<double2*>(out + off) = make_double2(v0, v1);
  }
}

template <int N, int MR>
void launch_fused01r(kp_ctx* ctx, const double* in, long long Q, const double* m1,
                     const double* m2, double alpha0, const Epilogue& e, double* out) {
  using C = F01R<N, MR>;
  auto kern = fused01r_kernel<N, MR>;
  ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), int(C::SMEM));
  const long long grid = Q * C::R;
  if (grid > 0x7fffffffLL) throw invalid_argument("fused01: too many slices");
  launch_pdl(ctx, kern, dim3(unsigned(grid)), dim3(C::NT), C::SMEM, in, m1, m2, alpha0, e, out);
  KP_CUDA(cudaGetLastError());
}

template <int N>
void launch_fused01(kp_ctx* ctx, const double* in, long long Q, const double* m1,
                    const double* m2, double alpha0, const Epilogue& e, double* out) {
  auto kern = fused01_kernel<N>;
  ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), int(F01<N>::SMEM));
  launch_pdl(ctx, kern, dim3(unsigned(Q)), dim3(F01<N>::NT), F01<N>::SMEM, in, m1, m2, alpha0, e,
             out);
  KP_CUDA(cudaGetLastError());
}

bool fused01_enabled() {
  static const bool on = [] {
    const char* v = getenv("KP_FUSE01");
    return !(v && std::string(v) == "0");
  }();
  return on;
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) % 16) == 0; }

}  // namespace

// out = epi1((alpha0 * in x_0 m0) x_1 m1) for order >= 3 real tensors whose
// first two modes are N x N slices, N in {64, 128}, with square factors.
// false = not applicable (the caller runs the two mode products).  The
// mode-1 epilogue must be a plain store (alpha/beta).
bool fused01_f64(kp_ctx* ctx, const double* in, const std::vector<int>& dims, const double* m0,
                 int rows0, const double* m1, int rows1, double alpha0, const Epilogue& e1,
                 double* out) {
  if (!fused01_enabled() || dims.size() < 3) return false;
  const int n = dims[0];
  if (dims[1] != n || rows0 != n || rows1 != n || (n != 64 && n != 128)) return false;
  if (e1.kind != EPI_STORE || e1.sc_dir != 0 || e1.bad_step) return false;
  if (!al16(in) || !al16(out) || !al16(m0) || !al16(m1) || in == out) return false;
  long long Q = 1;
  for (size_t mu = 2; mu < dims.size(); ++mu) Q *= dims[mu];
  if (Q < 1 || Q > 0x7fffffffLL) return false;
  static const int variant = [] {  // KP_FUSE01=slice: one CTA per slice at N = 128 (A/B)
    const char* v = getenv("KP_FUSE01");
    return (v && std::string(v) == "slice") ? 1 : 0;
  }();
  if (n == 128 && variant == 0)
    launch_fused01r<128, 64>(ctx, in, Q, m0, m1, alpha0, e1, out);
  else if (n == 128)
    launch_fused01<128>(ctx, in, Q, m0, m1, alpha0, e1, out);
  else
    launch_fused01<64>(ctx, in, Q, m0, m1, alpha0, e1, out);
  return true;
}

}  // namespace kp
