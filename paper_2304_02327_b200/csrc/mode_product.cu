// mode_product.cu -- FP64 mu-mode product on sm_100a DMMA tensor cores.
//
// Replaces the reference's CPU GEMM core of the Tucker operator:
//   mode_product_into (inc/mode_product.hpp:61-87) -> gemm (inc/kernels.hpp:279-327)
//   and gemm_batch_shared_b (inc/kernels.hpp:332-392).
//
// Contraction contract: out[p, i, q] = sum_j M[i, j] in[p, j, q]
// with p fastest.  Two permute-free GEMM views, never an explicit unfolding:
//   mode 0      : C(i, c)   = sum_j L(i, j) V(j, c)      A = L (M-contig),  B = V (K-contig)
//   mode mu >= 1: C_q(p, i) = sum_j V_q(p, j) L(i, j)    A = V_q (M-contig), B = L^T (N-contig)
// The tensor is always the streamed operand, the n x n factor the resident one.
//
// sm_100a has no FP64 tcgen05 kind (ptxas rejects .kind::f64), so the FP64
// tensor-core path is warp-level mma.sync m8n8k4 (SASS DMMA.8x8x4), measured
// at 37.1 TFLOP/s on B200 vs 34.2 for DFMA (profiles/fp64_peak_r01.txt).
//
// Kernel structure (one CTA = one BM x BN output tile of one batch slab):
//   * STAGES-deep cp.async (LDGSTS) ring of BK-wide K slices of A and B, with
//     16-byte copies along the contiguous index, zero-filled at ragged edges;
//   * warp tile WM x WN of 8x8 DMMA tiles; fragment loads are LDS.128: the
//     k index inside each group of 8 is permuted (thread tig owns k = 2tig,
//     2tig+1) and, on the contiguous operand index, pairs of 8-row/col MMA
//     tiles are interleaved so each thread's two values are adjacent.  Row
//     strides (BM+2, BN+2 doubles; BK+8 for the K-contiguous B) make every
//     quarter-warp touch all 32 banks exactly once;
//   * fused epilogue (Epilogue in kp_internal.h): alpha/beta, add_scaled,
//     kronsum+g and the ETD2RK stage/difference, written as 16-byte stores.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "kp_epilogue.cuh"

namespace kp {
namespace {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <int VEC>
__device__ __forceinline__ void cp_async(double* smem, const double* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (VEC == 2) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
  }
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool B_KCONTIG, int VEC>
struct Cfg {
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  static constexpr int MI = WM / 8, NI = WN / 8;
  static constexpr int LDA = BM + 2;                       // = 2 (mod 16) doubles
  static constexpr int LDB = B_KCONTIG ? BK + 8 : BN + 2;  // = 8 / 2 (mod 16)
  static constexpr int A_STAGE = BK * LDA;
  static constexpr int B_STAGE = B_KCONTIG ? BN * LDB : BK * LDB;
  static constexpr size_t SMEM = size_t(STAGES) * (A_STAGE + B_STAGE) * sizeof(double);
  static_assert(MI % 2 == 0 && NI % 2 == 0, "paired 8x8 tiles");
  static_assert(BK % 8 == 0, "k groups of 8");
};

// CPLX: 0 = real; 1 = complex, output rows are interleaved (re, im) pairs
// (mode 0 with the real 2n x 2n factor); 2 = complex "combine" (mode >= 1):
// rows 2p/2p+1 are re/im of the tensor, columns 2i/2i+1 re/im of the factor,
// and the epilogue forms out(p,i) = (C(2p,2i) - C(2p+1,2i+1), C(2p,2i+1) +
// C(2p+1,2i)) at complex offset p + i*P (ldc is then the complex row pitch
// in doubles, 2P).
template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool B_KCONTIG, int VEC,
          int CPLX, int MINB, bool SCAT>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32, MINB)
    dmma_gemm_kernel(GemmProblem p, Epilogue e, int tiles_m, int tiles_n, int n_fastest,
                     int c_vec2, long long species_half) {
  using CF = Cfg<BM, BN, BK, WARPS_M, WARPS_N, STAGES, B_KCONTIG, VEC>;
  constexpr int NT = CF::NT, MI = CF::MI, NI = CF::NI, LDA = CF::LDA, LDB = CF::LDB;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * CF::A_STAGE;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int wm0 = (warp % WARPS_M) * CF::WM;
  const int wn0 = (warp / WARPS_M) * CF::WN;

  // tile decode: the small dimension runs fastest so CTAs sharing a slab of
  // the streamed tensor are co-resident and the re-reads hit L2.
  const long long per_q = (long long)tiles_m * tiles_n;
  const long long tile = blockIdx.x;
  const long long q = tile / per_q;
  const int r = int(tile - q * per_q);
  int tm, tn;
  if (n_fastest) {
    tn = r % tiles_n;
    tm = r / tiles_n;
  } else {
    tm = r % tiles_m;
    tn = r / tiles_m;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const double* __restrict__ Ab = p.A + q * p.sA;
  const double* __restrict__ Bb = p.B + q * p.sB;
  const int M = p.M, N = p.N, K = p.K;
  const int KT = (K + BK - 1) / BK;

  // Per-thread copy plan, fixed for the whole tile: every thread owns the
  // same contiguous-index offset in each of its chunks, so a stage costs one
  // pointer bump + predicate per 16-byte copy (no divisions, no branches).
  constexpr int A_ROW = BM / VEC;  // chunks per k row of A
  static_assert(NT % A_ROW == 0, "A copy plan");
  constexpr int A_KSTEP = NT / A_ROW, A_PER = BK / A_KSTEP;
  const int a_col = (tid % A_ROW) * VEC, a_kk0 = tid / A_ROW;
  const int a_bytes = max(0, min(VEC, M - (m0 + a_col))) * 8;
  const double* a_src0 = Ab + m0 + a_col + (long long)a_kk0 * p.lda;
  const int a_dst0 = a_kk0 * LDA + a_col;

  constexpr int B_ROW = B_KCONTIG ? BK / VEC : BN / VEC;
  static_assert(NT % B_ROW == 0, "B copy plan");
  constexpr int B_STEP = NT / B_ROW;
  constexpr int B_PER = B_KCONTIG ? BN / B_STEP : BK / B_STEP;
  const int b_in = (tid % B_ROW) * VEC, b_out0 = tid / B_ROW;  // contiguous / strided index
  const double* b_src0;
  int b_dst0, b_bytes_n = 0;
  if constexpr (B_KCONTIG) {
    b_src0 = Bb + b_in + (long long)(n0 + b_out0) * p.sBn;
    b_dst0 = b_out0 * LDB + b_in;
  } else {
    b_src0 = Bb + n0 + b_in + (long long)b_out0 * p.sBk;
    b_dst0 = b_out0 * LDB + b_in;
    b_bytes_n = max(0, min(VEC, N - (n0 + b_in))) * 8;
  }

  auto load_stage = [&](int slot, int kt) {
    const int k0 = kt * BK;
    double* as = As + slot * CF::A_STAGE;
    double* bs = Bs + slot * CF::B_STAGE;
    const double* a_src = a_src0 + (long long)k0 * p.lda;
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
      const int bytes = (k0 + a_kk0 + i * A_KSTEP < K) ? a_bytes : 0;
      cp_async<VEC>(as + a_dst0 + i * A_KSTEP * LDA,
                    bytes ? a_src + (long long)i * A_KSTEP * p.lda : Ab, bytes);
    }
    if constexpr (B_KCONTIG) {
      const int kv = max(0, min(VEC, K - (k0 + b_in))) * 8;
#pragma unroll
      for (int i = 0; i < B_PER; ++i) {
        const int bytes = (n0 + b_out0 + i * B_STEP < N) ? kv : 0;
        cp_async<VEC>(bs + b_dst0 + i * B_STEP * LDB,
                      bytes ? b_src0 + k0 + (long long)i * B_STEP * p.sBn : Bb, bytes);
      }
    } else {
      const double* b_src = b_src0 + (long long)k0 * p.sBk;
#pragma unroll
      for (int i = 0; i < B_PER; ++i) {
        const int bytes = (k0 + b_out0 + i * B_STEP < K) ? b_bytes_n : 0;
        cp_async<VEC>(bs + b_dst0 + i * B_STEP * LDB,
                      bytes ? b_src + (long long)i * B_STEP * p.sBk : Bb, bytes);
      }
    }
  };

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_commit();
    }
    const double* as = As + (kt % STAGES) * CF::A_STAGE;
    const double* bs = Bs + (kt % STAGES) * CF::B_STAGE;
#pragma unroll
    for (int kb = 0; kb < BK; kb += 8) {
      double2 af[MI / 2][2];
#pragma unroll
      for (int pi = 0; pi < MI / 2; ++pi)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          af[pi][h] = *reinterpret_cast<const double2*>(as + (kb + 2 * tig + h) * LDA + wm0 +
                                                        16 * pi + 2 * g);
      double2 bf[NI][1];  // K-contig: one LDS.128 per n tile covers both halves
      double2 bn[NI / 2][2];
      if constexpr (B_KCONTIG) {
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
          bf[ni][0] = *reinterpret_cast<const double2*>(bs + (wn0 + 8 * ni + g) * LDB + kb +
                                                        2 * tig);
      } else {
#pragma unroll
        for (int pj = 0; pj < NI / 2; ++pj)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            bn[pj][h] = *reinterpret_cast<const double2*>(bs + (kb + 2 * tig + h) * LDB + wn0 +
                                                          16 * pj + 2 * g);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          const double a = (mi & 1) ? af[mi >> 1][h].y : af[mi >> 1][h].x;
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            double b;
            if constexpr (B_KCONTIG)
              b = h ? bf[ni][0].y : bf[ni][0].x;
            else
              b = (ni & 1) ? bn[ni >> 1][h].y : bn[ni >> 1][h].x;
            dmma(acc[mi][ni][0], acc[mi][ni][1], a, b);
          }
        }
    }
  }
  cp_wait<0>();

  // ---- epilogue ----
  double* __restrict__ Cb = p.C + q * p.sC;
  const long long cq = q * p.sC;
  bool nonfinite = false;
  if constexpr (CPLX == 2) {
    // pairs of n tiles (2pj, 2pj+1) hold the re/im columns of one factor row
#pragma unroll
    for (int pi = 0; pi < MI / 2; ++pi) {
      const int mrow = m0 + wm0 + 16 * pi + 2 * g;  // = 2p (even); M is even
      if (mrow >= M) continue;
#pragma unroll
      for (int pj = 0; pj < NI / 2; ++pj)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int ncol = n0 + wn0 + 16 * pj + 4 * tig + 2 * i;  // = 2 icol (even)
          if (ncol >= N) continue;
          const double c_rr = acc[2 * pi][2 * pj][i], c_ri = acc[2 * pi][2 * pj + 1][i];
          const double c_ir = acc[2 * pi + 1][2 * pj][i], c_ii = acc[2 * pi + 1][2 * pj + 1][i];
          const double2 v = make_double2(e.alpha * __dsub_rn(c_rr, c_ii),
                                         e.alpha * __dadd_rn(c_ri, c_ir));
          const long long off = mrow + (long long)(ncol >> 1) * p.ldc;
          double2 dv = make_double2(0.0, 0.0);
          const double2 rr = epi_pair_c(e, v, p.C, cq + off, &dv);
          double* dst = Cb + off;
          if constexpr (SCAT) dst = scatter_ptr(e, unsigned((cq + off) >> 1), 2);
          *reinterpret_cast<double2*>(dst) = rr;
          nonfinite |= !isfinite(rr.x) || !isfinite(rr.y);
          if (e.kind == EPI_STAGE_D) *reinterpret_cast<double2*>(e.D + cq + off) = dv;
        }
    }
    if (e.bad_step && nonfinite) atomicMin(e.bad_step, *e.step_ctr + 1);
  if (e.step_next && blockIdx.x == 0 && threadIdx.x == 0) *e.step_next = *e.step_ctr + 1;
    return;
  }
#pragma unroll
  for (int pi = 0; pi < MI / 2; ++pi) {
    const int mrow = m0 + wm0 + 16 * pi + 2 * g;  // rows mrow (tile 2pi), mrow+1 (tile 2pi+1)
    if (mrow >= M) continue;
    const bool two = (mrow + 1 < M);
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        int ncol;
        if constexpr (B_KCONTIG)
          ncol = n0 + wn0 + 8 * ni + 2 * tig + i;
        else
          ncol = n0 + wn0 + 16 * (ni >> 1) + 4 * tig + 2 * i + (ni & 1);
        if (ncol >= N) continue;
        const long long off = mrow + (long long)ncol * p.ldc;
        const double v0 = e.alpha * acc[2 * pi][ni][i];
        const double v1 = e.alpha * acc[2 * pi + 1][ni][i];
        if constexpr (CPLX == 1) {
          // rows (mrow, mrow+1) are (re, im) of one complex entry
          double2 dv = make_double2(0.0, 0.0);
          const double2 rr = epi_pair_c(e, make_double2(v0, v1), p.C, cq + off, &dv);
          double* dst = Cb + off;
          if constexpr (SCAT) dst = scatter_ptr(e, unsigned((cq + off) >> 1), 2);
          *reinterpret_cast<double2*>(dst) = rr;
          nonfinite |= !isfinite(rr.x) || !isfinite(rr.y);
          if (e.kind == EPI_STAGE_D) *reinterpret_cast<double2*>(e.D + cq + off) = dv;
          continue;
        }
        double d0 = 0.0, d1 = 0.0;
        const double r0 = epi_one(e, v0, p.C, cq + off, species_half, &d0);
        nonfinite |= !isfinite(r0);
        if constexpr (SCAT) {
          double r1 = 0.0;
          if (two) {
            r1 = epi_one(e, v1, p.C, cq + off + 1, species_half, &d1);
            nonfinite |= !isfinite(r1);
          }
          store_pair<SCAT>(e, Cb + off, (unsigned long long)(cq + off), r0, r1, two, c_vec2);
          if (e.kind == EPI_STAGE_D) {
            e.D[cq + off] = d0;
            if (two) e.D[cq + off + 1] = d1;
          }
        } else if (two) {
          const double r1 = epi_one(e, v1, p.C, cq + off + 1, species_half, &d1);
          nonfinite |= !isfinite(r1);
          if (c_vec2) {
            *reinterpret_cast<double2*>(Cb + off) = make_double2(r0, r1);
            if (e.kind == EPI_STAGE_D)
              *reinterpret_cast<double2*>(e.D + cq + off) = make_double2(d0, d1);
          } else {
            Cb[off] = r0;
            Cb[off + 1] = r1;
            if (e.kind == EPI_STAGE_D) {
              e.D[cq + off] = d0;
              e.D[cq + off + 1] = d1;
            }
          }
        } else {
          Cb[off] = r0;
          if (e.kind == EPI_STAGE_D) e.D[cq + off] = d0;
        }
      }
  }
  if (e.bad_step && nonfinite) atomicMin(e.bad_step, *e.step_ctr + 1);
  if (e.step_next && blockIdx.x == 0 && threadIdx.x == 0) *e.step_next = *e.step_ctr + 1;
}

template <int BM, int BN, int WARPS_M, int WARPS_N, bool B_KCONTIG, int VEC, int CPLX, int VAR,
          bool SCAT = false>
void launch_cfg(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, long long half) {
  // 128x128 with 8 warps of 64x32: one CTA per SM, BK=32 x 3 stages.
  // Every other tile uses 32x32 warp tiles (<= 128 registers) so that two or
  // more CTAs share an SM and hide each other's barrier/load phases: the
  // measured winner (tools/tucker_sweep.py, profiles/gemm_tiles_r01.txt).
  constexpr bool BIG = (BM == 128 && BN == 128 && WARPS_M * WARPS_N == 8);
  // VAR 1: 3-stage ring and >= 4 CTAs per SM (<= 128 registers) -- more
  // independent DMMA streams per SM partition
  constexpr int BK = BIG ? 32 : 16, STAGES = BIG ? 3 : (VAR == 1 ? 3 : 4);
  constexpr int MINB = BIG ? 1 : (VAR == 1 ? 4 : (WARPS_M * WARPS_N * 32 >= 512 ? 1 : 2));
  using CF = Cfg<BM, BN, BK, WARPS_M, WARPS_N, STAGES, B_KCONTIG, VEC>;
  auto kern = dmma_gemm_kernel<BM, BN, BK, WARPS_M, WARPS_N, STAGES, B_KCONTIG, VEC, CPLX, MINB,
                               SCAT>;
  ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), int(CF::SMEM));
  const int tiles_m = (p.M + BM - 1) / BM;
  const int tiles_n = (p.N + BN - 1) / BN;
  const long long total = (long long)tiles_m * tiles_n * p.batch;
  if (total > 0x7fffffffLL) throw invalid_argument("mode_product: problem too large");
  // run the dimension with fewer tiles fastest (see kernel comment)
  const int n_fastest = tiles_n <= tiles_m ? 1 : 0;
  const int c_vec2 = ((p.ldc % 2) == 0 && (p.sC % 2) == 0 &&
                      (reinterpret_cast<uintptr_t>(p.C) % 16) == 0 &&
                      (e.D == nullptr || (reinterpret_cast<uintptr_t>(e.D) % 16) == 0))
                         ? 1
                         : 0;
  kern<<<unsigned(total), CF::NT, CF::SMEM, ctx->stream>>>(p, e, tiles_m, tiles_n, n_fastest,
                                                           c_vec2, half);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int VAR = 0, bool SCAT = false>
void launch_layout(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, bool kcontig, bool vec2,
                   int cplx, long long half) {
  if (cplx == 1) {
    launch_cfg<BM, BN, WARPS_M, WARPS_N, true, 2, 1, VAR, SCAT>(ctx, p, e, half);
  } else if (cplx == 2) {
    launch_cfg<BM, BN, WARPS_M, WARPS_N, false, 2, 2, VAR, SCAT>(ctx, p, e, half);
  } else if (kcontig) {
    if (vec2)
      launch_cfg<BM, BN, WARPS_M, WARPS_N, true, 2, 0, VAR, SCAT>(ctx, p, e, half);
    else
      launch_cfg<BM, BN, WARPS_M, WARPS_N, true, 1, 0, VAR, SCAT>(ctx, p, e, half);
  } else {
    if (vec2)
      launch_cfg<BM, BN, WARPS_M, WARPS_N, false, 2, 0, VAR, SCAT>(ctx, p, e, half);
    else
      launch_cfg<BM, BN, WARPS_M, WARPS_N, false, 1, 0, VAR, SCAT>(ctx, p, e, half);
  }
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) % 16) == 0; }

}  // namespace

void launch_gemm(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, int cplx) {
  if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return;
  const bool kcontig = (p.sBk == 1);
  if (!kcontig && p.sBn != 1) throw invalid_argument("launch_gemm: B must be K- or N-contiguous");
  if ((cplx == 1 && !kcontig) || (cplx == 2 && kcontig))
    throw invalid_argument("launch_gemm: complex layout mismatch");
  // 16-byte copies need every streamed row start 16-byte aligned.
  bool vec2 = aligned16(p.A) && aligned16(p.B) && (p.lda % 2 == 0) && (p.sA % 2 == 0) &&
              (p.sB % 2 == 0);
  vec2 = vec2 && (kcontig ? (p.sBn % 2 == 0) : (p.sBk % 2 == 0));
  if (cplx && !vec2) throw invalid_argument("launch_gemm: complex operands must be 16-byte aligned");
  long long half = 0;
  if (e.kind == EPI_ADD_G && e.g.kind == KP_G_BRUSSELATOR)
    half = (long long)p.M * p.N * p.batch / 2;  // callers pass the whole stacked tensor
  static const bool native = [] {  // KP_GEMM=native: the hand-written mainloop
    const char* v = getenv("KP_GEMM");
    return v && std::string(v) == "native";
  }();
  if (!native) {
    launch_gemm_cutlass(ctx, p, e, cplx, kcontig, half);
    return;
  }
  const bool bm_small = p.M <= 64, bn_small = p.N <= 64;
  const long long tiles128 =
      (long long)((p.M + 127) / 128) * ((p.N + 127) / 128) * p.batch;
  const bool few = tiles128 < ctx->num_sms;
  // Tile menu (round 1): 1: 128x64 (8 warps), 5: 32x32, 6: 64x32 (4 warps),
  // 8/9: 64x64 / 32x64 with a 3-stage ring and >= 4 CTAs per SM.
  // Chosen from the measured sweep (profiles/gemm_tiles_r01.txt): small tiles
  // (many co-resident CTAs hide latency, fewer idle slots in the last wave)
  // win until the problem is large; long K (d=2, n >= 1024) favours big tiles.
  (void)few;
  (void)bm_small;
  (void)bn_small;
  const long long tiles64 = (long long)((p.M + 63) / 64) * ((p.N + 63) / 64) * p.batch;
  int tile;
  if (tiles64 * 2 < ctx->num_sms)
    tile = 5;
  else if (kcontig)
    tile = (p.K >= 1024 && p.M > 64) ? 1 : 9;
  else
    tile = (tiles64 >= 16LL * ctx->num_sms || p.K >= 1024) ? 8 : 6;
  if (e.sc_dir) {
    // fused exchange: a separate instantiation with the scatter stores (the
    // plain kernels carry no trace of them), two tile shapes
    if (tile == 5)
      launch_layout<32, 32, 2, 2, 0, true>(ctx, p, e, kcontig, vec2, cplx, half);
    else
      launch_layout<64, 64, 2, 2, 1, true>(ctx, p, e, kcontig, vec2, cplx, half);
    return;
  }
  static const int forced = [] {  // benchmarking override
    const char* v = getenv("KP_GEMM_TILE");
    return v ? atoi(v) : -1;
  }();
  if (forced >= 0 && forced <= 10) tile = forced;
  // (the hand-written mainloop is the KP_GEMM=native alternative; its
  // round-1 tile menu is trimmed to the shapes rule v2 selects)
  switch (tile) {
    case 1: launch_layout<128, 64, 4, 2>(ctx, p, e, kcontig, vec2, cplx, half); break;
    case 5: launch_layout<32, 32, 2, 2>(ctx, p, e, kcontig, vec2, cplx, half); break;
    case 6: launch_layout<64, 32, 2, 2>(ctx, p, e, kcontig, vec2, cplx, half); break;
    case 9: launch_layout<32, 64, 2, 2, 1>(ctx, p, e, kcontig, vec2, cplx, half); break;
    default: launch_layout<64, 64, 2, 2, 1>(ctx, p, e, kcontig, vec2, cplx, half); break;
  }
}

// out = epi(t x_mode m): the two permute-free GEMM views of
// mode_product_into (inc/mode_product.hpp:61-87).
void mode_product_f64(kp_ctx* ctx, const double* t, const std::vector<int>& dims, int mode,
                      const double* m, int rows, const Epilogue& e, double* out) {
  const int d = int(dims.size());
  long long P = 1, Q = 1;
  for (int mu = 0; mu < mode; ++mu) P *= dims[mu];
  for (int mu = mode + 1; mu < d; ++mu) Q *= dims[mu];
  const int nm = dims[mode];
  GemmProblem p;
  if (mode == 0) {
    // C(i, c) = sum_j L(i, j) V(j, c): A = L (lda = rows), B = V (K-contig, ldb = n0)
    if (Q > 0x7fffffffLL) throw invalid_argument("mode_product: tensor too large");
    p.M = rows;
    p.N = int(Q);
    p.K = nm;
    p.A = m;
    p.lda = rows;
    p.B = t;
    p.sBk = 1;
    p.sBn = nm;
    p.C = out;
    p.ldc = rows;
  } else {
    // C_q(p, i) = sum_j V_q(p, j) L(i, j): A = V_q (lda = P), B(k=j, n=i) = L[i + j*rows]
    if (P > 0x7fffffffLL || Q > 0x7fffffffLL) throw invalid_argument("mode_product: tensor too large");
    p.M = int(P);
    p.N = rows;
    p.K = nm;
    p.batch = int(Q);
    p.A = t;
    p.lda = P;
    p.sA = P * nm;
    p.B = m;
    p.sBk = rows;
    p.sBn = 1;
    p.C = out;
    p.ldc = P;
    p.sC = P * rows;
  }
  launch_gemm(ctx, p, e, 0);
}

}  // namespace kp
