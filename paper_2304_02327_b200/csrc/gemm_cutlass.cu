// gemm_cutlass.cu -- the mode-product GEMM on CUTLASS's sm80 multistage DMMA
// mainloop (header-only threadblock templates instantiated inside our own
// kernel) with our fused epilogues (kp_epilogue.cuh).  This is the GEMM every
// mode product and phi-builder product runs (mode_product.cu launch_gemm);
// the hand-written mainloop there remains selectable with KP_GEMM=native.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "cutlass/cutlass.h"
#include "cutlass/gemm/threadblock/default_mma.h"

#include "kp_epilogue.cuh"
#include "kp_launch.cuh"

namespace kp {
namespace {

// ------------------------------------------------------------------------
// Real GEMMs on CUTLASS's sm80 multistage DMMA mainloop (the header-only
// threadblock templates, instantiated inside our own kernel) with our
// epilogues.  The column-major C = A B is computed as the row-major
// C' = C^T = B^T A^T: A' = B^T (N x K), B' = A^T (K x M).  Tile menu (all
// BK = 16, 3 stages, 4 warps): 64 x 64 at 4 CTAs/SM for K <= 1024 (the
// cubes), 64 x 128 of C' with 32 x 64 warp tiles at 2 CTAs/SM for longer K
// (the configuration cuBLAS selects for DGEMM on this part), 128 x 64 for
// short M and 32 x 32 when the grid would not fill the SMs.  Every
// accumulator sums k in the same order in all of them (BK slices in order,
// DMMA k-groups of four in order), so the tile choice never changes a bit.
namespace cg_dmma {
using InstShape = cutlass::gemm::GemmShape<8, 8, 4>;
constexpr int kStages = 3;
// large problems: 64 x 128 tiles of C' (4 warps of 32 x 64, 2 CTAs/SM)
struct Big {
  using TB = cutlass::gemm::GemmShape<64, 128, 16>;
  using Warp = cutlass::gemm::GemmShape<32, 64, 16>;
  static constexpr int kMinBlocks = 2;
};
// short M (M <= 64, e.g. the block rows of the LU solves): 128 x 64 tiles of
// C' (64 rows of C), 4 warps of 64 x 32
struct Narrow {
  using TB = cutlass::gemm::GemmShape<128, 64, 16>;
  using Warp = cutlass::gemm::GemmShape<64, 32, 16>;
  static constexpr int kMinBlocks = 2;
};
// small problems (fewer 64 x 128 tiles than SMs): 32 x 32 tiles, 4 warps of 16 x 16
struct Small {
  using TB = cutlass::gemm::GemmShape<32, 32, 16>;
  using Warp = cutlass::gemm::GemmShape<16, 16, 16>;
  static constexpr int kMinBlocks = 2;
};
// short-K problems (K <= 256): 64 x 64 tiles, 4 warps of 32 x 32, 4 CTAs/SM --
// one CTA's epilogue overlaps three others' mainloops
struct Medium {
  using TB = cutlass::gemm::GemmShape<64, 64, 16>;
  using Warp = cutlass::gemm::GemmShape<32, 32, 16>;
  static constexpr int kMinBlocks = 4;
};
template <bool B_KCONTIG, typename CFG>
using MmaOf = typename cutlass::gemm::threadblock::DefaultMma<
    double,
    typename std::conditional<B_KCONTIG, cutlass::layout::RowMajor,
                              cutlass::layout::ColumnMajor>::type,  // A' = B^T
    1, double, cutlass::layout::RowMajor, 1,                        // B' = A^T
    double, cutlass::layout::RowMajor, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80,
    typename CFG::TB, typename CFG::Warp, InstShape, kStages,
    cutlass::arch::OpMultiplyAdd>::ThreadblockMma;
}  // namespace cg_dmma

template <bool B_KCONTIG, bool SCAT, typename CFG, int CPLX>
__global__ void __launch_bounds__(128, CFG::kMinBlocks)
    cutlass_dmma_kernel(GemmProblem p, Epilogue e,
                        typename cg_dmma::MmaOf<B_KCONTIG, CFG>::IteratorA::Params pa,
                        typename cg_dmma::MmaOf<B_KCONTIG, CFG>::IteratorB::Params pb, int tiles_m2,
                        int tiles_n2, int n_fastest, int c_vec2, long long species_half) {
  pdl_wait();
  using Mma = cg_dmma::MmaOf<B_KCONTIG, CFG>;
  using TBShape = typename CFG::TB;
  using WarpShape = typename CFG::Warp;
  extern __shared__ __align__(16) char smem_raw[];
  auto& ss = *reinterpret_cast<typename Mma::SharedStorage*>(smem_raw);
  // tiles of C' (M' = our N, N' = our M)
  const long long per_q = (long long)tiles_m2 * tiles_n2;
  const long long tile = blockIdx.x;
  const long long q = tile / per_q;
  const int r = int(tile - q * per_q);
  int t_m2, t_n2;
  if (n_fastest) {
    t_n2 = r % tiles_n2;
    t_m2 = r / tiles_n2;
  } else {
    t_m2 = r % tiles_m2;
    t_n2 = r / tiles_m2;
  }
  const int m2_0 = t_m2 * TBShape::kM, n2_0 = t_n2 * TBShape::kN;
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  typename Mma::IteratorA it_a(pa, const_cast<double*>(p.B + q * p.sB), {p.N, p.K}, tid,
                               {m2_0, 0});
  typename Mma::IteratorB it_b(pb, const_cast<double*>(p.A + q * p.sA), {p.K, p.M}, tid,
                               {0, n2_0});
  Mma mma(ss, tid, warp, lane);
  typename Mma::FragmentC acc;
  acc.clear();
  const int kiters = (p.K + TBShape::kK - 1) / TBShape::kK;
  mma(kiters, acc, it_a, it_b, acc);
  pdl_trigger();  // the next kernel may start its prologue during our epilogue

  // epilogue, staged through shared memory: the fragment element
  // D[(mi + ni * kRow) * 2 + i] is C'(row' = 8 mi + g, col' = 8 ni + 2 tig + i) of
  // the warp tile, i.e. C(m = col', n = row').  The tile is written to smem as
  // a column-major 128 x 64 block of C, then every thread walks (m, m+1)
  // pairs with consecutive threads on consecutive m: coalesced 16-byte
  // stores and ONE copy of the epilogue code (no per-fragment inlining).
  constexpr int kRow = WarpShape::kM / 8, kCol = WarpShape::kN / 8;
  constexpr int kWarpsM = TBShape::kM / WarpShape::kM;
  constexpr int TM = TBShape::kN, TN = TBShape::kM;  // C tile: TM rows x TN cols
  constexpr int LDS_C = TM + 2;
  static_assert(sizeof(double) * LDS_C * TN <= sizeof(typename Mma::SharedStorage),
                "C tile fits in the mainloop's shared memory");
  const int wm = warp % kWarpsM, wn = warp / kWarpsM;
  const int g = lane >> 2, tig = lane & 3;
  const double* accp = reinterpret_cast<const double*>(&acc);
  double* cs = reinterpret_cast<double*>(smem_raw);
  __syncthreads();  // mainloop smem reads are done
#pragma unroll
  for (int mi = 0; mi < kRow; ++mi)
#pragma unroll
    for (int ni = 0; ni < kCol; ++ni) {
      const int nl = wm * WarpShape::kM + 8 * mi + g;
      const int ml = wn * WarpShape::kN + 8 * ni + 2 * tig;
      *reinterpret_cast<double2*>(cs + ml + nl * LDS_C) =
          make_double2(accp[(mi + ni * kRow) * 2], accp[(mi + ni * kRow) * 2 + 1]);
    }
  __syncthreads();
  const int m0 = n2_0, n0 = m2_0;  // tile origin in C
  double* __restrict__ Cb = p.C + q * p.sC;
  const long long cq = q * p.sC;
  bool nonfinite = false;
  if constexpr (CPLX == 2) {
    // rows 2p / 2p+1 = re / im of the tensor, columns 2i / 2i+1 = re / im of
    // the factor: out(p, i) = (C(2p,2i) - C(2p+1,2i+1), C(2p,2i+1) + C(2p+1,2i))
    // at complex offset p + i * P (ldc = 2P doubles)
#pragma unroll 1
    for (int e2 = tid; e2 < (TM / 2) * (TN / 2); e2 += 128) {
      const int pl = e2 % (TM / 2), il = e2 / (TM / 2);
      const int mrow = m0 + 2 * pl, ncol = n0 + 2 * il;
      if (mrow >= p.M || ncol >= p.N) continue;
      const double* c0 = cs + 2 * pl + 2 * il * LDS_C;
      const double c_rr = c0[0], c_ir = c0[1], c_ri = c0[LDS_C], c_ii = c0[LDS_C + 1];
      const double2 v = make_double2(e.alpha * __dsub_rn(c_rr, c_ii), e.alpha * __dadd_rn(c_ri, c_ir));
      const long long off = mrow + (long long)(ncol >> 1) * p.ldc;
      double2 dv = make_double2(0.0, 0.0);
      const double2 rr = epi_pair_c(e, v, p.C, cq + off, &dv);
      double* dst = Cb + off;
      if constexpr (SCAT) dst = scatter_ptr(e, unsigned((cq + off) >> 1), 2);
      *reinterpret_cast<double2*>(dst) = rr;
      nonfinite |= !isfinite(rr.x) || !isfinite(rr.y);
      if (e.kind == EPI_STAGE_D) *reinterpret_cast<double2*>(e.D + cq + off) = dv;
    }
    if (e.bad_step && nonfinite) atomicMin(e.bad_step, *e.step_ctr + 1);
  if (e.step_next && blockIdx.x == 0 && threadIdx.x == 0) *e.step_next = *e.step_ctr + 1;
    return;
  }
#pragma unroll 1
  for (int e2 = tid; e2 < TM * TN / 2; e2 += 128) {
    const int ml = 2 * (e2 % (TM / 2)), nl = e2 / (TM / 2);
    const int mrow = m0 + ml, ncol = n0 + nl;
    if (mrow >= p.M || ncol >= p.N) continue;
    const bool two = (mrow + 1 < p.M);
    const long long off = mrow + (long long)ncol * p.ldc;
    const double2 a2 = *reinterpret_cast<const double2*>(cs + ml + nl * LDS_C);
    const double v0 = e.alpha * a2.x, v1 = e.alpha * a2.y;
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
    double r1 = 0.0;
    if (two) {
      r1 = epi_one(e, v1, p.C, cq + off + 1, species_half, &d1);
      nonfinite |= !isfinite(r1);
    }
    store_pair<SCAT>(e, Cb + off, (unsigned long long)(cq + off), r0, r1, two, c_vec2);
    if (e.kind == EPI_STAGE_D) {
      if (two && c_vec2) {
        *reinterpret_cast<double2*>(e.D + cq + off) = make_double2(d0, d1);
      } else {
        e.D[cq + off] = d0;
        if (two) e.D[cq + off + 1] = d1;
      }
    }
  }
  if (e.bad_step && nonfinite) atomicMin(e.bad_step, *e.step_ctr + 1);
  if (e.step_next && blockIdx.x == 0 && threadIdx.x == 0) *e.step_next = *e.step_ctr + 1;
}

template <bool B_KCONTIG, bool SCAT, typename CFG, int CPLX>
void launch_cutlass(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, long long half) {
  using Mma = cg_dmma::MmaOf<B_KCONTIG, CFG>;
  using LA = typename std::conditional<B_KCONTIG, cutlass::layout::RowMajor,
                                       cutlass::layout::ColumnMajor>::type;
  auto kern = cutlass_dmma_kernel<B_KCONTIG, SCAT, CFG, CPLX>;
  constexpr int smem = int(sizeof(typename Mma::SharedStorage));
  ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), smem);
  // A' = B^T: element (n, k) at B[k*sBk + n*sBn]
  typename Mma::IteratorA::Params pa(LA(B_KCONTIG ? p.sBn : p.sBk));
  // B' = A^T: element (k, m) at A[m + k*lda] -> row-major K x M, ld = lda
  typename Mma::IteratorB::Params pb(cutlass::layout::RowMajor(p.lda));
  const int tiles_m2 = (p.N + CFG::TB::kM - 1) / CFG::TB::kM;
  const int tiles_n2 = (p.M + CFG::TB::kN - 1) / CFG::TB::kN;
  const long long total = (long long)tiles_m2 * tiles_n2 * p.batch;
  if (total > 0x7fffffffLL) throw invalid_argument("mode_product: problem too large");
  const int n_fastest = tiles_n2 <= tiles_m2 ? 1 : 0;
  const int c_vec2 = ((p.ldc % 2) == 0 && (p.sC % 2) == 0 &&
                      (reinterpret_cast<uintptr_t>(p.C) % 16) == 0 &&
                      (e.D == nullptr || (reinterpret_cast<uintptr_t>(e.D) % 16) == 0))
                         ? 1
                         : 0;
  launch_pdl(ctx, kern, dim3(unsigned(total)), dim3(128), size_t(smem), p, e, pa, pb, tiles_m2,
             tiles_n2, n_fastest, c_vec2, half);
  KP_CUDA(cudaGetLastError());
}

// Real GEMMs: one mainloop (CUTLASS's), two tile shapes.  The k order of
// every accumulator is the same in both (BK = 16 slices in order, DMMA k
// groups of 4 in order), so results do not depend on the shape chosen.
template <bool B_KCONTIG, bool SCAT, int CPLX = 0>
void launch_cutlass_any(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, long long half) {
  const long long big_tiles = (long long)((p.N + 63) / 64) * ((p.M + 127) / 128) * p.batch;
  static const int forced = [] {  // benchmarking override: 1 small, 2 big, 3 medium
    const char* v = getenv("KP_CUTLASS_TILE");
    return v ? atoi(v) : 0;
  }();
  // small tiles when the big ones leave SMs idle, or give under ~8 waves of
  // short-K work (n = 128 cubes: 20.4 vs 17.1 TFLOP/s; n = 256: 29.3 vs 30.4)
  const bool small = big_tiles < ctx->num_sms || (big_tiles < 8LL * ctx->num_sms && p.K <= 256);
  const long long narrow_tiles = (long long)((p.N + 127) / 128) * ((p.M + 63) / 64) * p.batch;
  if (forced == 3) {  // benchmarking override: 64 x 64 tiles, 4 CTAs/SM
    launch_cutlass<B_KCONTIG, SCAT, cg_dmma::Medium, CPLX>(ctx, p, e, half);
    return;
  }
  if (forced == 1 || (forced != 2 && small && !(p.M <= 64 && narrow_tiles >= ctx->num_sms)))
    launch_cutlass<B_KCONTIG, SCAT, cg_dmma::Small, CPLX>(ctx, p, e, half);
  else if (p.M <= 64 && forced != 2)
    launch_cutlass<B_KCONTIG, SCAT, cg_dmma::Narrow, CPLX>(ctx, p, e, half);
  else if (forced != 2 && p.K <= 1024)
    // K <= 1024 (every cube of the sweep and the integrators): 64 x 64 tiles
    // at 4 CTAs/SM hide each CTA's prologue / epilogue behind three
    // mainloops: n=256 Tucker 30.6 -> 31.9 TFLOP/s, Brusselator ETD2RK
    // 247 -> 272 steps/s, n=512 34.4 -> 34.6 (tools/tucker_sweep.py A/B)
    launch_cutlass<B_KCONTIG, SCAT, cg_dmma::Medium, CPLX>(ctx, p, e, half);
  else
    launch_cutlass<B_KCONTIG, SCAT, cg_dmma::Big, CPLX>(ctx, p, e, half);
}

}  // namespace

void launch_gemm_cutlass(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, int cplx,
                         bool kcontig, long long half) {
  if (cplx == 1) {  // mode 0 with the real 2n x 2n factor (B K-contiguous)
    e.sc_dir ? launch_cutlass_any<true, true, 1>(ctx, p, e, half)
             : launch_cutlass_any<true, false, 1>(ctx, p, e, half);
  } else if (cplx == 2) {  // modes >= 1, re/im combine (B N-contiguous)
    e.sc_dir ? launch_cutlass_any<false, true, 2>(ctx, p, e, half)
             : launch_cutlass_any<false, false, 2>(ctx, p, e, half);
  } else if (e.sc_dir) {
    kcontig ? launch_cutlass_any<true, true>(ctx, p, e, half)
            : launch_cutlass_any<false, true>(ctx, p, e, half);
  } else {
    kcontig ? launch_cutlass_any<true, false>(ctx, p, e, half)
            : launch_cutlass_any<false, false>(ctx, p, e, half);
  }
}

}  // namespace kp
