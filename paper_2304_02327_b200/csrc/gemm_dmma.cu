// gemm_dmma.cu -- the mode-product GEMM: a hand-written, persistent,
// warp-specialized FP64 DMMA kernel for sm_100a with TMA tile staging.
//
// Replaces the reference's CPU GEMM cores of the Tucker operator:
//   gemm                (inc/kernels.hpp:279-327)  C = alpha A op(B) + beta C
//   gemm_batch_shared_b (inc/kernels.hpp:332-392)  C_q = alpha A_q op(B) + beta C_q
// reached from mode_product_into (inc/mode_product.hpp:61-87) through the two
// permute-free views of mode_product.cu (A M-contiguous; B K-contiguous for
// mode 0, N-contiguous for modes >= 1; C M-contiguous; batched over q).
//
// sm_100a has no FP64 tcgen05 kind (ptxas rejects .kind::f64), so the FP64
// tensor path is warp-level mma.sync m8n8k4 (SASS DMMA.8x8x4; 37.1 TFLOP/s
// measured on the pool's B200, profiles/fp64_peak_r01.txt).  What IS
// Blackwell-native here is the data movement and the schedule:
//
//   * one producer warp per CTA: one elected lane streams BK = 16 slices of
//     the A and B tiles into a STAGES-deep shared-memory ring with TMA
//     (cp.async.bulk.tensor, SASS UTMALDG), 128-byte hardware swizzle, and
//     arms the slot's "full" mbarrier with the expected byte count;
//   * NC consumer warps wait on "full", run the DMMAs straight from the
//     swizzled tiles, and release the slot with one arrive per warp on its
//     "empty" mbarrier -- no __syncthreads in the mainloop;
//   * persistent CTAs (grid = SMs x resident CTAs) walk the tiles with a
//     static stride; the producer runs ahead into the next tile while the
//     consumers stage the accumulators through a separate shared buffer
//     and run the fused epilogue (kp_epilogue.cuh), so the ring never
//     drains between tiles.
//
// Fragment layout (no padding is possible under TMA, so the swizzle and the
// fragment-to-index maps are chosen together to make every shared load
// conflict-free): element (row r, col c) of a 16-double-wide box sits at
// r*16 + 2*((c/2) ^ (r%8)) + c%2.  An M- (or N-) contiguous operand is read
// as LDS.128 pairs (m, m+1) that feed two 8x8 DMMA tiles at once, thread g of
// the pair owning m = 2*perm(g); the K-contiguous B (mode 0) is read as
// LDS.64 with DMMA column g on tile row rperm(g).  perm/rperm spread each
// quarter-/half-warp over all 32 banks for every k (derivation in DESIGN.md
// section 4.1).  The epilogue undoes the maps when it stages C.
//
// Arithmetic order: DMMA k-slot t of k-step s holds k = 16 kt + 4 s + t, the
// k-steps and slices in increasing order -- the order of fused01.cu and of
// every tile shape here, so results never depend on the tile chosen, on TMA
// vs the cp.async producer, or on which path (fused or not) ran.
//
// Operands that TMA cannot describe (a base or stride not 16-byte aligned:
// odd leading dimensions) take the SAME kernel with a cp.async producer warp
// (LDGSTS with zero-fill into the same swizzled layout, completion through
// cp.async.mbarrier.arrive) -- same consumer code, bit-identical results.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>

#include "kp_epilogue.cuh"
#include "kp_launch.cuh"

namespace kp {
namespace {

// ------------------------------------------------------------ PTX helpers

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map,
                                            unsigned long long* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void consumer_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 128-byte swizzle of a 16-double-wide box: (row r, col c) -> offset in doubles
__device__ __forceinline__ int swz(int r, int c) {
  return r * 16 + ((((c >> 1) ^ (r & 7))) << 1) + (c & 1);
}
// thread g's pair slot in a 16-wide (m, m+1) pair row, and the K-contiguous
// tile row of DMMA column g (see the file comment)
__device__ __forceinline__ int perm8(int g) { return ((g & 1) << 2) | (g >> 1); }
__device__ __forceinline__ int rperm8(int g) { return ((g & 3) << 1) | (g >> 2); }

// ------------------------------------------------------------ configuration

template <int BM_, int BN_, int WARPS_M, int WARPS_N, int STAGES_, int MINB, int STG_COLS = BN_,
          int NE_ = 0>
struct TileCfg {
  static constexpr int BM = BM_, BN = BN_, STAGES = STAGES_;
  static constexpr int BK = 16;
  static constexpr int NC = WARPS_M * WARPS_N;  // consumer (DMMA) warps
  static constexpr int NE = NE_;                // epilogue warps (0: consumers do it)
  static constexpr int NT = (NC + NE + 1) * 32;  // + one producer warp
  static constexpr int WARPS_M_ = WARPS_M;
  static constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  static constexpr int MI = WM / 8, NI = WN / 8;
  static constexpr int A_DBL = BM * BK, B_DBL = BN * BK;
  static constexpr int STAGE_DBL = A_DBL + B_DBL;
  static constexpr unsigned STAGE_BYTES = unsigned(STAGE_DBL) * 8u;
  static constexpr int LDS_C = BM + 2;  // staged C tile pitch (doubles)
  static constexpr int SC = STG_COLS;    // columns staged per epilogue pass
  static constexpr int STG_DBL = LDS_C * SC;
  static constexpr size_t SMEM =
      1024 + size_t(STAGES) * STAGE_BYTES + size_t(STG_DBL) * 8 + (2 * STAGES + 2) * 8;
  static constexpr int kMinBlocks = MINB;
  // entries per thread batched in the inline epilogue (kp_epilogue.cuh):
  // 1 for the 32 x 32 tiles, whose latency is hidden by 5 resident CTAs per
  // SM (a batch's registers would cost two of them); 2 for 64 x 64
  static constexpr int EU = (MI * NI <= 4) ? 1 : 2;
  static_assert(WM % 16 == 0 && WN % 16 == 0, "warp tiles are pairs of 8x8 DMMA tiles");
  static_assert(BM % 16 == 0 && BN % 16 == 0 && BN <= 256, "TMA boxes");
  static_assert(BN % SC == 0, "staging passes");
  static_assert(NE == 0 || SC == BN, "epilogue warps take the whole staged tile");
};

// The tile menu (measured; profiles/ncu_r02_summary.md).
// G: 64 x 64 tiles, 4 DMMA warps of 32 x 32 + 2 epilogue warps + the
//    producer, 2 CTAs per SM -- plain products with K > 256 (the headline)
using CfgG = TileCfg<64, 64, 2, 2, 4, 2, 64, 2>;
// N: 64 x 64, 3-stage ring, inline epilogue in two 32-column passes, 3 CTAs
//    per SM -- plain products with K <= 256
using CfgN = TileCfg<64, 64, 2, 2, 3, 3, 32>;
// M: 64 x 64, 4 stages, inline epilogue, 2 CTAs per SM -- the fused-scatter
//    (peer store) epilogues of the sharded path
using CfgM = TileCfg<64, 64, 2, 2, 4, 2>;
// S: 32 x 32, 4 warps of 16 x 16 -- small problems and FP64-heavy fused
//    epilogues at short K (the integrators)
using CfgS = TileCfg<32, 32, 2, 2, 4, 5>;
// L: 128 x 64, 4 warps of 64 x 32, one CTA per SM (KP_GEMM_TILE=L)
using CfgL = TileCfg<128, 64, 2, 2, 4, 1>;
// B / C: balanced single-wave tiles.  A mode product of a 128-cube has
//    16384 rows (or columns) to share among 148 SMs: 64-row tiles leave
//    3.46 per SM (one SM in two does a 4th while the rest idle), 112-row
//    tiles give 147 x 2 = 294 CTAs, two per SM, all resident at once.
//    B: 112 x 64 (4 DMMA warps of 112 x 16), rows taken from the STACKED
//    (batch x M) matrix for batched products (FLAT: 16-row TMA boxes, each
//    with its own batch coordinate), C: 64 x 112 for the K-contiguous B
//    of mode 0 (4 DMMA warps of 16 x 112).
using CfgB = TileCfg<112, 64, 1, 4, 3, 2, 32>;
using CfgC = TileCfg<64, 112, 4, 1, 3, 2, 56>;
// (measured and dropped: 128x64 / 64x128 with 8 DMMA + 3 epilogue warps at 1
// CTA/SM, 64x64 with 8 DMMA warps of 32x16 / 16x32, 64x32 / 32x64 at 4
// CTAs/SM, 32x32 / 32x64 with epilogue warps: all at or below G / N / S)

// ------------------------------------------------------------ the kernel

template <class CF, bool B_KCONTIG, bool TMA, int CPLX, bool SCAT, bool FLAT = false>
__global__ void __launch_bounds__(CF::NT, CF::kMinBlocks)
    dmma_tile_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, GemmProblem p, Epilogue e,
                     int tiles_m, int tiles_n, int n_fastest, int c_vec2, long long half) {
  constexpr int BM = CF::BM, BN = CF::BN, BK = CF::BK, STAGES = CF::STAGES, NC = CF::NC;
  constexpr int MI = CF::MI, NI = CF::NI;
  pdl_wait();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned for the 128-byte swizzle; pointer arithmetic (not an
  // integer round trip) keeps the shared address space visible to the
  // compiler, so fragment loads are LDS, not generic loads
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* ring = reinterpret_cast<double*>(base);
  double* stg = ring + STAGES * CF::STAGE_DBL;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(stg + CF::STG_DBL);
  unsigned long long* empty = full + STAGES;
  unsigned long long* stg_full = empty + STAGES;  // NE > 0: staged tile ready
  unsigned long long* stg_empty = stg_full + 1;   // NE > 0: staging buffer free
  constexpr int NE = CF::NE;

  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], TMA ? 1u : 32u);
      mbar_init(&empty[s], unsigned(NC));
    }
    mbar_init(stg_full, 1u);
    mbar_init(stg_empty, 1u);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  const long long per_q = (long long)tiles_m * tiles_n;
  // FLAT: tiles_m counts row blocks of the stacked (batch x M) matrix
  const long long total = FLAT ? per_q : per_q * p.batch;
  const int KT = (p.K + BK - 1) / BK;
  auto decode = [&](long long tile, long long& q, int& m0, int& n0) {
    q = tile / per_q;
    const int r = int(tile - q * per_q);
    int tm, tn;
    if (n_fastest) {
      tn = r % tiles_n;
      tm = r / tiles_n;
    } else {
      tm = r % tiles_m;
      tn = r / tiles_m;
    }
    m0 = tm * BM;
    n0 = tn * BN;
  };

  if (NE > 0 && warp >= NC && warp < NC + NE) {
    // ------------------------------------------------ epilogue warps
    const int etid = tid - NC * 32;
    unsigned ph = 0;
    bool nonfinite = false;
    for (long long tile = blockIdx.x; tile < total; tile += gridDim.x) {
      long long q;
      int m0, n0;
      decode(tile, q, m0, n0);
      mbar_wait(stg_full, ph);
      int rb = 0;
      if constexpr (FLAT) {
        q = m0 / p.M;
        m0 -= int(q) * p.M;
        rb = p.M - m0;
      }
      nonfinite |= staged_epilogue<BM, BN, CF::LDS_C, NE * 32, CPLX, SCAT, 4, FLAT>(
          p, e, stg, m0, n0, q, etid, c_vec2, half, rb);
      // bar.sync completes this group's shared loads before the release
      asm volatile("bar.sync 2, %0;\n" ::"r"(NE * 32) : "memory");
      if (etid == 0) mbar_arrive(stg_empty);
      ph ^= 1u;
    }
    if (e.bad_step && nonfinite) atomicMin(e.bad_step, *e.step_ctr + 1);
    return;
  }
  if (warp == NC + NE) {
    // ------------------------------------------------ producer warp
    int stage = 0;
    unsigned phase = 0;
    if constexpr (TMA) {
      if (lane != 0) return;
      for (long long tile = blockIdx.x; tile < total; tile += gridDim.x) {
        long long q;
        int m0, n0;
        decode(tile, q, m0, n0);
        int qa = int(q);
        const int qb = p.sB ? int(q) : 0;
        if constexpr (FLAT) {
          qa = m0 / p.M;
          m0 -= qa * p.M;
        }
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1u);
          double* as = ring + stage * CF::STAGE_DBL;
          double* bs = as + CF::A_DBL;
          mbar_expect_tx(&full[stage], CF::STAGE_BYTES);
#pragma unroll
          for (int c = 0; c < BM / 16; ++c) {
            int mc = m0 + 16 * c, qc = qa;
            if (FLAT && mc >= p.M) {  // the tile runs on into the next batch
              mc -= p.M;              // (past the last batch: out of bounds, zero-filled)
              ++qc;
            }
            tma_load_3d(as + c * 16 * BK, &mapA, &full[stage], mc, kt * BK, qc);
          }
          if constexpr (B_KCONTIG) {
            tma_load_3d(bs, &mapB, &full[stage], kt * BK, n0, qb);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 16; ++c)
              tma_load_3d(bs + c * 16 * BK, &mapB, &full[stage], n0 + 16 * c, kt * BK, qb);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    } else {
      // cp.async producer (operands TMA cannot describe): all 32 lanes
      for (long long tile = blockIdx.x; tile < total; tile += gridDim.x) {
        long long q;
        int m0, n0;
        decode(tile, q, m0, n0);
        const double* Ab = p.A + q * p.sA;
        const double* Bb = p.B + q * p.sB;
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1u);
          double* as = ring + stage * CF::STAGE_DBL;
          double* bs = as + CF::A_DBL;
          const int k0 = kt * BK;
          for (int idx = lane; idx < BM * BK; idx += 32) {
            const int m = idx % BM, k = idx / BM;
            const bool ok = (m0 + m < p.M) && (k0 + k < p.K);
            cp_async8(as + (m >> 4) * 16 * BK + swz(k, m & 15),
                      ok ? Ab + (m0 + m) + (long long)(k0 + k) * p.lda : p.A, ok ? 8 : 0);
          }
          if constexpr (B_KCONTIG) {
            for (int idx = lane; idx < BN * BK; idx += 32) {
              const int k = idx % BK, n = idx / BK;
              const bool ok = (n0 + n < p.N) && (k0 + k < p.K);
              cp_async8(bs + swz(n, k), ok ? Bb + (k0 + k) + (long long)(n0 + n) * p.sBn : p.B,
                        ok ? 8 : 0);
            }
          } else {
            for (int idx = lane; idx < BN * BK; idx += 32) {
              const int n = idx % BN, k = idx / BN;
              const bool ok = (n0 + n < p.N) && (k0 + k < p.K);
              cp_async8(bs + (n >> 4) * 16 * BK + swz(k, n & 15),
                        ok ? Bb + (n0 + n) + (long long)(k0 + k) * p.sBk : p.B, ok ? 8 : 0);
            }
          }
          cp_async_mbar_arrive(&full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------- consumer warps
  const int g = lane >> 2, tig = lane & 3;
  const int wm0 = (warp % CF::WARPS_M_) * CF::WM, wn0 = (warp / CF::WARPS_M_) * CF::WN;
  const int pg = perm8(g);
  // per-thread fragment offsets inside a stage (doubles), k-step s adds 64 (A, B
  // N-contiguous: 4 rows of 16) -- the swizzle depends only on (4s + tig) & 7,
  // which is tig or tig + 4
  int a_off[2], b_off[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = 4 * h + tig;
    a_off[h] = (wm0 >> 4) * 16 * BK + swz(r, 2 * pg);
    b_off[h] = B_KCONTIG ? 0 : CF::A_DBL + (wn0 >> 4) * 16 * BK + swz(r, 2 * pg);
  }
  // K-contiguous B: row rperm(g) of n tile ni, k = 4s + tig; k + 8 flips
  // bit 2 of the 16-byte chunk index, i.e. bit 3 of the offset (XOR 8)
  int bk_off[NI][2];
#pragma unroll
  for (int ni = 0; ni < NI; ++ni)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      bk_off[ni][h] = CF::A_DBL + swz(wn0 + 8 * ni + rperm8(g), 4 * h + tig);

  int stage = 0;
  unsigned phase = 0, stg_phase = 0;
  bool nonfinite = false;
  for (long long tile = blockIdx.x; tile < total; tile += gridDim.x) {
    long long q;
    int m0, n0;
    decode(tile, q, m0, n0);
    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // A slot is released one stage late: the DMMAs that consumed its
    // fragments sit before this iteration's full-barrier wait loop (a basic
    // block boundary the scheduler does not move instructions across), and a
    // DMMA cannot issue before its LDS operands have landed -- so every read
    // of the slot has completed before its "empty" arrive lets TMA overwrite
    // it.  (Releasing right after the last LDS let the arrive overtake the
    // loads in flight: a write-after-read race under TMA.)
    int prev = -1;
    for (int kt = 0; kt < KT; ++kt) {
      mbar_wait(&full[stage], phase);
      if (prev >= 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[prev]);
      }
      const double* st = ring + stage * CF::STAGE_DBL;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int h = s & 1, kofs = (s >> 1) * 128;  // rows 8..15: +8 rows of 16
        double2 af[MI / 2];
#pragma unroll
        for (int pi = 0; pi < MI / 2; ++pi)
          af[pi] = *reinterpret_cast<const double2*>(st + a_off[h] + kofs + pi * 16 * BK);
        double bv[NI];
        if constexpr (B_KCONTIG) {
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) bv[ni] = st[bk_off[ni][h] ^ ((s >> 1) << 3)];
        } else {
#pragma unroll
          for (int pj = 0; pj < NI / 2; ++pj) {
            const double2 b2 =
                *reinterpret_cast<const double2*>(st + b_off[h] + kofs + pj * 16 * BK);
            bv[2 * pj] = b2.x;
            bv[2 * pj + 1] = b2.y;
          }
        }
        if constexpr (CPLX == 2 && !B_KCONTIG) {
          // complex modes >= 1: rows (m, m+1) = (re, im) of a tensor entry,
          // columns (n, n+1) = (re, im) of a factor entry.  Three products
          // per complex block instead of four (the 3M form):
          //   P1 = re re -> acc[even][even], P2 = im im -> acc[odd][odd],
          //   P3 = (re + im)(re + im) -> acc[even][odd];
          // the epilogue forms (P1 - P2, P3 - P1 - P2).  acc[odd][even] stays 0.
          double as[MI / 2], bs[NI / 2];
#pragma unroll
          for (int pi = 0; pi < MI / 2; ++pi) as[pi] = __dadd_rn(af[pi].x, af[pi].y);
#pragma unroll
          for (int pj = 0; pj < NI / 2; ++pj) bs[pj] = __dadd_rn(bv[2 * pj], bv[2 * pj + 1]);
#pragma unroll
          for (int pi = 0; pi < MI / 2; ++pi)
#pragma unroll
            for (int pj = 0; pj < NI / 2; ++pj) {
              dmma(acc[2 * pi][2 * pj][0], acc[2 * pi][2 * pj][1], af[pi].x, bv[2 * pj]);
              dmma(acc[2 * pi + 1][2 * pj + 1][0], acc[2 * pi + 1][2 * pj + 1][1], af[pi].y,
                   bv[2 * pj + 1]);
              dmma(acc[2 * pi][2 * pj + 1][0], acc[2 * pi][2 * pj + 1][1], as[pi], bs[pj]);
            }
        } else {
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) {
            const double a = (mi & 1) ? af[mi >> 1].y : af[mi >> 1].x;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a, bv[ni]);
          }
        }
      }
      prev = stage;
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    // the last slot: bar.sync orders (waits for) this thread's shared loads
    consumer_bar(NC * 32);
    if (prev >= 0 && lane == 0) mbar_arrive(&empty[prev]);

    // ---- epilogue: stage C (undoing the fragment maps), then the fused
    // pass -- by the epilogue warps (NE > 0), or here in BN / SC passes
    auto stage_acc = [&](int c0) {
#pragma unroll
      for (int pi = 0; pi < MI / 2; ++pi) {
        const int ml = wm0 + 16 * pi + 2 * pg;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int c = 2 * tig + j;  // DMMA column
            const int nl = (B_KCONTIG ? wn0 + 8 * ni + rperm8(c)
                                      : wn0 + 16 * (ni >> 1) + 2 * perm8(c) + (ni & 1)) - c0;
            if (CF::SC == BN || (nl >= 0 && nl < CF::SC))
              *reinterpret_cast<double2*>(stg + ml + nl * CF::LDS_C) =
                  make_double2(acc[2 * pi][ni][j], acc[2 * pi + 1][ni][j]);
          }
      }
    };
    if constexpr (NE > 0) {
      mbar_wait(stg_empty, stg_phase ^ 1u);  // the epilogue warps drained it
      stage_acc(0);
      consumer_bar(NC * 32);  // all staging stores done before the release
      if (tid == 0) mbar_arrive(stg_full);
      stg_phase ^= 1u;
    } else {
      int rb = 0;
      if constexpr (FLAT) {
        q = m0 / p.M;
        m0 -= int(q) * p.M;
        rb = p.M - m0;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += CF::SC) {
        if (c0 > 0) consumer_bar(NC * 32);  // the previous pass has read stg
        stage_acc(c0);
        consumer_bar(NC * 32);
        nonfinite |= staged_epilogue<BM, CF::SC, CF::LDS_C, NC * 32, CPLX, SCAT, CF::EU, FLAT>(
            p, e, stg, m0, n0 + c0, q, tid, c_vec2, half, rb);
      }
    }
  }
  if (e.bad_step && nonfinite) atomicMin(e.bad_step, *e.step_ctr + 1);
  if (e.step_next && blockIdx.x == 0 && tid == 0) *e.step_next = *e.step_ctr + 1;
}

// ------------------------------------------------------------ host side

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    KP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f)
      throw cuda_error("cuTensorMapEncodeTiled is not available from the driver");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// A 3-D FP64 tensor map (dims d0 fastest) with a {b0, b1, 1} box and the
// 128-byte swizzle.  s1, s2 = strides of dims 1 and 2 in elements.
void make_map(CUtensorMap* m, const double* ptr, long long d0, long long d1, long long d2,
              long long s1, long long s2, int b0, int b1) {
  cuuint64_t dims[3] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(d2)};
  cuuint64_t strides[2] = {cuuint64_t(s1) * 8u, cuuint64_t(s2) * 8u};
  cuuint32_t box[3] = {cuuint32_t(b0), cuuint32_t(b1), 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  const CUresult r = tensor_map_encoder()(
      m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw cuda_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

bool a16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) % 16) == 0; }

// Can TMA describe both operands?  (16-byte aligned bases and strides, 32-bit dims)
bool tma_ok(const GemmProblem& p, bool kcontig) {
  static const bool off = [] {
    const char* v = getenv("KP_TMA");
    return v && std::string(v) == "0";
  }();
  if (off) return false;
  if (!a16(p.A) || !a16(p.B)) return false;
  if (p.lda % 2 || (p.batch > 1 && p.sA % 2) || (p.sB % 2)) return false;
  if (kcontig ? (p.sBn % 2) : (p.sBk % 2)) return false;
  const long long big = 0xffffffffLL;
  return p.M <= big && p.N <= big && p.K <= big && p.batch <= big;
}

int resident_ctas(const void* kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<const void*, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(kern);
  if (it != cache.end()) return it->second;
  int n = 0;
  KP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem));
  n = std::max(1, n);
  cache[kern] = n;
  return n;
}

template <class CF, bool KC, bool TMA, int CPLX, bool SCAT, bool FLAT = false>
void launch_tile(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, long long half) {
  auto kern = dmma_tile_kernel<CF, KC, TMA, CPLX, SCAT, FLAT>;
  ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), int(CF::SMEM));
  const int tiles_m =
      int((FLAT ? (long long)p.M * p.batch + CF::BM - 1 : (long long)p.M + CF::BM - 1) / CF::BM);
  const int tiles_n = (p.N + CF::BN - 1) / CF::BN;
  const long long total = (long long)tiles_m * tiles_n * (FLAT ? 1 : p.batch);
  const int n_fastest = tiles_n <= tiles_m ? 1 : 0;
  const int c_vec2 = ((p.ldc % 2) == 0 && (p.sC % 2) == 0 && a16(p.C) &&
                      (e.D == nullptr || a16(e.D)))
                         ? 1
                         : 0;
  CUtensorMap ma{}, mb{};
  if constexpr (TMA) {
    const long long qa_stride = p.batch > 1 ? p.sA : p.lda * std::max(1, p.K);
    make_map(&ma, p.A, p.M, p.K, p.batch, p.lda, (qa_stride + 1) & ~1LL, 16, CF::BK);
    const long long bb = p.sB ? p.batch : 1;
    if (KC) {
      const long long qs = p.sB ? p.sB : p.sBn * std::max(1, p.N);
      make_map(&mb, p.B, p.K, p.N, bb, p.sBn, (qs + 1) & ~1LL, CF::BK, CF::BN);
    } else {
      const long long qs = p.sB ? p.sB : p.sBk * std::max(1, p.K);
      make_map(&mb, p.B, p.N, p.K, bb, p.sBk, (qs + 1) & ~1LL, 16, CF::BK);
    }
  }
  const int per_sm = resident_ctas(reinterpret_cast<const void*>(kern), CF::NT, CF::SMEM);
  const long long grid = std::min<long long>(total, (long long)ctx->num_sms * per_sm);
  launch_pdl(ctx, kern, dim3(unsigned(grid)), dim3(CF::NT), CF::SMEM, ma, mb, p, e, tiles_m,
             tiles_n, n_fastest, c_vec2, half);
  KP_CUDA(cudaGetLastError());
}

template <class CF, int CPLX, bool SCAT>
void launch_layout(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, bool kcontig,
                   long long half) {
  const bool tma = tma_ok(p, kcontig);
  if (kcontig)
    tma ? launch_tile<CF, true, true, CPLX, SCAT>(ctx, p, e, half)
        : launch_tile<CF, true, false, CPLX, SCAT>(ctx, p, e, half);
  else
    tma ? launch_tile<CF, false, true, CPLX, SCAT>(ctx, p, e, half)
        : launch_tile<CF, false, false, CPLX, SCAT>(ctx, p, e, half);
}

template <class CF, bool SCAT>
void launch_cplx(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, bool kcontig, int cplx,
                 long long half) {
  if (cplx == 1)
    launch_layout<CF, 1, SCAT>(ctx, p, e, kcontig, half);
  else if (cplx == 2)
    launch_layout<CF, 2, SCAT>(ctx, p, e, kcontig, half);
  else
    launch_layout<CF, 0, SCAT>(ctx, p, e, kcontig, half);
}

}  // namespace

// Tile menu: 32 x 32 when 64 x 64 tiles would not give every resident CTA
// a few tiles; 128 x 64 for long K; 64 x 64 otherwise.  The k order is the
// same in all of them (see the file comment), so the choice never changes a
// bit.  KP_GEMM_TILE=G|N|M|S|L forces one, KP_GEMM_TILE_FUSED one for the
// fused-epilogue launches only (testing / benchmarking).
void launch_gemm_dmma(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, int cplx,
                      bool kcontig, long long half) {
  static const char forced = [] {
    const char* v = getenv("KP_GEMM_TILE");
    return v && *v ? v[0] : '\0';
  }();
  const long long tiles64 = (long long)((p.M + 63) / 64) * ((p.N + 63) / 64) * p.batch;
  // fused epilogues (stage updates, g, accumulation) carry FP64 work that
  // competes with the DMMAs for the FP64 datapath: at short K they run best
  // spread over many small CTAs (measured on the integrator configs)
  const bool fused = !(e.kind == EPI_STORE && e.beta == 0.0 && e.bad_step == nullptr);
  char cfg = 'G';
  if (tiles64 < 4LL * ctx->num_sms || (fused && p.K <= 256))
    cfg = 'S';
  else if (p.K <= 256)
    cfg = 'N';
  else if (!fused && p.K >= 1024) {
    // few rounds of 64 x 64 tiles with a short last round (d = 2, n = 2048:
    // 1024 tiles on 296 slots = 3.46 rounds, and the last round's lone CTAs,
    // one DMMA warp per scheduler, run at ~2/3 of an SM's rate): the 32 x 32
    // tiles spread the tail over every SM -- measured 32.2 vs 30.3 TFLOP/s
    const double rounds = double(tiles64) / (2.0 * ctx->num_sms);
    const double fr = rounds - double((long long)rounds);
    if (rounds < 6.0 && fr > 0.05 && fr < 0.6) cfg = 'S';
  }
  // balanced tiles (B / C), opt-in: KP_GEMM_BAL=2 for real, unscattered,
  // TMA-describable products whose 112-row (-column) tiles fill one wave of
  // two CTAs per SM, KP_GEMM_BAL=1 also for any product they spread more
  // evenly than 64 x 64 tiles.  Measured (B200, n = 128 cube): the wave is
  // balanced (294 CTAs) but nothing overlaps a CTA's TMA ramp and epilogue,
  // 26.9 vs 25.8 us per mode product (DMMA pipe 66 vs 74 % of active cycles),
  // AC3D 5.30k vs 5.97k steps/s; n = 256 29.7 vs 31.5 TFLOP/s -- so S / N / G
  // stay the defaults.
  const bool flat = !kcontig && p.batch > 1;
  const bool bal_ok = cplx == 0 && !e.sc_dir && tma_ok(p, kcontig) &&
                      (!flat || (p.sB == 0 && p.M % 16 == 0 && p.M >= CfgB::BM &&
                                 (long long)p.M * p.batch < (1LL << 31)));
  if (bal_ok) {
    const long long tb = kcontig ? (long long)((p.M + 63) / 64) * ((p.N + 111) / 112) * p.batch
                                 : (((long long)p.M * p.batch + 111) / 112) * ((p.N + 63) / 64);
    const long long slots = 2LL * ctx->num_sms;
    static const int bal_mode = [] {
      const char* v = getenv("KP_GEMM_BAL");
      return v && *v ? atoi(v) : 0;
    }();
    if (bal_mode != 0 && tb <= slots && 4 * tb >= 3 * slots && p.K >= 64) cfg = 'B';
    if (bal_mode == 1 && tb > slots) {
      const long long s64 = (long long)ctx->num_sms * (cfg == 'S' ? 5 : cfg == 'N' ? 3 : 2);
      const long long t64 = cfg == 'S' ? (long long)((p.M + 31) / 32) * ((p.N + 31) / 32) * p.batch
                                       : tiles64;
      const double eff64 = double(t64) / double((t64 + s64 - 1) / s64 * s64);
      const double effb = double(tb) / double((tb + slots - 1) / slots * slots);
      if (effb > eff64 + 0.03) cfg = 'B';
    }
  }
  if (forced) cfg = forced;
  if (cfg == 'B' && !bal_ok) cfg = 'S';
  static const char forced_fused = [] {
    const char* v = getenv("KP_GEMM_TILE_FUSED");
    return v && *v ? v[0] : '\0';
  }();
  if (fused && forced_fused && (forced_fused != 'B' || bal_ok)) cfg = forced_fused;
  // the fused exchange's peer-store epilogues take the same menu (the
  // epilogue warps of G overlap the scattered stores with the mainloop)
  auto go = [&](auto scat) {
    constexpr bool SC = decltype(scat)::value;
    switch (cfg) {
      case 'S': launch_cplx<CfgS, SC>(ctx, p, e, kcontig, cplx, half); break;
      case 'N': launch_cplx<CfgN, SC>(ctx, p, e, kcontig, cplx, half); break;
      case 'M': launch_cplx<CfgM, SC>(ctx, p, e, kcontig, cplx, half); break;
      case 'L': launch_cplx<CfgL, SC>(ctx, p, e, kcontig, cplx, half); break;
      default: launch_cplx<CfgG, SC>(ctx, p, e, kcontig, cplx, half); break;
    }
  };
  if (cfg == 'B') {
    if (kcontig)
      launch_tile<CfgC, true, true, 0, false>(ctx, p, e, half);
    else if (flat)
      launch_tile<CfgB, false, true, 0, false, true>(ctx, p, e, half);
    else
      launch_tile<CfgB, false, true, 0, false>(ctx, p, e, half);
    return;
  }
  if (e.sc_dir)
    go(std::true_type{});
  else
    go(std::false_type{});
}

}  // namespace kp
