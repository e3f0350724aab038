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
// The GEMM itself is gemm_dmma.cu (hand-written, warp-specialized, TMA-fed
// DMMA kernel); this file holds the views and the launch checks.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "kp_epilogue.cuh"

namespace kp {
namespace {

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) % 16) == 0; }

}  // namespace

void launch_gemm(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, int cplx) {
  if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return;
  const bool kcontig = (p.sBk == 1);
  if (!kcontig && p.sBn != 1) throw invalid_argument("launch_gemm: B must be K- or N-contiguous");
  if ((cplx == 1 && !kcontig) || (cplx == 2 && kcontig))
    throw invalid_argument("launch_gemm: complex layout mismatch");
  if (cplx) {
    const bool vec2 = aligned16(p.A) && aligned16(p.B) && (p.lda % 2 == 0) &&
                      (p.sA % 2 == 0) && (p.sB % 2 == 0) &&
                      (kcontig ? (p.sBn % 2 == 0) : (p.sBk % 2 == 0));
    if (!vec2) throw invalid_argument("launch_gemm: complex operands must be 16-byte aligned");
  }
  long long half = 0;
  if (e.kind == EPI_ADD_G && e.g.kind == KP_G_BRUSSELATOR)
    half = (long long)p.M * p.N * p.batch / 2;  // callers pass the whole stacked tensor
  launch_gemm_dmma(ctx, p, e, cplx, kcontig, half);
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
