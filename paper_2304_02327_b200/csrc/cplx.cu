// cplx.cu -- complex128 mu-mode products (the NLS config, BASELINE config 5).
//
// The reference runs complex Tucker operators through its generic scalar
// micro-kernel (inc/kernels.hpp:174-186; 9.6 real-GFLOP/s on 8 vCPUs).  Here
// both GEMM views become REAL DMMA GEMMs over the interleaved storage
// (4M convention: 4 real multiply-adds per complex one, no extra pass):
//   mode 0      : out(2i+b, c) = sum_{j,a} Lbig(2i+b, 2j+a) V(2j+a, c) with the
//                 2rows x 2n real factor Lbig = [[Lr, -Li], [Li, Lr]] (interleaved),
//                 built once per call; epilogue sees (re, im) as a row pair.
//   mode mu >= 1: C(2p+a, 2i+c) = sum_j V_a(p, j) L_c(i, j) reading the tensor and
//                 the factor in place as real matrices; the epilogue combines
//                 (rr - ii, ri + ir) and writes the complex entry (p, i).
#include <string>

#include "kp_internal.h"

namespace kp {
namespace {

// Lbig[(2i+b) + 2r*(2j+a)] for L (r x n complex, column-major interleaved)
__global__ void build_lbig_kernel(const double2* __restrict__ L, int r, int n,
                                  double* __restrict__ big) {
  const long long total = (long long)r * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = int(idx % r), j = int(idx / r);
    const double2 v = L[idx];
    const long long ld = 2LL * r;
    const long long c0 = (2LL * j) * ld, c1 = (2LL * j + 1) * ld;
    big[2 * i + c0] = v.x;       // (re row, re col):  Lr
    big[2 * i + 1 + c0] = v.y;   // (im row, re col):  Li
    big[2 * i + c1] = -v.y;      // (re row, im col): -Li
    big[2 * i + 1 + c1] = v.x;   // (im row, im col):  Lr
  }
}

constexpr int SLOT_LBIG = 12;

}  // namespace

void mode_product_c128(kp_ctx* ctx, const double* t, const std::vector<int>& dims, int mode,
                       const double* m, int rows, const Epilogue& e, double* out) {
  const int d = int(dims.size());
  long long P = 1, Q = 1;
  for (int mu = 0; mu < mode; ++mu) P *= dims[mu];
  for (int mu = mode + 1; mu < d; ++mu) Q *= dims[mu];
  const int nm = dims[mode];
  GemmProblem p;
  if (mode == 0) {
    if (Q > 0x7fffffffLL || 2LL * nm > 0x7fffffffLL) throw invalid_argument("mode_product: tensor too large");
    double* big = static_cast<double*>(ctx->ws.get(SLOT_LBIG, 4ull * rows * nm * sizeof(double)));
    const long long total = (long long)rows * nm;
    const unsigned grid = unsigned(std::min<long long>((total + 255) / 256, ctx->num_sms * 8LL));
    build_lbig_kernel<<<grid, 256, 0, ctx->stream>>>(reinterpret_cast<const double2*>(m), rows,
                                                     nm, big);
    ctx->launches++;
    KP_CUDA(cudaGetLastError());
    p.M = 2 * rows;
    p.N = int(Q);
    p.K = 2 * nm;
    p.A = big;
    p.lda = 2LL * rows;
    p.B = t;
    p.sBk = 1;
    p.sBn = 2LL * nm;
    p.C = out;
    p.ldc = 2LL * rows;
    launch_gemm(ctx, p, e, 1);
  } else {
    if (2 * P > 0x7fffffffLL || Q > 0x7fffffffLL) throw invalid_argument("mode_product: tensor too large");
    p.M = int(2 * P);
    p.N = 2 * rows;
    p.K = nm;
    p.batch = int(Q);
    p.A = t;
    p.lda = 2 * P;
    p.sA = 2 * P * nm;
    p.B = m;
    p.sBk = 2LL * rows;
    p.sBn = 1;
    p.C = out;
    p.ldc = 2 * P;
    p.sC = 2 * P * rows;
    launch_gemm(ctx, p, e, 2);
  }
}

}  // namespace kp
