// gemm_api.cu -- the reference's GEMM cores and LU as C ABI entry points
// (SURVEY.md 8(a) rows a3/a4, 8(b) signatures), on device pointers:
//   gemm                 inc/kernels.hpp:279-327  C = alpha A op(B) + beta C
//   gemm_batch_shared_b  inc/kernels.hpp:332-392  C_q = alpha A_q op(B) + beta C_q
//   lu_factor / lu_solve inc/linsolve.hpp:95-146
// Real GEMMs are the DMMA GEMM of the mode products (launch_gemm: A
// M-contiguous, B K-contiguous for Op::none or N-contiguous for
// Op::transpose).  Complex GEMMs (interleaved complex128) are four real DMMA
// GEMMs on de-interleaved planes (rr, ii, ri, ir) plus one combine pass
// c = alpha (rr - ii, ri + ir) + beta c -- same products and sums as the
// reference's complex micro-kernel up to rounding order (tolerance-tested).
#include <algorithm>
#include <string>

#include "kp_internal.h"

namespace kp {
namespace {

// planes of a column-major complex (rows x cols, ld) block, batch stride bs
__global__ void deinterleave_kernel(const double2* __restrict__ x, int rows, int cols, long long ld,
                                    long long bs, int batch, double* __restrict__ re,
                                    double* __restrict__ im) {
  const long long per = (long long)rows * cols, tot = per * batch;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long q = t / per, r = t - q * per;
    const long long j = r / rows, i = r - j * rows;
    const double2 v = x[q * bs + i + j * ld];
    re[t] = v.x;
    im[t] = v.y;
  }
}

// c = alpha * (rr - ii, ri + ir) + beta * c   (c: rows x cols, ldc, batch stride cs)
__global__ void combine_kernel(const double* __restrict__ rr, const double* __restrict__ ii,
                               const double* __restrict__ ri, const double* __restrict__ ir,
                               int rows, int cols, double2 alpha, double2 beta,
                               double2* __restrict__ c, long long ldc, long long cs, int batch) {
  const long long per = (long long)rows * cols, tot = per * batch;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long q = t / per, r = t - q * per;
    const long long j = r / rows, i = r - j * rows;
    const double pr = __dsub_rn(rr[t], ii[t]), pi = __dadd_rn(ri[t], ir[t]);
    double2 out = make_double2(__dsub_rn(__dmul_rn(alpha.x, pr), __dmul_rn(alpha.y, pi)),
                               __dadd_rn(__dmul_rn(alpha.x, pi), __dmul_rn(alpha.y, pr)));
    double2* cp = c + q * cs + i + j * ldc;
    if (beta.x != 0.0 || beta.y != 0.0) {
      const double2 cv = *cp;
      out.x = __dadd_rn(out.x, __dsub_rn(__dmul_rn(beta.x, cv.x), __dmul_rn(beta.y, cv.y)));
      out.y = __dadd_rn(out.y, __dadd_rn(__dmul_rn(beta.x, cv.y), __dmul_rn(beta.y, cv.x)));
    }
    *cp = out;
  }
}

// The reference's scale_only (inc/kernels.hpp:266-272, taken when k <= 0 or
// alpha == 0, :283-286): C = beta * C, or exactly 0 when beta == 0 -- A and B
// are never read, so an Inf/NaN in them cannot reach C.
__global__ void scale_only_kernel(double* __restrict__ c, int rows, int cols, long long ldc,
                                  long long cs, int batch, int cplx, double2 beta) {
  const long long per = (long long)rows * cols, tot = per * batch;
  const bool zero = beta.x == 0.0 && beta.y == 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long q = t / per, r = t - q * per;
    const long long j = r / rows, i = r - j * rows;
    if (cplx) {
      double2* cp = reinterpret_cast<double2*>(c) + q * cs + i + j * ldc;
      const double2 v = *cp;
      *cp = zero ? make_double2(0.0, 0.0)
                 : make_double2(__dsub_rn(__dmul_rn(beta.x, v.x), __dmul_rn(beta.y, v.y)),
                                __dadd_rn(__dmul_rn(beta.x, v.y), __dmul_rn(beta.y, v.x)));
    } else {
      double* cp = c + q * cs + i + j * ldc;
      *cp = zero ? 0.0 : __dmul_rn(beta.x, *cp);
    }
  }
}

void scale_only(kp_ctx* ctx, int m, int n, double2 beta, double* c, long long ldc, long long sc,
                int batch, int cplx) {
  if (m <= 0 || n <= 0 || batch <= 0) return;
  const long long tot = (long long)m * n * batch;
  const unsigned g = unsigned(std::max<long long>(
      1, std::min<long long>((tot + 255) / 256, ctx->num_sms * 8LL)));
  scale_only_kernel<<<g, 256, 0, ctx->stream>>>(c, m, n, ldc, sc, batch, cplx, beta);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
}

// C_q = alpha * A_q * op(B_q) + beta * C_q, q < batch (real)
void gemm_real(kp_ctx* ctx, int m, int n, int k, double alpha, const double* a, long long lda,
               long long sa, const double* b, long long ldb, long long sb, int opb, double beta,
               double* c, long long ldc, long long sc, int batch) {
  if (m <= 0 || n <= 0 || batch <= 0) return;
  GemmProblem p;
  p.M = m;
  p.N = n;
  p.K = k;
  p.batch = batch;
  p.A = a;
  p.lda = lda;
  p.sA = sa;
  p.B = b;
  p.sB = sb;
  if (opb == 0) {  // op(B)(k, n) = B[k + n ldb]
    p.sBk = 1;
    p.sBn = ldb;
  } else {  // op(B)(k, n) = B[n + k ldb]
    p.sBk = ldb;
    p.sBn = 1;
  }
  p.C = c;
  p.ldc = ldc;
  p.sC = sc;
  Epilogue e;
  e.alpha = alpha;
  e.beta = beta;
  launch_gemm(ctx, p, e, 0);
}

void gemm_cplx(kp_ctx* ctx, int m, int n, int k, double2 alpha, const double* a, long long lda,
               long long sa, const double* b, long long ldb, int opb, double2 beta, double* c,
               long long ldc, long long sc, int batch) {
  if (m <= 0 || n <= 0 || batch <= 0) return;
  const int br = opb == 0 ? k : n, bc = opb == 0 ? n : k;  // stored shape of B
  const long long na = (long long)m * k * batch, nb = (long long)br * bc,
                  nc = (long long)m * n * batch;
  double* ws = static_cast<double*>(
      ctx->ws.get(66, sizeof(double) * size_t(2 * na + 2 * nb + 4 * nc + 4)));
  double *ar = ws, *ai = ar + na, *bre = ai + na, *bim = bre + nb;
  double *rr = bim + nb, *ii = rr + nc, *ri = ii + nc, *ir = ri + nc;
  auto grid = [&](long long t) {
    return unsigned(std::max<long long>(1, std::min<long long>((t + 255) / 256, ctx->num_sms * 8LL)));
  };
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  if (k > 0) {
    deinterleave_kernel<<<grid(na), 256, 0, ctx->stream>>>(a2, m, k, lda, sa, batch, ar, ai);
    deinterleave_kernel<<<grid(nb), 256, 0, ctx->stream>>>(b2, br, bc, ldb, 0, 1, bre, bim);
    ctx->launches += 2;
  }
  const long long sA = (long long)m * k, sC = (long long)m * n;
  // dense planes: A m x k (ld m), B br x bc (ld br), products m x n (ld m)
  gemm_real(ctx, m, n, k, 1.0, ar, m, sA, bre, br, 0, opb, 0.0, rr, m, sC, batch);
  gemm_real(ctx, m, n, k, 1.0, ai, m, sA, bim, br, 0, opb, 0.0, ii, m, sC, batch);
  gemm_real(ctx, m, n, k, 1.0, ar, m, sA, bim, br, 0, opb, 0.0, ri, m, sC, batch);
  gemm_real(ctx, m, n, k, 1.0, ai, m, sA, bre, br, 0, opb, 0.0, ir, m, sC, batch);
  combine_kernel<<<grid(nc), 256, 0, ctx->stream>>>(rr, ii, ri, ir, m, n, alpha, beta,
                                                    reinterpret_cast<double2*>(c), ldc, sc, batch);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
}

void check_gemm(int m, int n, int k, long long lda, long long ldb, int opb, long long ldc) {
  if (m < 0 || n < 0 || k < 0) throw invalid_argument("gemm: negative dimension");
  if (opb != 0 && opb != 1) throw invalid_argument("gemm: opb must be 0 (none) or 1 (transpose)");
  if (lda < std::max(1, m) || ldc < std::max(1, m) ||
      ldb < std::max(1, opb == 0 ? k : n))
    throw invalid_argument("gemm: leading dimension too small");
}

template <typename F>
int guard(F&& f) {
  try {
    f();
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

void need(kp_ctx* ctx) {
  if (!ctx) throw invalid_argument("kronphi_b200: null context");
  KP_CUDA(cudaSetDevice(ctx->device));
}

double2 cscalar(const double* v, const char* what) {
  if (!v) throw invalid_argument(std::string("gemm: null ") + what);
  return make_double2(v[0], v[1]);
}

}  // namespace
}  // namespace kp

using namespace kp;

extern "C" {

int kp_gemm_f64(kp_ctx* ctx, int m, int n, int k, double alpha, const double* a, int lda,
                const double* b, int ldb, int opb, double beta, double* c, int ldc) {
  return guard([&] {
    need(ctx);
    check_gemm(m, n, k, lda, ldb, opb, ldc);
    if (k == 0 || alpha == 0.0)
      return scale_only(ctx, m, n, make_double2(beta, 0.0), c, ldc, 0, 1, 0);
    gemm_real(ctx, m, n, k, alpha, a, lda, 0, b, ldb, 0, opb, beta, c, ldc, 0, 1);
  });
}

int kp_gemm_batch_shared_b_f64(kp_ctx* ctx, int m, int n, int k, double alpha, const double* a,
                               int lda, long long a_stride, const double* b, int ldb, int opb,
                               double beta, double* c, int ldc, long long c_stride, int batch) {
  return guard([&] {
    need(ctx);
    check_gemm(m, n, k, lda, ldb, opb, ldc);
    if (batch < 0) throw invalid_argument("gemm_batch_shared_b: negative batch");
    if (k == 0 || alpha == 0.0)
      return scale_only(ctx, m, n, make_double2(beta, 0.0), c, ldc, c_stride, batch, 0);
    gemm_real(ctx, m, n, k, alpha, a, lda, a_stride, b, ldb, 0, opb, beta, c, ldc, c_stride,
              batch);
  });
}

int kp_gemm_c128(kp_ctx* ctx, int m, int n, int k, const double* alpha2, const double* a, int lda,
                 const double* b, int ldb, int opb, const double* beta2, double* c, int ldc) {
  return guard([&] {
    need(ctx);
    check_gemm(m, n, k, lda, ldb, opb, ldc);
    const double2 al = cscalar(alpha2, "alpha");
    if (k == 0 || (al.x == 0.0 && al.y == 0.0))
      return scale_only(ctx, m, n, cscalar(beta2, "beta"), c, ldc, 0, 1, 1);
    gemm_cplx(ctx, m, n, k, al, a, lda, 0, b, ldb, opb, cscalar(beta2, "beta"), c, ldc, 0, 1);
  });
}

int kp_gemm_batch_shared_b_c128(kp_ctx* ctx, int m, int n, int k, const double* alpha2,
                                const double* a, int lda, long long a_stride, const double* b,
                                int ldb, int opb, const double* beta2, double* c, int ldc,
                                long long c_stride, int batch) {
  return guard([&] {
    need(ctx);
    check_gemm(m, n, k, lda, ldb, opb, ldc);
    if (batch < 0) throw invalid_argument("gemm_batch_shared_b: negative batch");
    const double2 al = cscalar(alpha2, "alpha");
    if (k == 0 || (al.x == 0.0 && al.y == 0.0))
      return scale_only(ctx, m, n, cscalar(beta2, "beta"), c, ldc, c_stride, batch, 1);
    gemm_cplx(ctx, m, n, k, al, a, lda, a_stride, b, ldb, opb, cscalar(beta2, "beta"), c, ldc,
              c_stride, batch);
  });
}

int kp_lu_factor_f64(kp_ctx* ctx, double* a, int n, int* piv) {
  return guard([&] {
    need(ctx);
    if (n <= 0 || !a || !piv) throw invalid_argument("lu_factor: bad arguments");
    lu_factor_dev(ctx, a, n, piv);
  });
}

int kp_lu_solve_f64(kp_ctx* ctx, const double* lu, const int* piv, int n, double* b, int nrhs) {
  return guard([&] {
    need(ctx);
    if (n <= 0 || !lu || !piv || !b || nrhs < 0) throw invalid_argument("lu_solve: bad arguments");
    if (nrhs > 0) lu_solve_dev(ctx, lu, piv, n, b, nrhs);
  });
}

}  // extern "C"
