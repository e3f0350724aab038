// riccati.cu -- the reference's LQR differential Riccati problem on the device.
//
// src/problems.cpp:130-284 (build_riccati, riccati_rhs, riccati_jacobian_factors,
// to_problem_spec): U' = A^T U + U A + C + U B U with B = -b b^T, C = alpha c c^T,
// in Kronecker form K = A^T (+) A^T on the n x n state (d = 2) and the
// nonlinearity g(U) = C + U B U = C - w z^T, w = U b, z = U^T b (the
// "control products", :188-200, two GEMV-shaped reductions).
// Rosenbrock-Euler (inc/integrators.hpp:166-194) needs the per-step Jacobian
// factors J_1 = A^T - w b^T, J_2 = A^T - z b^T (:212-250; one shared factor
// when U is symmetric to 1e-8).
//
// Rounding follows the reference: each dot product is its gemm's FMA chain in
// KC = 256 slices (inc/kernels.hpp:297), g = fma(-w_i, z_j, c_ij) and the
// rank-1 Jacobian update fma(-col_i, b_j, a_ij), which is how g++ contracts
// `c - w*z` and `a -= col*b` there.
#include <algorithm>
#include <cmath>
#include <vector>

#include "kp_internal.h"

namespace kp {
namespace {

constexpr int KC = 256;

// w_i = sum_p U(i,p) b_p  and  z_j = sum_p b_p U(p,j), KC-sliced FMA chains
__global__ void control_products_kernel(const double* __restrict__ u, int n,
                                        const double* __restrict__ b, double* __restrict__ w,
                                        double* __restrict__ z) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {  // w_t: rows of U, coalesced across threads
    double c = 0.0, acc = 0.0;
    for (int p0 = 0; p0 < n; p0 += KC) {
      acc = 0.0;
      const int p1 = min(n, p0 + KC);
      for (int p = p0; p < p1; ++p) acc = __fma_rn(u[t + (size_t)p * n], b[p], acc);
      c = (p0 == 0) ? acc : __dadd_rn(c, acc);
    }
    w[t] = c;
  } else if (t < 2 * n) {  // z_j: columns of U
    const int j = t - n;
    const double* col = u + (size_t)j * n;
    double c = 0.0, acc = 0.0;
    for (int p0 = 0; p0 < n; p0 += KC) {
      acc = 0.0;
      const int p1 = min(n, p0 + KC);
      for (int p = p0; p < p1; ++p) acc = __fma_rn(b[p], col[p], acc);
      c = (p0 == 0) ? acc : __dadd_rn(c, acc);
    }
    z[j] = c;
  }
}

// out_ij = c_ij - w_i z_j
__global__ void riccati_g_kernel(int n, const double* __restrict__ cm,
                                 const double* __restrict__ w, const double* __restrict__ z,
                                 double* __restrict__ out) {
  const long long total = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = int(e % n), j = int(e / n);
    out[e] = __fma_rn(-w[i], z[j], cm[e]);
  }
}

// J = A^T - col b^T on the columns where b != 0
__global__ void jacobian_kernel(int n, const double* __restrict__ at,
                                const double* __restrict__ col, const double* __restrict__ b,
                                double* __restrict__ j) {
  const long long total = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ii = int(e % n), jj = int(e / n);
    const double bj = b[jj];
    j[e] = (bj == 0.0) ? at[e] : __fma_rn(-col[ii], bj, at[e]);
  }
}

unsigned grid_for(kp_ctx* ctx, long long n) {
  return unsigned(std::max<long long>(1, std::min<long long>((n + 255) / 256, ctx->num_sms * 16LL)));
}

}  // namespace

// g(U) for the Riccati kind: aux[0] = b (n), aux[1] = C (n x n); w/z scratch
// of 2n doubles.
void riccati_g(kp_ctx* ctx, const kp_gfun& g, const double* u, int n, double* wz, double* out) {
  control_products_kernel<<<(2 * n + 127) / 128, 128, 0, ctx->stream>>>(u, n, g.aux[0], wz,
                                                                         wz + n);
  riccati_g_kernel<<<grid_for(ctx, (long long)n * n), 256, 0, ctx->stream>>>(n, g.aux[1], wz,
                                                                               wz + n, out);
  ctx->launches += 2;
  KP_CUDA(cudaGetLastError());
}

// Jacobian factors (src/problems.cpp:212-250).  Returns 1 when one factor
// serves both modes (symmetric state), 2 otherwise (j2 filled too).
int riccati_jacobians(kp_ctx* ctx, const kp_gfun& g, const double* u, const double* at, int n,
                      double* wz, double* j1, double* j2) {
  control_products_kernel<<<(2 * n + 127) / 128, 128, 0, ctx->stream>>>(u, n, g.aux[0], wz,
                                                                         wz + n);
  ctx->launches++;
  std::vector<double> h(2 * size_t(n));
  KP_CUDA(cudaMemcpyAsync(h.data(), wz, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  KP_CUDA(cudaStreamSynchronize(ctx->stream));
  double asym = 0.0, scale_wz = 0.0;
  for (int i = 0; i < n; ++i) {
    asym = std::max(asym, std::abs(h[i] - h[n + i]));
    scale_wz = std::max({scale_wz, std::abs(h[i]), std::abs(h[n + i])});
  }
  const long long total = (long long)n * n;
  jacobian_kernel<<<grid_for(ctx, total), 256, 0, ctx->stream>>>(n, at, wz, g.aux[0], j1);
  ctx->launches++;
  if (asym <= 1e-8 * std::max(scale_wz, 1e-300)) {
    KP_CUDA(cudaGetLastError());
    return 1;
  }
  jacobian_kernel<<<grid_for(ctx, total), 256, 0, ctx->stream>>>(n, at, wz + n, g.aux[0], j2);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
  return 2;
}

}  // namespace kp
