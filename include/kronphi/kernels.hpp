// Forwarding header: code written against the reference's
// "kronphi/kernels.hpp" compiles unchanged against the B200 drop-in:
// kronphi::Op, gemm and gemm_batch_shared_b (device DMMA GEMM, kronphi.hpp).
#pragma once
#include <cstddef>

#include "kronphi_b200/kronphi.hpp"

namespace kronphi {

// The reference's unblocked host GEMM (C = alpha A op(B) + beta C), kept for
// tests written against it -- TEST SUPPORT ONLY: nothing in the library
// calls it, the product path is gemm() above.
template <typename T>
void gemm_naive(int m, int n, int k, T alpha, const T* a, int lda, const T* b, int ldb, Op opb,
                T beta, T* c, int ldc) {
  for (int col = 0; col < n; ++col)
    for (int row = 0; row < m; ++row) {
      T sum{};
      for (int p = 0; p < k; ++p) {
        const T bv = opb == Op::none ? b[p + std::size_t(col) * ldb] : b[col + std::size_t(p) * ldb];
        sum += a[row + std::size_t(p) * lda] * bv;
      }
      T& dst = c[row + std::size_t(col) * ldc];
      dst = beta == T{} ? alpha * sum : alpha * sum + beta * dst;
    }
}

}  // namespace kronphi
