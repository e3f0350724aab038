// exchange.cu -- the slab <-> pencil re-partition of the sharded integrators
// as device-initiated stores into peer memory.
//
// The all-to-all that follows (or precedes) the last mode product is not a
// separate collective: mode products store their results straight into the
// owners' receive buffers (mode_product.cu, Epilogue::sc_*), and this plain
// scatter kernel covers the re-partitions with no producing GEMM.  The
// buffers are CUDA IPC mappings of the other ranks' allocations, so over
// NVLink every store is a P2P write; completion is the caller's stream
// synchronize + barrier (no kernel ever waits on another rank).
#include <algorithm>

#include "kp_internal.h"

namespace kp {
namespace {

// same index map as scatter_ptr in mode_product.cu (kept separate: that one
// is inlined into the GEMM epilogue)
__device__ __forceinline__ double* dest(const Epilogue& e, unsigned elem, int comps) {
  const unsigned A = e.sc_A, B = e.sc_B, C = e.sc_C, P = unsigned(e.sc_P), r = unsigned(e.sc_rank);
  const unsigned Bp = B / P, Cl = C / P;
  const unsigned t = elem / A, a = elem - t * A;
  unsigned s;
  unsigned long long idx;
  if (e.sc_dir == 1) {
    const unsigned t2 = t / B, b = t - t2 * B;
    const unsigned sp = t2 / Cl, cl = t2 - sp * Cl;
    s = b / Bp;
    idx = a + (unsigned long long)A *
                  ((b - s * Bp) + (unsigned long long)Bp * (r * Cl + cl + (unsigned long long)C * sp));
  } else {
    const unsigned t2 = t / Bp, bl = t - t2 * Bp;
    const unsigned sp = t2 / C, c = t2 - sp * C;
    s = c / Cl;
    idx = a + (unsigned long long)A *
                  ((r * Bp + bl) + (unsigned long long)B * ((c - s * Cl) + (unsigned long long)Cl * sp));
  }
  return e.sc_peers[s] + idx * comps;
}

__global__ void scatter_copy_kernel(const double* __restrict__ x, unsigned n, int comps,
                                    Epilogue e) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double* d = dest(e, i, comps);
    if (comps == 2) {
      *reinterpret_cast<double2*>(d) = reinterpret_cast<const double2*>(x)[i];
    } else {
      *d = x[i];
    }
  }
}

}  // namespace

void scatter_copy(kp_ctx* ctx, const double* x, long long n, int comps, const Epilogue& e) {
  if (n <= 0) return;
  if (n > 0xffffffffLL) throw invalid_argument("scatter: tensor too large");
  const unsigned grid = unsigned(std::min<long long>((n + 255) / 256, ctx->num_sms * 16LL));
  scatter_copy_kernel<<<grid, 256, 0, ctx->stream>>>(x, unsigned(n), comps, e);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
}

}  // namespace kp
