// kp_launch.cuh -- programmatic dependent launch (PDL) for the kernels of the
// integrators' time loop.
//
// A step is a chain of short, dependent kernels (stencil, 2d GEMMs,
// elementwise passes); each boundary costs a launch plus a ramp-up.  Kernels
// launched through launch_pdl carry the programmatic-stream-serialization
// attribute (kept as programmatic edges when the loop is captured into a
// CUDA graph): the next kernel's CTAs are scheduled once every CTA of the
// current one has triggered (the GEMMs after their mainloop, the other
// kernels implicitly at exit), run their setup, and block in pdl_wait()
// until the predecessor has completed and its writes are visible.  (A
// trigger at kernel start -- dependents parked on the SMs for the whole
// predecessor -- made the small ADR / Riccati loops up to 1.6x slower.)  Every
// kernel launched this way calls pdl_wait() before touching global memory,
// so the data dependencies are exactly those of plain stream order.
// OFF by default, KP_PDL=1 enables it: measured neutral within +-5 % on the
// configs, ADR 80^3 ETD2RK 10 % slower, and the first launch of a captured
// graph with programmatic edges cost ~0.4 s.  griddepcontrol.wait is a no-op
// without the attribute.
#pragma once

#include <cstdlib>
#include <string>

#include "kp_internal.h"

namespace kp {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("KP_PDL");
    return v && std::string(v) == "1";
  }();
  return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(kp_ctx* ctx, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KP_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
  ctx->launches++;
}

}  // namespace kp
