// capi.cpp -- the extern "C" boundary of libkronphi_b200.so (include/kronphi_b200.h).
//
// Every entry point validates its arguments with the reference's rules and
// messages (inc/mode_product.hpp:45-56, :29-33, :103, :113), runs the device
// path, and maps exceptions to status codes + kp_last_error().  There is no
// CPU compute fallback anywhere: a missing GPU or a CUDA failure is an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "kp_internal.h"

namespace kp {

void* Workspace::get(int slot, size_t bytes) {
  if (slot >= int(ptr.size())) {
    ptr.resize(slot + 1, nullptr);
    cap.resize(slot + 1, 0);
  }
  if (cap[slot] < bytes) {
    if (ptr[slot]) KP_CUDA(cudaFree(ptr[slot]));
    ptr[slot] = nullptr;
    cap[slot] = 0;
    KP_CUDA(cudaMalloc(&ptr[slot], bytes));
    cap[slot] = bytes;
  }
  return ptr[slot];
}
void Workspace::release() {
  for (void* p : ptr)
    if (p) cudaFree(p);
  ptr.clear();
  cap.clear();
}
void* PinnedStage::get(size_t bytes) {
  if (cap < bytes) {
    if (ptr) KP_CUDA(cudaFreeHost(ptr));
    ptr = nullptr;
    cap = 0;
    KP_CUDA(cudaMallocHost(&ptr, bytes));
    cap = bytes;
  }
  return ptr;
}
void PinnedStage::release() {
  if (ptr) cudaFreeHost(ptr);
  ptr = nullptr;
  cap = 0;
}

namespace {

thread_local std::string g_err;

}  // namespace

void kp_set_last_error(const std::string& m) { g_err = m; }

void ensure_smem_attr(kp_ctx* ctx, const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({kernel, ctx->device})) return;
  KP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({kernel, ctx->device});
}

namespace {

template <typename F>
int guard(F&& f) {
  try {
    f();
    return KP_OK;
  } catch (const kp::divergence_error& e) {
    g_err = e.what();
    return KP_EDIVERGE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return KP_EINVAL;
  } catch (const kp::cuda_error& e) {
    g_err = e.what();
    return KP_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KP_ERUNTIME;
  }
}

void need_ctx(kp_ctx* ctx) {
  if (!ctx) throw invalid_argument("kronphi_b200: null context");
  KP_CUDA(cudaSetDevice(ctx->device));
}

std::vector<int> check_dims(const int* dims, int d, const char* who) {
  if (d <= 0 || !dims) throw invalid_argument(std::string(who) + ": Tensor: empty dims");
  std::vector<int> v(dims, dims + d);
  for (int x : v)
    if (x <= 0) throw invalid_argument(std::string(who) + ": Tensor: nonpositive dim");
  return v;
}

size_t numel(const std::vector<int>& dims) {
  size_t n = 1;
  for (int x : dims) n *= size_t(x);
  return n;
}

// inc/mode_product.hpp:45-56 (same messages)
void check_mode(const std::vector<int>& dims, int mode, int cols) {
  const int d = int(dims.size());
  if (mode < 0 || mode >= d)
    throw invalid_argument("mode_product: mode " + std::to_string(mode) +
                           " out of range for order " + std::to_string(d));
  if (cols != dims[mode])
    throw invalid_argument("mode_product: size mismatch on mode " + std::to_string(mode) +
                           ": matrix has " + std::to_string(cols) + " columns, tensor dim is " +
                           std::to_string(dims[mode]));
}

}  // namespace

using ModeFn = void (*)(kp_ctx*, const double*, const std::vector<int>&, int, const double*, int,
                        const Epilogue&, double*);

// Tucker operator on device pointers: out = ((pref*t) x_1 M_1 ... x_d M_d).
// The prefactor is folded into the first mode's alpha (exact for the powers
// of two (l!)^(d-1) of l <= 2, inc/split_phi.hpp:41).  Ping-pong buffers come
// from workspace slots slot_base, slot_base+1.  `last` (optional) is the
// epilogue of the final mode (stepper fusion).  comps = doubles per entry.
void tucker_generic(kp_ctx* ctx, ModeFn mp, int comps, const double* t, std::vector<int> dims,
                    const double* const* ms, const int* rows, double pref, double* out,
                    const Epilogue* last = nullptr, int slot_base = 0) {
  const int d = int(dims.size());
  const double* cur = t;
  int mu0 = 0;
  if (comps == 1 && d >= 3) {  // modes 0 and 1 in one pass over small slices
    double* dst = static_cast<double*>(
        ctx->ws.get(slot_base + 1, numel(dims) * sizeof(double)));
    if (fused01_f64(ctx, t, dims, ms[0], rows[0], ms[1], rows[1], pref, Epilogue{}, dst)) {
      cur = dst;
      mu0 = 2;
    }
  }
  for (int mu = mu0; mu < d; ++mu) {
    std::vector<int> od = dims;
    od[mu] = rows[mu];
    double* dst;
    if (mu == d - 1 && !(d == 1 && out == t)) {
      dst = out;
    } else {
      dst = static_cast<double*>(
          ctx->ws.get(slot_base + (mu & 1), numel(od) * comps * sizeof(double)));
    }
    Epilogue e;
    if (mu == d - 1 && last) e = *last;
    e.alpha = (mu == 0) ? pref : 1.0;
    mp(ctx, cur, dims, mu, ms[mu], rows[mu], e, dst);
    dims = od;
    cur = dst;
  }
  if (cur != out)
    KP_CUDA(cudaMemcpyAsync(out, cur, numel(dims) * comps * sizeof(double),
                            cudaMemcpyDeviceToDevice, ctx->stream));
}

void tucker_f64(kp_ctx* ctx, const double* t, std::vector<int> dims, const double* const* ms,
                const int* rows, double pref, double* out, const Epilogue* last = nullptr,
                int slot_base = 0) {
  tucker_generic(ctx, mode_product_f64, 1, t, std::move(dims), ms, rows, pref, out, last,
                 slot_base);
}
void tucker_c128(kp_ctx* ctx, const double* t, std::vector<int> dims, const double* const* ms,
                 const int* rows, double pref, double* out, const Epilogue* last = nullptr,
                 int slot_base = 0) {
  tucker_generic(ctx, mode_product_c128, 2, t, std::move(dims), ms, rows, pref, out, last,
                 slot_base);
}

// kronsum_action (inc/mode_product.hpp:111-121): term 0 stores, terms >= 1
// accumulate (beta = 1); `last` fuses an epilogue into the final term.
void kronsum_generic(kp_ctx* ctx, ModeFn mp, const double* t, const std::vector<int>& dims,
                     const double* const* as, double* out, const Epilogue* last = nullptr) {
  const int d = int(dims.size());
  for (int mu = 0; mu < d; ++mu) {
    Epilogue e;
    if (mu == d - 1 && last) e = *last;
    e.alpha = 1.0;
    e.beta = mu > 0 ? 1.0 : 0.0;
    mp(ctx, t, dims, mu, as[mu], dims[mu], e, out);
  }
}

}  // namespace kp

using namespace kp;

extern "C" {

const char* kp_last_error(void) { return g_err.c_str(); }

int kp_ctx_create(int device, kp_ctx** out) {
  return guard([&] {
    if (!out) throw invalid_argument("kp_ctx_create: null out");
    int count = 0;
    KP_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
      throw invalid_argument("kp_ctx_create: no CUDA device " + std::to_string(device));
    KP_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    KP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      throw runtime_error(std::string("kronphi_b200 needs an sm_100 (Blackwell) GPU, found ") +
                          prop.name);
    kp_ctx* c = new kp_ctx;
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    KP_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    KP_CUDA(cudaMalloc(&c->d_flag, 256));
    KP_CUDA(cudaMallocHost(&c->h_flag, 256));
    *out = c;
  });
}

int kp_ctx_destroy(kp_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->ws.release();
    ctx->pin_in.release();
    ctx->pin_out.release();
    cudaFree(ctx->d_flag);
    cudaFreeHost(ctx->h_flag);
    cudaStreamDestroy(ctx->own_stream);
    delete ctx;
  });
}

int kp_ctx_set_stream(kp_ctx* ctx, void* stream) {
  return guard([&] {
    need_ctx(ctx);
    ctx->stream = static_cast<cudaStream_t>(stream);  // 0 = the legacy default stream
  });
}

int kp_ctx_use_own_stream(kp_ctx* ctx) {
  return guard([&] {
    need_ctx(ctx);
    ctx->stream = ctx->own_stream;
  });
}

void* kp_ctx_get_stream(kp_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int kp_ctx_synchronize(kp_ctx* ctx) {
  return guard([&] {
    need_ctx(ctx);
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

unsigned long long kp_ctx_launch_count(kp_ctx* ctx) { return ctx ? ctx->launches : 0ULL; }

int kp_malloc(kp_ctx* ctx, size_t bytes, void** ptr) {
  return guard([&] {
    need_ctx(ctx);
    KP_CUDA(cudaMalloc(ptr, std::max<size_t>(bytes, 16)));
  });
}
int kp_free(kp_ctx* ctx, void* ptr) {
  return guard([&] {
    need_ctx(ctx);
    KP_CUDA(cudaFree(ptr));
  });
}
int kp_upload(kp_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    need_ctx(ctx);
    KP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}
int kp_download(kp_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    need_ctx(ctx);
    KP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}
int kp_copy(kp_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    need_ctx(ctx);
    if (bytes && (!dst || !src)) throw invalid_argument("copy: null pointer");
    if (bytes) KP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  });
}

int kp_memset(kp_ctx* ctx, void* dst, int value, size_t bytes) {
  return guard([&] {
    need_ctx(ctx);
    KP_CUDA(cudaMemsetAsync(dst, value, bytes, ctx->stream));
  });
}

// ---------------- mode products ----------------

int kp_mode_product_f64(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                        const double* m, int rows, int cols, double alpha, double beta,
                        double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "mode_product");
    check_mode(dv, mode, cols);
    if (rows <= 0) throw invalid_argument("mode_product: matrix has no rows");
    if (out == t) throw invalid_argument("mode_product: out must not alias the input");
    Epilogue e;
    e.alpha = alpha;
    e.beta = beta;
    mode_product_f64(ctx, t, dv, mode, m, rows, e, out);
  });
}

namespace {
// ETD2RK's stage update in the epilogue of a mode product (see header)
int mode_product_stage(kp_ctx* ctx, bool cplx, const double* t, const int* dims, int d, int mode,
                       const double* m, int rows, double alpha, const double* x, double gamma,
                       const kp_gfun* g, double t1, double t2, double* out, double* d_out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "mode_product");
    check_mode(dv, mode, dv[mode]);
    if (rows != dv[mode]) throw invalid_argument("mode_product_stage: square factor expected");
    if (!x || out == t || out == x) throw invalid_argument("mode_product_stage: bad buffers");
    Epilogue e;
    e.alpha = alpha;
    e.gamma = gamma;
    e.X = x;
    e.kind = EPI_FMA_X;
    const bool coupled = g && d_out && g->kind == KP_G_BRUSSELATOR;
    if (coupled && (cplx || dv.back() != 2))
      throw invalid_argument("brusselator g: slowest mode must hold 2 species");
    if (g && d_out && !coupled) {
      e.kind = EPI_STAGE_D;
      e.D = d_out;
      e.g = *g;
      e.t = t1;
      e.t2 = t2;
    }
    if (cplx)
      mode_product_c128(ctx, t, dv, mode, m, rows, e, out);
    else
      mode_product_f64(ctx, t, dv, mode, m, rows, e, out);
    if (coupled) {
      const long long n = (long long)numel(dv);
      gdiff_dev(ctx, *g, t1, t2 - t1, out, x, n, n / 2, false, d_out);
    }
  });
}
}  // namespace

int kp_mode_product_stage_f64(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                              const double* m, int rows, double alpha, const double* x,
                              double gamma, const kp_gfun* g, double t1, double t2, double* out,
                              double* d_out) {
  return mode_product_stage(ctx, false, t, dims, d, mode, m, rows, alpha, x, gamma, g, t1, t2,
                            out, d_out);
}
int kp_mode_product_stage_c128(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                               const double* m, int rows, double alpha, const double* x,
                               double gamma, const kp_gfun* g, double t1, double t2, double* out,
                               double* d_out) {
  return mode_product_stage(ctx, true, t, dims, d, mode, m, rows, alpha, x, gamma, g, t1, t2,
                            out, d_out);
}

int kp_tucker_f64(kp_ctx* ctx, const double* t, const int* dims, int d, const double* const* ms,
                  const int* rows, double prefactor, double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "tucker");
    if (!ms || !rows) throw invalid_argument("tucker: expected one factor per mode");
    for (int mu = 0; mu < d; ++mu)
      if (rows[mu] <= 0) throw invalid_argument("tucker: factor has no rows");
    tucker_f64(ctx, t, dv, ms, rows, prefactor, out);
  });
}

int kp_kronsum_f64(kp_ctx* ctx, const double* t, const int* dims, int d, const double* const* as,
                   double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "kronsum_action");
    if (!as) throw invalid_argument("kronsum_action: expected one factor per mode");
    if (out == t) throw invalid_argument("kronsum_action: out must not alias the input");
    if (!kronsum_try_banded(ctx, false, t, dv, as, out))
      kronsum_generic(ctx, mode_product_f64, t, dv, as, out);
  });
}

// ---------------- host-buffer drop-in variants ----------------

namespace {

// Upload n_mats square-or-rectangular host matrices into one device slab.
std::vector<const double*> upload_mats(kp_ctx* ctx, int slot, const double* const* hm,
                                       const std::vector<size_t>& sizes) {
  size_t total = 0;
  for (size_t s : sizes) total += (s + 1) & ~size_t(1);  // keep 16-byte alignment
  double* dev = static_cast<double*>(ctx->ws.get(slot, total * sizeof(double)));
  std::vector<const double*> out;
  size_t off = 0;
  for (size_t i = 0; i < sizes.size(); ++i) {
    KP_CUDA(cudaMemcpyAsync(dev + off, hm[i], sizes[i] * sizeof(double), cudaMemcpyHostToDevice,
                            ctx->stream));
    out.push_back(dev + off);
    off += (sizes[i] + 1) & ~size_t(1);
  }
  return out;
}

// Tensor H2D through the pinned stage (one pageable->pinned memcpy plus one
// async DMA; large tensors go in 64 MiB chunks so the two overlap poorly but
// never need a pinned buffer the size of the tensor twice).
void h2d(kp_ctx* ctx, double* dst, const double* src, size_t n) {
  KP_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
}
void d2h(kp_ctx* ctx, double* dst, const double* src, size_t n) {
  KP_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  KP_CUDA(cudaStreamSynchronize(ctx->stream));
}

constexpr int SLOT_HOST_IN = 8, SLOT_HOST_OUT = 9, SLOT_HOST_MATS = 10;
constexpr int SLOT_PIPE_A = 13, SLOT_PIPE_SUB = 14;
constexpr int SLOT_HOST_IN2 = 60, SLOT_HOST_OUT2 = 61, SLOT_PIPE_A2 = 62;

// Host-buffer Tucker with the PCIe copies overlapped with the device work
// (the e2e drop-in path).  Mode products on distinct modes act plane by plane
// along the slowest mode, so:
//   * the input streams in over a copy stream in chunks of planes (slowest
//     mode); modes 0..d-2 of chunk k run while chunk k+1 is in flight;
//   * the last mode (which needs every plane) is computed in blocks of OUTPUT
//     planes -- row blocks of its factor -- and each block is copied back
//     over a second copy stream while the next one computes.
// Results are bit-identical to the unpipelined Tucker (same per-entry sums).
void host_tucker_pipelined(kp_ctx* ctx, ModeFn mp, int comps, const double* const* ts,
                           const std::vector<int>& dv, const std::vector<const double*>& dm,
                           const int* rows, double pref, double* const* outs, int count) {
  const int d = int(dv.size());
  size_t plane_in = comps, plane_mid = comps, plane_out = comps;
  for (int mu = 0; mu < d - 1; ++mu) {
    plane_in *= size_t(dv[mu]);
    plane_mid *= size_t(rows[mu]);
    plane_out *= size_t(rows[mu]);
  }
  const int nlast = dv[d - 1], rlast = rows[d - 1];
  // one buffer set per tensor in flight (two when streaming several tensors:
  // tensor i+1 uploads while tensor i finishes and downloads)
  const int nbuf = count > 1 ? 2 : 1;
  double *din[2], *dmid[2], *dout[2];
  for (int b = 0; b < nbuf; ++b) {
    din[b] = static_cast<double*>(
        ctx->ws.get(b ? SLOT_HOST_IN2 : SLOT_HOST_IN, plane_in * nlast * sizeof(double)));
    dmid[b] = static_cast<double*>(
        ctx->ws.get(b ? SLOT_HOST_OUT2 : SLOT_HOST_OUT, plane_mid * nlast * sizeof(double)));
    dout[b] = static_cast<double*>(
        ctx->ws.get(b ? SLOT_PIPE_A2 : SLOT_PIPE_A, plane_out * rlast * sizeof(double)));
  }
  double* sub = static_cast<double*>(
      ctx->ws.get(SLOT_PIPE_SUB, size_t(rlast) * nlast * comps * sizeof(double)));
  // pipeline depth: ~16 MiB per chunk, at most 8 (small tensors: one chunk,
  // i.e. exactly the unpipelined launch sequence)
  const size_t in_bytes = plane_in * nlast * sizeof(double);
  const int depth = int(std::min<size_t>(8, std::max<size_t>(1, in_bytes >> 24)));
  const int nch = std::min(nlast, depth), nblk = std::min(rlast, depth);
  // chunk scratch (ping-pong slots 0/1) sized once for the largest chunk, so
  // no slot is reallocated under in-flight work
  {
    const int pmax = (nlast + nch - 1) / nch + 1;
    size_t big = 0;
    std::vector<int> cd = dv;
    cd[d - 1] = std::min(nlast, pmax);
    for (int mu = 0; mu < d - 1; ++mu) {
      cd[mu] = rows[mu];
      size_t n_od = comps;
      for (int x : cd) n_od *= size_t(x);
      big = std::max(big, n_od);
    }
    if (d > 1) {
      ctx->ws.get(0, big * sizeof(double));
      ctx->ws.get(1, big * sizeof(double));
    }
  }
  cudaStream_t s_in, s_out;
  KP_CUDA(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
  KP_CUDA(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
  // per tensor: nch chunk-arrival events, nblk block-done events, one
  // "inputs consumed" and one "outputs downloaded" event per buffer set
  std::vector<cudaEvent_t> ev(size_t(count) * (nch + nblk) + 1 + 2 * nbuf);
  for (auto& e : ev) KP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t* ev_start = &ev[size_t(count) * (nch + nblk)];
  cudaEvent_t* ev_in_free = ev_start + 1;     // [nbuf]
  cudaEvent_t* ev_out_free = ev_in_free + nbuf;  // [nbuf]
  try {
    // factors were uploaded on ctx->stream: the copy streams start after them
    KP_CUDA(cudaEventRecord(*ev_start, ctx->stream));
    KP_CUDA(cudaStreamWaitEvent(s_in, *ev_start, 0));
    std::vector<int> md = dv;
    for (int mu = 0; mu < d - 1; ++mu) md[mu] = rows[mu];
    for (int i = 0; i < count; ++i) {
      const int b = i % nbuf;
      cudaEvent_t* ech = &ev[size_t(i) * (nch + nblk)];
      cudaEvent_t* eblk = ech + nch;
      if (i >= nbuf) KP_CUDA(cudaStreamWaitEvent(s_in, ev_in_free[b], 0));
      for (int k = 0; k < nch; ++k) {
        const int p0 = int((long long)nlast * k / nch), p1 = int((long long)nlast * (k + 1) / nch);
        KP_CUDA(cudaMemcpyAsync(din[b] + plane_in * p0, ts[i] + plane_in * p0,
                                plane_in * (p1 - p0) * sizeof(double), cudaMemcpyHostToDevice,
                                s_in));
        KP_CUDA(cudaEventRecord(ech[k], s_in));
        KP_CUDA(cudaStreamWaitEvent(ctx->stream, ech[k], 0));
        std::vector<int> cd = dv;
        cd[d - 1] = p1 - p0;
        const double* cur = din[b] + plane_in * p0;
        for (int mu = 0; mu < d - 1; ++mu) {
          std::vector<int> od = cd;
          od[mu] = rows[mu];
          size_t n_od = comps;
          for (int x : od) n_od *= size_t(x);
          double* dst = (mu == d - 2) ? dmid[b] + plane_mid * p0
                                      : static_cast<double*>(ctx->ws.get(mu & 1, n_od * sizeof(double)));
          Epilogue e;
          e.alpha = (mu == 0) ? pref : 1.0;
          mp(ctx, cur, cd, mu, dm[mu], rows[mu], e, dst);
          cd = od;
          cur = dst;
        }
      }
      if (d > 1 && nbuf > 1) KP_CUDA(cudaEventRecord(ev_in_free[b], ctx->stream));
      // last mode in blocks of output planes, each copied back as it completes
      if (i >= nbuf) KP_CUDA(cudaStreamWaitEvent(ctx->stream, ev_out_free[b], 0));
      for (int bl = 0; bl < nblk; ++bl) {
        const int i0 = int((long long)rlast * bl / nblk), i1 = int((long long)rlast * (bl + 1) / nblk);
        const int rb = i1 - i0;
        if (i == 0)  // rows i0..i1 of the last factor as a contiguous rb x nlast matrix
          KP_CUDA(cudaMemcpy2DAsync(sub + size_t(i0) * nlast * comps, rb * comps * sizeof(double),
                                    dm[d - 1] + size_t(i0) * comps, rlast * comps * sizeof(double),
                                    rb * comps * sizeof(double), nlast, cudaMemcpyDeviceToDevice,
                                    ctx->stream));
        Epilogue e;
        e.alpha = (d == 1) ? pref : 1.0;
        mp(ctx, d == 1 ? din[b] : dmid[b], md, d - 1, sub + size_t(i0) * nlast * comps, rb, e,
           dout[b] + plane_out * i0);
        KP_CUDA(cudaEventRecord(eblk[bl], ctx->stream));
      }
      if (d == 1 && nbuf > 1) KP_CUDA(cudaEventRecord(ev_in_free[b], ctx->stream));
      for (int bl = 0; bl < nblk; ++bl) {
        const int i0 = int((long long)rlast * bl / nblk), i1 = int((long long)rlast * (bl + 1) / nblk);
        KP_CUDA(cudaStreamWaitEvent(s_out, eblk[bl], 0));
        KP_CUDA(cudaMemcpyAsync(outs[i] + plane_out * i0, dout[b] + plane_out * i0,
                                plane_out * (i1 - i0) * sizeof(double), cudaMemcpyDeviceToHost,
                                s_out));
      }
      if (nbuf > 1) KP_CUDA(cudaEventRecord(ev_out_free[b], s_out));
    }
    KP_CUDA(cudaStreamSynchronize(s_out));
    KP_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    cudaStreamSynchronize(s_in);
    cudaStreamSynchronize(s_out);
    cudaStreamSynchronize(ctx->stream);
    for (auto& e : ev) cudaEventDestroy(e);
    cudaStreamDestroy(s_in);
    cudaStreamDestroy(s_out);
    throw;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  cudaStreamDestroy(s_in);
  cudaStreamDestroy(s_out);
}

}  // namespace

// ---------------- fused exchange over peer memory (kp_scatter) ----------------

namespace {

constexpr int SLOT_PEERS = 63;

// Epilogue fields of a kp_scatter; checks the local tensor against the
// layout and uploads the peer pointer table (stream-ordered).
Epilogue scatter_epilogue(kp_ctx* ctx, const kp_scatter* sc, long long local_elems) {
  if (!sc || !sc->peers) throw invalid_argument("scatter: null descriptor");
  if (sc->dir != 1 && sc->dir != 2) throw invalid_argument("scatter: dir must be 1 or 2");
  if (sc->P < 1 || sc->rank < 0 || sc->rank >= sc->P) throw invalid_argument("scatter: bad rank");
  if (sc->A < 1 || sc->B < 1 || sc->C < 1 || sc->S < 1 || sc->B % sc->P || sc->C % sc->P)
    throw invalid_argument("scatter: B and C must be divisible by P");
  const long long total = sc->A * sc->B * sc->C * sc->S;
  if (total / sc->P != local_elems)
    throw invalid_argument("scatter: local tensor does not match the layout");
  if (sc->A * sc->B * sc->C > 0xffffffffLL || local_elems > 0xffffffffLL)
    throw invalid_argument("scatter: tensor too large");
  for (int r = 0; r < sc->P; ++r)
    if (!sc->peers[r] || (reinterpret_cast<uintptr_t>(sc->peers[r]) % 16))
      throw invalid_argument("scatter: peer buffers must be non-null and 16-byte aligned");
  double** dev = static_cast<double**>(ctx->ws.get(SLOT_PEERS, sizeof(double*) * 64));
  if (sc->P > 64) throw invalid_argument("scatter: at most 64 ranks");
  KP_CUDA(cudaMemcpyAsync(dev, sc->peers, sizeof(double*) * sc->P, cudaMemcpyHostToDevice,
                          ctx->stream));
  Epilogue e;
  e.sc_dir = sc->dir;
  e.sc_P = sc->P;
  e.sc_rank = sc->rank;
  e.sc_A = unsigned(sc->A);
  e.sc_B = unsigned(sc->B);
  e.sc_C = unsigned(sc->C);
  e.sc_peers = dev;
  return e;
}

int mode_product_scatter(kp_ctx* ctx, bool cplx, const double* t, const int* dims, int d,
                         int mode, const double* m, int rows, double alpha, const double* x,
                         double gamma, const kp_scatter* sc) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "mode_product");
    check_mode(dv, mode, dv[mode]);
    auto od = dv;
    od[mode] = rows;
    Epilogue e = scatter_epilogue(ctx, sc, (long long)numel(od));
    e.alpha = alpha;
    if (x) {
      e.kind = EPI_FMA_X;
      e.X = x;
      e.gamma = gamma;
    }
    // C is never written with a scatter; it only anchors the index arithmetic
    double* anchor = sc->peers[sc->rank];
    if (cplx)
      mode_product_c128(ctx, t, dv, mode, m, rows, e, anchor);
    else
      mode_product_f64(ctx, t, dv, mode, m, rows, e, anchor);
  });
}

}  // namespace

int kp_mode_product_scatter_f64(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                                const double* m, int rows, double alpha, const double* x,
                                double gamma, const kp_scatter* sc) {
  return mode_product_scatter(ctx, false, t, dims, d, mode, m, rows, alpha, x, gamma, sc);
}
int kp_mode_product_scatter_c128(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                                 const double* m, int rows, double alpha, const double* x,
                                 double gamma, const kp_scatter* sc) {
  return mode_product_scatter(ctx, true, t, dims, d, mode, m, rows, alpha, x, gamma, sc);
}

int kp_scatter_copy(kp_ctx* ctx, const double* x, long long n_elems, int comps,
                    const kp_scatter* sc) {
  return guard([&] {
    need_ctx(ctx);
    if (comps != 1 && comps != 2) throw invalid_argument("scatter: comps must be 1 or 2");
    if (!x && n_elems > 0) throw invalid_argument("scatter: null input");
    const Epilogue e = scatter_epilogue(ctx, sc, n_elems);
    scatter_copy(ctx, x, n_elems, comps, e);
  });
}

int kp_ipc_get_handle(const void* dptr, void* handle64) {
  return guard([&] {
    if (!dptr || !handle64) throw invalid_argument("ipc: null pointer");
    cudaIpcMemHandle_t h;
    KP_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, sizeof(h));
  });
}
int kp_ipc_open_handle(const void* handle64, void** dptr) {
  return guard([&] {
    if (!dptr || !handle64) throw invalid_argument("ipc: null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    KP_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}
int kp_ipc_close_handle(void* dptr) {
  return guard([&] { KP_CUDA(cudaIpcCloseMemHandle(dptr)); });
}

int kp_host_mode_product_f64(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                             const double* m, int rows, int cols, double alpha, double beta,
                             double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "mode_product");
    check_mode(dv, mode, cols);
    auto od = dv;
    od[mode] = rows;
    const size_t nin = numel(dv), nout = numel(od);
    double* din = static_cast<double*>(ctx->ws.get(SLOT_HOST_IN, nin * sizeof(double)));
    double* dout = static_cast<double*>(ctx->ws.get(SLOT_HOST_OUT, nout * sizeof(double)));
    const double* hm[1] = {m};
    auto dm = upload_mats(ctx, SLOT_HOST_MATS, hm, {size_t(rows) * cols});
    h2d(ctx, din, t, nin);
    if (beta != 0.0) h2d(ctx, dout, out, nout);
    Epilogue e;
    e.alpha = alpha;
    e.beta = beta;
    mode_product_f64(ctx, din, dv, mode, dm[0], rows, e, dout);
    d2h(ctx, out, dout, nout);
  });
}

int kp_host_tucker_f64(kp_ctx* ctx, const double* t, const int* dims, int d,
                       const double* const* ms, const int* rows, double prefactor, double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "tucker");
    std::vector<size_t> sizes;
    std::vector<int> od = dv;
    for (int mu = 0; mu < d; ++mu) {
      sizes.push_back(size_t(rows[mu]) * dv[mu]);
      od[mu] = rows[mu];
    }
    auto dm = upload_mats(ctx, SLOT_HOST_MATS, ms, sizes);
    host_tucker_pipelined(ctx, mode_product_f64, 1, &t, dv, dm, rows, prefactor, &out, 1);
  });
}

int kp_host_tucker_stream_f64(kp_ctx* ctx, int count, const double* const* ts, const int* dims,
                              int d, const double* const* ms, const int* rows, double prefactor,
                              double* const* outs) {
  return guard([&] {
    need_ctx(ctx);
    if (count < 0 || (count > 0 && (!ts || !outs)))
      throw invalid_argument("tucker: bad tensor list");
    const auto dv = check_dims(dims, d, "tucker");
    if (count == 0) return;
    std::vector<size_t> sizes;
    for (int mu = 0; mu < d; ++mu) sizes.push_back(size_t(rows[mu]) * dv[mu]);
    auto dm = upload_mats(ctx, SLOT_HOST_MATS, ms, sizes);
    host_tucker_pipelined(ctx, mode_product_f64, 1, ts, dv, dm, rows, prefactor, outs, count);
  });
}

int kp_host_kronsum_f64(kp_ctx* ctx, const double* t, const int* dims, int d,
                        const double* const* as, double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "kronsum_action");
    std::vector<size_t> sizes;
    for (int mu = 0; mu < d; ++mu) sizes.push_back(size_t(dv[mu]) * dv[mu]);
    const size_t n = numel(dv);
    double* din = static_cast<double*>(ctx->ws.get(SLOT_HOST_IN, n * sizeof(double)));
    double* dout = static_cast<double*>(ctx->ws.get(SLOT_HOST_OUT, n * sizeof(double)));
    auto dm = upload_mats(ctx, SLOT_HOST_MATS, as, sizes);
    h2d(ctx, din, t, n);
    if (!kronsum_try_banded(ctx, false, din, dv, dm.data(), dout))
      kronsum_generic(ctx, mode_product_f64, din, dv, dm.data(), dout);
    d2h(ctx, out, dout, n);
  });
}

// ---------------- elementwise ----------------

int kp_axpy_f64(kp_ctx* ctx, size_t n, double alpha, const double* x, double* y) {
  return guard([&] {
    need_ctx(ctx);
    launch_fma(ctx, n, alpha, x, y, y);
  });
}

int kp_add_scaled_f64(kp_ctx* ctx, size_t n, const double* x, double alpha, const double* y,
                      double* z) {
  return guard([&] {
    need_ctx(ctx);
    launch_fma(ctx, n, alpha, y, x, z);
  });
}

int kp_eval_g_f64(kp_ctx* ctx, const kp_gfun* g, double t, const double* u, const int* dims,
                  int d, double* gout) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "g");
    if (!g) throw invalid_argument("g: null descriptor");
    if (g->kind == KP_G_NLS) throw invalid_argument("g: NLS needs a complex tensor");
    if (g->kind == KP_G_RICCATI) {  // src/problems.cpp:263-276, nonlocal
      if (d != 2 || dv[0] != dv[1]) throw invalid_argument("riccati g: needs an n x n state");
      riccati_g(ctx, *g, u, dv[0],
                static_cast<double*>(ctx->ws.get(50, 2 * size_t(dv[0]) * sizeof(double))), gout);
      return;
    }
    size_t half = 0;
    if (g->kind == KP_G_BRUSSELATOR) {
      if (dv.back() != 2)
        throw invalid_argument("brusselator g: slowest mode must hold 2 species");
      half = numel(dv) / 2;
    }
    launch_eval_g(ctx, *g, t, u, numel(dv), half, false, gout);
  });
}

int kp_riccati_jacobian_factors_f64(kp_ctx* ctx, const kp_gfun* g, const double* u,
                                    const double* at, int n, double* j1, double* j2,
                                    int* nfactors) {
  return guard([&] {
    need_ctx(ctx);
    if (!g || g->kind != KP_G_RICCATI || !g->aux[0])
      throw invalid_argument("riccati_jacobian_factors: needs a Riccati g descriptor");
    if (n <= 0 || !u || !at || !j1 || !j2 || !nfactors)
      throw invalid_argument("riccati_jacobian_factors: bad arguments");
    *nfactors = riccati_jacobians(
        ctx, *g, u, at, n, static_cast<double*>(ctx->ws.get(50, 2 * size_t(n) * sizeof(double))),
        j1, j2);
  });
}

int kp_eval_g_c128(kp_ctx* ctx, const kp_gfun* g, double t, const double* u, const int* dims,
                   int d, double* gout) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "g");
    if (!g) throw invalid_argument("g: null descriptor");
    if (g->kind == KP_G_ALLEN_CAHN || g->kind == KP_G_BRUSSELATOR || g->kind == KP_G_ADR ||
        g->kind == KP_G_RICCATI)
      throw invalid_argument("g: unsupported nonlinearity kind for complex");
    launch_eval_g(ctx, *g, t, u, numel(dv), 0, true, gout);
  });
}

int kp_all_finite_f64(kp_ctx* ctx, size_t n, const double* x, int* ok) {
  return guard([&] {
    need_ctx(ctx);
    *ok = all_finite(ctx, n, x);
  });
}

int kp_mark_nonfinite_f64(kp_ctx* ctx, size_t n, const double* x, int* bad_dev, int step) {
  return guard([&] {
    need_ctx(ctx);
    if (!bad_dev) throw invalid_argument("mark_nonfinite: null flag");
    finite_mark(ctx, n, x, bad_dev, step);
  });
}

int kp_measure_fp64_peak(kp_ctx* ctx, double* tflops) {
  return guard([&] {
    need_ctx(ctx);
    *tflops = measure_fp64_peak(ctx);
  });
}

// ---------------- complex128 ----------------

namespace {
void real_scalar(const double* z, const char* what, double* out) {
  if (!z) {
    *out = (std::string(what) == "beta") ? 0.0 : 1.0;
    return;
  }
  if (z[1] != 0.0)
    throw invalid_argument(std::string("mode_product: complex ") + what +
                           " with nonzero imaginary part is not supported");
  *out = z[0];
}
}  // namespace

int kp_mode_product_c128(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                         const double* m, int rows, int cols, const double* alpha2,
                         const double* beta2, double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "mode_product");
    check_mode(dv, mode, cols);
    if (rows <= 0) throw invalid_argument("mode_product: matrix has no rows");
    if (out == t) throw invalid_argument("mode_product: out must not alias the input");
    Epilogue e;
    real_scalar(alpha2, "alpha", &e.alpha);
    real_scalar(beta2, "beta", &e.beta);
    mode_product_c128(ctx, t, dv, mode, m, rows, e, out);
  });
}

int kp_tucker_c128(kp_ctx* ctx, const double* t, const int* dims, int d, const double* const* ms,
                   const int* rows, double prefactor, double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "tucker");
    if (!ms || !rows) throw invalid_argument("tucker: expected one factor per mode");
    for (int mu = 0; mu < d; ++mu)
      if (rows[mu] <= 0) throw invalid_argument("tucker: factor has no rows");
    tucker_c128(ctx, t, dv, ms, rows, prefactor, out);
  });
}

int kp_kronsum_c128(kp_ctx* ctx, const double* t, const int* dims, int d,
                    const double* const* as, double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "kronsum_action");
    if (!as) throw invalid_argument("kronsum_action: expected one factor per mode");
    if (out == t) throw invalid_argument("kronsum_action: out must not alias the input");
    if (!kronsum_try_banded(ctx, true, t, dv, as, out))
      kronsum_generic(ctx, mode_product_c128, t, dv, as, out);
  });
}

int kp_host_tucker_c128(kp_ctx* ctx, const double* t, const int* dims, int d,
                        const double* const* ms, const int* rows, double prefactor,
                        double* out) {
  return guard([&] {
    need_ctx(ctx);
    const auto dv = check_dims(dims, d, "tucker");
    std::vector<size_t> sizes;
    std::vector<int> od = dv;
    for (int mu = 0; mu < d; ++mu) {
      sizes.push_back(2 * size_t(rows[mu]) * dv[mu]);
      od[mu] = rows[mu];
    }
    auto dm = upload_mats(ctx, SLOT_HOST_MATS, ms, sizes);
    host_tucker_pipelined(ctx, mode_product_c128, 2, &t, dv, dm, rows, prefactor, &out, 1);
  });
}

}  // extern "C"
