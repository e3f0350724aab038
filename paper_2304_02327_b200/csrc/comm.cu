// comm.cu -- the native multi-GPU plumbing of the C ABI: an NCCL communicator
// created from an ncclUniqueId (SURVEY.md 8(b) replacement contract) and the
// two exchanges the slab-sharded integrators need:
//   * the slab <-> pencil re-partition around the last mode product (option
//     A: all-to-all pencil transpose), as pack kernel -> grouped
//     ncclSend/ncclRecv -> unpack kernel on the context's stream;
//   * the one-plane halo exchange of the banded Kronecker sum.
// The pack / unpack halves are exported on their own so a host with another
// transport (MPI, its own IPC) can drive the same layout.  NCCL is loaded
// with dlopen on first use, so the library itself has no link-time NCCL
// dependency (torch's bundled libnccl is reused when it is already loaded).
//
// Layouts (same as kp_scatter): slab (A, B, C/P, S), pencil (A, B/P, C, S),
// column-major.  The block rank r sends to rank s is the sub-tensor
// (a, bl, cl, sp) of size A x B/P x C/P x S, contiguous in that order:
//   dir 1 (slab -> pencil): slab entry (a, b = s Bp + bl, cl, sp)
//                           lands at pencil (a, bl, c = r Cl + cl, sp) of s;
//   dir 2 (pencil -> slab): pencil entry (a, bl, c = s Cl + cl, sp)
//                           lands at slab (a, b = r Bp + bl, cl, sp) of s.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "kp_internal.h"

struct kp_comm {
  ncclComm_t nc = nullptr;
  int P = 1, rank = 0, device = 0;
};

namespace kp {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("NCCL not found: ") + dlerror();
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ReduceScatter = reinterpret_cast<decltype(a.ReduceScatter)>(sym("ncclReduceScatter"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GroupStart &&
           a.GroupEnd && a.GetErrorString && a.ReduceScatter && a.AllReduce && a.AllGather;
    if (!a.ok) a.why = "NCCL library lacks the point-to-point API";
    return a;
  }();
  return api;
}

const NcclApi& need_nccl() {
  const NcclApi& a = nccl();
  if (!a.ok) throw runtime_error(a.why);
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw runtime_error(std::string(what) + ": " + nccl().GetErrorString(r));
}

struct Part {
  unsigned A, B, C, S, P, rank;
};

// local linear index of the packed/unpacked entry `i` (i runs over the
// local tensor); returns the index on the other side of the map.
//   pack   : local (slab/pencil) index i -> send-buffer index
//   unpack : recv-buffer index i        -> local (pencil/slab) index
__device__ __forceinline__ unsigned long long pack_index(const Part& p, int dir, unsigned i) {
  const unsigned Bp = p.B / p.P, Cl = p.C / p.P;
  const unsigned long long blk = (unsigned long long)p.A * Bp * Cl * p.S;
  const unsigned t = i / p.A, a = i - t * p.A;
  unsigned s, bl, cl, sp;
  if (dir == 1) {  // slab (a, b, cl, sp)
    const unsigned t2 = t / p.B, b = t - t2 * p.B;
    sp = t2 / Cl;
    cl = t2 - sp * Cl;
    s = b / Bp;
    bl = b - s * Bp;
  } else {  // pencil (a, bl, c, sp)
    const unsigned t2 = t / Bp;
    bl = t - t2 * Bp;
    sp = t2 / p.C;
    const unsigned c = t2 - sp * p.C;
    s = c / Cl;
    cl = c - s * Cl;
  }
  return s * blk + a + (unsigned long long)p.A * (bl + (unsigned long long)Bp * (cl + (unsigned long long)Cl * sp));
}

__device__ __forceinline__ unsigned long long unpack_index(const Part& p, int dir, unsigned i) {
  const unsigned Bp = p.B / p.P, Cl = p.C / p.P;
  const unsigned blk = p.A * Bp * Cl * p.S;
  const unsigned r = i / blk, w = i - r * blk;
  const unsigned t = w / p.A, a = w - t * p.A;
  const unsigned bl = t % Bp, t2 = t / Bp;
  const unsigned cl = t2 % Cl, sp = t2 / Cl;
  if (dir == 1)  // -> pencil (a, bl, c = r Cl + cl, sp)
    return a + (unsigned long long)p.A * (bl + (unsigned long long)Bp * (r * Cl + cl + (unsigned long long)p.C * sp));
  // -> slab (a, b = r Bp + bl, cl, sp)
  return a + (unsigned long long)p.A * ((r * Bp + bl) + (unsigned long long)p.B * (cl + (unsigned long long)Cl * sp));
}

// y[map(i)] = x[i] (pack) or y[map(i)] = x[i] with the unpack map; reads
// coalesced, writes in runs of A entries
template <int COMPS, bool PACK>
__global__ void repartition_kernel(Part p, int dir, unsigned n, const double* __restrict__ x,
                                   double* __restrict__ y) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long j = PACK ? pack_index(p, dir, i) : unpack_index(p, dir, i);
    if constexpr (COMPS == 2)
      reinterpret_cast<double2*>(y)[j] = reinterpret_cast<const double2*>(x)[i];
    else
      y[j] = x[i];
  }
}

Part make_part(int dir, int P, int rank, long long A, long long B, long long C, long long S,
               int comps, long long* n_local) {
  if (dir != 1 && dir != 2) throw invalid_argument("repartition: dir must be 1 or 2");
  if (P < 1 || rank < 0 || rank >= P) throw invalid_argument("repartition: bad rank");
  if (comps != 1 && comps != 2) throw invalid_argument("repartition: comps must be 1 or 2");
  if (A < 1 || B < 1 || C < 1 || S < 1 || B % P || C % P)
    throw invalid_argument("repartition: B and C must be divisible by P");
  const long long n = A * B * C * S / P;
  if (A * B * C * S > 0xffffffffLL) throw invalid_argument("repartition: tensor too large");
  *n_local = n;
  return Part{unsigned(A), unsigned(B), unsigned(C), unsigned(S), unsigned(P), unsigned(rank)};
}

void launch_repartition(kp_ctx* ctx, const Part& p, int dir, bool pack, int comps, long long n,
                        const double* x, double* y) {
  if (n <= 0) return;
  const unsigned grid = unsigned(std::min<long long>((n + 255) / 256, ctx->num_sms * 16LL));
  if (comps == 2)
    pack ? repartition_kernel<2, true><<<grid, 256, 0, ctx->stream>>>(p, dir, unsigned(n), x, y)
         : repartition_kernel<2, false><<<grid, 256, 0, ctx->stream>>>(p, dir, unsigned(n), x, y);
  else
    pack ? repartition_kernel<1, true><<<grid, 256, 0, ctx->stream>>>(p, dir, unsigned(n), x, y)
         : repartition_kernel<1, false><<<grid, 256, 0, ctx->stream>>>(p, dir, unsigned(n), x, y);
  ctx->launches++;
  KP_CUDA(cudaGetLastError());
}

// equal-block all-to-all of `count` doubles per rank on ctx's stream
void alltoall(kp_ctx* ctx, kp_comm* c, const double* send, double* recv, size_t count) {
  const NcclApi& a = need_nccl();
  nccl_check(a.GroupStart(), "ncclGroupStart");
  for (int s = 0; s < c->P; ++s) {
    nccl_check(a.Send(send + size_t(s) * count, count, ncclFloat64, s, c->nc, ctx->stream),
               "ncclSend");
    nccl_check(a.Recv(recv + size_t(s) * count, count, ncclFloat64, s, c->nc, ctx->stream),
               "ncclRecv");
  }
  nccl_check(a.GroupEnd(), "ncclGroupEnd");
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

void need(kp_ctx* ctx, kp_comm* c) {
  if (!ctx) throw invalid_argument("kronphi_b200: null context");
  if (!c) throw invalid_argument("kronphi_b200: null communicator");
  if (c->device != ctx->device)
    throw invalid_argument("kronphi_b200: communicator and context are on different devices");
  KP_CUDA(cudaSetDevice(ctx->device));
}

constexpr int SLOT_SEND = 64, SLOT_RECV = 65;  // distinct from every other slot (phi.cu uses 20..58)

}  // namespace

// ---- internal entry points for the sharded integrator (stepper.cu) ----
int comm_size(const kp_comm* c) { return c->P; }
int comm_rank(const kp_comm* c) { return c->rank; }

void repartition_pack(kp_ctx* ctx, int dir, int P, int rank, long long A, long long B,
                      long long C, long long S, int comps, const double* x, double* send,
                      bool pack) {
  long long n = 0;
  const Part p = make_part(dir, P, rank, A, B, C, S, comps, &n);
  launch_repartition(ctx, p, dir, pack, comps, n, x, send);
}

void comm_repartition(kp_ctx* ctx, kp_comm* c, int dir, long long A, long long B, long long C,
                      long long S, int comps, const double* x, double* y, double* send,
                      double* recv) {
  long long n = 0;
  const Part p = make_part(dir, c->P, c->rank, A, B, C, S, comps, &n);
  if (c->P == 1) {
    if (x != y)
      KP_CUDA(cudaMemcpyAsync(y, x, size_t(n) * comps * sizeof(double), cudaMemcpyDeviceToDevice,
                              ctx->stream));
    return;
  }
  launch_repartition(ctx, p, dir, true, comps, n, x, send);
  alltoall(ctx, c, send, recv, size_t(n / c->P) * comps);
  launch_repartition(ctx, p, dir, false, comps, n, recv, y);
}

// grouped send/recv of `count` doubles from each (src, dst) pair below:
// sends[i] -> rank to[i], recvs[i] <- rank from[i]
void comm_sendrecv(kp_ctx* ctx, kp_comm* c, const std::vector<const double*>& sends,
                   const std::vector<int>& to, const std::vector<double*>& recvs,
                   const std::vector<int>& from, size_t count) {
  const NcclApi& a = need_nccl();
  nccl_check(a.GroupStart(), "ncclGroupStart");
  for (size_t i = 0; i < sends.size(); ++i)
    nccl_check(a.Send(sends[i], count, ncclFloat64, to[i], c->nc, ctx->stream), "ncclSend");
  for (size_t i = 0; i < recvs.size(); ++i)
    nccl_check(a.Recv(recvs[i], count, ncclFloat64, from[i], c->nc, ctx->stream), "ncclRecv");
  nccl_check(a.GroupEnd(), "ncclGroupEnd");
}

// recv (count doubles) = sum over ranks of chunk `rank` of send (P chunks)
void comm_reduce_scatter(kp_ctx* ctx, kp_comm* c, const double* send, double* recv,
                         size_t count) {
  nccl_check(need_nccl().ReduceScatter(send, recv, count, ncclFloat64, ncclSum, c->nc,
                                       ctx->stream),
             "ncclReduceScatter");
}

// recv = the P ranks' `bytes`-long send blocks, rank order (device buffers)
void comm_allgather_bytes(kp_ctx* ctx, kp_comm* c, const void* send, void* recv, size_t bytes) {
  nccl_check(need_nccl().AllGather(send, recv, bytes, ncclUint8, c->nc, ctx->stream),
             "ncclAllGather");
}

// in place: x = op over ranks (op 0 min, 1 max), n doubles
void comm_allreduce(kp_ctx* ctx, kp_comm* c, double* x, size_t n, int op) {
  nccl_check(need_nccl().AllReduce(x, x, n, ncclFloat64, op == 0 ? ncclMin : ncclMax, c->nc,
                                   ctx->stream),
             "ncclAllReduce");
}

}  // namespace kp

using namespace kp;

extern "C" {

int kp_comm_unique_id(void* id128) {
  return guard([&] {
    if (!id128) throw invalid_argument("comm: null id buffer");
    ncclUniqueId id;
    nccl_check(need_nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id128, &id, sizeof(id));
  });
}

int kp_comm_create(kp_ctx* ctx, int nranks, int rank, const void* id128, kp_comm** out) {
  return guard([&] {
    if (!ctx || !out || !id128) throw invalid_argument("comm: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw invalid_argument("comm: bad rank");
    KP_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    auto* c = new kp_comm;
    c->P = nranks;
    c->rank = rank;
    c->device = ctx->device;
    const ncclResult_t r = need_nccl().CommInitRank(&c->nc, nranks, id, rank);
    if (r != ncclSuccess) {
      delete c;
      nccl_check(r, "ncclCommInitRank");
    }
    *out = c;
  });
}

int kp_comm_destroy(kp_comm* c) {
  return guard([&] {
    if (!c) return;
    if (c->nc) nccl_check(need_nccl().CommDestroy(c->nc), "ncclCommDestroy");
    delete c;
  });
}

int kp_comm_alltoall_f64(kp_ctx* ctx, kp_comm* c, const double* send, double* recv,
                         long long count) {
  return guard([&] {
    need(ctx, c);
    if (count < 0 || (count > 0 && (!send || !recv)))
      throw invalid_argument("alltoall: bad buffers");
    if (count > 0) alltoall(ctx, c, send, recv, size_t(count));
  });
}

int kp_repartition_pack(kp_ctx* ctx, int dir, int P, int rank, long long A, long long B,
                        long long C, long long S, int comps, const double* x, double* send) {
  return guard([&] {
    if (!ctx) throw invalid_argument("kronphi_b200: null context");
    KP_CUDA(cudaSetDevice(ctx->device));
    long long n = 0;
    const Part p = make_part(dir, P, rank, A, B, C, S, comps, &n);
    launch_repartition(ctx, p, dir, true, comps, n, x, send);
  });
}

int kp_repartition_unpack(kp_ctx* ctx, int dir, int P, int rank, long long A, long long B,
                          long long C, long long S, int comps, const double* recv, double* y) {
  return guard([&] {
    if (!ctx) throw invalid_argument("kronphi_b200: null context");
    KP_CUDA(cudaSetDevice(ctx->device));
    long long n = 0;
    const Part p = make_part(dir, P, rank, A, B, C, S, comps, &n);
    launch_repartition(ctx, p, dir, false, comps, n, recv, y);
  });
}

int kp_comm_repartition(kp_ctx* ctx, kp_comm* c, int dir, long long A, long long B, long long C,
                        long long S, int comps, const double* x, double* y) {
  return guard([&] {
    need(ctx, c);
    long long n = 0;
    const Part p = make_part(dir, c->P, c->rank, A, B, C, S, comps, &n);
    const size_t bytes = size_t(n) * comps * sizeof(double);
    if (c->P == 1) {  // slab == pencil: the map is the identity
      if (x != y) KP_CUDA(cudaMemcpyAsync(y, x, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      return;
    }
    double* send = static_cast<double*>(ctx->ws.get(SLOT_SEND, bytes));
    double* recv = static_cast<double*>(ctx->ws.get(SLOT_RECV, bytes));
    launch_repartition(ctx, p, dir, true, comps, n, x, send);
    alltoall(ctx, c, send, recv, size_t(n / c->P) * comps);
    launch_repartition(ctx, p, dir, false, comps, n, recv, y);
  });
}

int kp_comm_halo_f64(kp_ctx* ctx, kp_comm* c, const double* first, const double* last,
                     long long count, double* left, double* right) {
  return guard([&] {
    need(ctx, c);
    if (count <= 0) return;
    const NcclApi& a = need_nccl();
    const int P = c->P, up = (c->rank + 1) % P, down = (c->rank + P - 1) % P;
    nccl_check(a.GroupStart(), "ncclGroupStart");
    nccl_check(a.Send(last, size_t(count), ncclFloat64, up, c->nc, ctx->stream), "ncclSend");
    nccl_check(a.Recv(left, size_t(count), ncclFloat64, down, c->nc, ctx->stream), "ncclRecv");
    nccl_check(a.Send(first, size_t(count), ncclFloat64, down, c->nc, ctx->stream), "ncclSend");
    nccl_check(a.Recv(right, size_t(count), ncclFloat64, up, c->nc, ctx->stream), "ncclRecv");
    nccl_check(a.GroupEnd(), "ncclGroupEnd");
  });
}

}  // extern "C"
