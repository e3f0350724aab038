// kp_internal.h -- shared host-side declarations of the kronphi_b200 library.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "kronphi_b200.h"

namespace kp {

// Exceptions thrown inside the library and mapped to status codes at the C
// boundary (capi.cpp).  Same taxonomy as the reference's exceptions.
struct invalid_argument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct runtime_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct divergence_error : std::runtime_error {
  long step;
  divergence_error(const std::string& m, long s) : std::runtime_error(m), step(s) {}
};

void kp_set_last_error(const std::string& m);

#define KP_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::kp::cuda_error(std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per device, so a process driving several GPUs needs it
// on each (capi.cpp).
void ensure_smem_attr(kp_ctx* ctx, const void* kernel, int bytes);

// Grow-only device scratch with a few named slots (ping-pong buffers of the
// Tucker operator, stepper temporaries).  No cudaMalloc on the hot path after
// the first call at a given size.
struct Workspace {
  std::vector<void*> ptr;
  std::vector<size_t> cap;
  void* get(int slot, size_t bytes);
  void release();
};

struct PinnedStage {
  void* ptr = nullptr;
  size_t cap = 0;
  void* get(size_t bytes);
  void release();
};

}  // namespace kp

struct kp_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  unsigned long long launches = 0;
  kp::Workspace ws;
  kp::PinnedStage pin_in, pin_out;
  double* d_flag = nullptr;  // small device scratch (finite flag etc.)
  int* h_flag = nullptr;     // pinned host mirror
};

namespace kp {

// ---- GEMM-shaped mode-product core (mode_product.cu) ----
// C_q(m,n) = epi(alpha * sum_k A_q(m,k) B_q(k,n), ...), q < batch, with
//   A_q(m,k) = A[q*sA + m + k*lda]                 (M-contiguous)
//   B_q(k,n) = B[q*sB + k*sBk + n*sBn]             (sBk==1 or sBn==1)
//   C_q(m,n) = C[q*sC + m + n*ldc]                 (M-contiguous)
enum EpiKind : int {
  EPI_STORE = 0,    // C = alpha*acc + beta*C
  EPI_FMA_X = 1,    // C = fma(gamma, alpha*acc, X)             (add_scaled)
  EPI_ADD_G = 2,    // C = (alpha*acc + beta*C) + g(t, X)        (kronsum + g)
  EPI_STAGE_D = 3,  // S = fma(gamma, alpha*acc, X); C = S; D = g(t2, S) - g(t, X)
  EPI_ADD_X = 4,    // C = (alpha*acc + beta*C) + X   (kronsum + a precomputed g)
};

struct Epilogue {
  int kind = EPI_STORE;
  double alpha = 1.0, beta = 0.0, gamma = 0.0;
  const double* X = nullptr;  // same layout as C
  double* D = nullptr;        // second output (EPI_STAGE_D)
  kp_gfun g{};
  double t = 0.0, t2 = 0.0;
  // divergence tracking (inc/integrators.hpp:364): when set, any non-finite
  // value written by this epilogue records atomicMin(*bad_step, *step_ctr + 1)
  int* bad_step = nullptr;
  const int* step_ctr = nullptr;
  // step counter of the NEXT step (integrate's two alternating slots): the
  // last kernel of a step writes *step_next = *step_ctr + 1 (one thread), so
  // no separate counter kernel is launched per step
  int* step_next = nullptr;
  // fused exchange (kp_scatter): C's entries go to peer buffers instead
  int sc_dir = 0;  // 0: store into C; 1: slab -> pencil; 2: pencil -> slab
  int sc_P = 1, sc_rank = 0;
  unsigned sc_A = 1, sc_B = 1, sc_C = 1;
  double* const* sc_peers = nullptr;  // device array of P pointers
};

struct GemmProblem {
  int M = 0, N = 0, K = 0, batch = 1;
  const double* A = nullptr;
  long long lda = 0, sA = 0;
  const double* B = nullptr;
  long long sBk = 0, sBn = 0, sB = 0;
  double* C = nullptr;
  long long ldc = 0, sC = 0;
};

// The plain re-partition (exchange.cu): entry i of x (comps doubles) stored at
// its kp_scatter destination (e.sc_*).
void scatter_copy(kp_ctx* ctx, const double* x, long long n, int comps, const Epilogue& e);

// The hand-written warp-specialized TMA/DMMA GEMM (gemm_dmma.cu): launch_gemm's path.
void launch_gemm_dmma(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, int cplx,
                      bool kcontig, long long half);

// cplx: 0 real, 1 complex rows (mode 0), 2 complex combine (mode >= 1); see mode_product.cu
void launch_gemm(kp_ctx* ctx, const GemmProblem& p, const Epilogue& e, int cplx = 0);

// Real mode product out = epi(t x_mode M) on device pointers.
void mode_product_f64(kp_ctx* ctx, const double* t, const std::vector<int>& dims, int mode,
                      const double* m, int rows, const Epilogue& e, double* out);

// Modes 0 and 1 of a Tucker operator fused per N x N slice (fused01.cu):
// out = e1((alpha0 * in x_0 m0) x_1 m1).  false = not applicable.
bool fused01_f64(kp_ctx* ctx, const double* in, const std::vector<int>& dims, const double* m0,
                 int rows0, const double* m1, int rows1, double alpha0, const Epilogue& e1,
                 double* out);

// Complex mode product (interleaved complex128, cplx.cu).  m is rows x dims[mode].
void mode_product_c128(kp_ctx* ctx, const double* t, const std::vector<int>& dims, int mode,
                       const double* m, int rows, const Epilogue& e, double* out);

// ---- matrix functions (phi.cu, gll_rule.cpp) ----
void gll_rule_host(int q, double* nodes, double* weights);
// expm of `batch` consecutive n x n matrices (inc/matrix_functions.hpp:76-95)
void expm_batch(kp_ctx* ctx, const double* x, int n, int batch, double* out);
// x = a^{-1} b (lu_factor + lu_solve, inc/linsolve.hpp:95-151); a n x n, b/x n x nrhs
void solve_dev(kp_ctx* ctx, const double* a, int n, const double* b, int nrhs, double* x);
// lu_factor / lu_solve (inc/linsolve.hpp:95-146) split: a factored in place,
// piv = n device ints; b (n x nrhs) overwritten with the solution
void lu_factor_dev(kp_ctx* ctx, double* a, int n, int* piv);
void lu_solve_dev(kp_ctx* ctx, const double* lu, const int* piv, int n, double* b, int nrhs);
// phiquad (inc/matrix_functions.hpp:146-199): phis = ell_max+1 consecutive
// n x n matrices; returns the scaling exponent
int phiquad_dev(kp_ctx* ctx, const double* x, int n, int ell_max, int q, int forced, double* phis);
// complex128 (interleaved) versions through the real 2n x 2n representation
void expm_batch_c128(kp_ctx* ctx, const double* x, int n, int batch, double* out);
int phiquad_dev_c128(kp_ctx* ctx, const double* x, int n, int ell_max, int q, int forced,
                     double* phis);

// ---- Riccati problem (riccati.cu) ----
void riccati_g(kp_ctx* ctx, const kp_gfun& g, const double* u, int n, double* wz, double* out);
int riccati_jacobians(kp_ctx* ctx, const kp_gfun& g, const double* u, const double* at, int n,
                      double* wz, double* j1, double* j2);

// ---- banded Kronecker sum (banded.cu) ----
bool banded_kronsum_enabled();  // KP_KRONSUM=dense disables
bool band_of(kp_ctx* ctx, const double* a, int n, bool cplx, int** cols, double** vals);
bool kronsum_try_banded(kp_ctx* ctx, bool cplx, const double* t, const std::vector<int>& dims,
                        const double* const* as, double* out);
// half > 0: Brusselator g (species = last mode).  slab >= 0: the input holds
// `halo` extra planes on each side of mode `slab`, whose interior starts at
// global plane k0 of n_glob (sharded runs); slab = -1: plain tensor.
void kronsum_banded(kp_ctx* ctx, bool cplx, const double* u, const std::vector<int>& dims,
                    const std::vector<const int*>& cols, const std::vector<const double*>& vals,
                    const std::vector<char>& active, double* r, bool with_g, const kp_gfun& g,
                    long long half, int slab = -1, int k0 = 0, int n_glob = 0, int halo = 0,
                    double t = 0.0);

// ---- communicator internals (comm.cu), used by the sharded integrator ----
int comm_size(const kp_comm* c);
int comm_rank(const kp_comm* c);
// pack (slab/pencil -> send blocks) or unpack (recv blocks -> pencil/slab)
void repartition_pack(kp_ctx* ctx, int dir, int P, int rank, long long A, long long B,
                      long long C, long long S, int comps, const double* x, double* y,
                      bool pack);
void comm_repartition(kp_ctx* ctx, kp_comm* c, int dir, long long A, long long B, long long C,
                      long long S, int comps, const double* x, double* y, double* send,
                      double* recv);
void comm_sendrecv(kp_ctx* ctx, kp_comm* c, const std::vector<const double*>& sends,
                   const std::vector<int>& to, const std::vector<double*>& recvs,
                   const std::vector<int>& from, size_t count);
void comm_reduce_scatter(kp_ctx* ctx, kp_comm* c, const double* send, double* recv,
                         size_t count);
void comm_allreduce(kp_ctx* ctx, kp_comm* c, double* x, size_t n, int op);
void comm_allgather_bytes(kp_ctx* ctx, kp_comm* c, const void* send, void* recv, size_t bytes);

// the whole exp-Euler loop of a 128 x 128 real state in one cluster launch
// (banded.cu small2d_expeuler_kernel); false = not applicable
bool small2d_expeuler(kp_ctx* ctx, const std::vector<int>& dims,
                      const std::vector<const int*>& cols, const std::vector<const double*>& vals,
                      const double* L, const kp_gfun& g, double tau, long n_steps, double* u,
                      int* bad);

// ---- steppers (stepper.cu) ----
// d = g(t + tau, s) - g(t, u); half > 0: Brusselator species offset
void gdiff_dev(kp_ctx* ctx, const kp_gfun& g, double t, double tau, const double* s,
               const double* u, long long n, long long half, bool cplx, double* dd);

// ---- elementwise (elementwise.cu) ----
// z = fma(b, y, x): axpy is (b=alpha, y=x, x=y, z=y), add_scaled is (b=alpha, y=y, x=x)
void launch_fma(kp_ctx* ctx, size_t n, double b, const double* y, const double* x, double* z);
// out = g(t, u); n entries (complex: n complex entries); half > 0 = Brusselator
// species offset (u = [0, half), v = [half, 2 half)).
void launch_eval_g(kp_ctx* ctx, const kp_gfun& g, double t, const double* u, size_t n,
                   size_t half, bool cplx, double* out);
void launch_scale(kp_ctx* ctx, size_t n, double a, const double* x, double* y);
int all_finite(kp_ctx* ctx, size_t n, const double* x);
// atomicMin(*bad, step) if x has a non-finite entry (no host sync)
void finite_mark(kp_ctx* ctx, size_t n, const double* x, int* bad, int step);
// device divergence flag: atomicMin(*bad, *ctr + 1) if x has a non-finite entry
void finite_flag(kp_ctx* ctx, size_t n, const double* x, int* bad, const int* ctr);
double measure_fp64_peak(kp_ctx* ctx);

}  // namespace kp
