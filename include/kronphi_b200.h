/*
 * kronphi_b200.h -- C ABI of the B200-native direction-split phi library.
 *
 * Drop-in boundary for the hot path of the reference library `kronphi`
 * (arXiv 2304.02327, /root/reference/proj; prefix inc/ = proj/include/kronphi/).
 * The reference has no FFI; its boundary is the C++ template API in inc/.
 * Each entry point below names the reference function it replaces.  The C++
 * layer include/kronphi_b200/kronphi.hpp re-exposes the reference's C++
 * signatures on top of this ABI (same names, argument meaning, exceptions).
 *
 * Conventions
 *  - Column-major tensors, first index fastest (inc/tensor.hpp:1-2); matrices
 *    column-major (inc/matrix.hpp:58-59).  Complex data is interleaved
 *    (re, im) exactly like std::complex<double>.
 *  - kp_* compute calls take DEVICE pointers and are stream-ordered on the
 *    context's stream; kp_host_* calls take HOST pointers, stage through the
 *    context's pinned buffers and return when the result is on the host.
 *  - Arrays of per-mode pointers (ms, as, factors) are HOST arrays holding
 *    device (kp_*) or host (kp_host_*) pointers.
 *  - Status codes map to the reference's exception types:
 *      KP_EINVAL   -> std::invalid_argument (message names the mode, as
 *                     inc/mode_product.hpp:51-55)
 *      KP_ERUNTIME -> std::runtime_error (singular LU, inc/linsolve.hpp:39)
 *      KP_EDIVERGE -> kronphi::DivergenceError (inc/integrators.hpp:86-97)
 *      KP_ECUDA    -> CUDA failure (message carries cudaGetErrorString)
 *    kp_last_error() returns the calling thread's last message.
 *  - One context is not thread-safe across threads sharing its stream (the
 *    reference's functions are reentrant per call; here reentrancy is per
 *    context).
 */
#ifndef KRONPHI_B200_H
#define KRONPHI_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KP_OK 0
#define KP_EINVAL 1
#define KP_ERUNTIME 2
#define KP_EDIVERGE 3
#define KP_ECUDA 4

typedef struct kp_ctx kp_ctx;

/* Methods: same order as kronphi::Method (inc/integrators.hpp:24-31). */
#define KP_LAWSON_EULER 0
#define KP_LAWSON2B 1
#define KP_EXP_EULER 2
#define KP_EXP_EULER_LS 3
#define KP_ETD2RK 4
#define KP_ROSENBROCK_EULER 5 /* per-step phi_1 of the Jacobian factors (RICCATI g only) */

/* Closed set of device nonlinearities g(t,u) replacing the reference's host
 * std::function (inc/integrators.hpp:60,112). */
#define KP_G_ZERO 0
#define KP_G_SQUARE 1
#define KP_G_CONST 2       /* p[0] */
#define KP_G_ALLEN_CAHN 3  /* u - u^3 */
#define KP_G_BRUSSELATOR 4 /* species stacked as the slowest mode (size 2); p[0]=a, p[1]=b */
#define KP_G_NLS 5         /* -i |u|^2 u, complex */
#define KP_G_ADR 6         /* 1/(1+u^2) + e^t psi_a - 1/(1+e^{2t} u0^2): the reference's
                              ADR source (src/problems.cpp:101-115); aux[0] = psi_a,
                              aux[1] = u0^2 (device arrays shaped like u) */

#define KP_G_RICCATI 7     /* C + U B U = C - (U b)(U^T b)^T on an n x n state (d = 2):
                              the reference's LQR Riccati g (src/problems.cpp:263-276);
                              aux[0] = b (n), aux[1] = C (n x n); Rosenbrock-Euler's
                              Jacobian factors J = A^T - w b^T (:212-250) need the K
                              factors to be {A^T, A^T} */

/* step_ctr/t0/tau: when step_ctr is set (the integrators do this), a
 * time-dependent g reads t = t0 + (*step_ctr) * tau (+ the stage offset) from
 * the device step counter, so captured CUDA-graph steps see the right t. */
typedef struct {
  int kind;
  double p[4];
  const double* aux[2];
  const int* step_ctr;
  double t0, tau;
} kp_gfun;

/* ---------------- context, memory, errors ---------------- */
const char* kp_last_error(void);
int kp_ctx_create(int device, kp_ctx** out);
int kp_ctx_destroy(kp_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL means the legacy default stream, as in CUDA. */
int kp_ctx_set_stream(kp_ctx* ctx, void* stream);
/* Go back to the context's own non-blocking stream (the initial state). */
int kp_ctx_use_own_stream(kp_ctx* ctx);
void* kp_ctx_get_stream(kp_ctx* ctx);
int kp_ctx_synchronize(kp_ctx* ctx);
/* Number of kernels this context has launched (bench.py's gpu_launches). */
unsigned long long kp_ctx_launch_count(kp_ctx* ctx);

int kp_malloc(kp_ctx* ctx, size_t bytes, void** ptr);
int kp_free(kp_ctx* ctx, void* ptr);
int kp_upload(kp_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);
int kp_download(kp_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);
int kp_memset(kp_ctx* ctx, void* dst_dev, int value, size_t bytes);
/* Device-to-device copy on the context's stream; either side may be a peer
 * mapping (CUDA IPC) of another GPU's memory (NVLink P2P). */
int kp_copy(kp_ctx* ctx, void* dst_dev, const void* src_dev, size_t bytes);

/* ---------------- mu-mode / Tucker / Kronecker sum ---------------- */
/* out = alpha * (t x_mode M) + beta * out.
 * Replaces mode_product_into (inc/mode_product.hpp:61-87; beta = 1 is its
 * accumulate=true) and mode_product (:89-97).  M is rows x cols with
 * cols == dims[mode]; out has dims with dims[mode] -> rows.  out must not
 * alias t. */
int kp_mode_product_f64(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                        const double* m, int rows, int cols, double alpha, double beta,
                        double* out);
int kp_mode_product_c128(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                         const double* m, int rows, int cols, const double* alpha2,
                         const double* beta2, double* out);

/* ETD2RK's stage in the epilogue of the last mode product
 * (inc/integrators.hpp:157-162): out = fma(gamma, alpha * (t x_mode M), x)
 * and, when g and d_out are given, d_out = g(t2, out) - g(t1, x) in the same
 * pass (the coupled Brusselator g as one extra paired pass).  M square
 * (rows = dims[mode]).  Used by the slab-sharded integrators, whose last mode
 * runs in the pencil layout; the single-GPU integrate fuses it internally. */
int kp_mode_product_stage_f64(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                              const double* m, int rows, double alpha, const double* x,
                              double gamma, const kp_gfun* g, double t1, double t2, double* out,
                              double* d_out);
int kp_mode_product_stage_c128(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                               const double* m, int rows, double alpha, const double* x,
                               double gamma, const kp_gfun* g, double t1, double t2,
                               double* out, double* d_out);

/* C = alpha * A * op(B) + beta * C on device pointers, column-major.
 * Replaces gemm (inc/kernels.hpp:279-327): A m x k (lda), op(B) k x n with
 * opb 0 = Op::none (B k x n, ldb) or 1 = Op::transpose (B n x k, ldb), C m x n
 * (ldc).  _c128: interleaved complex128, alpha2/beta2 = (re, im). */
int kp_gemm_f64(kp_ctx* ctx, int m, int n, int k, double alpha, const double* a, int lda,
                const double* b, int ldb, int opb, double beta, double* c, int ldc);
int kp_gemm_c128(kp_ctx* ctx, int m, int n, int k, const double* alpha2, const double* a,
                 int lda, const double* b, int ldb, int opb, const double* beta2, double* c,
                 int ldc);
/* C_q = alpha * A_q * op(B) + beta * C_q for q < batch, A_q = a + q*a_stride,
 * C_q = c + q*c_stride (strides in elements).  Replaces gemm_batch_shared_b
 * (inc/kernels.hpp:332-392). */
int kp_gemm_batch_shared_b_f64(kp_ctx* ctx, int m, int n, int k, double alpha, const double* a,
                               int lda, long long a_stride, const double* b, int ldb, int opb,
                               double beta, double* c, int ldc, long long c_stride, int batch);
int kp_gemm_batch_shared_b_c128(kp_ctx* ctx, int m, int n, int k, const double* alpha2,
                                const double* a, int lda, long long a_stride, const double* b,
                                int ldb, int opb, const double* beta2, double* c, int ldc,
                                long long c_stride, int batch);
/* lu_factor (inc/linsolve.hpp:95-117): a (n x n) factored in place (unit
 * lower L below the diagonal, U on and above), piv = n device ints; a
 * singular matrix -> KP_ERUNTIME "lu_factor: matrix is singular".
 * lu_solve (:119-146): b (n x nrhs) overwritten with the solution. */
int kp_lu_factor_f64(kp_ctx* ctx, double* a, int n, int* piv);
int kp_lu_solve_f64(kp_ctx* ctx, const double* lu, const int* piv, int n, double* b, int nrhs);

/* out = ((prefactor * t) x_1 M_1 x_2 ... x_d M_d).
 * Replaces tucker (inc/mode_product.hpp:101-108) with prefactor = 1 and
 * apply_split_phi (inc/split_phi.hpp:53-62) with prefactor = (l!)^(d-1).
 * M_mu is rows[mu] x dims[mu].  Intermediates live in the context's
 * workspace; out may alias t. */
int kp_tucker_f64(kp_ctx* ctx, const double* t, const int* dims, int d,
                  const double* const* ms, const int* rows, double prefactor, double* out);
int kp_tucker_c128(kp_ctx* ctx, const double* t, const int* dims, int d,
                   const double* const* ms, const int* rows, double prefactor, double* out);

/* out = sum_mu t x_mu A_mu.  Replaces kronsum_action (inc/mode_product.hpp:111-121).
 * out must not alias t. */
int kp_kronsum_f64(kp_ctx* ctx, const double* t, const int* dims, int d,
                   const double* const* as, double* out);
int kp_kronsum_c128(kp_ctx* ctx, const double* t, const int* dims, int d,
                    const double* const* as, double* out);

/* The Kronecker-sum action on one slab of a slab-sharded tensor, for banded
 * factors (at most three nonzeros per row: the configs' tridiagonal and
 * periodic operators) -- kronsum_action (inc/mode_product.hpp:111-121) as a
 * stencil with the reference's rounding.  u_ext holds the rank's slab of
 * mode `slab_mode` (interior dims `dims`) plus one halo plane on each side
 * (global planes k0-1 and k0+dims[slab_mode], modulo n_glob); r receives
 * the interior.  as[mu] are the full n x n factors (n_glob for slab_mode).
 * g (nullable) is added as in r = K u + g(u); the Brusselator's species mode
 * must be the last mode. */
int kp_kronsum_slab_f64(kp_ctx* ctx, const double* u_ext, const int* dims, int d,
                        const double* const* as, int slab_mode, int k0, int n_glob,
                        const kp_gfun* g, double* r);
int kp_kronsum_slab_c128(kp_ctx* ctx, const double* u_ext, const int* dims, int d,
                         const double* const* as, int slab_mode, int k0, int n_glob,
                         const kp_gfun* g, double* r);

/* The same slab action with the band structures scanned once up front
 * (kp_kronsum_slab_* rescans every call, one host sync each): a loop that
 * applies the same factors every step creates one kp_band per factor and
 * calls the _banded form, which never synchronizes.  bands[mu] must hold the
 * n x n factor of mode mu (n_glob for slab_mode); more than three nonzeros
 * in a row -> KP_EINVAL. */
typedef struct kp_band kp_band;
int kp_band_create(kp_ctx* ctx, const double* a, int n, int cplx, kp_band** out);
int kp_band_destroy(kp_band* band);
int kp_kronsum_slab_banded_f64(kp_ctx* ctx, const double* u_ext, const int* dims, int d,
                               const kp_band* const* bands, int slab_mode, int k0, int n_glob,
                               const kp_gfun* g, double* r);
int kp_kronsum_slab_banded_c128(kp_ctx* ctx, const double* u_ext, const int* dims, int d,
                                const kp_band* const* bands, int slab_mode, int k0, int n_glob,
                                const kp_gfun* g, double* r);

/* ---------------- multi-GPU: fused exchange over peer memory ----------------
 * The slab-sharded integrators re-partition the state
 * between the slab layout (last spatial mode split over P ranks) and the
 * pencil layout (second-to-last mode split) around the last mode product.
 * Instead of a GEMM followed by an all-to-all, the GEMM epilogue stores every
 * output entry straight into the destination rank's buffer (NVLink P2P
 * stores through CUDA IPC mappings); a plain scatter kernel does the same
 * for the transposes with no producing GEMM.  Local tensors are column-major
 *   slab   (A, B,   C/P, S)      pencil (A, B/P, C, S)
 * with A = prod(n_1..n_{d-2}), B = n_{d-1}, C = n_d (global sizes), S the
 * species count.  peers[s] is rank s's receive buffer mapped in this process
 * (peers[rank] = own buffer).  Completion: the caller synchronizes its stream
 * and barriers with the other ranks before the receivers read. */
typedef struct {
  int dir; /* 1: slab -> pencil, 2: pencil -> slab */
  int P, rank;
  long long A, B, C, S;
  double* const* peers; /* host array of P device pointers */
} kp_scatter;
/* out = fma(gamma, alpha * (t x_mode m), x) (x == NULL: alpha * (t x_mode m)),
 * each entry stored at its destination rank/index (real / complex128). */
int kp_mode_product_scatter_f64(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                                const double* m, int rows, double alpha, const double* x,
                                double gamma, const kp_scatter* sc);
int kp_mode_product_scatter_c128(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                                 const double* m, int rows, double alpha, const double* x,
                                 double gamma, const kp_scatter* sc);
/* The transpose alone: the local tensor x (n_elems entries of comps doubles,
 * 1 = real, 2 = complex) scattered to its destinations. */
int kp_scatter_copy(kp_ctx* ctx, const double* x, long long n_elems, int comps,
                    const kp_scatter* sc);
/* CUDA IPC for the receive buffers (64-byte opaque handles). */
int kp_ipc_get_handle(const void* dptr, void* handle64);
int kp_ipc_open_handle(const void* handle64, void** dptr);
int kp_ipc_close_handle(void* dptr);

/* ---------------- multi-GPU: NCCL communicator (native plumbing) ----------------
 * "the multi-GPU communicator init from ncclUniqueId".  One
 * process per GPU; rank 0 calls kp_comm_unique_id and the caller broadcasts
 * the 128 bytes (any side channel), then every rank calls kp_comm_create
 * with its context (device).  NCCL is dlopen'ed on first use.  All
 * operations are stream-ordered on the context's stream.
 *   kp_comm_repartition: the slab <-> pencil transpose of the sharded
 *     integrators (layouts as kp_scatter above; dir 1 slab -> pencil, 2 back;
 *     comps 1 real / 2 complex) = pack -> grouped ncclSend/Recv -> unpack;
 *     bit-identical to the peer-memory scatter (pure data movement).
 *   kp_repartition_pack / _unpack: its two local halves (send buffer =
 *     P blocks of A*B/P*C/P*S entries, block s for rank s) for callers with
 *     their own transport.
 *   kp_comm_halo_f64: left <- last plane of rank-1, right <- first plane of
 *     rank+1 (cyclic): the one-plane halo of kp_kronsum_slab_*. */
typedef struct kp_comm kp_comm;
int kp_comm_unique_id(void* id128);
int kp_comm_create(kp_ctx* ctx, int nranks, int rank, const void* id128, kp_comm** out);
int kp_comm_destroy(kp_comm* comm);
int kp_comm_alltoall_f64(kp_ctx* ctx, kp_comm* comm, const double* send, double* recv,
                         long long count_per_rank);
int kp_comm_repartition(kp_ctx* ctx, kp_comm* comm, int dir, long long A, long long B,
                        long long C, long long S, int comps, const double* x, double* y);
int kp_repartition_pack(kp_ctx* ctx, int dir, int P, int rank, long long A, long long B,
                        long long C, long long S, int comps, const double* x, double* send);
int kp_repartition_unpack(kp_ctx* ctx, int dir, int P, int rank, long long A, long long B,
                          long long C, long long S, int comps, const double* recv, double* y);
int kp_comm_halo_f64(kp_ctx* ctx, kp_comm* comm, const double* first, const double* last,
                     long long count, double* left, double* right);

/* Host-buffer variants (the drop-in path: host in, host out, H2D/D2H inside). */
int kp_host_mode_product_f64(kp_ctx* ctx, const double* t, const int* dims, int d, int mode,
                             const double* m, int rows, int cols, double alpha, double beta,
                             double* out);
int kp_host_tucker_f64(kp_ctx* ctx, const double* t, const int* dims, int d,
                       const double* const* ms, const int* rows, double prefactor,
                       double* out);
/* Streamed host Tucker: count tensors (same dims and factors), ts[i] ->
 * outs[i] (host, column-major).  Uploads of tensor i+1 overlap the last mode
 * and the download of tensor i (two device buffer sets), so a sequence of
 * tucker() calls costs ~max(H2D, D2H, compute) per tensor instead of their
 * sum.  Results are bitwise those of kp_host_tucker_f64 per tensor. */
int kp_host_tucker_stream_f64(kp_ctx* ctx, int count, const double* const* ts, const int* dims,
                              int d, const double* const* ms, const int* rows, double prefactor,
                              double* const* outs);
int kp_host_tucker_c128(kp_ctx* ctx, const double* t, const int* dims, int d,
                        const double* const* ms, const int* rows, double prefactor,
                        double* out);
int kp_host_kronsum_f64(kp_ctx* ctx, const double* t, const int* dims, int d,
                        const double* const* as, double* out);

/* ---------------- elementwise (inc/tensor.hpp:123-155) ---------------- */
/* y = alpha * x + y  (axpy) */
int kp_axpy_f64(kp_ctx* ctx, size_t n, double alpha, const double* x, double* y);
/* z = x + alpha * y  (add_scaled) */
int kp_add_scaled_f64(kp_ctx* ctx, size_t n, const double* x, double alpha, const double* y,
                      double* z);
/* gout = g(t, u) over a tensor of shape dims */
int kp_eval_g_f64(kp_ctx* ctx, const kp_gfun* g, double t, const double* u, const int* dims,
                  int d, double* gout);
int kp_eval_g_c128(kp_ctx* ctx, const kp_gfun* g, double t, const double* u, const int* dims,
                   int d, double* gout);
/* Jacobian factors of the Riccati problem at the n x n state u
 * (riccati_jacobian_factors, src/problems.cpp:212-250): J = A^T - (U b) b^T;
 * one factor serves both modes when U is symmetric to 1e-8 (then *nfactors =
 * 1 and j2 is untouched), else j2 = A^T - (U^T b) b^T and *nfactors = 2.
 * g: a KP_G_RICCATI descriptor (aux[0] = b); at, u, j1, j2: device, n x n. */
int kp_riccati_jacobian_factors_f64(kp_ctx* ctx, const kp_gfun* g, const double* u,
                                    const double* at, int n, double* j1, double* j2,
                                    int* nfactors);
/* *all_finite = 1 if every entry is finite (inc/integrators.hpp:101-108) */
int kp_all_finite_f64(kp_ctx* ctx, size_t n, const double* x, int* all_finite);
/* Stream-ordered, no host sync: atomicMin(*bad_dev, step) when x (n doubles)
 * holds a non-finite value -- the per-step finite check of host-driven loops
 * (inc/integrators.hpp:364), read once after the loop. */
int kp_mark_nonfinite_f64(kp_ctx* ctx, size_t n, const double* x, int* bad_dev, int step);

/* ---------------- matrix functions (inc/matrix_functions.hpp) ---------------- */
/* q-point Gauss-Legendre-Lobatto rule on [0,1] (host; src/gll_rule.cpp:35-72) */
int kp_gll_rule(int q, double* nodes, double* weights);
/* x = a^{-1} b by blocked LU with partial pivoting (solve = lu_factor +
 * lu_solve, inc/linsolve.hpp:95-151); a: n x n, b and x: n x nrhs, device,
 * column-major (x may alias b).  Singular a -> KP_ERUNTIME. */
int kp_solve_f64(kp_ctx* ctx, const double* a, int n, const double* b, int nrhs, double* x);
/* out = e^x, n x n (expm, inc/matrix_functions.hpp:76-95) */
int kp_expm_f64(kp_ctx* ctx, const double* x, int n, double* out);
int kp_expm_c128(kp_ctx* ctx, const double* x, int n, double* out);
/* phis = [phi_0(x), ..., phi_ell_max(x)], ell_max+1 consecutive n x n
 * matrices (phiquad, :146-199; PhiTable::phis); forced_scaling < 0 = none. */
int kp_phiquad_f64(kp_ctx* ctx, const double* x, int n, int ell_max, int q, int forced_scaling,
                   double* phis, int* scaling_exponent);
int kp_phiquad_c128(kp_ctx* ctx, const double* x, int n, int ell_max, int q, int forced_scaling,
                    double* phis, int* scaling_exponent);

/* ---------------- direction splitting (inc/split_phi.hpp) ---------------- */
/* factors[mu] = phi_ell(tau*A_mu) (expm for ell = 0), *prefactor = (ell!)^(d-1)
 * (build_split_phi, :25-48).  Apply with kp_tucker_* (prefactor argument). */
int kp_build_split_phi_f64(kp_ctx* ctx, const double* const* as, const int* dims, int d,
                           double tau, int ell, int q, double* const* factors, double* prefactor);
int kp_build_split_phi_c128(kp_ctx* ctx, const double* const* as, const int* dims, int d,
                            double tau, int ell, int q, double* const* factors,
                            double* prefactor);

/* ---------------- steppers (inc/integrators.hpp) ---------------- */
/* One step out = step(u).  f1/f2 as in the reference's step functions:
 * Lawson methods f1 = exp factors; ExpEuler f1 = phi1; ExpEulerLS f1 = exp,
 * f2 = phi1; ETD2RK f1 = phi1, f2 = phi2 (pref1/pref2 = split prefactors);
 * RosenbrockEuler f1 = the Jacobian factors J_mu (phi_1(tau J_mu) built in the
 * call, equal pointers share one build, :166-194; f2 unused).
 * Replaces lawson_euler_step, lawson2b_step, exp_euler_step,
 * exp_euler_linear_split_step, etd2rk_step, rosenbrock_euler_step (:116-194).
 * out must not alias u. */
int kp_step_f64(kp_ctx* ctx, int method, const double* u, const int* dims, int d, double t,
                double tau, const double* const* as, const double* const* f1, double pref1,
                const double* const* f2, double pref2, const kp_gfun* g, double* out);
int kp_step_c128(kp_ctx* ctx, int method, const double* u, const int* dims, int d, double t,
                 double tau, const double* const* as, const double* const* f1, double pref1,
                 const double* const* f2, double pref2, const kp_gfun* g, double* out);
/* integrate (:219-373, Split backend): tau = (t_final-t0)/n_steps, factors
 * built once on the device, n_steps steps on device-resident state u (in:
 * u0, out: final state), per-step finite check.  On divergence returns
 * KP_EDIVERGE with *diverged_step = first non-finite step (1-based).
 * RosenbrockEuler needs g = KP_G_RICCATI (its jacobian_factors are rebuilt on
 * the device every step), otherwise KP_EINVAL like the reference (:223-225).
 * *loop_seconds (may be NULL) = device time of the time loop. */
int kp_integrate_f64(kp_ctx* ctx, int method, double* u, const int* dims, int d,
                     const double* const* as, const kp_gfun* g, double t0, double t_final,
                     long n_steps, int q, long* diverged_step, double* loop_seconds);
int kp_integrate_c128(kp_ctx* ctx, int method, double* u, const int* dims, int d,
                      const double* const* as, const kp_gfun* g, double t0, double t_final,
                      long n_steps, int q, long* diverged_step, double* loop_seconds);
/* integrate with trajectory sampling (StepperConfig::sample_every,
 * IntegrateResult::trajectory, :284-287,:365-366): after every sample_every
 * steps fn(user, step, u_host) receives the state (a library-owned pinned
 * host buffer of prod(dims) (x2 complex) doubles, valid during the call);
 * the caller records (t0, u0) itself, as the reference does before the loop.
 * sample_every = 0 is kp_integrate_*. */
typedef void (*kp_sample_fn)(void* user, long step, const double* u_host);
int kp_integrate_sampled_f64(kp_ctx* ctx, int method, double* u, const int* dims, int d,
                             const double* const* as, const kp_gfun* g, double t0,
                             double t_final, long n_steps, int q, int sample_every,
                             kp_sample_fn fn, void* user, long* diverged_step,
                             double* loop_seconds);
int kp_integrate_sampled_c128(kp_ctx* ctx, int method, double* u, const int* dims, int d,
                              const double* const* as, const kp_gfun* g, double t0,
                              double t_final, long n_steps, int q, int sample_every,
                              kp_sample_fn fn, void* user, long* diverged_step,
                              double* loop_seconds);
/* Slab-sharded integrate across the GPUs of one node (the
 * reference is single-node CPU).  u_local: this rank's slab of the state on
 * the context's device (dims_local: the last spatial mode holds n_d / P
 * planes; a stacked Brusselator keeps its species mode last); as: the FULL
 * factors (device).  Exchanges over comm (NCCL on the context's stream, no
 * host sync inside a step; the step is a replayed CUDA graph).  mode_d: how
 * the last mode crosses the slabs -- 1 = all-to-all pencil transpose (bitwise
 * equal to the single-GPU integrate), 2 = partial products + reduce-scatter,
 * 0 = pick by measurement (one step of each, max over ranks); *mode_used
 * reports the choice.  Divergence: KP_EDIVERGE with the first bad step over
 * all ranks.  *loop_seconds = device time of the loop, max over ranks.
 * g: the pointwise set (not ADR / Riccati); methods lawson_euler, lawson2b,
 * exp_euler, etd2rk. */
int kp_integrate_sharded_f64(kp_ctx* ctx, kp_comm* comm, int method, double* u_local,
                             const int* dims_local, int d, const double* const* as,
                             const kp_gfun* g, double t0, double t_final, long n_steps, int q,
                             int mode_d, int* mode_used, long* diverged_step,
                             double* loop_seconds);
int kp_integrate_sharded_c128(kp_ctx* ctx, kp_comm* comm, int method, double* u_local,
                              const int* dims_local, int d, const double* const* as,
                              const kp_gfun* g, double t0, double t_final, long n_steps, int q,
                              int mode_d, int* mode_used, long* diverged_step,
                              double* loop_seconds);
/* The same sharded integrator with all P ranks driven by this process on one
 * device (u_slabs[r] = rank r's slab; the exchanges become device copies):
 * the data movement of a P-GPU run, testable on one GPU. */
int kp_integrate_sharded_local_f64(kp_ctx* ctx, int P, int method, double* const* u_slabs,
                                   const int* dims_local, int d, const double* const* as,
                                   const kp_gfun* g, double t0, double t_final, long n_steps,
                                   int q, int mode_d, int* mode_used, long* diverged_step,
                                   double* loop_seconds);
int kp_integrate_sharded_local_c128(kp_ctx* ctx, int P, int method, double* const* u_slabs,
                                    const int* dims_local, int d, const double* const* as,
                                    const kp_gfun* g, double t0, double t_final, long n_steps,
                                    int q, int mode_d, int* mode_used, long* diverged_step,
                                    double* loop_seconds);
/* The mode-d-sharded Tucker operator (real): V x_1 M_1 ... x_d M_d with V
 * slab-sharded along mode d (t_slab: this rank's n_1 x .. x n_d/P slab;
 * square, full factors).  Modes 1..d-1 on the slab; mode d across the slabs:
 * mode_d 1 = all-to-all, result in the PENCIL layout (n_1 .. n_(d-1)/P x n_d,
 * bitwise the rank's block of the single-GPU result); 2 = partial products +
 * reduce-scatter, result in the SLAB layout; 3 = fused: mode d-1's GEMM
 * epilogue stores every entry straight into its owner's pencil buffer (peer
 * memory, CUDA IPC over NVLink; mappings cached), result as for 1. */
int kp_tucker_sharded_f64(kp_ctx* ctx, kp_comm* comm, const double* t_slab,
                          const int* dims_local, int d, const double* const* ms,
                          double prefactor, int mode_d, double* out);
int kp_tucker_sharded_local_f64(kp_ctx* ctx, int P, const double* const* t_slabs,
                                const int* dims_local, int d, const double* const* ms,
                                double prefactor, int mode_d, double* const* outs);
/* Host-buffer drop-in: u0/as on the host, u_final written on the host. */
int kp_host_integrate_f64(kp_ctx* ctx, int method, const double* u0, const int* dims, int d,
                          const double* const* as, const kp_gfun* g, double t0, double t_final,
                          long n_steps, int q, double* u_final, long* diverged_step,
                          double* loop_seconds);
int kp_host_integrate_c128(kp_ctx* ctx, int method, const double* u0, const int* dims, int d,
                           const double* const* as, const kp_gfun* g, double t0, double t_final,
                           long n_steps, int q, double* u_final, long* diverged_step,
                           double* loop_seconds);

/* Measured FP64 peak of this device: a DMMA (mma.sync m8n8k4 f64) loop over
 * all SMs; returns TFLOP/s.  Used as the roofline denominator. */
int kp_measure_fp64_peak(kp_ctx* ctx, double* tflops);

#ifdef __cplusplus
}
#endif
#endif
