/*
 * nenmf_b200.h -- C ABI of libnenmf_b200.so, the sm_100a (B200) hot path of
 * compressed NeNMF (arXiv 1812.04315).
 *
 * The reference (/root/reference/pkg/src/nenmf) is pure Python/NumPy and has
 * no FFI; its hot path sits behind the public Python API.  Each entry point
 * below replaces the NumPy/OpenBLAS/LAPACK work of one reference function and
 * is what a ctypes binding of that function calls:
 *
 *   nenmf_solve_nnls        nnls.py:119-227       solve_nnls (whole inner solve)
 *   nenmf_spectral_norm_sq  matrix.py:131-174     spectral_norm_sq (+ power iteration)
 *   nenmf_gradient          nnls.py:72-86         gradient
 *   nenmf_pg_norm_sq        nnls.py:89-107        projected_gradient_norm
 *   nenmf_rsi               compression.py:120-141 subspace_iteration_pair
 *   nenmf_compress          compression.py:179-188 compress_problem
 *   nenmf_abt               factorize.py:110,113  F @ R, L @ G (skinny, long K)
 *   nenmf_residual_sumsq    factorize.py:139, tracing.py:45-57  ||X - G F||^2
 *   nenmf_sumsq             matrix.py:177-179     frobenius_norm^2
 *   nenmf_dual_pass         compression.py:134-139 X @ A and X.T @ B in one pass
 *   nenmf_orthonormalize    compression.py:88-106 _orthonormal_columns (CholeskyQR2;
 *                           Householder TSQR for k > 32)
 *   nenmf_power_iteration   compression.py:144-176 power_iteration_pair
 *   nenmf_sketch_draws      compression.py:130-132 default_rng(seed).standard_normal
 *   nenmf_panel_gram/_factor/_trsm  compression.py:88-106 split for row shards
 *   nenmf_prepare_x + *_prepared    one X preparation shared by the sketch,
 *                           the compression and the vanilla V products
 *   nenmf_solve_nnls_prepared  nnls.py:119-227 with V = X F^T / X^T G from Xp
 *   nenmf_solve_nnls_next   nnls.py:119-227 + factorize.py:110,113 (the solve
 *                           also forms the next half-step operand)
 *   nenmf_convert_f64       matrix.py:194-214 read_nmfb payload -> device dtype
 *   nenmf_uniform_draws     synthetic.py:62-64 / matrix.py:73-82 G, F draws of generate_problem
 *
 * Conventions
 *  - All array pointers are DEVICE pointers, row-major, allocated by the
 *    caller.  Nothing is allocated or freed inside the library.
 *  - "skinny" matrices are stored short-dimension-major: a tall n x k panel
 *    P is passed as Pt (k x n, row-major), i.e. P in column-major order.
 *  - dtype: NENMF_F64 (parity mode) or NENMF_F32; every array of one call has
 *    that element type; scalar results are always double.
 *  - Every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *    default) and returns a launch status.  Data-dependent failures (zero
 *    matrix, non-finite iterates, sketch collapse) are written by the kernels
 *    into a caller-provided device nenmf_device_status and surface when the
 *    caller reads it back, exactly where the reference raises.
 *  - Workspace: each op reports its scratch size via *_workspace_bytes;
 *    pass at least that many bytes (256-byte aligned) in `ws`.
 *  - No global mutable state; calls on different streams/threads are safe.
 */
#ifndef NENMF_B200_H
#define NENMF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NENMF_ABI_VERSION 1

typedef enum { NENMF_F64 = 0, NENMF_F32 = 1 } nenmf_dtype;

/* maps 1:1 onto errors.py classes (see paper_1812_04315_b200/errors.py) */
typedef enum {
  NENMF_OK = 0,
  NENMF_ERR_DIM = 1,                 /* DimensionError          errors.py:10 */
  NENMF_ERR_ZERO_MATRIX = 2,         /* ZeroMatrixError         errors.py:14 */
  NENMF_ERR_NUMERICAL_FAILURE = 3,   /* NumericalFailureError   errors.py:30 */
  NENMF_ERR_NUMERICAL_COLLAPSE = 4,  /* NumericalCollapseError  errors.py:43 */
  NENMF_ERR_VALUE = 5,               /* ValueError                            */
  NENMF_ERR_CUDA = 6,
  NENMF_ERR_WORKSPACE = 7,
  NENMF_ERR_UNSUPPORTED = 8,
  NENMF_ERR_WATCHDOG = 9             /* a persistent solve made no progress for NENMF_WATCHDOG_S seconds */
} nenmf_status_code;

/* Written by the kernels (device memory, 64 bytes).  Zero it before use. */
typedef struct {
  int32_t code;          /* nenmf_status_code of the first failure, 0 if none */
  int32_t iteration;     /* inner iteration of a NUMERICAL_FAILURE            */
  int32_t inner_iters;   /* inner iterations executed by the last solve       */
  int32_t returned_best; /* 1: best iterate returned, 0: start returned       */
  double lipschitz;      /* L used by the last solve                           */
  double best_partial;   /* Gram-form objective of the returned iterate       */
  double pg_ref;         /* projected-gradient norm at the start point        */
  double resid[2];       /* 1/2||A best - B||^2, 1/2||A start - B||^2         */
  double pad;
} nenmf_device_status;

int nenmf_abi_version(void);
const char* nenmf_status_string(int code);
/* number of SMs of the current device (0 if no device) */
int nenmf_device_sm_count(void);
/* kernels this library has launched in this process (diagnostic counter) */
unsigned long long nenmf_launch_count(void);
/* development aid: per-iteration timeline of the last traced solve
 * (NENMF_NNLS_TRACE=1 in the environment), 4 x 4096 globaltimer stamps */
int nenmf_debug_nnls_trace(unsigned long long* host_out, int count);

/* ---- inner solver (nnls.py:119-227) -------------------------------------
 * Solves min_{F>=0} 1/2||B - A F||^2 from F0.  A (r x p) is passed as
 * At (p x r).  B is (r x c): row-major with leading dimension ldb when
 * trans_b == 0, or the transpose of a row-major (c x r) matrix with leading
 * dimension ldb when trans_b == 1 (this is how vanilla NeNMF's G-half reads
 * X^T without materialising it, factorize.py:92).  F0 and F_out are (p x c)
 * and must not alias.  power_vectors: device array of power_count
 * normalised start vectors of length min(r, p), the reference's seeded
 * stream in draw order (matrix.py:24,138-149): vector 0 starts the power
 * iteration, the next one is taken whenever ||W v|| == 0 (past power_count
 * the re-draw is the zero vector); power_max_iters / power_tol are the
 * reference's max_iters (100) and tol (1e-9).
 * Writes status->{code, iteration, inner_iters, returned_best, lipschitz}. */
size_t nenmf_solve_nnls_workspace_bytes(int dtype, int64_t r, int64_t p, int64_t c);
int nenmf_solve_nnls(int dtype, const void* At, int64_t r, int64_t p,
                     const void* B, int64_t c, int64_t ldb, int trans_b,
                     const void* F0, void* F_out,
                     int max_iter, double grad_tol, double lipschitz_safety,
                     const double* power_vectors, int power_count, int power_max_iters,
                     double power_tol, nenmf_device_status* status, void* ws, size_t ws_bytes,
                     void* stream);

/* nenmf_solve_nnls plus the operand of the next half-step of the outer loop:
 * next_out (p x next_k) = F_out next_bt^T with next_bt (next_k x c), i.e.
 * F R (factorize.py:110) after an F-half and L G (factorize.py:113) after a
 * G-half.  Formed inside the solver launch when it is fused (r <= 64); same
 * result as a separate nenmf_abt(F_out, next_bt) up to summation order. */
size_t nenmf_solve_nnls_next_workspace_bytes(int dtype, int64_t r, int64_t p, int64_t c, int64_t next_k);

/* Vanilla half-steps on FP32 data (factorize.py:94-98): as nenmf_solve_nnls,
 * with Xp = nenmf_prepare_x(X) of the X that B is (trans_b = 0: B = X, r x c)
 * or whose transpose B is (trans_b = 1: X is c x r).  V = A^T B then comes
 * from one tensor-core pass over Xp; B itself is still read by the
 * explicit-residual tie-break (nnls.py:219-227).  Xp = NULL: plain solve. */
size_t nenmf_solve_nnls_prepared_workspace_bytes(int dtype, int64_t r, int64_t p, int64_t c);
int nenmf_solve_nnls_prepared(int dtype, const void* At, int64_t r, int64_t p, const void* B,
                              int64_t c, int64_t ldb, int trans_b, const void* Xp, const void* F0,
                              void* F_out, int max_iter, double grad_tol, double lipschitz_safety,
                              const double* power_vectors, int power_count, int power_max_iters,
                              double power_tol, nenmf_device_status* status, void* ws,
                              size_t ws_bytes, void* stream);
int nenmf_solve_nnls_next(int dtype, const void* At, int64_t r, int64_t p,
                          const void* B, int64_t c, int64_t ldb, int trans_b,
                          const void* F0, void* F_out,
                          int max_iter, double grad_tol, double lipschitz_safety,
                          const double* power_vectors, int power_count, int power_max_iters,
                          double power_tol, const void* next_bt, int64_t next_k, void* next_out,
                          nenmf_device_status* status, void* ws, size_t ws_bytes, void* stream);

/* sigma_max(A)^2 by power iteration on the smaller Gram (matrix.py:158-174).
 * A (r x p) passed as At (p x r).  Result (double) -> *out (device). */
/* ---- exact-SNR problem generator (synthetic.py:47-95), fused -----------
 * G (n x p), F (p x m), N (n x m) fp64 on the device (the draws of
 * generate_problem, bit-identical streams).  nenmf_generate_norms: out2[0] =
 * ||G F||^2 (G F formed on the fly, not stored), out2[1] = ||N||^2, one read
 * of N.  nenmf_generate_write: X = G F + scale N in dtype (N may be NULL for
 * the noiseless case). */
size_t nenmf_generate_workspace_bytes(void);
int nenmf_generate_norms(const double* G, const double* F, const double* N, int64_t n, int64_t m, int64_t p,
                         double* out2, void* ws, size_t ws_bytes, void* stream);
int nenmf_generate_write(int dtype, const double* G, const double* F, const double* N, int64_t n, int64_t m,
                         int64_t p, double scale, void* X, void* stream);

/* ---- rank groups ------------------------------------------
 * A compressed half-step whose columns are split over R ranks (X row-sharded
 * across GPUs: the G-half owns this rank's rows of G, the F-half a slice of
 * F's columns).  Each rank launches the same persistent solver on its own
 * columns; the per-iteration sums of the stopping/best decisions (nnls.py:
 * 177,196-203) and the tie-break residuals (nnls.py:219-227) are exchanged
 * inside the kernel through an exchange buffer on every rank (peer memory
 * over NVLink, epoch-tagged, summed in rank order), so all ranks take the
 * same decisions.  next_out receives nvr partial next products (p x next_k
 * each, this launch's virtual ranks in order); the caller all-reduces them.
 * With nvr = R one launch emulates the whole group on one GPU (its CTAs split
 * into R virtual ranks), which is how the exchange is tested on one device.
 * Replaces nnls.py:119-227 for the sharded compressed loop (factorize.py:
 * 197-213 run on row blocks). */
typedef struct nenmf_group {
  int ranks;        /* R, 2..8 */
  int rank0;        /* rank of this launch's first virtual rank */
  int nvr;          /* virtual ranks in this launch: 1 per GPU, or R to emulate the group */
  int watchdog_s;   /* > 0: this solve's no-progress limit in seconds (else NENMF_WATCHDOG_S / 60 s) */
  int64_t col0[9];  /* virtual rank v owns columns [col0[v], col0[v+1]) of this launch's arrays; col0[nvr] = c */
  void* xch[8];     /* every rank's exchange buffer (nenmf_group_xch_bytes() each, zeroed once) */
  uint64_t epoch;   /* the same on every rank, unique per solve over the buffers' lifetime, 0 < epoch < 2^40 */
} nenmf_group;
size_t nenmf_group_xch_bytes(void);
/* NENMF_OK when a solve of this shape runs as a group solve (ranks, nvr
 * virtual ranks in one launch), NENMF_ERR_UNSUPPORTED when the caller must
 * replicate it instead (columns beyond the register-resident solver). */
int nenmf_solve_nnls_group_check(int dtype, int64_t r, int64_t p, int64_t c, int64_t next_k, int ranks,
                                 int nvr, int max_iter);
int nenmf_solve_nnls_group(int dtype, const void* At, int64_t r, int64_t p, const void* B, int64_t c,
                           int64_t ldb, int trans_b, const void* F0, void* F_out, int max_iter,
                           double grad_tol, double lipschitz_safety, const double* power_vectors,
                           int power_count, int power_max_iters, double power_tol, const void* next_bt,
                           int64_t next_k, void* next_out, const nenmf_group* group,
                           nenmf_device_status* status, void* ws, size_t ws_bytes, void* stream);
/* CUDA IPC of the exchange buffers: a 64-byte handle of a device allocation,
 * and the peer mapping of a handle from another process. */
int nenmf_ipc_handle(const void* dev_ptr, void* handle64);
int nenmf_ipc_open(const void* handle64, void** dev_ptr);
int nenmf_ipc_close(void* dev_ptr);

size_t nenmf_spectral_norm_sq_workspace_bytes(int dtype, int64_t r, int64_t p);
int nenmf_spectral_norm_sq(int dtype, const void* At, int64_t r, int64_t p,
                           const double* power_vectors, int power_count, int max_iters, double tol,
                           double* out, nenmf_device_status* status,
                           void* ws, size_t ws_bytes, void* stream);

/* grad = A^T (A F - B) in Gram form (nnls.py:72-86); same operand forms as
 * nenmf_solve_nnls.  grad is (p x c). */
size_t nenmf_gradient_workspace_bytes(int dtype, int64_t r, int64_t p, int64_t c);
int nenmf_gradient(int dtype, const void* At, int64_t r, int64_t p,
                   const void* B, int64_t c, int64_t ldb, int trans_b,
                   const void* F, void* grad, void* ws, size_t ws_bytes, void* stream);

/* sum over entries of (F > 0 ? g : min(g, 0))^2 -> *out (nnls.py:89-107) */
size_t nenmf_reduce_workspace_bytes(int64_t count);
int nenmf_pg_norm_sq(int dtype, const void* F, const void* g, int64_t count,
                     double* out, void* ws, size_t ws_bytes, void* stream);
/* sum of squares of `count` contiguous entries -> *out (matrix.py:177-179) */
int nenmf_sumsq(int dtype, const void* M, int64_t count, double* out,
                void* ws, size_t ws_bytes, void* stream);
/* One read of M (rows x cols, leading dimension ld): *nonzero = 1 if some
 * entry is nonzero (compression.py:109-117, X.any()), *negative = 1 if some
 * entry is < 0 (the FactorPair sign check, factorize.py:44-48, for factors
 * already on the device).  Flags are only raised (the caller zeroes them);
 * either may be NULL.  No synchronisation. */
int nenmf_scan_flags(int dtype, const void* M, int64_t rows, int64_t cols, int64_t ld,
                     int* nonzero, int* negative, void* stream);
/* dst (cols x rows, contiguous) = src (rows x cols, leading dimension ld)^T:
 * an n x p factor G brought into the p x n panel layout of the solver
 * (factorize.py:92,109 transpose G / F for the half-steps). */
int nenmf_transpose(int dtype, const void* src, int64_t rows, int64_t cols, int64_t ld, void* dst,
                    void* stream);
/* cudaMemsetAsync(ptr, 0, bytes) on `stream`: zeroes status words and flags
 * without a kernel launch. */
int nenmf_zero(void* ptr, size_t bytes, void* stream);

/* ||X - G F||_F^2 -> *out, X (n x m, ld ldx), G passed as Gt (p x n),
 * F (p x m) (factorize.py:139; tracing.py:45-57) */
size_t nenmf_residual_sumsq_workspace_bytes(int dtype, int64_t n, int64_t m, int64_t p);
int nenmf_residual_sumsq(int dtype, const void* X, int64_t n, int64_t m, int64_t ldx,
                         const void* Gt, const void* F, int64_t p, double* out,
                         void* ws, size_t ws_bytes, void* stream);

/* nenmf_residual_sumsq reading X from its prepared copy Xp (FP32, p <= 32):
 * one tensor-core pass (tcgen05, BF16x3 products, fp32 accumulators) per
 * 128 x 128 tile computes G F and accumulates (x - (G F))^2 in fp64.  Falls
 * back to the plain call on X when Xp is NULL or the shape has no prepared
 * form (X may then not be NULL).  Workspace: *_prepared_workspace_bytes. */
size_t nenmf_residual_sumsq_prepared_workspace_bytes(int dtype, int64_t n, int64_t m, int64_t p);
int nenmf_residual_sumsq_prepared(int dtype, const void* X, const void* Xp, int64_t n, int64_t m,
                                  int64_t ldx, const void* Gt, const void* F, int64_t p,
                                  double* out, void* ws, size_t ws_bytes, void* stream);

/* C (p x q) = A (p x K) B (q x K)^T, long K (factorize.py:110,113). */
size_t nenmf_abt_workspace_bytes(int dtype, int64_t p, int64_t q, int64_t K);
int nenmf_abt(int dtype, const void* A, int64_t p, const void* B, int64_t q, int64_t K,
              void* C, void* ws, size_t ws_bytes, void* stream);

/* ---- randomized subspace iteration (compression.py:120-188) ------------- */

/* One streaming pass over X (n x m, ld ldx) computing, when the operand is
 * non-NULL, Yt = At X^T (k x n; At is k x m) and Zt = Bt X (k x m; Bt is
 * k x n), i.e. X @ A and X.T @ B of the reference (compression.py:134-139)
 * stored transposed.  Deterministic (fixed-order reduction). */
size_t nenmf_dual_pass_workspace_bytes(int dtype, int64_t n, int64_t m, int64_t k);
int nenmf_dual_pass(int dtype, const void* X, int64_t n, int64_t m, int64_t ldx,
                    const void* At, const void* Bt, int64_t k, void* Yt, void* Zt,
                    void* ws, size_t ws_bytes, void* stream);

/* In-place orthonormal basis of a tall rows x k panel given as Pt (k x rows):
 * reduced Householder QR (TSQR), rank deficiency tolerated, collapse (non-
 * finite input or all-zero diag R) -> status NUMERICAL_COLLAPSE
 * (compression.py:88-106). */
size_t nenmf_orthonormalize_workspace_bytes(int64_t rows, int64_t k);
int nenmf_orthonormalize(int dtype, void* Pt, int64_t rows, int64_t k,
                         nenmf_device_status* status, void* ws, size_t ws_bytes,
                         void* stream);

/* Algorithm 2: L (nu x n) and Rt (nu x m, i.e. R transposed) from the
 * reference's Gaussian draws: omega_l_t = Omega_L^T (nu x m), omega_r
 * (nu x n) (compression.py:130-141). */
size_t nenmf_rsi_workspace_bytes(int dtype, int64_t n, int64_t m, int64_t nu);
int nenmf_rsi(int dtype, const void* X, int64_t n, int64_t m, int64_t ldx,
              const void* omega_l_t, const void* omega_r, int64_t nu, int q,
              void* L, void* Rt, nenmf_device_status* status,
              void* ws, size_t ws_bytes, void* stream);

/* X_L = L X (nu x m) and X_R^T = (X R)^T (nu x n) (compression.py:179-188) */
int nenmf_compress(int dtype, const void* X, int64_t n, int64_t m, int64_t ldx,
                   const void* L, const void* Rt, int64_t nu, void* XL, void* XRt,
                   void* ws, size_t ws_bytes, void* stream);

/* ---- the reference's Gaussian sketch draws, on the device ----------------
 * Omega_L (m x nu) then Omega_R (nu x n) from ONE numpy.random.default_rng
 * (seed).standard_normal stream (compression.py:130-132), bit-identical to
 * NumPy: PCG64 state/increment as 128-bit halves (numpy PCG64(seed).state),
 * `tables` = NumPy's ziggurat tables fi[256], wi[256] (double), ki[256]
 * (uint64) in device memory.  Writes omega_l_t = Omega_L^T (nu x m) and
 * omega_r (nu x n) in `dtype`; *ok (device int) = 1 on success, 0 if the
 * chunked walk could not be stitched (the caller redraws on the host).
 * tails (device, 1 + 2 * nenmf_sketch_tail_capacity entries): [count] then
 * (draw index, u53 << 1 | negative) of every draw from the ziggurat tail;
 * the caller rewrites those values as +-(r + (-log1p(-u53 2^-53)) / r) with
 * the C library's log1p (CUDA's log1p may differ from it by one ulp). */
size_t nenmf_sketch_draws_workspace_bytes(int64_t n, int64_t m, int64_t nu);
int64_t nenmf_sketch_tail_capacity(int64_t n, int64_t m, int64_t nu);
int nenmf_sketch_draws(int dtype, const void* tables, uint64_t state_lo, uint64_t state_hi,
                       uint64_t inc_lo, uint64_t inc_hi, int64_t n, int64_t m, int64_t nu,
                       void* omega_l_t, void* omega_r, int* ok, unsigned long long* tails,
                       void* ws, size_t ws_bytes, void* stream);

/* NumPy Generator.random (float64) draws from the PCG64 state/increment
 * (128-bit halves): out[i] = (next64 >> 11) 2^-53 for count values, as the
 * reference's open_uniform (matrix.py:73-82) takes them; *zero (device int)
 * = 1 if a draw is exactly 0 (the caller then redraws like open_uniform). */
int nenmf_uniform_draws(uint64_t state_lo, uint64_t state_hi, uint64_t inc_lo, uint64_t inc_hi, int64_t count,
                        double* out, int* zero, void* stream);

/* ---- stages of the orthonormalisation, for row-sharded panels ----------
 * nenmf_orthonormalize is CholeskyQR2 (rank-revealing first pass).  When a
 * tall panel is split by rows across ranks, the caller runs its stages with
 * an all-reduce of the k x k Gram matrix in between:
 *   nenmf_panel_gram    G = P^T P of the local rows (fp64, fixed order)
 *   (all-reduce G over ranks)
 *   nenmf_panel_factor  (pivoted) Cholesky of G -> R (k x k), meta (1 + k
 *                       ints: rank, pivot order); identical on every rank
 *   nenmf_panel_trsm    local rows: Pout = Pin Pi R^-1; columns past the rank
 *                       get fixed pseudo-random values keyed by the GLOBAL row
 *                       index row0 + i (so shards reproduce the 1-GPU panel);
 *                       full_rank_only skips the solve when rank < k
 * Pass 1: pivot = 1 on P (-> Q1); pass 2: pivot = 0 on Q1 (-> Q). */
size_t nenmf_panel_gram_workspace_bytes(int dtype, int64_t rows, int64_t k);
int nenmf_panel_gram(int dtype, const void* Pt, int64_t rows, int64_t k, double* G,
                     void* ws, size_t ws_bytes, void* stream);
int nenmf_panel_factor(const double* G, int64_t k, int pivot, double* R, int* meta,
                       nenmf_device_status* status, void* stream);
int nenmf_panel_trsm(int dtype, const void* Pin_t, int64_t rows, int64_t k, const double* R,
                     const int* meta, void* Pout_t, int64_t row0, int full_rank_only,
                     void* stream);

/* ---- prepared X (FP32 tensor-core passes) -------------------------------
 * The FP32 passes read X in a "prepared" tile-major form: every 128 x 128
 * tile as bf16 hi/lo planes in the tensor-core shared-memory layout, the
 * same 4 bytes per element as X.  nenmf_rsi/nenmf_compress prepare X
 * internally on every call; the *_prepared variants take a copy made once
 * by nenmf_prepare_x (Xp may be NULL: then they behave like the plain call),
 * so one preparation serves the sketch and the compression of the same X
 * (compression.py:120-141 followed by :179-188).  nenmf_prepared_x_bytes
 * returns 0 when the dtype/shape has no prepared form (FP64, k > 32). */
size_t nenmf_prepared_x_bytes(int dtype, int64_t n, int64_t m, int64_t k);
int nenmf_prepare_x(int dtype, const void* X, int64_t n, int64_t m, int64_t ldx, int64_t k,
                    void* Xp, void* stream);
/* nenmf_prepare_x that also raises *nonzero (zeroed by the caller) when X has
 * a nonzero entry: subspace_iteration_pair's X != 0 check (compression.py:
 * 109-117) folded into the one read of X the preparation makes. */
int nenmf_prepare_x_checked(int dtype, const void* X, int64_t n, int64_t m, int64_t ldx, int64_t k,
                            void* Xp, int* nonzero, void* stream);
size_t nenmf_dual_pass_prepared_workspace_bytes(int dtype, int64_t n, int64_t m, int64_t k);
int nenmf_dual_pass_prepared(int dtype, const void* Xp, int64_t n, int64_t m,
                             const void* At, const void* Bt, int64_t k, void* Yt, void* Zt,
                             void* ws, size_t ws_bytes, void* stream);
size_t nenmf_rsi_prepared_workspace_bytes(int dtype, int64_t n, int64_t m, int64_t nu);
int nenmf_rsi_prepared(int dtype, const void* X, const void* Xp, int64_t n, int64_t m,
                       int64_t ldx, const void* omega_l_t, const void* omega_r, int64_t nu,
                       int q, void* L, void* Rt, nenmf_device_status* status,
                       void* ws, size_t ws_bytes, void* stream);
/* Randomized power iteration (compression.py:144-176): the products of
 * nenmf_rsi without the intermediate orthonormalisations, one at the end.
 * Status NUMERICAL_COLLAPSE with iteration k when an iterate overflows at
 * step k (FP32 tracks power-of-two scale factors so the fp64 overflow point
 * is reproduced) or, with iteration q, when a column is entirely zero.  Xp
 * may be NULL; workspace: nenmf_rsi_prepared_workspace_bytes (Xp given) or
 * nenmf_rsi_workspace_bytes. */
int nenmf_power_iteration(int dtype, const void* X, const void* Xp, int64_t n, int64_t m, int64_t ldx,
                          const void* omega_l_t, const void* omega_r, int64_t nu, int q, void* L,
                          void* Rt, nenmf_device_status* status, void* ws, size_t ws_bytes,
                          void* stream);
int nenmf_compress_prepared(int dtype, const void* X, const void* Xp, int64_t n, int64_t m,
                            int64_t ldx, const void* L, const void* Rt, int64_t nu,
                            void* XL, void* XRt, void* ws, size_t ws_bytes, void* stream);

/* ---- NMFB payload conversion (matrix.py:180-214) -------------------------
 * dst[i] = (dtype) src[i] for count float64 values already on the device (a
 * chunk of an NMFB file's little-endian payload; src 16-byte aligned); sets
 * *nonfinite (device int) to 1 if any value is NaN/Inf (read_nmfb's
 * require_finite, matrix.py:39-42).  dtype NENMF_F64 copies. */
int nenmf_convert_f64(int dtype, const double* src, int64_t count, void* dst, int* nonfinite, void* stream);

/* ---- measurement hooks (not part of the reference interface) ------------
 * While enabled, every tensor-core X-pass kernel launch is bracketed by CUDA
 * events on its stream; nenmf_debug_xpass_ms waits for them and returns the
 * number of launches timed and their total duration (the roofline of
 * bench.py is computed from the kernel alone, not the small launches around
 * it).  Process-wide debug state. */
void nenmf_debug_xpass_timing(int on);
int nenmf_debug_xpass_ms(double* total_ms);

#ifdef __cplusplus
}
#endif
#endif /* NENMF_B200_H */
