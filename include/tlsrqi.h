/*
 * tlsrqi.h — C ABI of libtlsrqi.so, the B200 (sm_100a) hot path of
 * RQI-PCGTLS-MP (Oktay & Carson, arXiv 2305.19028).
 *
 * Problem (§1): total least squares
 *     min ||[E, r]||_F  subject to  (A + E) x = b + r,
 * solved through the smallest singular pair of [A, b]:  sigma_{n+1} and
 * x_TLS = -v_{1:n,n+1} / v_{n+1,n+1}.
 * Method: Rayleigh quotient iteration on [A,b]^T[A,b] (Alg. 4, l.221-258),
 * each step two PCGTLS solves with A^T A - sigma_k^2 I (Alg. 3, l.186-204)
 * preconditioned by P = R~ D, R~ an upper-triangular factor of the Gram of
 * A D^{-1} computed from data rounded to u_f and stored in u_f (l.213,
 * l.231, l.290-307).  The readings R1..R18 cited below are DESIGN.md §3.
 *
 * Conventions for every entry point
 *  - Pointers named *_dev are CUDA device pointers on the calling thread's
 *    current device; *_host are host pointers.  The caller owns all of them;
 *    the library never retains them after the call returns.
 *  - `stream` is a cudaStream_t (passed as void*); all device work of a call
 *    is enqueued on it.  Calls that return results to the host
 *    (tls_factor_precond, tls_rqi_pcgtls, tls_solve_host) synchronise it.
 *  - Scratch memory comes from the caller's workspace `ws_dev` of
 *    `ws_bytes` >= tls_workspace_size(...) bytes (256-byte aligned).  The only
 *    allocations the library makes itself belong to a tls_precond_t handle.
 *  - Return value: 0 = OK; > 0 = numerical outcome with partial results
 *    (TLS_CHOL_BREAKDOWN .. TLS_STAGNATED); < 0 = usage or runtime error
 *    (TLS_ERR_*).  tls_last_error() gives a thread-local message.
 *  - Multi-GPU (row sharding): every rank passes its own
 *    contiguous row block of A and b (m_local rows, row_offset = first global
 *    row) and the same comm; all ranks must make the same calls with the same
 *    scalar arguments.  n-vectors and results are replicated on every rank.
 *    comm = NULL means one GPU.
 */
#ifndef TLSRQI_H
#define TLSRQI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLSRQI_ABI_VERSION 6

#if defined(__GNUC__)
#define TLS_API __attribute__((visibility("default")))
#else
#define TLS_API
#endif

/* Number formats (Table 2 l.435-447; bf16 reading R12). */
typedef enum { TLS_FP16 = 0, TLS_BF16 = 1, TLS_FP32 = 2, TLS_FP64 = 3 } tls_prec_t;

/* Matrix layouts. */
typedef enum { TLS_DENSE_ROWMAJOR = 0, TLS_CSR = 1 } tls_layout_t;

/* Status codes. */
enum {
  TLS_OK = 0,
  TLS_CHOL_BREAKDOWN = 1, /* non-positive / non-finite Cholesky pivot */
  TLS_PCG_BREAKDOWN = 2,  /* delta_j <= 0 in PCGTLS (Alg. 3 l.192; reading R3) */
  TLS_MAX_OUTER = 3,      /* max_outer RQI steps without meeting a stop test (R6) */
  TLS_NONFINITE = 4,      /* sigma^2 or psi not finite */
  TLS_RANGE = 5,          /* A D^{-1} or R~ overflows u_f (reading R4) */
  TLS_NOT_MINIMAL = 6,    /* opts.minimal_check: A^T A - sigma^2 I not positive definite at the result (R28) */
  TLS_STAGNATED = 7,      /* psi rose before the tol crossing (R7) */
  TLS_ERR_ARG = -1, TLS_ERR_CUDA = -2, TLS_ERR_NCCL = -3, TLS_ERR_WORKSPACE = -4,
  TLS_ERR_UNSUPPORTED = -5
};

/* Termination reasons reported in tls_info_t.termination. */
enum {
  TLS_TERM_NONE = 0, TLS_TERM_CONVERGED_TOL = 1, TLS_TERM_PSI_INCREASE_CONVERGED = 2,
  TLS_TERM_STAGNATED = 3, TLS_TERM_MAX_OUTER = 4, TLS_TERM_BREAKDOWN = 5, TLS_TERM_NONFINITE = 6
};

/* The local row block of A (m_global x n).  Dense: `vals` is m_local x ld
 * fp64 row-major, ld >= n, ld even, vals 16-byte aligned (rows are streamed
 * with 16-byte bulk copies).  CSR: rowptr (m_local+1, int64, rowptr[0] = 0),
 * colidx (nnz_local, int32, ascending within a row), vals (nnz_local fp64). */
typedef struct {
  int32_t layout;       /* tls_layout_t */
  int32_t reserved;
  int64_t m_local, n, m_global, row_offset, ld;
  const double* vals;   /* device */
  const int64_t* rowptr;/* device, CSR only */
  const int32_t* colidx;/* device, CSR only */
  int64_t nnz_local;
} tls_matrix_t;

typedef struct tls_comm_s* tls_comm_t;       /* wraps an ncclComm_t */
typedef struct tls_precond_s* tls_precond_t; /* owns R~ (u_f), D, block inverses */

/* Options (defaults in brackets; tls_rqi_opts_default fills them). */
typedef struct {
  int32_t budget_rule;    /* 0: k+1 PCG steps at RQI step k [0]; 1: until tol, cap 400 */
  int32_t stop_rule;      /* 0: strict psi increase (l.265) [0]; 1: weak >= (l.532) */
  int32_t max_outer;      /* [50] */
  int32_t polish;         /* RQI steps after the tol crossing (R6) [1] */
  double tol_inner;       /* PCG early exit eta <= tol_inner^2 eta_0; <= 0 means tol [-1] */
  int32_t boot;           /* 0: x_LS by preconditioned CGLS (R5) [0]; 1: semi-normal */
  int32_t boot_max;       /* [200] */
  double boot_tol;        /* [1e-8] */
  int32_t op_variant;     /* 0: A-in-loop operator (R1) [0]; 1: the paper's A-free Alg. 3 as printed
                             (delta = p^T p - sigma^2 q^T q, w = p - sigma^2 P^{-T} q;
                             no pass over A inside PCGTLS; the sigma = 0 bootstrap stays A-in-loop) */
  int32_t breakdown_rule; /* 0: delta < 0 is a breakdown (R3) [0]; 1: only delta == 0 stops */
  int32_t gram_chunk;     /* K_t rows per fp32 accumulation chunk (R11) [64]; multiple of 64 for the tensor-core path */
  int32_t u_p;            /* precision of the PCGTLS operator A^T A q of the RQI's inner solves (R23):
                             0 or TLS_FP64 [0]; TLS_FP32 = the paper's experimental setting u_p = single
                              on an fp32 copy of A made by the solve and kept in the
                             precond handle (4 m_local ld32 bytes, dense A, n <= 2048, op_variant 0).
                             The bootstrap, the residual passes and all n-vector work stay fp64. */
  int32_t precond_apply;  /* how q = P^{-1} p and w = P^{-T} y are applied (R24): 1 = forward/back
                             substitution with the stored R~ ("Forward/Backward Subs",
                             l.427); 2 = products with W = R~^{-1} formed once per handle in fp64 (npad^2
                             doubles owned by the handle); 0 = auto [0]: 2 when comm has several ranks,
                             else 1 */
  int32_t certify;        /* 1: after the solve, sigma_certified = sqrt(||b - A x||^2 / (1 + ||x||^2)) with
                             every residual and sum by Dot2 (compensated; one more pass over A;
                             SURVEY §8(c) c2 step 8); 0 [0]: skipped, sigma_certified = NaN */
  int32_t minimal_check;  /* R28: after an OK solve, this many PCGTLS steps at the returned sigma^2 on a fixed
                             counter-based right-hand side; a curvature delta_j <= 0 shows A^T A - sigma^2 I is
                             not positive definite (sigma >= sigma'_n: not the TLS solution, PAPER.md
                             l.266-268) and the status becomes TLS_NOT_MINIMAL (x, sigma and the termination
                             are kept).  One pass over A per step.  0 [0]: off */
  int32_t reserved;
} tls_rqi_opts_t;

/* Results.  pcg_iters (2*max_outer ints), sigma2_trace, psi_trace
 * (max_outer+1 doubles each) are optional caller-owned host arrays. */
typedef struct {
  int32_t status, termination;
  int32_t rqi_iters;      /* k at which the loop stopped (number of residual evaluations) */
  int32_t boot_iters;     /* CGLS iterations of the bootstrap (R5) */
  int32_t* pcg_iters;     /* [2*(k-1)]: counts of solve (a) -f and (b) x_k per RQI step */
  double* sigma2_trace;   /* sigma_k^2, k = 1..rqi_iters */
  double* psi_trace;      /* psi_k */
  int32_t breakdown_k, breakdown_rhs, breakdown_j, chol_pivot;
  double sigma2;          /* sigma^2 of the returned iterate */
  int64_t passes;         /* passes over A made by the call */
  int32_t launches;       /* kernels launched by the call (this library's kernels only) */
  int32_t pcg_steps;      /* RQI steps whose PCGTLS counts are in pcg_iters */
  double sigma_certified; /* compensated sigma of the returned x (opts.certify), else NaN */
  double* delta_min_trace;/* optional [2*(k-1)]: smallest curvature delta_j = p_j^T C p_j seen by solve (a) and
                             (b) at each RQI step (the per-step trace of SURVEY §8(c) c2 step 9) */
} tls_info_t;

TLS_API int tls_abi_version(void);
TLS_API void tls_rqi_opts_default(tls_rqi_opts_t* opts);
TLS_API const char* tls_status_string(int status);
TLS_API const char* tls_last_error(void);

/* ---- communicator (NCCL over NVLink/NVSwitch; libnccl.so.2 is dlopen'ed) ---- */
/* Rank 0 creates the 128-byte unique id and broadcasts it (e.g. with
 * torch.distributed) before every rank calls tls_comm_init. */
TLS_API int tls_comm_get_unique_id(void* id_out_host /* 128 bytes */);
TLS_API int tls_comm_init(int nranks, int rank, const void* id_host, int device, tls_comm_t* out);
/* Host-staged communicator for ranks that are processes sharing ONE GPU (PAPER.md has no
 * multi-GPU design; this exercises the row-sharded path of SURVEY §8(e) on a single device).
 * Every rank calls it with the same `name` (a POSIX shared-memory name starting with '/',
 * unique per run: a stale segment of the same name is reused as is) and `slot_bytes` (the
 * per-rank staging slot, >= 4096 and a multiple of 256; larger all-reduces run in chunks).
 * Each collective synchronises the caller's stream, exchanges through the segment and sums
 * the ranks' contributions on the host in rank order 0..P-1, so every rank gets identical
 * bits; no kernel waits for another rank.  A rank that waits more than 120 s for the others
 * returns TLS_ERR_NCCL.  Returns after every rank has mapped the segment; rank 0 unlinks it in
 * tls_comm_destroy (which is collective for this backend). */
TLS_API int tls_comm_init_shm(int nranks, int rank, const char* name, size_t slot_bytes, int device,
                              tls_comm_t* out);
/* Peer-memory exchange of the operator pass's sums (the one-shot,
 * rank-ordered reduction over NVLink instead of ncclAllReduce for the 2n+2 (n+2) pass sums of
 * PAPER.md Alg. 3 / Alg. 4; k_peer.cu).  Attached to an existing communicator (NCCL or shm, which
 * still serves the other collectives):
 *   tls_comm_peer_prepare: allocates this rank's receive buffer (2 x nranks x wcap doubles, wcap >=
 *     2n + 2 of every solve that uses the communicator) and flags on the communicator's device and
 *     writes their two CUDA-IPC handles (128 bytes) to handles_out (host);
 *   every rank then gathers all ranks' 128-byte records in rank order (e.g. torch.distributed
 *     all_gather) and calls tls_comm_peer_connect(comm, all_handles) (nranks x 128 bytes, host),
 *     which maps the peers' buffers.
 * From then on each dense operator/residual pass ends with ONE kernel that reduces this rank's
 * per-CTA partial sums, stores them into every rank's buffer over peer memory, waits for all
 * ranks' (flags, system scope) and sums the ranks' contributions in rank order 0..P-1 (identical
 * bits on every rank; the same order as the shm backend).  The ranks' kernels wait for each
 * other, so every rank must run on its own GPU, concurrently.  A wait that times out makes the
 * call return TLS_ERR_NCCL.  Up to 8 ranks.  Errors: TLS_ERR_ARG (order of calls, sizes),
 * TLS_ERR_CUDA (allocation, IPC). */
TLS_API int tls_comm_peer_prepare(tls_comm_t comm, int64_t wcap, void* handles_out /* 128 bytes */);
TLS_API int tls_comm_peer_connect(tls_comm_t comm, const void* all_handles /* nranks x 128 bytes */);
/* Test hook for the exchange kernel on ONE GPU: nranks emulated ranks in one cooperative launch
 * (the pool forbids separate launches that wait for each other on one device).  partials: device,
 * [nranks][G][W] (rank r's G per-CTA rows); out: device, [nranks][W] (rank r's result); `reps`
 * exchanges in a row (epochs 1..reps: the double-buffered slots are reused).  Allocates and frees
 * its own buffers; synchronises `stream`. */
TLS_API int tls_peer_exchange_emulate(int nranks, const double* partials, int G, int W, int reps, double* out,
                                      void* stream);
TLS_API int tls_comm_nranks(tls_comm_t comm);   /* 1 for NULL */
TLS_API int tls_comm_rank(tls_comm_t comm);     /* 0 for NULL */
TLS_API int tls_comm_destroy(tls_comm_t comm);

/* Workspace bytes for tls_factor_precond and tls_rqi_pcgtls on this A. */
TLS_API size_t tls_workspace_size(const tls_matrix_t* A, int32_t max_outer);

/* ---- preconditioner build (§8 rows a1-a3) ----
 * d_j = 2^floor(log2 max_i |a_ij|) (reading R2);
 * G = sum over K_t-row chunks of fp32-accumulated A^_c^T A^_c, A^ = fl_uf(A D^{-1})
 * (u_f = fp16/bf16 on tensor cores; fp32/fp64 in fp64), summed in fp64 and
 * all-reduced over ranks (R10, R11); G = R^T R by a blocked fp64 Cholesky;
 * R~ = fl_uf(R) kept in the handle.  On TLS_CHOL_BREAKDOWN info->chol_pivot is
 * the 1-based pivot and *R_out is NULL. */
TLS_API int tls_factor_precond(const tls_matrix_t* A, int32_t u_f, const tls_rqi_opts_t* opts,
                       tls_comm_t comm, void* stream, void* ws_dev, size_t ws_bytes,
                       tls_precond_t* R_out, tls_info_t* info);

/* ---- the paper's preferred preconditioner: Householder QR in u_f ----
 * PAPER.md l.215-218 and Alg. 4 l.231 "Compute A = Q[R 0]^T in u_q"; readings R25, R26.
 * R~ = the R factor (diag >= 0) of a Householder QR of fl_uf(A D^{-1}), with the same D
 * and ||A||_F^2 as tls_factor_precond; every elementwise operation is rounded to u_f, inner
 * products are accumulated in fp64 and rounded once.  The returned handle is used exactly
 * like a Cholesky one.  Dense A only (CSR: TLS_ERR_ARG).
 * Row-sharded A (comm with nranks > 1) or TSQR leaves (environment TLS_QR_LEAVES = k,
 * default 1: each rank's rows split into k contiguous blocks [s m/k, (s+1) m/k)): every
 * leaf is factored as above, the leaf R's are stacked row-interleaved (row i of leaf L =
 * rank * k + s at stack row i * leaves + L; the stack all-reduced over the ranks, each rank
 * filling only its own rows), and R~ is the R factor of the stack, computed the same way
 * without further scaling and skipping the stack rows that are still zero (R26).  Every leaf
 * needs >= n rows (else TLS_ERR_ARG).  R~ is identical on every rank.
 * ws_dev: ws_bytes >= tls_qr_workspace_size(A, u_f, nranks) bytes (it holds an m_local x n
 * fp32 -- fp64 for u_f = TLS_FP64 -- working copy of the rows, and for TSQR the stack and
 * its working copy).  A column that becomes exactly zero in u_f: TLS_CHOL_BREAKDOWN,
 * info->chol_pivot = its 1-based index (within the leaf or stack factorization where it
 * happened), *R_out = NULL.  An inner product or reflector overflowing u_f (e.g. a column
 * with x^T x > 65504 in fp16): TLS_RANGE, *R_out = NULL.  The stream is synchronised once at
 * the end; the environment knobs TLS_QR_PDL=0 (plain launches) and TLS_QR_COOP=1 (one
 * cooperative kernel for the column loop) select measured-slower variants for comparison.
 * tls_qr_workspace_size returns 0 for CSR, a bad u_f or nranks < 1. */
TLS_API size_t tls_qr_workspace_size(const tls_matrix_t* A, int32_t u_f, int32_t nranks);
TLS_API int tls_factor_precond_qr(const tls_matrix_t* A, int32_t u_f, tls_comm_t comm, void* stream, void* ws_dev,
                                  size_t ws_bytes, tls_precond_t* R_out, tls_info_t* info);

/* The same preconditioner with the trailing updates blocked (reading R29; SURVEY §8(f) NEXT-2
 * "on tensor cores"): panels of 128 columns factored as tls_factor_precond_qr does (R25, D of
 * R27), the panel's 128 reflectors applied to the trailing columns at once in compact WY form
 * C <- C - V (T^T (V^T C)) with V^T C and V^T V on tcgen05 (fp32 sums per 64-row chunk, fp64
 * across, as R11), T in fp64, Y = T^T V^T C rounded to u_f and V Y on tcgen05 (fp32), the
 * difference rounded once to u_f.  In exact arithmetic the same R as the unblocked QR; in u_f
 * another backward-stable rounding sequence (oracle.qr.householder_qr_r_blocked).  u_f = fp16
 * or bf16, dense A, one rank (m_global == m_local), n <= 2048.  Workspace:
 * tls_qr_blocked_workspace_size (the unblocked QR's plus a 16-bit copy of A and the WY panels). */
TLS_API size_t tls_qr_blocked_workspace_size(const tls_matrix_t* A, int32_t u_f);
TLS_API int tls_factor_precond_qr_blocked(const tls_matrix_t* A, int32_t u_f, void* stream, void* ws_dev,
                                          size_t ws_bytes, tls_precond_t* R_out, tls_info_t* info);

/* Handle from host data (tests: import the oracle's R~ to isolate PCG/RQI
 * parity).  Rt_host: n x n row-major upper-triangular values already
 * representable in u_f; d_host: n powers of two; normA2 = ||A||_F^2 (global). */
TLS_API int tls_precond_import(int64_t n, int32_t u_f, const double* Rt_host, const double* d_host,
                       double normA2, void* stream, tls_precond_t* out);
/* Copy R~ (n x n row-major, upcast to fp64), d and ||A||_F^2 back to the host. */
TLS_API int tls_precond_export(tls_precond_t R, double* Rt_host, double* d_host, double* normA2_host);
TLS_API void tls_precond_destroy(tls_precond_t R);

/* ---- the RQI-PCGTLS-MP solve (§8 rows a4-a9) ----
 * R must come from this A (same n and, for a factored handle, the same m_global and the same
 * content: the handle keeps a checksum of 256 evenly spread rows of this rank's block, taken at
 * the factorization and compared at every solve -- an A rewritten in place is TLS_ERR_ARG;
 * imported handles are not checked).  u and u_r must be TLS_FP64 (north_star); tol is the
 * primary stop psi_k <= tol ||[A,b]||_F^2 (R6).  x_out_dev (n fp64) receives the returned
 * iterate on every rank, *sigma_out_host = sqrt(sigma^2) of that iterate.
 * Without per-launch profiling and on one rank, each PCG loop runs as a CUDA graph whose
 * trip count is decided on the device (TLS_PCG_GRAPH=0: host loop; same kernels, same bits).
 * Handle-owned allocations made by the first solve that needs them (freed or pooled by
 * tls_precond_destroy): the explicit inverse W (2 npad^2 doubles, precond_apply = 2 or a
 * sharded solve) and the fp32 copy of the local block (u_p = fp32); tls_precond_prepare makes
 * them beforehand, after which the solve allocates nothing.  An NCCL error raised
 * asynchronously is reported as TLS_ERR_NCCL at the end of the call. */
/* Makes the handle-owned buffers of R that a solve would otherwise allocate on first use, so that
 * tls_rqi_pcgtls then allocates nothing: what = 1 the explicit inverse W = R~^{-1} and W^T
 * (2 npad^2 doubles, reading R24), 2 the fp32 copy of this rank's block of A (u_p = fp32, R23;
 * checked against the handle's content checksum like a solve), 3 both.  ws_dev / ws_bytes as for
 * tls_rqi_pcgtls (used for what & 2).  Synchronises `stream`.  Errors: TLS_ERR_ARG (what, R of
 * another A), TLS_ERR_WORKSPACE, TLS_ERR_UNSUPPORTED (fp32 copy of a CSR A or n > 2048),
 * TLS_ERR_CUDA (allocation). */
TLS_API int tls_precond_prepare(const tls_matrix_t* A, tls_precond_t R, int32_t what, void* stream, void* ws_dev,
                                size_t ws_bytes);
TLS_API int tls_rqi_pcgtls(const tls_matrix_t* A, const double* b_local_dev, const tls_precond_t R,
                   int32_t u, int32_t u_r, double tol, const tls_rqi_opts_t* opts,
                   tls_comm_t comm, void* stream, void* ws_dev, size_t ws_bytes,
                   double* x_out_dev, double* sigma_out_host, tls_info_t* info);

/* End-to-end from HOST buffers: copies this rank's row block of A (m_local x ld
 * row-major, global rows [row_offset, row_offset + m_local) of m_global) and b
 * into the caller's device buffer `dev_buf` (>= tls_solve_host_bytes), factors,
 * solves (all-reducing over `comm` when not NULL) and copies x back to x_host.
 * Pinned host memory gives asynchronous copies. */
TLS_API size_t tls_solve_host_bytes(int64_t m_local, int64_t n, int64_t ld, int32_t max_outer);
TLS_API int tls_solve_host(const double* A_host, const double* b_host, int64_t m_local, int64_t n,
                           int64_t ld, int64_t m_global, int64_t row_offset, int32_t u_f, double tol,
                           const tls_rqi_opts_t* opts, tls_comm_t comm, void* stream, void* dev_buf,
                           size_t dev_bytes, double* x_host, double* sigma_out_host, tls_info_t* info);

/* ---- single steps, exposed for step-level parity tests and profiling ---- */
/* a1: per-column max |a_ij| and ||A||_F^2 of the local block (not reduced over ranks).
 * colmax_dev: n doubles; sumsq_dev: 1 double. */
TLS_API int tls_colstats(const tls_matrix_t* A, double* colmax_dev, double* sumsq_dev, void* stream,
                 void* ws_dev, size_t ws_bytes);
/* a2: G_dev (n x n fp64 row-major, full symmetric) = Gram of fl_uf(A D^{-1}) of the
 * local block with K_t-row fp32 chunks (u_f fp16/bf16) or fp64 (fp32/fp64). */
TLS_API int tls_gram(const tls_matrix_t* A, int32_t u_f, const double* d_dev, int32_t K_t,
             double* G_dev, void* stream, void* ws_dev, size_t ws_bytes);
/* a7 / a5: one pass over the local block with nrhs in {1,2}:
 *   mode 0 (operator): t_r = A q_r; v_r = A^T t_r; s[r] = t_r^T t_r
 *   mode 1 (residual): t = b - A q_0; v_0 = A^T t; s[0] = t^T t; s[1] = b^T t
 * q_dev: nrhs x n (row r at q_dev + r*n); v_dev: nrhs x n; s_dev: 2 doubles. */
TLS_API int tls_pass(const tls_matrix_t* A, int32_t mode, int32_t nrhs, const double* q_dev,
             const double* b_dev, double* v_dev, double* s_dev, void* stream, void* ws_dev,
             size_t ws_bytes);
/* a7 with u_p = fp32 (R23): the 2-RHS operator pass on R's fp32 copy of this A (made on
 * first use): t_r = fl32(A) fl32(q_r) and v_r = fl32(A)^T t_r accumulated in fp32, s[r] =
 * t_r^T t_r in fp64.  q_dev, v_dev: 2 x n fp64; s_dev: 2 doubles. */
TLS_API int tls_pass_fp32(const tls_matrix_t* A, tls_precond_t R, const double* q_dev, double* v_dev,
                          double* s_dev, void* stream, void* ws_dev, size_t ws_bytes);
/* a6: Y_dev (nrhs x n) <- P^{-1} Y (trans = 0: D^{-1} R~^{-1} Y, back substitution)
 * or P^{-T} Y (trans = 1: R~^{-T} D^{-1} Y, forward substitution), nrhs in {1,2}.
 * trans | 2: the same maps through the explicit inverse W = R~^{-1} (R24; W is formed
 * once and kept by the handle). */
TLS_API int tls_precond_apply(const tls_precond_t R, int32_t trans, int32_t nrhs, double* Y_dev,
                      void* stream);
/* fl_uf rounding of n fp64 values (reading R4), for bit-exact parity tests. */
TLS_API int tls_round(const double* x_dev, double* y_dev, int64_t n, int32_t prec, void* stream);

/* ---- per-kernel timing (CUDA events recorded on the launch stream around
 * each launch of the listed kernels; used by bench.py for the roofline) ---- */
enum {
  TLS_PROF_PASS_OP2 = 0,  /* operator pass, 2 RHS (a7) */
  TLS_PROF_PASS_OP1 = 1,  /* operator pass, 1 RHS (bootstrap CGLS) */
  TLS_PROF_PASS_RESID = 2,/* residual pass (a5, a1 at x = 0) */
  TLS_PROF_COLSTATS = 3,  /* column statistics pass (a1) */
  TLS_PROF_GRAM = 4,      /* u_f Gram incl. split reduction (a2) */
  TLS_PROF_CHOL = 5,      /* blocked Cholesky (a3) */
  TLS_PROF_PCG_STEP = 6,  /* fused PCG step: fwd solve + recurrences + back solve (a6, a8) */
  TLS_PROF_PCG_INIT = 7,  /* PCG initialisation: fwd + back solve (a6) */
  TLS_PROF_REDUCE = 8,    /* fixed-order partial reductions */
  TLS_PROF_PASS_OP2_FP32 = 9, /* operator pass on the fp32 copy of A (u_p = fp32, R23) */
  TLS_PROF_NCAT = 10
};
/* Enable (1) or disable (0) timing; both reset the accumulated totals. */
TLS_API int tls_profile_enable(int on);
/* Total milliseconds and launch counts per category (arrays of ncat entries).
 * Synchronises on the recorded events. */
TLS_API int tls_profile_read(double* ms_host, int64_t* count_host, int ncat);

#ifdef __cplusplus
}
#endif
#endif /* TLSRQI_H */
