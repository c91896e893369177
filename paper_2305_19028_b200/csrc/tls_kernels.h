// tls_kernels.h — host-side launchers of the libtlsrqi kernels (internal).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tls {

constexpr int kMaxDenseN = 4096;   // register-resident column ownership in k_pass (CPT <= 8)

int num_sms();
bool pass_pdl();   // programmatic dependent launch of passes and PCG steps (TLS_PDL=0: off)

// ---- streaming passes over A (k_pass.cu) ---------------------------------------------
enum PassMode { PASS_OPERATOR = 0, PASS_RESIDUAL = 1, PASS_COLSTATS = 2 };
struct DenseView {
  const double* A;
  int64_t m;
  int n;
  int64_t ld;
};
// CTAs used by one pass and the partial-buffer doubles it needs.
int pass_grid(const DenseView& A);
size_t pass_partials_doubles(const DenseView& A);
// Writes gridDim x W partials; W = nrhs*n + 2 (operator/residual) or 2n (colstats).
// `active` (may be NULL): int[2] of PCG activity flags; the kernel is a no-op when both are 0.
int launch_pass(const DenseView& A, int mode, int nrhs, const double* q, const double* b,
                double* partials, const int* active, cudaStream_t st, int* grid_out);
// u_p = fp32 operator pass (k_pass32.cu, R23): A32 = fl32(A) row-major with ld32 = p32_ld(n);
// 2 RHS, writes grid x (2n + 2) partials like launch_pass (grid <= pass_partials rows).
int p32_ld(int n);
int launch_round32(const DenseView& A, float* A32, cudaStream_t st);
int launch_pass32(const DenseView& A, const float* A32, const double* q, double* partials, const int* active,
                  cudaStream_t st, int* grid_out);
// fp64 operator (2 RHS) / residual passes in k_pass32.cu's team-per-row layout.
int launch_pass_team(const DenseView& A, int mode, const double* q, const double* b, double* partials,
                     const int* active, cudaStream_t st, int* grid_out);
// out[w] = sum_g partials[g][w] (max for w < nmax), fixed order.
// Peer-memory exchange (k_peer.cu, NEXT-3): receive buffers and flags of every rank, as this
// rank sees them (its own: local pointers; the others': CUDA-IPC peer mappings).
constexpr int kMaxPeers = 8;
constexpr int kXchCtas = 128;         // CTAs per rank of k_reduce_exchange (column slices of 32)
struct PeerTab {
  double* rbuf[kMaxPeers];            // rank p's receive buffer: [2 parities][P slots][wcap] doubles
  int* rflag[kMaxPeers];              // rank p's flags: [P ranks][kXchCtas]
};
// passout of `ranks_here` ranks (rank0 ..) = rank-ordered sum over all P ranks of each rank's
// fixed-order reduction of its G partial rows (k_reduce_partials' order); `cooperative` for the
// one-GPU emulation where all P ranks run in this launch.
int launch_reduce_exchange(const PeerTab& pt, int P, int rank0, int ranks_here, const double* partials, size_t pstride,
                           int G, int W, int wcap, double* out, size_t ostride, int epoch, const int* active, int* err,
                           bool cooperative, cudaStream_t st);
int launch_reduce(const double* partials, int G, int W, int nmax, double* out, const int* active,
                  cudaStream_t st);
// d_j = 2^floor(log2 colmax_j), dinv_j = 1/d_j, normA2 = sum_j sumsq_j; *flag = 1 on a zero or
// non-finite column.
int launch_scaling(const double* colmax, const double* sumsq, int n, double* d, double* dinv,
                   double* normA2, int* flag, cudaStream_t st, int mode = 0);
int launch_round(const double* x, double* y, int64_t n, int prec, cudaStream_t st);

// ---- CSR (k_csr.cu) --------------------------------------------------------------------
struct CsrView {
  const int64_t* rowptr;  // m + 1
  const int32_t* colidx;  // nnz, ascending within a row
  const double* vals;     // nnz
  int64_t m;
  int n;
  int64_t nnz;
};
// sampled content checksum of a local block (k_pass.cu): 256 evenly spread rows; scratch: 256 doubles
int launch_fingerprint(const DenseView* dv, const CsrView* cv, double* out, double* scratch, cudaStream_t st);

struct CscView {          // transpose of a CsrView, rows ascending within every column
  int64_t* colptr;        // n + 1
  int32_t* rowidx;        // nnz
  double* vals;           // nnz
};
// colstats[0..n) = per-column max |a_ij|, colstats[n] = ||A||_F^2, colstats[n+1..2n) = 0.
// partials: kCsrRowCTAs doubles.
int launch_csr_colstats(const CsrView& A, double* colstats, double* partials, cudaStream_t st);
// G (n x n, full symmetric) = Gram of fl_uf(A D^{-1}); fp16: exact fixed-point sum in ws
// (csr_gram_ws_bytes), rounded once; with fixed_point_out the limbs are left in ws (two
// n x n int64 arrays, for an exact all-reduce) and launch_csr_gram_fin converts them.
size_t csr_gram_ws_bytes(int n);
int launch_csr_gram(const CsrView& A, int u_f, const double* dinv, double* G, void* ws, size_t ws_bytes,
                    int* range_flag, cudaStream_t st, int* launches, bool fixed_point_out);
int launch_csr_gram_fin(const void* ws, int n, double* G, cudaStream_t st);
size_t csc_scratch_bytes(int64_t m, int n);
int launch_csc_build(const CsrView& A, CscView C, void* scratch, cudaStream_t st, int* launches);
size_t csr_pass_partials_doubles();
// out = [v_0 .. v_{nrhs-1} (stride n), s0, s1] as in launch_pass + launch_reduce;
// tbuf: nrhs * m doubles.
int launch_csr_pass(const CsrView& A, const CscView& C, int mode, int nrhs, const double* q, const double* b,
                    double* tbuf, double* partials, double* out, const int* active, cudaStream_t st);

// ---- Gram (k_gram.cu: CUDA-core fp64/fp32 path; k_gram_tc.cu: tcgen05 path) -------------
size_t gram_ws_doubles(const DenseView& A, int K_t);   // workspace of either path (doubles)
bool gram_tc_supported(int u_f, int K_t);
size_t gram_tc_ws_bytes(int64_t m, int n, int K_t);
int launch_gram_tc(const DenseView& A, int u_f, const double* dinv, int K_t, double* G, void* ws, size_t ws_bytes,
                   int* range_flag, cudaStream_t st, int* launches);
int launch_gram(const DenseView& A, int u_f, const double* dinv, int K_t, double* G, double* ws,
                size_t ws_doubles, int* range_flag, cudaStream_t st, int* launches);

// ---- Cholesky and R~ packing (k_chol.cu) -----------------------------------------------
// Cholesky G = R^T R (n x n row-major, input and output R in the upper triangle; the
// lower triangle is not touched) by the tile-DAG kernel of k_chol_dag.cu.  *pivot =
// 1-based index of the first failed pivot (0 if none).  ws: >= chol_ws_bytes(n).
size_t chol_ws_bytes(int n);
int launch_cholesky(double* G, int n, int* pivot, void* ws, size_t ws_bytes, cudaStream_t st, int* launches);
// R~ = fl_uf(R) into the handle layouts; *range = 1 on overflow or a zero diagonal.
struct PrecondDev {
  int n, npad, u_f;
  void* Rrow;       // npad x npad u_f, row-major R~ (lower part 0, padded diagonal 1)
  void* RTrow;      // npad x npad u_f, row-major R~^T
  double* DinvB;    // (npad/32) blocks of 32x32: DinvB[kb][l][i] = (R~_kk^{-1})[i][l]
  double* DinvF;    // (npad/32) blocks of 32x32: DinvF[kb][l][i] = (R~_kk^{-1})[l][i]
  double* EB;       // (npad/32) blocks: EB[kb][l][i] = (R~_kk^{-1} R~_{k,k+1})[i][l]     (back solve)
  double* EF;       // (npad/32) blocks: EF[kb][l][i] = (R~_kk^{-T} R~_{k-1,k}^T)[i][l]  (forward solve)
  double* d;        // npad (1 on padding)
  double* dinv;     // npad
  double* normA2;   // 1 (device)
  const double* W = nullptr;   // explicit inverse R~^{-1} (fp64 npad x npad, upper) when the solve applies it (R24)
  const double* WT = nullptr;  // its transpose (lower), so both products run over contiguous rows
};
// W = R~^{-1} and WT = W^T (k_trtri in k_trsv.cu): npad x npad fp64 each, zeroed by the launcher.
int launch_trtri(const PrecondDev& pc, double* W, double* WT, cudaStream_t st);
// lower = 0: R upper (R[i][j], j >= i, row-major); lower = 1: R^T in the lower triangle.
int launch_pack_R(const double* R, int ldR, int lower, PrecondDev& pc, int* range, cudaStream_t st,
                  int* launches);
size_t precond_bytes(int n, int u_f);

// ---- triangular solves, PCG and RQI vector kernels (k_trsv.cu) -------------------------
struct PcgState {
  double eta[2], eta0[2], qq[2], pp[2], delta_min[2];
  double sigma2, g, psi, xx, tol2;
  int active[2], count[2], brk[2], brk_j[2];
  int iter[2];    // iteration index j of the next step, per RHS
  double bb;      // b^T b of the local rows (all-reduced), from the setup pass
  // the graph-captured PCG loop (NEXT-3, tls_api.cu pcg_loop): iteration j, budget, whether
  // the step computes the next q, and the iterations run so far (launch accounting)
  int loop_j, loop_budget, loop_nextq, loop_total;
};
struct PcgVecs {  // device, each [2][n] (RHS r at offset r * n)
  double *omega, *s, *p, *q, *rhs;
  double* w;      // P^{-T}-solve result of a step (explicit-inverse path, R24)
};
int launch_precond_apply(const PrecondDev& pc, int trans, int nrhs, double* Y, int ldY,
                         cudaStream_t st);
int launch_pcg_init(const PrecondDev& pc, int nrhs, PcgVecs v, PcgState* S, cudaStream_t st);
// One CTA per RHS; an RHS whose active flag is 0 is left untouched.
// variant 0: A-in-loop operator (R1; passout = the operator pass); variant 1: the
// paper's A-free Alg. 3 (delta = p^T p - sigma^2 q^T q, w = p - sigma^2 P^{-T} q;
// passout unused).
// pass_nrhs: the RHS count of the operator pass that filled passout (layout [v_0..v_{pass_nrhs-1}, tau..]).
// partials != nullptr (explicit-inverse step only, NEXT-3): passout is computed in the step's
// first phase from the G per-CTA partial rows of the operator pass (k_reduce_partials' order).
int launch_pcg_step(const PrecondDev& pc, PcgVecs v, const double* passout, PcgState* S, int nrhs,
                    int breakdown_rule, int compute_next_q, int variant, int pass_nrhs, cudaStream_t st,
                    const double* partials = nullptr, int G = 0, const int* nq_dev = nullptr);
// step record: sigma2, f (stored as rhs0 = -f), g, psi; copies x into rhs1.
int launch_rqi_eval(const PrecondDev& pc, const double* passout, const double* x, PcgVecs v,
                    PcgState* S, cudaStream_t st);
int launch_rqi_update(const PrecondDev& pc, PcgVecs v, const PcgState* S, double* x,
                      double* x_prev, cudaStream_t st);
// x1 = x0 + sigma0^2 P^{-1} P^{-T} x0, sigma0^2 = rho0/(1 + x0^T x0) (Alg. 4 l.229-235).
int launch_boot_x1(const PrecondDev& pc, const double* passout_r0, const double* x0, double* x1,
                   cudaStream_t st);

// compensated certificate (k_certify.cu): out[0..1] = Dot2 pair of ||b - A x||^2 over the
// local rows, out[2] = ||x||^2; part: certify_grid() x 2 doubles of scratch.
int certify_grid();
int launch_certify(const DenseView* D, const CsrView* S, const double* b, const double* x, int n, double* part,
                   double* out, cudaStream_t st);

// ---- Householder QR in u_f (k_qr.cu, reading R25) ---------------
int qr_rows_per_cta(int64_t m, int n);
int qr_ldw(int n, int u_f);                        // row stride of the working copy
size_t qr_work_bytes(int64_t m, int n, int u_f);   // W copy + partials + w^T + scalars + flags
// dinv == nullptr: no scaling (the TSQR stack of already scaled leaf R's)
// row_stride > 0: A is the row-interleaved TSQR stack of row_stride leaf R's (rows >= (j+2)
// row_stride are zero in columns j, j+1 and are skipped, R26)
// leaf = 1: a TSQR leaf (R26): a column vanishing on these rows takes the identity reflector
// (R_jj = 0) instead of raising the breakdown flag
int launch_qr(const DenseView& A, int u_f, const double* dinv, void* Wbuf, double* partP, double* wT, double* scal,
              int* qflags, double* G, cudaStream_t st, int* launches, int row_stride = 0, int leaf = 0);
// ---- blocked QR with tensor-core trailing updates (k_qr.cu + k_gram_tc.cu; reading R29) ----
size_t qr_wy_bytes(int64_t m, int n);             // buffers beyond the unblocked ones (W16, V, T, Y, ...)
int launch_qr_blocked(const DenseView& A, int u_f, const double* dinv, void* Wbuf, double* partP, double* wT,
                      double* scal, int* qflags, double* G, void* wy, cudaStream_t st, int* launches);
size_t tc_atb_ws_bytes(int nb);
int launch_tc_atb(int u_f, const uint16_t* a, int64_t lda, const uint16_t* b, int64_t ldb, int64_t m, int nb,
                  double* out, int ldo, double* part, size_t part_bytes, cudaStream_t st);
int launch_qr_wy_update(int u_f, const uint16_t* Vt, int64_t ldv, const uint16_t* Y, int64_t ldy, float* W,
                        uint16_t* W16, int64_t ldw, int64_t ld16, int64_t r0, int c0, int64_t m, int n, cudaStream_t st);

}  // namespace tls
