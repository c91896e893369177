// k_pass.cu — the HBM-bound streaming passes over A.
//
// One persistent CTA per SM streams a contiguous block of rows of A through a
// 6-stage shared-memory ring filled by the TMA bulk-copy engine
// (cp.async.bulk, one elected producer lane, mbarrier completion); 8 consumer
// warps own fixed column chunks (16 B each) of every row, so q and the
// accumulator v = A^T t live in registers for the whole pass and A is read from
// HBM exactly once.  Per group of rows the row dot products t_i = a_i . q are
// reduced across the CTA (warp transpose-reduce + one shared-memory exchange),
// then v += t_i a_i.  Modes:
//   operator (a7):  t = A q_r (r < nrhs), v_r = A^T t_r, s_r = t_r^T t_r
//   residual (a5):  t = b - A x, v = A^T t, s0 = t^T t, s1 = b^T t
//   colstats (a1):  per column max |a_ij| and sum a_ij^2
// Each CTA writes a partial; k_reduce_partials sums them in fixed CTA order
// (deterministic).
#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

constexpr int kPassConsumers = 256;
constexpr int kPassWarps = kPassConsumers / 32;
constexpr int kPassThreads = kPassConsumers + 32;   // one consumer set
constexpr int kPassNS = 2;                             // max consumer sets (even / odd stages)
// consumer sets per instantiation (measured): the 1-RHS passes (residual, 1-RHS operator)
// gain from two sets; the 2-RHS operator pass is register-limited with two (96 regs).
// (measured per shape, tools/time_pass.py); the column-statistics pass uses one set
constexpr int pass_sets_rt(int nrhs, int mode, int cpt) {
  return (mode != 2 /*PASS_COLSTATS*/ && (nrhs == 1 || cpt == 1)) ? 2 : 1;
}
constexpr int kPassRedDoubles = kPassWarps * 16 + 16 + 32;   // red + tfin + sred of one set
// (round 2: 3 stages of 64 KB with 8-row reduction groups for the 2-RHS pass measured slower,
// 1.265 vs 1.234 ms at 2^20 x 1024)
constexpr int kPassStages = 6;
constexpr int kPassStageBytes = 32 * 1024;
constexpr size_t kPassSmem = (size_t)kPassStages * kPassStageBytes + 2 * kPassStages * 8 +
                             (size_t)kPassNS * kPassRedDoubles * 8;

static int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// Programmatic dependent launch of the passes and the PCG steps (NEXT-3; TLS_PDL=0 disables).
bool pass_pdl() {
  static const bool on = [] { const char* e = getenv("TLS_PDL"); return !(e && e[0] == '0'); }();
  return on;
}

static int rows_per_stage(const DenseView& A) {
  int64_t r = kPassStageBytes / (A.ld * 8);
  return (int)(r < 1 ? 1 : r);
}

int pass_grid(const DenseView& A) {
  const int rps = rows_per_stage(A);
  int64_t stages = (A.m + rps - 1) / rps;
  int64_t g = num_sms();
  if (stages < g) g = stages;
  return (int)(g < 1 ? 1 : g);
}

size_t pass_partials_doubles(const DenseView& A) {
  return (size_t)pass_grid(A) * kPassNS * (size_t)(2 * A.n + 2);
}

// One group of RB rows of the current stage: row dot products t_r = a_i . q_r (thread
// partials over its column chunks, warp transpose-reduce, one shared-memory exchange
// across the consumer warps), then v_r += t_r a_i.  FULL: all RB rows and all column
// chunks exist (no predicates).  `stt` = this thread's first element of row rb.
template <int NRHS, int MODE, int CPT, int RB, bool FULL>
__device__ __forceinline__ void pass_group(const double* __restrict__ stt, int64_t ld, int rb, int rows, int64_t rs,
                                           const double* __restrict__ b, const double2 (&qr)[NRHS][CPT],
                                           double2 (&acc)[NRHS][CPT], const bool (&okc)[CPT], const bool (&ok1)[CPT],
                                           double* red, double* tfin, int warp, int lane, int tid, double& sacc,
                                           double& sacc2, int bar) {
  constexpr int V = RB * NRHS;
  double2 a[RB][CPT];
  double part[V];
  // residual mode: the thread that finishes row (rb + tid) loads b_i now, so the load is in
  // flight during the dot products instead of between the two barriers
  double bpre = 0.0;
  if (MODE == PASS_RESIDUAL && tid < V && (FULL || rb + tid < rows)) bpre = b[rs + rb + tid];
#pragma unroll
  for (int rr = 0; rr < RB; ++rr) {
    const double2* rowp = reinterpret_cast<const double2*>(stt + (size_t)rr * ld);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (FULL) {
        a[rr][c] = rowp[c * kPassConsumers];
      } else {
        double2 v = make_double2(0.0, 0.0);
        if (rb + rr < rows && okc[c]) {
          v = rowp[c * kPassConsumers];
          if (!ok1[c]) v.y = 0.0;
        }
        a[rr][c] = v;
      }
    }
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        d0 = fma(a[rr][c].x, qr[r][c].x, d0);
        d1 = fma(a[rr][c].y, qr[r][c].y, d1);
      }
      part[rr * NRHS + r] = d0 + d1;
    }
  }
  warp_transpose_reduce<V>(part, lane);
  if ((lane & (32 / V - 1)) == 0) red[warp * 16 + transpose_reduce_index<V>(lane)] = part[0];
  named_bar_sync(bar, kPassConsumers);
  if (tid < V) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kPassWarps; ++w) t += red[w * 16 + tid];
    const int row = rb + tid / NRHS;
    if (!FULL && row >= rows) {
      t = 0.0;
    } else if (MODE == PASS_RESIDUAL) {
      const double bi = bpre;   // NRHS == 1: row = rb + tid
      t = bi - t;
      sacc2 = fma(bi, t, sacc2);
    }
    sacc = fma(t, t, sacc);
    tfin[tid] = t;
  }
  named_bar_sync(bar, kPassConsumers);
#pragma unroll
  for (int rr = 0; rr < RB; ++rr) {
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      const double t = tfin[rr * NRHS + r];
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        acc[r][c].x = fma(t, a[rr][c].x, acc[r][c].x);
        acc[r][c].y = fma(t, a[rr][c].y, acc[r][c].y);
      }
    }
  }
}

// NS consumer sets of 8 warps take alternate stages (latency: a set's two barriers per
// row group serialise its stage, two sets overlap them); each set keeps its own v
// accumulators and writes its own partial row (the reduce sums grid * NS rows).
template <int NRHS, int MODE, int CPT, bool FC, int NS>
__global__ void __launch_bounds__(NS * kPassConsumers + 32, 1)
k_pass(const double* __restrict__ A, int64_t m, int n, int64_t ld, int rps,
       const double* __restrict__ q, const double* __restrict__ b,
       double* __restrict__ partials, int W, const int* __restrict__ active) {
  // launched with programmatic stream serialization after a PCG step (NEXT-3): everything
  // below reads the step's results (active, q), so wait for it first; the launch itself (CTA
  // rasterisation, shared-memory carve-out) overlaps the step's tail.  A no-op otherwise.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (active != nullptr && (active[0] | active[1]) == 0) return;
  extern __shared__ __align__(128) unsigned char smem[];
  double* ring = reinterpret_cast<double*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kPassStages * kPassStageBytes);
  uint64_t* empty = full + kPassStages;
  const int warp_all = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int set = warp_all / kPassWarps;                         // NS for the producer warp
  double* red = reinterpret_cast<double*>(empty + kPassStages) + (size_t)(set < NS ? set : 0) * kPassRedDoubles;
  double* tfin = red + kPassWarps * 16;                           // [16]
  double* sred = tfin + 16;                                       // [32]
  constexpr int kStageDoubles = kPassStageBytes / 8;
  const int tid = threadIdx.x - set * kPassConsumers, warp = warp_all - set * kPassWarps;
  const int bar = 1 + set;
  const int64_t G = gridDim.x;
  const int64_t r0 = m * (int64_t)blockIdx.x / G;
  const int64_t r1 = m * (int64_t)(blockIdx.x + 1) / G;
  const int nst = (int)((r1 - r0 + rps - 1) / rps);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPassStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPassWarps);   // the 8 warps of the set that consumes the stage
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (set == NS) {  // ---------------- producer: TMA bulk copies of row blocks
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int it = 0; it < nst; ++it) {
        const int s = it % kPassStages;
        const uint32_t ph = (uint32_t)(it / kPassStages) & 1u;
        if (it >= kPassStages) mbar_wait(&empty[s], ph ^ 1u);
        const int64_t rs = r0 + (int64_t)it * rps;
        const int rows = (int)min((int64_t)rps, r1 - rs);
        const uint32_t bytes = (uint32_t)(rows * ld * 8);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(ring + (size_t)s * kStageDoubles, A + rs * ld, bytes, &full[s], pol);
      }
    }
    return;
  }

  // ---------------- consumers
  // rows per reduction group (divides rows per stage); two consumer sets with 2 RHS halve it
  // to stay within the 96-register budget of the 17-warp CTA
  constexpr int RB = ((CPT >= 8) ? 1 : 8 / CPT) / ((NS == 2 && NRHS == 2 && CPT < 8) ? 2 : 1);
  constexpr int V = RB * NRHS;
  const int nchunks = (n + 1) >> 1;

  double2 qr[NRHS][CPT];
  double2 acc[NRHS][CPT];
  bool okc[CPT], ok1[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int ch = tid + c * kPassConsumers;
    const int col = 2 * ch;
    okc[c] = ch < nchunks;
    ok1[c] = col + 1 < n;
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      acc[r][c] = make_double2(0.0, 0.0);
      if (MODE != PASS_COLSTATS) {
        const double qx = okc[c] ? q[(size_t)r * n + col] : 0.0;
        const double qy = ok1[c] ? q[(size_t)r * n + col + 1] : 0.0;
        qr[r][c] = make_double2(qx, qy);
      }
    }
  }
  double sacc = 0.0, sacc2 = 0.0;

  for (int it = set; it < nst; it += NS) {
    const int s = it % kPassStages;
    const uint32_t ph = (uint32_t)(it / kPassStages) & 1u;
    mbar_wait(&full[s], ph);
    const double* st = ring + (size_t)s * kStageDoubles;
    const int64_t rs = r0 + (int64_t)it * rps;
    const int rows = (int)min((int64_t)rps, r1 - rs);

    if (MODE == PASS_COLSTATS) {
      for (int rr = 0; rr < rows; ++rr) {
        const double2* rowp = reinterpret_cast<const double2*>(st + (size_t)rr * ld);
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          if (!okc[c]) continue;
          double2 a = rowp[tid + c * kPassConsumers];
          if (!ok1[c]) a.y = 0.0;
          acc[0][c].x = fmax(acc[0][c].x, fabs(a.x));
          acc[0][c].y = fmax(acc[0][c].y, fabs(a.y));
          acc[1][c].x = fma(a.x, a.x, acc[1][c].x);
          acc[1][c].y = fma(a.y, a.y, acc[1][c].y);
        }
      }
    } else {
      // full row groups without predicates (FC: every column chunk exists), then the tail
      int rb = 0;
      if (FC) {
        for (; rb + RB <= rows; rb += RB)
          pass_group<NRHS, MODE, CPT, RB, true>(st + (size_t)rb * ld + 2 * tid, ld, rb, rows, rs, b, qr, acc, okc, ok1,
                                               red, tfin, warp, lane, tid, sacc, sacc2, bar);
      }
      for (; rb < rows; rb += RB)
        pass_group<NRHS, MODE, CPT, RB, false>(st + (size_t)rb * ld + 2 * tid, ld, rb, rows, rs, b, qr, acc, okc, ok1,
                                              red, tfin, warp, lane, tid, sacc, sacc2, bar);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- write this set's partial
  double* out = partials + ((size_t)blockIdx.x * NS + set) * W;
#pragma unroll
  for (int r = 0; r < NRHS; ++r) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!okc[c]) continue;
      const int col = 2 * (tid + c * kPassConsumers);
      out[(size_t)r * n + col] = acc[r][c].x;
      if (ok1[c]) out[(size_t)r * n + col + 1] = acc[r][c].y;
    }
  }
  if (MODE != PASS_COLSTATS) {
    if (tid < 16) {
      sred[tid] = tid < V ? sacc : 0.0;
      sred[16 + tid] = tid < V ? sacc2 : 0.0;
    }
    named_bar_sync(bar, kPassConsumers);
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int i = 0; i < V; ++i) {
        if (NRHS == 2) {
          if (i % 2 == 0) s0 += sred[i]; else s1 += sred[i];
        } else {
          s0 += sred[i];
          s1 += sred[16 + i];
        }
      }
      out[(size_t)NRHS * n] = s0;
      out[(size_t)NRHS * n + 1] = s1;
    }
  }
}

template <int NRHS, int MODE, int CPT>
static int launch_pass_t(const DenseView& A, const double* q, const double* b, double* partials,
                         int W, const int* active, cudaStream_t st, int G) {
  // FC: n fills every thread's CPT column chunks exactly (n = 2 * CPT * consumers)
  const bool fc = (A.n == 2 * CPT * kPassConsumers);
  constexpr int NS = pass_sets_rt(NRHS, MODE, CPT);
  auto kern = fc ? k_pass<NRHS, MODE, CPT, true, NS> : k_pass<NRHS, MODE, CPT, false, NS>;
  static bool attr[2] = {false, false};
  if (!attr[fc]) {
    TLS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPassSmem));
    attr[fc] = true;
  }
  if (pass_pdl()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(NS * kPassConsumers + 32);
    cfg.dynamicSmemBytes = kPassSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TLS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, A.A, A.m, A.n, A.ld, rows_per_stage(A), q, b, partials, W, active));
    return 0;
  }
  kern<<<G, NS * kPassConsumers + 32, kPassSmem, st>>>(A.A, A.m, A.n, A.ld, rows_per_stage(A), q, b, partials,
                                                             W, active);
  TLS_LAUNCH_CHECK();
  return 0;
}

template <int NRHS, int MODE>
static int launch_pass_cpt(const DenseView& A, const double* q, const double* b, double* partials,
                           int W, const int* active, cudaStream_t st, int G) {
  const int chunks = (A.n + 1) / 2;
  if (chunks <= kPassConsumers) return launch_pass_t<NRHS, MODE, 1>(A, q, b, partials, W, active, st, G);
  if (chunks <= 2 * kPassConsumers) return launch_pass_t<NRHS, MODE, 2>(A, q, b, partials, W, active, st, G);
  if (chunks <= 4 * kPassConsumers) return launch_pass_t<NRHS, MODE, 4>(A, q, b, partials, W, active, st, G);
  return launch_pass_t<NRHS, MODE, 8>(A, q, b, partials, W, active, st, G);
}

int launch_pass(const DenseView& A, int mode, int nrhs, const double* q, const double* b,
                double* partials, const int* active, cudaStream_t st, int* grid_out) {
  if (A.n > kMaxDenseN || (A.ld & 1) || A.ld < A.n) {
    set_error("dense pass: need n <= %d and even ld >= n", kMaxDenseN);
    return TLS_ERR_UNSUPPORTED;
  }
  // TLS_PASS_TEAM=1: the team-per-row layout of k_pass32.cu for the fp64 operator (2 RHS)
  // and residual passes (A/B switch)
  static const int team = [] { const char* e = getenv("TLS_PASS_TEAM"); return e ? atoi(e) : 0; }();
  if (team && A.n <= 2048 && (mode == PASS_RESIDUAL || (mode == PASS_OPERATOR && nrhs == 2)))
    return launch_pass_team(A, mode, q, b, partials, active, st, grid_out);
  const int G = pass_grid(A);
  // partial rows for the fixed-order reduce: one per consumer set (pass_sets_rt of the
  // instantiation launch_pass_cpt picks)
  const int chunks = (A.n + 1) / 2;
  const int cpt = chunks <= kPassConsumers ? 1 : chunks <= 2 * kPassConsumers ? 2 : chunks <= 4 * kPassConsumers ? 4 : 8;
  const int kn = mode == PASS_COLSTATS ? 2 : (mode == PASS_RESIDUAL ? 1 : nrhs);
  if (grid_out) *grid_out = G * pass_sets_rt(kn, mode, cpt);
  if (A.m == 0) return 0;
  if (mode == PASS_COLSTATS)
    return launch_pass_cpt<2, PASS_COLSTATS>(A, q, b, partials, 2 * A.n, active, st, G);
  if (mode == PASS_RESIDUAL)
    return launch_pass_cpt<1, PASS_RESIDUAL>(A, q, b, partials, A.n + 2, active, st, G);
  if (nrhs == 1) return launch_pass_cpt<1, PASS_OPERATOR>(A, q, b, partials, A.n + 2, active, st, G);
  return launch_pass_cpt<2, PASS_OPERATOR>(A, q, b, partials, 2 * A.n + 2, active, st, G);
}

// --------------------------------------------------------------------------- partial reduction
constexpr int kRedBatch = 20;   // partial rows in flight per thread: a row group of G = 148 CTAs in one batch
__global__ void k_reduce_partials(const double* __restrict__ partials, int G, int W, int nmax,
                                  double* __restrict__ out, const int* __restrict__ active) {
  // launched with programmatic dependent launch after a pass (round 2 continued): wait for it
  // before reading anything (a no-op otherwise), let the PCG step that follows launch at once
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (active != nullptr && (active[0] | active[1]) == 0) return;
  __shared__ double sm[8][33];
  const int tx = threadIdx.x, grp = threadIdx.y;
  const int w = blockIdx.x * 32 + tx;
  const int g0 = G * grp / 8, g1 = G * (grp + 1) / 8;
  const bool ismax = w < nmax;
  double acc = 0.0;
  if (w < W) {
    // a group's rows (<= kRedBatch of them for G <= 8 * kRedBatch) all in flight, combined in
    // row order (the same bits as one at a time; the dependent one-load-per-add loop was
    // L2-latency bound: 9.4 us for 296 x 2050 partials; 8 in flight plus a serial tail, round 2)
    for (int g = g0; g < g1; g += kRedBatch) {
      double v[kRedBatch];
#pragma unroll
      for (int k = 0; k < kRedBatch; ++k) v[k] = g + k < g1 ? partials[(size_t)(g + k) * W + w] : 0.0;
#pragma unroll
      for (int k = 0; k < kRedBatch; ++k)
        if (g + k < g1) acc = ismax ? fmax(acc, v[k]) : acc + v[k];
    }
  }
  sm[grp][tx] = acc;
  __syncthreads();
  if (grp == 0 && w < W) {
    double r = sm[0][tx];
    for (int k = 1; k < 8; ++k) r = ismax ? fmax(r, sm[k][tx]) : r + sm[k][tx];
    out[w] = r;
  }
}

int launch_reduce(const double* partials, int G, int W, int nmax, double* out, const int* active,
                  cudaStream_t st) {
  dim3 blk(32, 8);
  if (pass_pdl()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((W + 31) / 32);
    cfg.blockDim = blk;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TLS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_reduce_partials, partials, G, W, nmax, out, active));
    return 0;
  }
  k_reduce_partials<<<(W + 31) / 32, blk, 0, st>>>(partials, G, W, nmax, out, active);
  TLS_LAUNCH_CHECK();
  return 0;
}

// --------------------------------------------------------------------------- scaling D
// mode 0 (Cholesky route, R2): d_j = 2^floor(log2 max_i |a_ij|).
// mode 1 (QR route, R27): the paper's D = diag(A^T A)^{1/2} rounded to a
// power of two: k = floor(log2 c_j), d_j = 2^ceil(k/2), decided on c_j's exponent alone.
__global__ void k_scaling(const double* __restrict__ colmax, const double* __restrict__ sumsq, int n,
                          double* __restrict__ d, double* __restrict__ dinv, double* __restrict__ normA2,
                          int* __restrict__ flag, int mode) {
  __shared__ double red[32];
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double cm = mode == 0 ? colmax[j] : sumsq[j];
    if (!(cm > 0.0) || !isfinite(cm)) atomicExch(flag, 1);
    int e = 0;
    frexp(cm, &e);
    const int p = mode == 0 ? e - 1 : -((1 - e) >> 1);   // mode 1: ceil((e - 1) / 2)
    d[j] = scalbn(1.0, p);
    dinv[j] = scalbn(1.0, -p);
    s += sumsq[j];
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) *normA2 = s;
}

int launch_scaling(const double* colmax, const double* sumsq, int n, double* d, double* dinv,
                   double* normA2, int* flag, cudaStream_t st, int mode) {
  k_scaling<<<1, 1024, 0, st>>>(colmax, sumsq, n, d, dinv, normA2, flag, mode);
  TLS_LAUNCH_CHECK();
  return 0;
}

// --------------------------------------------------------------------------- content fingerprint
// A sampled checksum of the local block of A (the handle remembers what it was
// factored from): 256 rows spread evenly over the block (first and last included), each row's
// entries weighted by fixed pseudo-random column weights, summed per row in column order and
// over rows in thread order (deterministic).  CSR also weighs the column indices.  An A rewritten
// in place, or another A of the same shape, changes it unless the rewrite misses every sampled
// row (2 MB read at n = 1024: a few microseconds).
__device__ __forceinline__ double fp_weight(int64_t j) {
  const uint64_t h = (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ull;
  return 1.0 + (double)(h >> 40) * 0x1p-24;
}
// One CTA per sampled row (coalesced), the row's weighted sum by a fixed-order block
// reduction into part[r]; k_fingerprint_fin adds the 256 row sums in a fixed order.
__global__ void __launch_bounds__(256) k_fingerprint(const double* __restrict__ A, int64_t m, int n, int64_t ld,
                                                     const int64_t* __restrict__ rowptr,
                                                     const int32_t* __restrict__ colidx, double* __restrict__ part) {
  __shared__ double red[32];
  const int r = blockIdx.x, t = threadIdx.x;
  double acc = 0.0;
  if (m > 0 && (m >= 256 || r < m)) {
    const int64_t i = m >= 256 ? (int64_t)r * (m - 1) / 255 : r;
    if (rowptr) {
      for (int64_t k = rowptr[i] + t; k < rowptr[i + 1]; k += blockDim.x)
        acc += A[k] * fp_weight(colidx[k]) + (double)colidx[k] * 0x1p-20;
    } else {
      for (int j = t; j < n; j += blockDim.x) acc += A[i * ld + j] * fp_weight(j);
    }
  }
  acc = block_sum(acc, red);
  if (t == 0) part[r] = acc;
}
// one warp: lane l sums the row sums 8l .. 8l+7 in order (all eight loads in flight), then a
// fixed butterfly (deterministic; round 2 continued: one thread's 256 dependent adds took ~11 us)
__global__ void k_fingerprint_fin(const double* __restrict__ part, double* __restrict__ out) {
  const int l = threadIdx.x;
  double v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = part[8 * l + u];
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += v[u];
  s = warp_sum(s);
  if (l == 0) out[0] = s;
}

int launch_fingerprint(const DenseView* dv, const CsrView* cv, double* out, double* scratch, cudaStream_t st) {
  if (cv) k_fingerprint<<<256, 256, 0, st>>>(cv->vals, cv->m, cv->n, 0, cv->rowptr, cv->colidx, scratch);
  else k_fingerprint<<<256, 256, 0, st>>>(dv->A, dv->m, dv->n, dv->ld, nullptr, nullptr, scratch);
  k_fingerprint_fin<<<1, 32, 0, st>>>(scratch, out);
  TLS_LAUNCH_CHECK();
  return 0;
}

__global__ void k_round(const double* __restrict__ x, double* __restrict__ y, int64_t n, int prec) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = round_uf(x[i], prec);
}

int launch_round(const double* x, double* y, int64_t n, int prec, cudaStream_t st) {
  if (n == 0) return 0;
  int64_t g = (n + 255) / 256;
  if (g > 4096) g = 4096;
  k_round<<<(int)g, 256, 0, st>>>(x, y, n, prec);
  TLS_LAUNCH_CHECK();
  return 0;
}

}  // namespace tls
