// k_pass32.cu — team-per-row streaming passes over A:
//   * the PCGTLS operator pass with u_p = fp32 (reading R23), and
//   * the same layout for the fp64 operator (2 RHS) and residual (1 RHS) passes
//     (a5, a7), selectable against k_pass (launch_pass_team).
//
// The paper's experiments run the inner PCG in single precision with u = u_r = double
// ("single precision for u_p was sufficient for all included
// examples").  On the A-in-loop operator (R1) the only O(mn) work of PCGTLS is
//   t_r = A q_r,  v_r = A^T t_r,  s_r = t_r^T t_r      (r = 0, 1: the two batched solves)
// and at u_p = fp32 it runs on an fp32 copy A32 = fl32(A) (row-major, ld32 = n rounded
// up to 4, zero padded) held by the preconditioner handle: q_r is rounded to fp32 on
// load, t_r and v_r are accumulated in fp32, s_r in fp64 from the fp32 t_r.  It reads
// 4mn bytes instead of 8mn.  The residual mode (fp64 only) computes t = b - A x,
// v = A^T t, s = (t^T t, b^T t).
//
// Layout (different from k_pass, whose 8 warps cooperate on every row): a TEAM of
// G warps owns whole rows, each warp a slice of 32 * CPL 16-byte vectors (up to 1024
// fp32 or 512 fp64 columns), so q and the accumulator v stay in registers and a row's
// dot product needs only a warp butterfly (plus, for G > 1, one team barrier).  Each
// team streams its own chunks of RS consecutive rows (>= 4 KB) through a private
// 6-slot shared-memory ring with TMA bulk copies issued by its leader lane; there is
// no producer warp and no CTA-wide synchronisation until the final fixed-order
// reduction of the teams' v into the CTA partial.
#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

constexpr int kTWarps = 8;
constexpr int kTSlots = 6;
constexpr int kTSlotMin = 4096;   // bytes per slot (at least one row)

static int t_slot_bytes(int row_bytes) { return row_bytes > kTSlotMin ? row_bytes : kTSlotMin; }
static int t_rows_per_slot(int row_bytes) { return t_slot_bytes(row_bytes) / row_bytes; }
// one ring per team of G warps, its full barriers, tpart (128 doubles), tsum (16 doubles)
static size_t t_smem(int row_bytes, int G) {
  const int T = kTWarps / G;
  return (size_t)T * kTSlots * t_slot_bytes(row_bytes) + (size_t)T * kTSlots * 8 + 128 * 8 + 16 * 8;
}

template <typename E> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int N = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int N = 2; };

template <typename E>
__device__ __forceinline__ void vload(E (&dst)[Vec16<E>::N], const E* src) {
  const typename Vec16<E>::type v = *reinterpret_cast<const typename Vec16<E>::type*>(src);
  if constexpr (Vec16<E>::N == 4) { dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w; }
  else { dst[0] = v.x; dst[1] = v.y; }
}

template <typename E>
__device__ __forceinline__ E shfl_xor(E v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
template <typename E>
__device__ __forceinline__ E shfl_idx(E v, int l) { return __shfl_sync(0xffffffffu, v, l); }

// MODE: PASS_OPERATOR (2 RHS, q = 2 x n) or PASS_RESIDUAL (1 RHS, q = x, b).
template <typename E, int MODE, int CPL, int G>
__global__ void __launch_bounds__(kTWarps * 32, 1)
    k_pass_team(const E* __restrict__ A, int64_t m, int n, int64_t ld, int RS, int slot_bytes,
                const double* __restrict__ q, const double* __restrict__ b, double* __restrict__ partials, int W,
                const int* __restrict__ active) {
  if (active != nullptr && (active[0] | active[1]) == 0) return;
  constexpr int NR = MODE == PASS_OPERATOR ? 2 : 1;
  constexpr int EV = Vec16<E>::N;
  constexpr int T = kTWarps / G;        // teams
  constexpr int SW = 32 * CPL * EV;     // columns per warp slice
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)T * kTSlots * slot_bytes);
  E* tpart = reinterpret_cast<E*>(full + T * kTSlots);                       // [T][2 buf][G][2]
  double* tsum = reinterpret_cast<double*>(full + T * kTSlots) + 128;        // [T][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / G, wt = warp % G;
  const bool leader = (wt == 0) && (lane == 0);
  const int64_t Gc = gridDim.x;
  const int64_t r0 = m * (int64_t)blockIdx.x / Gc;
  const int64_t r1 = m * (int64_t)(blockIdx.x + 1) / Gc;
  const int64_t nchunk = (r1 - r0 + RS - 1) / RS;
  // this team's chunks: team, team + T, team + 2T, ...
  const int nt = (int)(nchunk > team ? (nchunk - team + T - 1) / T : 0);
  unsigned char* tring = ring + (size_t)team * kTSlots * slot_bytes;
  uint64_t* tfull = full + team * kTSlots;

  if (threadIdx.x == 0) {
    for (int s = 0; s < T * kTSlots; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  auto issue = [&](int i) {   // chunk i of this team into slot i % kTSlots
    const int64_t rs = r0 + ((int64_t)i * T + team) * RS;
    const int rows = (int)min((int64_t)RS, r1 - rs);
    const uint32_t bytes = (uint32_t)rows * (uint32_t)ld * (uint32_t)sizeof(E);
    const int s = i % kTSlots;
    mbar_arrive_expect_tx(&tfull[s], bytes);
    bulk_g2s(tring + (size_t)s * slot_bytes, A + rs * ld, bytes, &tfull[s], pol);
  };
  if (leader)
    for (int i = 0; i < kTSlots && i < nt; ++i) issue(i);

  // q_r (rounded to E), this lane's columns wt*SW + EV*(lane + 32c) .. + EV-1
  E qv[NR][CPL][EV], acc[NR][CPL][EV];
  bool okc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int col = wt * SW + EV * (lane + 32 * c);
    okc[c] = col < ld;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
#pragma unroll
      for (int k = 0; k < EV; ++k) {
        qv[r][c][k] = (col + k < n) ? (E)q[(size_t)r * n + col + k] : (E)0;
        acc[r][c][k] = (E)0;
      }
    }
  }
  double s0 = 0.0, s1 = 0.0;
  int rowctr = 0;

  for (int i = 0; i < nt; ++i) {
    const int s = i % kTSlots;
    const int64_t rs = r0 + ((int64_t)i * T + team) * RS;
    const int rows = (int)min((int64_t)RS, r1 - rs);
    mbar_wait(&tfull[s], (uint32_t)(i / kTSlots) & 1u);
    const E* slot = reinterpret_cast<const E*>(tring + (size_t)s * slot_bytes);
    for (int rr = 0; rr < rows; ++rr, ++rowctr) {
      double bi = 0.0;
      if (MODE == PASS_RESIDUAL) bi = __ldg(b + rs + rr);
      const E* row = slot + (size_t)rr * ld + wt * SW;
      E a[CPL][EV];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        if (okc[c]) vload<E>(a[c], row + EV * (lane + 32 * c));
        else {
#pragma unroll
          for (int k = 0; k < EV; ++k) a[c][k] = (E)0;
        }
      }
      // t_r = a . q_r: EV independent accumulators per RHS
      E d[2];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        E p[EV];
#pragma unroll
        for (int k = 0; k < EV; ++k) p[k] = (E)0;
#pragma unroll
        for (int c = 0; c < CPL; ++c)
#pragma unroll
          for (int k = 0; k < EV; ++k) p[k] = fma(a[c][k], qv[r][c][k], p[k]);
        if constexpr (EV == 4) d[r] = (p[0] + p[1]) + (p[2] + p[3]);
        else d[r] = p[0] + p[1];
      }
      // butterfly; 2 RHS: lanes 0-15 end with the warp's sum for RHS 0, 16-31 for RHS 1
      E keep;
      if (NR == 2) {
        const bool lo = lane < 16;
        keep = lo ? d[0] : d[1];
        keep += shfl_xor<E>(lo ? d[1] : d[0], 16);
      } else {
        keep = d[0];
        keep += shfl_xor<E>(keep, 16);
      }
      keep += shfl_xor<E>(keep, 8);
      keep += shfl_xor<E>(keep, 4);
      keep += shfl_xor<E>(keep, 2);
      keep += shfl_xor<E>(keep, 1);
      E t0, t1 = (E)0;
      if (G == 1) {
        t0 = (NR == 2) ? shfl_idx<E>(keep, 0) : keep;
        if (NR == 2) t1 = shfl_idx<E>(keep, 16);
      } else {
        // the team's warps exchange their slice sums (double-buffered by row parity)
        E* tp = tpart + ((team * 2 + (rowctr & 1)) * G) * 2;
        if (lane == 0) tp[wt * 2 + 0] = keep;
        if (NR == 2 && lane == 16) tp[wt * 2 + 1] = keep;
        named_bar_sync(1 + team, G * 32);
        t0 = tp[0];
        if (NR == 2) t1 = tp[1];
#pragma unroll
        for (int g = 1; g < G; ++g) {
          t0 += tp[g * 2];
          if (NR == 2) t1 += tp[g * 2 + 1];
        }
      }
      if (MODE == PASS_RESIDUAL) {
        t0 = (E)(bi - (double)t0);
        if (wt == 0) {
          s0 = fma((double)t0, (double)t0, s0);
          s1 = fma(bi, (double)t0, s1);
        }
      } else if (wt == 0) {
        s0 = fma((double)t0, (double)t0, s0);
        s1 = fma((double)t1, (double)t1, s1);
      }
#pragma unroll
      for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int k = 0; k < EV; ++k) {
          acc[0][c][k] = fma(t0, a[c][k], acc[0][c][k]);
          if (NR == 2) acc[NR - 1][c][k] = fma(t1, a[c][k], acc[NR - 1][c][k]);
        }
    }
    // every warp of the team has this slot's rows in registers: refill it
    if (G == 1) __syncwarp();
    else named_bar_sync(1 + team, G * 32);
    if (leader && i + kTSlots < nt) issue(i + kTSlots);
  }

  // ---- fixed-order reduction of the teams' v (fp64) into this CTA's partial
  __syncthreads();
  double* vsum = reinterpret_cast<double*>(ring);    // [NR][ld], the ring is free now
  for (int tm = 0; tm < T; ++tm) {
    if (team == tm) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        if (!okc[c]) continue;
        const int col = wt * SW + EV * (lane + 32 * c);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          double* dst = vsum + (size_t)r * ld + col;
#pragma unroll
          for (int k = 0; k < EV; ++k) dst[k] = (tm == 0) ? (double)acc[r][c][k] : dst[k] + (double)acc[r][c][k];
        }
      }
      if (wt == 0 && lane == 0) { tsum[tm * 2] = s0; tsum[tm * 2 + 1] = s1; }
    }
    __syncthreads();
  }
  double* out = partials + (size_t)blockIdx.x * W;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
#pragma unroll
    for (int r = 0; r < NR; ++r) out[(size_t)r * n + j] = vsum[(size_t)r * ld + j];
  }
  if (threadIdx.x == 0) {
    double a0 = 0.0, a1 = 0.0;
    for (int tm = 0; tm < T; ++tm) { a0 += tsum[tm * 2]; a1 += tsum[tm * 2 + 1]; }
    out[(size_t)NR * n] = a0;
    out[(size_t)NR * n + 1] = a1;
  }
}

// A32 = fl32(A) (RNE), zero padded to ld32 columns.
__global__ void k_round32(const double* __restrict__ A, int64_t m, int n, int64_t ld, float* __restrict__ A32,
                          int ld32) {
  const int64_t total = m * (int64_t)ld32;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ld32;
    const int j = (int)(e - i * ld32);
    A32[e] = j < n ? __double2float_rn(__ldcs(A + i * ld + j)) : 0.0f;
  }
}

int p32_ld(int n) { return (n + 3) & ~3; }

int launch_round32(const DenseView& A, float* A32, cudaStream_t st) {
  if (A.m == 0) return 0;
  const int ld32 = p32_ld(A.n);
  k_round32<<<num_sms() * 8, 256, 0, st>>>(A.A, A.m, A.n, A.ld, A32, ld32);
  TLS_LAUNCH_CHECK();
  return 0;
}

// CTAs of a team pass: at least a few chunks per team, never more partial rows than
// k_pass reserves (pass_partials_doubles).
static int team_grid(const DenseView& A, int row_bytes, int W) {
  const int64_t rs = t_rows_per_slot(row_bytes);
  const int64_t chunks = (A.m + rs - 1) / rs;
  int64_t g = num_sms();
  const int64_t by_rows = (chunks + 2 * kTWarps - 1) / (2 * kTWarps);
  if (by_rows < g) g = by_rows;
  const int64_t cap = (int64_t)pass_partials_doubles(A) / W;
  if (cap < g) g = cap;
  return (int)(g < 1 ? 1 : g);
}

template <typename E, int MODE, int CPL, int G>
static int launch_team_t(const DenseView& A, const E* Ap, int64_t ld, const double* q, const double* b,
                         double* partials, const int* active, cudaStream_t st, int grid, int W) {
  const int row_bytes = (int)(ld * sizeof(E));
  const size_t sm = t_smem(row_bytes, G);
  auto kern = k_pass_team<E, MODE, CPL, G>;
  static size_t attr = 0;
  if (attr < sm) {
    TLS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = sm;
  }
  kern<<<grid, kTWarps * 32, sm, st>>>(Ap, A.m, A.n, ld, t_rows_per_slot(row_bytes), t_slot_bytes(row_bytes), q, b,
                                        partials, W, active);
  TLS_LAUNCH_CHECK();
  return 0;
}

int launch_pass32(const DenseView& A, const float* A32, const double* q, double* partials, const int* active,
                  cudaStream_t st, int* grid_out) {
  const int ld32 = p32_ld(A.n);
  if (A.n > 2048) { set_error("u_p = fp32 pass: n <= 2048"); return TLS_ERR_UNSUPPORTED; }
  const int W = 2 * A.n + 2;
  const int grid = team_grid(A, ld32 * 4, W);
  if (grid_out) *grid_out = grid;
  if (A.m == 0) return 0;
  constexpr int OP = PASS_OPERATOR;
  if (ld32 <= 128) return launch_team_t<float, OP, 1, 1>(A, A32, ld32, q, nullptr, partials, active, st, grid, W);
  if (ld32 <= 256) return launch_team_t<float, OP, 2, 1>(A, A32, ld32, q, nullptr, partials, active, st, grid, W);
  if (ld32 <= 512) return launch_team_t<float, OP, 4, 1>(A, A32, ld32, q, nullptr, partials, active, st, grid, W);
  if (ld32 <= 1024) return launch_team_t<float, OP, 8, 1>(A, A32, ld32, q, nullptr, partials, active, st, grid, W);
  return launch_team_t<float, OP, 8, 2>(A, A32, ld32, q, nullptr, partials, active, st, grid, W);
}

// fp64 operator (2 RHS) / residual (1 RHS) passes in the team layout.
template <int MODE>
static int launch_team64(const DenseView& A, const double* q, const double* b, double* partials, const int* active,
                         cudaStream_t st, int grid, int W) {
  const int64_t ld = A.ld;
  if (ld <= 64) return launch_team_t<double, MODE, 1, 1>(A, A.A, ld, q, b, partials, active, st, grid, W);
  if (ld <= 128) return launch_team_t<double, MODE, 2, 1>(A, A.A, ld, q, b, partials, active, st, grid, W);
  if (ld <= 256) return launch_team_t<double, MODE, 4, 1>(A, A.A, ld, q, b, partials, active, st, grid, W);
  if (ld <= 512) return launch_team_t<double, MODE, 8, 1>(A, A.A, ld, q, b, partials, active, st, grid, W);
  if (ld <= 1024) return launch_team_t<double, MODE, 8, 2>(A, A.A, ld, q, b, partials, active, st, grid, W);
  return launch_team_t<double, MODE, 8, 4>(A, A.A, ld, q, b, partials, active, st, grid, W);
}

int launch_pass_team(const DenseView& A, int mode, const double* q, const double* b, double* partials,
                     const int* active, cudaStream_t st, int* grid_out) {
  if (A.n > 2048 || (A.ld & 1)) { set_error("team pass: n <= 2048, even ld"); return TLS_ERR_UNSUPPORTED; }
  const int W = mode == PASS_OPERATOR ? 2 * A.n + 2 : A.n + 2;
  const int grid = team_grid(A, (int)(A.ld * 8), W);
  if (grid_out) *grid_out = grid;
  if (A.m == 0) return 0;
  if (mode == PASS_OPERATOR) return launch_team64<PASS_OPERATOR>(A, q, b, partials, active, st, grid, W);
  return launch_team64<PASS_RESIDUAL>(A, q, b, partials, active, st, grid, W);
}

}  // namespace tls
