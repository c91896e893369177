// k_pass32.cu — the PCGTLS operator pass with u_p = fp32 (reading R23).
//
// The paper's experiments run the inner PCG in single precision with u = u_r = double
// ("single precision for u_p was sufficient for all included
// examples").  On the A-in-loop operator (R1) the only O(mn) work of PCGTLS is
//   t_r = A q_r,  v_r = A^T t_r,  s_r = t_r^T t_r      (r = 0, 1: the two batched solves)
// and this kernel does it on an fp32 copy A32 = fl32(A) (row-major, ld32 = n rounded
// up to 4, zero padded) held by the preconditioner handle: q_r is rounded to fp32 on
// load, t_r and v_r are accumulated in fp32, s_r in fp64 from the fp32 t_r.  It reads
// 4mn bytes instead of 8mn.
//
// Layout (different from k_pass, whose 8 warps cooperate on every row): a TEAM of
// G warps owns whole rows (G = 1 for n <= 1024, 2 for n <= 2048), each warp a slice of
// up to 1024 columns held as 8 float4 per lane, so q and the accumulator v stay in
// registers and a row's dot product needs only a warp butterfly (plus, for G = 2, one
// 64-thread barrier).  Each team streams its own chunks of rows (RS consecutive rows,
// about 4 KB) through a private 6-slot shared-memory ring with TMA bulk copies issued
// by its leader lane; there is no producer warp and no CTA-wide synchronisation until
// the final fixed-order reduction of the teams' v into the CTA partial.
#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

constexpr int kP32Warps = 8;
constexpr int kP32Slots = 6;
constexpr int kP32SlotMin = 4096;   // bytes per slot (at least one row)

static int p32_slot_bytes(int ld32) { return ld32 * 4 > kP32SlotMin ? ld32 * 4 : kP32SlotMin; }
static int p32_rows_per_slot(int ld32) { return p32_slot_bytes(ld32) / (ld32 * 4); }
// one ring of kP32Slots slots per team of G warps, its full barriers, tpart (128 floats),
// tsum (16 doubles)
static size_t p32_smem(int ld32, int G) {
  const int T = kP32Warps / G;
  return (size_t)T * kP32Slots * p32_slot_bytes(ld32) + (size_t)T * kP32Slots * 8 + 128 * 4 + 16 * 8;
}

template <int CPL, int G>
__global__ void __launch_bounds__(kP32Warps * 32, 1)
    k_pass32(const float* __restrict__ A32, int64_t m, int n, int ld32, int RS, int slot_bytes,
             const double* __restrict__ q, double* __restrict__ partials, int W, const int* __restrict__ active) {
  if (active != nullptr && (active[0] | active[1]) == 0) return;
  constexpr int T = kP32Warps / G;      // teams
  constexpr int SW = 32 * CPL * 4;      // columns per warp slice
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)T * kP32Slots * slot_bytes);
  float* tpart = reinterpret_cast<float*>(full + T * kP32Slots);           // [T][2 buf][G][2] (<= 128)
  double* tsum = reinterpret_cast<double*>(tpart + 128);                   // [T][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / G, wt = warp % G;
  const bool leader = (wt == 0) && (lane == 0);
  const int64_t Gc = gridDim.x;
  const int64_t r0 = m * (int64_t)blockIdx.x / Gc;
  const int64_t r1 = m * (int64_t)(blockIdx.x + 1) / Gc;
  const int64_t nchunk = (r1 - r0 + RS - 1) / RS;
  // this team's chunks: team, team + T, team + 2T, ...
  const int nt = (int)(nchunk > team ? (nchunk - team + T - 1) / T : 0);
  unsigned char* tring = ring + (size_t)team * kP32Slots * slot_bytes;
  uint64_t* tfull = full + team * kP32Slots;

  if (threadIdx.x == 0) {
    for (int s = 0; s < T * kP32Slots; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  auto issue = [&](int i) {   // chunk i of this team into slot i % kP32Slots
    const int64_t rs = r0 + ((int64_t)i * T + team) * RS;
    const int rows = (int)min((int64_t)RS, r1 - rs);
    const uint32_t bytes = (uint32_t)rows * (uint32_t)ld32 * 4u;
    const int s = i % kP32Slots;
    mbar_arrive_expect_tx(&tfull[s], bytes);
    bulk_g2s(tring + (size_t)s * slot_bytes, A32 + rs * ld32, bytes, &tfull[s], pol);
  };
  if (leader)
    for (int i = 0; i < kP32Slots && i < nt; ++i) issue(i);

  // q_r rounded to fp32 (R23), this lane's columns wt*SW + 4*(lane + 32c) .. +3
  float4 qv[2][CPL], acc[2][CPL];
  bool okc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int col = wt * SW + 4 * (lane + 32 * c);
    okc[c] = col < ld32;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float e[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) e[k] = (col + k < n) ? (float)q[(size_t)r * n + col + k] : 0.0f;
      qv[r][c] = make_float4(e[0], e[1], e[2], e[3]);
      acc[r][c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  double s0 = 0.0, s1 = 0.0;
  int rowctr = 0;

  for (int i = 0; i < nt; ++i) {
    const int s = i % kP32Slots;
    mbar_wait(&tfull[s], (uint32_t)(i / kP32Slots) & 1u);
    const int64_t rs = r0 + ((int64_t)i * T + team) * RS;
    const int rows = (int)min((int64_t)RS, r1 - rs);
    const float* slot = reinterpret_cast<const float*>(tring + (size_t)s * slot_bytes);
    for (int rr = 0; rr < rows; ++rr, ++rowctr) {
      const float4* row = reinterpret_cast<const float4*>(slot + (size_t)rr * ld32 + wt * SW);
      float4 a[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) a[c] = okc[c] ? row[lane + 32 * c] : make_float4(0.f, 0.f, 0.f, 0.f);
      // t_r = a . q_r: four independent fp32 accumulators per RHS
      float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f), p1 = p0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        p0.x = fmaf(a[c].x, qv[0][c].x, p0.x); p0.y = fmaf(a[c].y, qv[0][c].y, p0.y);
        p0.z = fmaf(a[c].z, qv[0][c].z, p0.z); p0.w = fmaf(a[c].w, qv[0][c].w, p0.w);
        p1.x = fmaf(a[c].x, qv[1][c].x, p1.x); p1.y = fmaf(a[c].y, qv[1][c].y, p1.y);
        p1.z = fmaf(a[c].z, qv[1][c].z, p1.z); p1.w = fmaf(a[c].w, qv[1][c].w, p1.w);
      }
      const float d0 = (p0.x + p0.y) + (p0.z + p0.w);
      const float d1 = (p1.x + p1.y) + (p1.z + p1.w);
      // butterfly: lanes 0-15 end with the warp's t_0, lanes 16-31 with t_1
      const bool lo = lane < 16;
      float keep = lo ? d0 : d1;
      keep += __shfl_xor_sync(0xffffffffu, lo ? d1 : d0, 16);
      keep += __shfl_xor_sync(0xffffffffu, keep, 8);
      keep += __shfl_xor_sync(0xffffffffu, keep, 4);
      keep += __shfl_xor_sync(0xffffffffu, keep, 2);
      keep += __shfl_xor_sync(0xffffffffu, keep, 1);
      float t0, t1;
      if (G == 1) {
        t0 = __shfl_sync(0xffffffffu, keep, 0);
        t1 = __shfl_sync(0xffffffffu, keep, 16);
      } else {
        // the team's warps exchange their slice sums (double-buffered by row parity)
        float* tp = tpart + ((team * 2 + (rowctr & 1)) * G) * 2;
        if (lane == 0) tp[wt * 2 + 0] = keep;
        if (lane == 16) tp[wt * 2 + 1] = keep;
        named_bar_sync(1 + team, G * 32);
        t0 = tp[0];
        t1 = tp[1];
#pragma unroll
        for (int g = 1; g < G; ++g) { t0 += tp[g * 2]; t1 += tp[g * 2 + 1]; }
      }
      if (wt == 0) {
        s0 = fma((double)t0, (double)t0, s0);
        s1 = fma((double)t1, (double)t1, s1);
      }
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        acc[0][c].x = fmaf(t0, a[c].x, acc[0][c].x); acc[0][c].y = fmaf(t0, a[c].y, acc[0][c].y);
        acc[0][c].z = fmaf(t0, a[c].z, acc[0][c].z); acc[0][c].w = fmaf(t0, a[c].w, acc[0][c].w);
        acc[1][c].x = fmaf(t1, a[c].x, acc[1][c].x); acc[1][c].y = fmaf(t1, a[c].y, acc[1][c].y);
        acc[1][c].z = fmaf(t1, a[c].z, acc[1][c].z); acc[1][c].w = fmaf(t1, a[c].w, acc[1][c].w);
      }
    }
    // every warp of the team has this slot's rows in registers: refill it
    if (G == 1) __syncwarp();
    else named_bar_sync(1 + team, G * 32);
    if (leader && i + kP32Slots < nt) issue(i + kP32Slots);
  }

  // ---- fixed-order reduction of the teams' v (fp64) into this CTA's partial
  __syncthreads();
  double* vsum = reinterpret_cast<double*>(ring);    // [2][ld32], the ring is free now
  for (int tm = 0; tm < T; ++tm) {
    if (team == tm) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        if (!okc[c]) continue;
        const int col = wt * SW + 4 * (lane + 32 * c);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          double* dst = vsum + (size_t)r * ld32 + col;
          const float e[4] = {acc[r][c].x, acc[r][c].y, acc[r][c].z, acc[r][c].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) dst[k] = (tm == 0) ? (double)e[k] : dst[k] + (double)e[k];
        }
      }
      if (wt == 0 && lane == 0) { tsum[tm * 2] = s0; tsum[tm * 2 + 1] = s1; }
    }
    __syncthreads();
  }
  double* out = partials + (size_t)blockIdx.x * W;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    out[j] = vsum[j];
    out[(size_t)n + j] = vsum[(size_t)ld32 + j];
  }
  if (threadIdx.x == 0) {
    double a0 = 0.0, a1 = 0.0;
    for (int tm = 0; tm < T; ++tm) { a0 += tsum[tm * 2]; a1 += tsum[tm * 2 + 1]; }
    out[2 * (size_t)n] = a0;
    out[2 * (size_t)n + 1] = a1;
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

int pass32_grid(const DenseView& A) {
  const int64_t rs = p32_rows_per_slot(p32_ld(A.n));
  const int64_t chunks = (A.m + rs - 1) / rs;
  int64_t g = num_sms();
  // at least a few chunks per team, and never more partial rows than k_pass reserves
  const int64_t by_rows = (chunks + 2 * kP32Warps - 1) / (2 * kP32Warps);
  if (by_rows < g) g = by_rows;
  const int64_t cap = (int64_t)pass_partials_doubles(A) / (2 * A.n + 2);
  if (cap < g) g = cap;
  return (int)(g < 1 ? 1 : g);
}

template <int CPL, int G>
static int launch_p32_t(const DenseView& A, const float* A32, const double* q, double* partials, const int* active,
                        cudaStream_t st, int grid) {
  const int ld32 = p32_ld(A.n);
  const size_t sm = p32_smem(ld32, G);
  auto kern = k_pass32<CPL, G>;
  static size_t attr = 0;
  if (attr < sm) {
    TLS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = sm;
  }
  kern<<<grid, kP32Warps * 32, sm, st>>>(A32, A.m, A.n, ld32, p32_rows_per_slot(ld32), p32_slot_bytes(ld32), q,
                                          partials, 2 * A.n + 2, active);
  TLS_LAUNCH_CHECK();
  return 0;
}

int launch_pass32(const DenseView& A, const float* A32, const double* q, double* partials, const int* active,
                  cudaStream_t st, int* grid_out) {
  const int ld32 = p32_ld(A.n);
  if (A.n > 2048) { set_error("u_p = fp32 pass: n <= 2048"); return TLS_ERR_UNSUPPORTED; }
  const int grid = pass32_grid(A);
  if (grid_out) *grid_out = grid;
  if (A.m == 0) return 0;
  if (ld32 <= 128) return launch_p32_t<1, 1>(A, A32, q, partials, active, st, grid);
  if (ld32 <= 256) return launch_p32_t<2, 1>(A, A32, q, partials, active, st, grid);
  if (ld32 <= 512) return launch_p32_t<4, 1>(A, A32, q, partials, active, st, grid);
  if (ld32 <= 1024) return launch_p32_t<8, 1>(A, A32, q, partials, active, st, grid);
  return launch_p32_t<8, 2>(A, A32, q, partials, active, st, grid);
}

}  // namespace tls
