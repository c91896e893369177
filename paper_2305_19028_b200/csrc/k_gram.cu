// k_gram.cu — the u_f Gram matrix G = A^^T A^, A^ = fl_uf(A D^{-1})  (
// PAPER.md l.231, l.290-307; readings R10, R11).
//
// This file holds the CUDA-core SYRK path: 64x64 upper tiles, split-K over
// chunks of K_t rows.  For u_f in {fp16, bf16} each chunk is accumulated in
// fp32 (products of u_f values are exact in fp32, as on the tensor cores) and
// drained into fp64 registers at the chunk end; for u_f in {fp32, fp64} the
// accumulation is fp64.  Partial tiles are summed over splits in fixed order.
#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

constexpr int kGT = 64;    // tile edge
constexpr int kGKB = 32;   // rows per smem step

static void gram_shape(const DenseView& A, int K_t, int& TT, int& ntiles, int& nchunks, int& nsplit) {
  TT = (A.n + kGT - 1) / kGT;
  ntiles = TT * (TT + 1) / 2;
  nchunks = (int)((A.m + K_t - 1) / K_t);
  if (nchunks < 1) nchunks = 1;
  const int target = 4 * num_sms();
  nsplit = (target + ntiles - 1) / ntiles;
  if (nsplit > nchunks) nsplit = nchunks;
  if (nsplit < 1) nsplit = 1;
}

static void gram_shape_f64(const DenseView& A, int& TT, int& ntiles, int& nsplit);
constexpr int kGT2_ = 128;
size_t gram_ws_doubles(const DenseView& A, int K_t) {
  int TT, nt, nc, ns;
  gram_shape(A, K_t, TT, nt, nc, ns);
  int T2, nt2, ns2;
  gram_shape_f64(A, T2, nt2, ns2);
  size_t cc = (size_t)ns * nt * kGT * kGT;
  const size_t c2 = (size_t)ns2 * nt2 * kGT2_ * kGT2_;
  if (c2 > cc) cc = c2;
  const size_t tc = (gram_tc_ws_bytes(A.m, A.n, 64) + 7) / 8;
  return cc > tc ? cc : tc;
}

template <typename ACC, int PREC>
__global__ void __launch_bounds__(256)
k_gram_cc(const double* __restrict__ A, int64_t m, int n, int64_t ld, const double* __restrict__ dinv,
          int K_t, int nchunks, int nsplit, int TT, double* __restrict__ part, int* __restrict__ range) {
  __shared__ ACC As[kGKB][kGT + 4];
  __shared__ ACC Bs[kGKB][kGT + 4];
  // tile index -> (I, J), I <= J, row-major over the upper triangle of tiles
  int t = blockIdx.x, I = 0;
  while (t >= TT - I) { t -= TT - I; ++I; }
  const int J = I + t;
  const bool diag = (I == J);
  const int s = blockIdx.y;
  const int c0 = (int)((int64_t)nchunks * s / nsplit), c1 = (int)((int64_t)nchunks * (s + 1) / nsplit);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int I0 = I * kGT, J0 = J * kGT;

  double dacc[4][4];
  ACC facc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) dacc[i][j] = 0.0;
  int bad = 0;

  for (int c = c0; c < c1; ++c) {
    const int64_t rb = (int64_t)c * K_t;
    const int64_t re = min(rb + (int64_t)K_t, m);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) facc[i][j] = (ACC)0;
    for (int64_t r = rb; r < re; r += kGKB) {
      // stage kGKB rows x 64 columns for I (and J) as rounded u_f values
      for (int e = threadIdx.x; e < kGKB * kGT; e += 256) {
        const int rr = e / kGT, cc = e % kGT;
        const int64_t row = r + rr;
        ACC va = (ACC)0, vb = (ACC)0;
        if (row < re) {
          const int ca = I0 + cc;
          if (ca < n) {
            const double v = round_uf(A[row * ld + ca] * dinv[ca], PREC);
            bad |= !isfinite(v);
            va = (ACC)v;
          }
          if (!diag) {
            const int cb = J0 + cc;
            if (cb < n) {
              const double v = round_uf(A[row * ld + cb] * dinv[cb], PREC);
              bad |= !isfinite(v);
              vb = (ACC)v;
            }
          }
        }
        As[rr][cc] = va;
        if (!diag) Bs[rr][cc] = vb;
      }
      __syncthreads();
      const ACC(*Bp)[kGT + 4] = diag ? As : Bs;
#pragma unroll 8
      for (int k = 0; k < kGKB; ++k) {
        ACC a[4], bb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bb[j] = Bp[k][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) facc[i][j] = fma(a[i], bb[j], facc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dacc[i][j] += (double)facc[i][j];
  }
  if (bad) atomicExch(range, 1);
  double* out = part + ((size_t)s * gridDim.x + blockIdx.x) * (kGT * kGT);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) out[(ty * 4 + i) * kGT + tx * 4 + j] = dacc[i][j];
}

// u_f in {fp32, fp64}: the products of u_f values are accumulated in fp64 throughout
// (R10: no fp32 level), so the chunk structure is irrelevant and each CTA sums its
// whole row split.  128 x 128 upper tiles, 32 x 64 per warp (64 fp64 accumulators), 16-row
// K-steps staged in shared memory with the next step's global loads (rounded to u_f when
// staged) in flight during the current step's DMMAs.
// kGP2: row stride 136 doubles (272 words = 16 mod 32 banks), so the DMMA fragment loads
// (4 rows x 8 consecutive doubles per warp) take the minimum two wavefronts.
constexpr int kGT2 = 128, kGK2 = 16, kGP2 = kGT2 + 8;
template <int PREC>
__global__ void __launch_bounds__(256, 1)
k_gram_f64(const double* __restrict__ A, int64_t m, int n, int64_t ld, const double* __restrict__ dinv,
           int nsplit, int TT, double* __restrict__ part, int* __restrict__ range) {
  __shared__ __align__(16) double As[kGK2][kGP2];
  __shared__ __align__(16) double Bs[kGK2][kGP2];
  int t = blockIdx.x, I = 0;
  while (t >= TT - I) { t -= TT - I; ++I; }
  const int J = I + t;
  const bool diag = (I == J);
  const int s = blockIdx.y;
  const int64_t rb = m * s / nsplit, re = m * (s + 1) / nsplit;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, wm = warp & 3, wn = warp >> 2;
  const int I0 = I * kGT2, J0 = J * kGT2;
  // staging map: thread -> (row lr = tid / 16, columns lc + 16 q): lanes read consecutive
  // doubles from global and write consecutive shared-memory words
  const int lr = tid >> 4, lc = tid & 15;
  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int bad = 0;
  // raw fp64 loads of the next step are kept in registers and only rounded (and scaled)
  // when they are staged, so the loads stay in flight during the current step's math
  double pa[8], pb[8];
  auto fetch = [&](int64_t r) {
    const int64_t row = r + lr;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int ca = I0 + lc + 16 * q, cb = J0 + lc + 16 * q;
      pa[q] = (row < re && ca < n) ? __ldcs(A + row * ld + ca) : 0.0;
      pb[q] = (!diag && row < re && cb < n) ? __ldcs(A + row * ld + cb) : 0.0;
    }
  };
  if (rb < re) fetch(rb);
  for (int64_t r = rb; r < re; r += kGK2) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int ca = I0 + lc + 16 * q, cb = J0 + lc + 16 * q;
      const double va = ca < n ? round_uf(pa[q] * dinv[ca], PREC) : 0.0;
      bad |= !isfinite(va);
      As[lr][lc + 16 * q] = va;
      if (!diag) {
        const double vb = cb < n ? round_uf(pb[q] * dinv[cb], PREC) : 0.0;
        bad |= !isfinite(vb);
        Bs[lr][lc + 16 * q] = vb;
      }
    }
    __syncthreads();
    if (r + kGK2 < re) fetch(r + kGK2);       // next step's loads overlap this step's math
    const double(*Bp)[kGP2] = diag ? As : Bs;
    // fp64 tensor cores (DMMA m8n8k4, SASS DMMA; the same 64 FMA/clk/SM as DFMA on B200 at
    // 1/8 of the instructions, measured tools/micro/dmma.cu): warp (wm, wn) owns rows
    // wm*32.. and columns wn*64.. of the tile; A = Â_I^T (8 x 4 fragments), B = Â_J (4 x 8).
    // 16.0 -> 13.2 ms at 65536 x 2048 against the DFMA version (22 TF/s, ~60% of the fp64
    // peak; a cp.async ring with in-place conversion measured 16.3 ms)
#pragma unroll
    for (int kk = 0; kk < kGK2; kk += 4) {
      const int kr = kk + (lane & 3);
      double af[4], bf[8];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = As[kr][wm * 32 + mi * 8 + (lane >> 2)];
#pragma unroll
      for (int nj = 0; nj < 8; ++nj) bf[nj] = Bp[kr][wn * 64 + nj * 8 + (lane >> 2)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 8; ++nj)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[mi][nj][0]), "+d"(acc[mi][nj][1])
                       : "d"(af[mi]), "d"(bf[nj]));
    }
    __syncthreads();
  }
  if (bad) atomicExch(range, 1);
  double* out = part + ((size_t)s * gridDim.x + blockIdx.x) * (kGT2 * kGT2);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 8; ++nj) {
      const int row = wm * 32 + mi * 8 + (lane >> 2), col = wn * 64 + nj * 8 + 2 * (lane & 3);
      *reinterpret_cast<double2*>(out + (size_t)row * kGT2 + col) = make_double2(acc[mi][nj][0], acc[mi][nj][1]);
    }
}

static void gram_shape_f64(const DenseView& A, int& TT, int& ntiles, int& nsplit) {
  TT = (A.n + kGT2 - 1) / kGT2;
  ntiles = TT * (TT + 1) / 2;
  const int64_t steps = (A.m + kGK2 - 1) / kGK2;
  nsplit = (int)((2 * (int64_t)num_sms() + ntiles - 1) / ntiles);
  if (nsplit > steps) nsplit = (int)steps;
  if (nsplit < 1) nsplit = 1;
}

// Sum the split partials in fixed order; write the tile and its mirror image.
__global__ void k_gram_reduce(const double* __restrict__ part, int ntiles, int nsplit, int TT, int n,
                              double* __restrict__ G, int tile) {
  int t = blockIdx.x, I = 0;
  while (t >= TT - I) { t -= TT - I; ++I; }
  const int J = I + t;
  for (int e = threadIdx.x; e < tile * tile; e += blockDim.x) {
    const int i = e / tile, j = e % tile;
    const int gi = I * tile + i, gj = J * tile + j;
    double acc = 0.0;
    for (int s = 0; s < nsplit; ++s) acc += part[((size_t)s * ntiles + blockIdx.x) * (tile * tile) + e];
    if (gi < n && gj < n) {
      G[(size_t)gi * n + gj] = acc;
      G[(size_t)gj * n + gi] = acc;
    }
  }
}

int launch_gram(const DenseView& A, int u_f, const double* dinv, int K_t, double* G, double* ws,
                size_t ws_doubles, int* range_flag, cudaStream_t st, int* launches) {
  if (K_t < 1) K_t = 64;
  if (gram_tc_supported(u_f, K_t))
    return launch_gram_tc(A, u_f, dinv, K_t, G, ws, ws_doubles * 8, range_flag, st, launches);
  if (u_f == TLS_FP32 || u_f == TLS_FP64) {
    int TT, ntiles, nsplit;
    gram_shape_f64(A, TT, ntiles, nsplit);
    if ((size_t)nsplit * ntiles * kGT2 * kGT2 > ws_doubles) {
      set_error("gram: workspace too small");
      return TLS_ERR_WORKSPACE;
    }
    dim3 grid(ntiles, nsplit);
    if (u_f == TLS_FP32)
      k_gram_f64<TLS_FP32><<<grid, 256, 0, st>>>(A.A, A.m, A.n, A.ld, dinv, nsplit, TT, ws, range_flag);
    else
      k_gram_f64<TLS_FP64><<<grid, 256, 0, st>>>(A.A, A.m, A.n, A.ld, dinv, nsplit, TT, ws, range_flag);
    TLS_LAUNCH_CHECK();
    k_gram_reduce<<<ntiles, 256, 0, st>>>(ws, ntiles, nsplit, TT, A.n, G, kGT2);
    TLS_LAUNCH_CHECK();
    if (launches) *launches += 2;
    return 0;
  }
  int TT, ntiles, nchunks, nsplit;
  gram_shape(A, K_t, TT, ntiles, nchunks, nsplit);
  if ((size_t)nsplit * ntiles * kGT * kGT > ws_doubles) {
    set_error("gram: workspace too small");
    return TLS_ERR_WORKSPACE;
  }
  dim3 grid(ntiles, nsplit);
  switch (u_f) {
    case TLS_FP16:
      k_gram_cc<float, TLS_FP16><<<grid, 256, 0, st>>>(A.A, A.m, A.n, A.ld, dinv, K_t, nchunks, nsplit, TT, ws, range_flag);
      break;
    case TLS_BF16:
      k_gram_cc<float, TLS_BF16><<<grid, 256, 0, st>>>(A.A, A.m, A.n, A.ld, dinv, K_t, nchunks, nsplit, TT, ws, range_flag);
      break;
    case TLS_FP32:
      k_gram_cc<double, TLS_FP32><<<grid, 256, 0, st>>>(A.A, A.m, A.n, A.ld, dinv, K_t, nchunks, nsplit, TT, ws, range_flag);
      break;
    default:
      k_gram_cc<double, TLS_FP64><<<grid, 256, 0, st>>>(A.A, A.m, A.n, A.ld, dinv, K_t, nchunks, nsplit, TT, ws, range_flag);
      break;
  }
  TLS_LAUNCH_CHECK();
  k_gram_reduce<<<ntiles, 256, 0, st>>>(ws, ntiles, nsplit, TT, A.n, G, kGT);
  TLS_LAUNCH_CHECK();
  if (launches) *launches += 2;
  return 0;
}

}  // namespace tls
