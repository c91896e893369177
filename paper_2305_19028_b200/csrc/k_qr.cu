// k_qr.cu — the paper's preferred preconditioner on the GPU: R~ = the R factor of a
// Householder QR of A D^{-1} computed in u_f (PAPER.md l.215-218,
// l.231 "Compute A = Q[R 0]^T in u_q", l.276-288; reading R25).
//
// Arithmetic (R25): every elementwise operation is rounded to u_f on its own, inner
// products are accumulated in fp64 and rounded once (a wide accumulator).  Per column j
// (x = W[j:, j]):
//     sigma = fl(sqrt(fl(x^T x))),  alpha = -sign(x_0) sigma,  v = x - alpha e_0 (v_0 rounded),
//     beta = fl(2 / fl(v^T v)),     w^T = fl(beta fl(v^T W[j:, j+1:])),
//     W[j:, j+1:] = fl(W - fl(v w^T))                      (each product and difference rounded)
// and R row j = sign(alpha) [alpha, W[j, j+1:]] (diag(R) >= 0).
//
// B200 design: W = fl_uf(A D^{-1}) lives row-major in HBM as fp32 (exact for fp16/bf16/fp32
// values) or fp64 (u_f = fp64).  One column costs ONE streaming pass over the trailing
// matrix: k_qr_step updates rows >= j with column j's reflector and, in the same pass,
// accumulates the fp64 partial inner products of the NEXT column (x'^T x' and x'^T W')
// per CTA, so column j+1's reflector needs no second pass; k_qr_fin reduces those partials
// (fixed order, deterministic), forms the column's scalars and w^T.  2 launches per column.
#include <cuda_bf16.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

namespace {
constexpr int kQrThreads = 256;
// update-pass CTA size: one CTA per SM, 512 threads (<= 8 columns per thread) or 256 (16)
template <int CPT> __host__ __device__ constexpr int qr_step_threads() { return CPT >= 16 ? 256 : 512; }

// Round an fp32 value to u_f (fp16 / bf16 hardware conversions; identity for fp32).
template <int PREC> __device__ __forceinline__ float qr_rdf(float x) {
  if constexpr (PREC == TLS_FP16) return __half2float(__float2half_rn(x));
  else if constexpr (PREC == TLS_BF16) return __bfloat162float(__float2bfloat16_rn(x));
  else return x;
}

template <typename T> __device__ __forceinline__ T qr_store(double v);
template <> __device__ __forceinline__ float qr_store<float>(double v) { return (float)v; }   // exact: v in u_f
template <> __device__ __forceinline__ double qr_store<double>(double v) { return v; }

// Team size for a pass over `ncols` columns with CPT columns per thread.
__host__ __device__ inline int qr_team(int ncols, int cpt) {
  int tg = (ncols + cpt - 1) / cpt;
  tg = (tg + 31) / 32 * 32;
  if (tg < 32) tg = 32;
  return tg > kQrThreads ? kQrThreads : tg;
}

// scal[j]: {alpha, v_0, sigma, beta}
// One pass.  LOAD: W = fl_uf(A D^{-1}) and the partials of column 0.  Otherwise: apply
// column j's reflector to rows >= j, columns > j, write R row j, and accumulate the partials
// of column c = j + 1 over rows > c: partP[b][k] = sum_i x'_i W'[i][k] for k >= c (k = c is
// the tail x'^T x' of the column below its diagonal).
// A CTA owns RB rows; it runs `teams` rows at a time, one team of TG threads per row (CPT
// columns per thread, k = c + tl + q TG), with the next row of each team loaded before the
// current one is stored.  Team partials are combined in shared memory in team order.
template <typename T, bool LOAD> struct QrSrc { using type = T; };
template <typename T> struct QrSrc<T, true> { using type = double; };   // LOAD reads A itself

// Loads of the next row keep the storage type: nothing waits on them until the row is used.
template <typename T, bool LOAD, int CPT>
__device__ __forceinline__ void qr_load_row(const T* __restrict__ W, const double* __restrict__ A, int64_t lda,
                                            int64_t i, int n, int ldw, int j, int c, int tl, int TG,
                                            typename QrSrc<T, LOAD>::type (&dst)[CPT],
                                            typename QrSrc<T, LOAD>::type& sj, typename QrSrc<T, LOAD>::type& sc) {
  using S = typename QrSrc<T, LOAD>::type;
  const S* src;
  if constexpr (LOAD) src = A + i * lda;
  else src = W + i * (int64_t)ldw;
  if (!LOAD) sj = (i == j) ? S(0) : src[j];
  sc = c < n ? src[c] : S(0);
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int k = c + tl + q * TG;
    dst[q] = k < n ? src[k] : S(0);
  }
}

template <typename T, bool LOAD, int CPT, int PREC>
__global__ void __launch_bounds__(qr_step_threads<CPT>(), 1) k_qr_step(T* __restrict__ W, const double* __restrict__ A, int64_t lda,
                                                         const double* __restrict__ dinv, int64_t m, int n, int ldw, int j,
                                                         int RB, int bfirst, int TG,
                                                         const double* __restrict__ wT,
                                                         const double* __restrict__ scal, double* __restrict__ partP,
                                                         double* __restrict__ G, const int* __restrict__ dead) {
  extern __shared__ double qsm[];
  // programmatic dependent launch: wait for the predecessor's writes before reading anything;
  // the next kernel is released after the row loop (below)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (!LOAD && *dead) return;
  const int c = j + 1;
  const int ncols = n - c;
  const int64_t rs = LOAD ? 0 : j;
  const int b = bfirst + (int)blockIdx.x;
  int64_t r0 = (int64_t)b * RB;
  const int64_t r1 = min(m, r0 + RB);
  if (r1 <= rs) return;                 // rows all above: k_qr_fin does not read this CTA
  if (r0 < rs) r0 = rs;
  const int t = threadIdx.x, tm = t / TG, tl = t % TG, teams = blockDim.x / TG;
  using S = typename QrSrc<T, LOAD>::type;
  constexpr int prec = PREC;
  double wk[CPT], acc[CPT];
  S cur[CPT], nxt[CPT];
  const double alpha = LOAD ? 0.0 : scal[4 * j + 0];
  const double v0 = LOAD ? 0.0 : scal[4 * j + 1];
  const double wc = LOAD ? (dinv ? dinv[0] : 1.0) : (c < n ? wT[c] : 0.0);   // LOAD: the scale of column 0
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int k = c + tl + q * TG;
    wk[q] = k < n ? (LOAD ? (dinv ? dinv[k] : 1.0) : wT[k]) : 0.0;   // LOAD: the column scales (none: 1)
    acc[q] = 0.0;
  }
  int64_t i = r0 + tm;
  bool have = i < r1;
  S nj = S(0), nc = S(0);
  if (have) qr_load_row<T, LOAD, CPT>(W, A, lda, i, n, ldw, j, c, tl, TG, nxt, nj, nc);
  while (have) {
#pragma unroll
    for (int q = 0; q < CPT; ++q) cur[q] = nxt[q];
    const double cj = (double)nj, cc = (double)nc;
    const int64_t inext = i + teams;
    const bool hn = inext < r1;
    if (hn) qr_load_row<T, LOAD, CPT>(W, A, lda, inext, n, ldw, j, c, tl, TG, nxt, nj, nc);
    // in-place update by a multi-warp team: see qr_update_v4 (the LOAD pass reads A, not W)
    if (!LOAD && TG > 32) asm volatile("bar.sync %0, %1;" ::"r"(1 + tm), "r"(TG) : "memory");
    T* row = W + i * (int64_t)ldw;
    const bool accum = i > c;
    if (LOAD && tl < ldw - n) row[n + tl] = T(0);      // padding columns of the working copy
    if constexpr (!LOAD && PREC != TLS_FP64) {
      // fp32 arithmetic, bit-identical to the fp64-then-round of the oracle: the products of
      // two u_f values are exact in fp32 (fp16: 22 bits, bf16: 16) or correctly rounded
      // (u_f = fp32), and a difference rounded to fp32 and then to u_f equals the difference
      // rounded once to u_f, as fp32's 24 bits >= 2p + 2 for p = 11 and 8 (double rounding is
      // innocuous; R25).  Conversions then stay off the XU pipe (packed F2FP / HADD2).
      const float vf = (i == j) ? (float)v0 : (float)cj;
      const float xf = qr_rdf<PREC>(__fsub_rn((float)cc, qr_rdf<PREC>(__fmul_rn(vf, (float)wc))));
      const double xd = (double)xf;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int k = c + tl + q * TG;
        if (k < n) {
          const float nf = qr_rdf<PREC>(__fsub_rn((float)cur[q], qr_rdf<PREC>(__fmul_rn(vf, (float)wk[q]))));
          row[k] = nf;
          if (accum) acc[q] = fma(xd, (double)nf, acc[q]);
          if (i == j) G[(int64_t)j * n + k] = alpha < 0.0 ? -(double)nf : (double)nf;
        }
      }
    } else {
      double xc, vi = 0.0;   // xc: new value of column c in this row (same bits in every thread)
      if (LOAD) {
        xc = round_uf(cc * wc, prec);
      } else {
        vi = (i == j) ? v0 : cj;
        xc = round_uf(__dsub_rn(cc, round_uf(__dmul_rn(vi, wc), prec)), prec);
      }
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int k = c + tl + q * TG;
        if (k < n) {
          const double cv = (double)cur[q];
          const double nv = LOAD ? round_uf(cv * wk[q], prec)
                                 : round_uf(__dsub_rn(cv, round_uf(__dmul_rn(vi, wk[q]), prec)), prec);
          row[k] = qr_store<T>(nv);
          if (accum) acc[q] = fma(xc, nv, acc[q]);
          if (!LOAD && i == j) G[(int64_t)j * n + k] = alpha < 0.0 ? -nv : nv;
        }
      }
    }
    i = inext;
    have = hn;
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (teams == 1) {
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int k = c + tl + q * TG;
      if (k < n) partP[(int64_t)b * n + k] = acc[q];
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int kk = tl + q * TG;
    if (kk < ncols) qsm[tm * ncols + kk] = acc[q];
  }
  __syncthreads();
  for (int kk = t; kk < ncols; kk += blockDim.x) {
    double sum = 0.0;
    for (int u = 0; u < teams; ++u) sum += qsm[u * ncols + kk];
    partP[(int64_t)b * n + c + kk] = sum;
  }
}

// The update pass on the fp32 working copy (u_f = fp16 / bf16 / fp32), 16-byte accesses:
// thread tl owns the 4-column groups g = tl + q TG starting at the aligned column c0 = c & ~3
// (ldw is a multiple of 4).  Columns k < c and k >= n carry w_k = 0, so they are rewritten
// with their own values (rd(x - rd(v 0)) = x) and need no masks.
// Row block b's share of column j's update pass (the body of k_qr_step_v4); `teams` teams of
// TG threads, threads beyond teams x TG only join the combine.
template <int CPT, int PREC>
__device__ __forceinline__ void qr_update_v4(float* __restrict__ W, int64_t m, int n, int ldw, int j, int RB, int b,
                                             int TG, int teams, const double* __restrict__ wT,
                                             const double* __restrict__ scal, double* __restrict__ partP,
                                             double* __restrict__ G, double* qsm, bool pdl_release) {
  constexpr int GPT = CPT / 4;
  const int c = j + 1, c0 = c & ~3;
  // columns up to n (rounded to 4): the whole row for the unblocked factorization (n = the
  // matrix's n, ldw = round4(n)), the panel for the blocked one (n = the panel's end, R29)
  const int lde = min(ldw, (n + 3) & ~3);
  const int ngroups = (lde - c0) >> 2;
  int64_t r0 = (int64_t)b * RB;
  const int64_t r1 = min(m, r0 + RB);
  if (r1 <= j) return;
  if (r0 < j) r0 = j;
  const int t = threadIdx.x, tm = t / TG, tl = t % TG;
  const double alpha = scal[4 * j + 0];
  const float v0f = (float)scal[4 * j + 1];
  const float wcf = (float)wT[c];
  float wk[CPT];
  double acc[CPT];
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = c0 + 4 * (tl + q * TG) + e;
      wk[4 * q + e] = (k >= c && k < n) ? (float)wT[k] : 0.f;
      acc[4 * q + e] = 0.0;
    }
  }
  // rows of this team in flight: a ring of QD rows (static slots, the loop unrolled by QD), so
  // each row's load is issued QD rows before its update (round 2 continued: with one row ahead
  // the pass was one L2/HBM round trip per row of a team -- the per-column chain of the QR was
  // load-latency bound; the arithmetic and its order are unchanged)
#ifdef TLS_QR_QD
  constexpr int QD = TLS_QR_QD;                  // build-time A/B (1 = round 2's one row ahead)
#else
  // measured (profiles/r02_qr_depth.log): 4 rows ahead 234 vs 287 ms for the unblocked QR at
  // 65536 x 2048, the same blocked (57.8 vs 56.8 ms) and 5% slower at 16384 x 1024 unblocked;
  // the blocked QR's panel passes (one 4-column group per thread) keep 8
  constexpr int QD = GPT == 1 ? 8 : 4;
#endif
  float4 buf[QD][GPT];
  float bj[QD], bc[QD];
  auto load = [&](int64_t ii, float4 (&dst)[GPT], float& dj, float& dc) {
    const float* src = W + ii * (int64_t)ldw;
    dj = src[j];
    dc = src[c];
#pragma unroll
    for (int q = 0; q < GPT; ++q) {
      const int g = tl + q * TG;
      if (g < ngroups) dst[q] = *reinterpret_cast<const float4*>(src + c0 + 4 * g);
    }
  };
  int64_t i = r0 + tm;
  const bool active_team = tm < teams;
#pragma unroll
  for (int d = 0; d < QD; ++d)
    if (active_team && i + (int64_t)d * teams < r1) load(i + (int64_t)d * teams, buf[d], bj[d], bc[d]);
  while (active_team && i < r1) {
#pragma unroll
    for (int d = 0; d < QD; ++d) {
      if (i < r1) {
        float4 cur[GPT];
#pragma unroll
        for (int q = 0; q < GPT; ++q) cur[q] = buf[d][q];
        const float cj = bj[d], cc = bc[d];
        const int64_t ifar = i + (int64_t)QD * teams;
        if (ifar < r1) load(ifar, buf[d], bj[d], bc[d]);
        // A team of several warps updates a row in place, and every thread reads the row's column
        // c (old value) while the thread owning column c's group writes its new value: all of the
        // team's loads of a row must be performed before any store to it (QD iterations later).
        // bar.sync orders them (its participants' prior accesses are performed first).  A one-warp
        // team needs none.  (Without it, teams of 3 warps -- n >= ~520 -- read already-updated
        // column-c values: round 1's QR differed from the oracle there.)
        if (TG > 32) asm volatile("bar.sync %0, %1;" ::"r"(1 + tm), "r"(TG) : "memory");
        float* row = W + i * (int64_t)ldw;
        const float vf = (i == j) ? v0f : cj;
        const double xd = (double)qr_rdf<PREC>(__fsub_rn(cc, qr_rdf<PREC>(__fmul_rn(vf, wcf))));
        const bool accum = i > c;
#pragma unroll
        for (int q = 0; q < GPT; ++q) {
          const int g = tl + q * TG;
          if (g < ngroups) {
            float x[4] = {cur[q].x, cur[q].y, cur[q].z, cur[q].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              x[e] = qr_rdf<PREC>(__fsub_rn(x[e], qr_rdf<PREC>(__fmul_rn(vf, wk[4 * q + e]))));
              if (accum) acc[4 * q + e] = fma(xd, (double)x[e], acc[4 * q + e]);
            }
            *reinterpret_cast<float4*>(row + c0 + 4 * g) = make_float4(x[0], x[1], x[2], x[3]);
            if (i == j) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int k = c0 + 4 * g + e;
                if (k >= c && k < n) G[(int64_t)j * n + k] = alpha < 0.0 ? -(double)x[e] : (double)x[e];
              }
            }
          }
        }
        i += teams;
      }
    }
  }
  if (pdl_release) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int ncv = ngroups * 4;
  if (teams > 1) {
#pragma unroll
    for (int q = 0; q < GPT; ++q) {
      const int g = tl + q * TG;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (tm < teams && g < ngroups) qsm[tm * ncv + 4 * g + e] = acc[4 * q + e];
    }
    __syncthreads();
    for (int kk = t; kk < ncv; kk += blockDim.x) {   // (teams x ncv doubles of qsm)
      const int k = c0 + kk;
      if (k < c || k >= n) continue;
      double sum = 0.0;
      for (int u = 0; u < teams; ++u) sum += qsm[u * ncv + kk];
      partP[(int64_t)b * n + k] = sum;
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int g = tl + q * TG;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = c0 + 4 * g + e;
      if (tm < teams && g < ngroups && k >= c && k < n) partP[(int64_t)b * n + k] = acc[4 * q + e];
    }
  }
}

template <int CPT, int PREC>
__global__ void __launch_bounds__(qr_step_threads<CPT>(), 1) k_qr_step_v4(
    float* __restrict__ W, int64_t m, int n, int ldw, int j, int RB, int bfirst, int TG,
    const double* __restrict__ wT, const double* __restrict__ scal, double* __restrict__ partP,
    double* __restrict__ G, const int* __restrict__ dead) {
  extern __shared__ double qsm[];
  // programmatic dependent launch: wait for the predecessor's writes before reading anything;
  // the next kernel is released after the row loop
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (*dead) return;
  qr_update_v4<CPT, PREC>(W, m, n, ldw, j, RB, bfirst + (int)blockIdx.x, TG, (int)blockDim.x / TG, wT, scal, partP, G,
                          qsm, true);
}

// Column j's scalars and w^T from the partials the previous pass left (CTAs b >= b0 wrote).
// A CTA reduces 32 columns: warp w sums partial rows b = b0 + w (mod 8), then the 8 warp
// sums are added in warp order (deterministic).
template <typename T, int PREC>
__global__ void __launch_bounds__(kQrThreads) k_qr_fin(const T* __restrict__ W, int n, int ldw, int j, int b0, int nb,
                                                        const double* __restrict__ partP, double* __restrict__ wT,
                                                        double* __restrict__ scal, double* __restrict__ G,
                                                        int* __restrict__ qflags, int leaf, int ldp) {
  // ldp: the row stride of the partials (the n of the pass that wrote them: the matrix's n, or the
  // panel's end in the blocked QR, whose first panel reads the full-width load pass)
  __shared__ double red[32];
  // programmatic dependent launch: the next kernel of the chain may be scheduled now; this
  // one waits for its predecessor's writes before reading anything
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ double cs[8][32];
  constexpr int prec = PREC;
  if (qflags[0]) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double tl = 0.0;
  for (int b = b0 + t; b < nb; b += kQrThreads) tl += partP[(int64_t)b * ldp + j];
  const double tail = block_sum(tl, red);                      // fixed order: same bits in every CTA
  const double x0 = (double)W[(int64_t)j * ldw + j];
  const double sigma = round_uf(sqrt(round_uf(fma(x0, x0, tail), prec)), prec);
  const bool ident = sigma == 0.0;
  if (ident && !leaf) {      // zero column in u_f (an overflowed inf/NaN goes on, as in the oracle: TLS_RANGE)
    if (blockIdx.x == 0 && t == 0) { qflags[0] = 1; qflags[1] = j + 1; }
    return;
  }
  // a TSQR leaf's vanishing column (R26): the identity reflector (alpha = v_0 = beta = 0 gives
  // w^T = 0, the update leaves every row as it is and R's row j is W[j, j:] with R_jj = 0)
  const double alpha = ident ? 0.0 : (x0 >= 0.0 ? -sigma : sigma);
  const double v0 = ident ? 0.0 : round_uf(x0 - alpha, prec);
  const double vv = ident ? 1.0 : round_uf(fma(v0, v0, tail), prec);
  const double beta = ident ? 0.0 : round_uf(2.0 / vv, prec);
  const int k = j + 1 + blockIdx.x * 32 + lane;
  // warp w sums the partial rows b0 + w + 16i into s0 and b0 + w + 8 + 16i into s1, in i order;
  // all of a batch's loads are issued before its adds (round 2 continued: the dependent
  // two-loads-per-step loop was ~9 L2 round trips per column; same order, same bits)
  double s0 = 0.0, s1 = 0.0;
  if (k < n) {
    constexpr int kB = 10;                    // rows per accumulator per batch: nb <= 160 in one batch
    for (int b = b0 + warp; b < nb; b += 16 * kB) {
      double pa[kB], pb[kB];
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int r0 = b + 16 * i, r1 = r0 + 8;
        pa[i] = r0 < nb ? partP[(int64_t)r0 * ldp + k] : 0.0;
        pb[i] = r1 < nb ? partP[(int64_t)r1 * ldp + k] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        if (b + 16 * i < nb) s0 += pa[i];
        if (b + 16 * i + 8 < nb) s1 += pb[i];
      }
    }
  }
  cs[warp][lane] = s0 + s1;
  __syncthreads();
  if (warp == 0 && k < n) {
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += cs[u][lane];
    const double w = round_uf(fma(v0, (double)W[(int64_t)j * ldw + k], s), prec);
    wT[k] = round_uf(beta * w, prec);
  }
  if (blockIdx.x == 0 && t == 0) {
    scal[4 * j + 0] = alpha;
    scal[4 * j + 1] = v0;
    scal[4 * j + 2] = sigma;
    scal[4 * j + 3] = beta;
    G[(int64_t)j * n + j] = sigma;                              // |alpha|: diag(R) >= 0
  }
}

// Launch with programmatic stream serialisation (PDL): the kernels of the per-column chain
// overlap their launch with the tail of the previous one (each waits on griddepcontrol).
template <typename... KArgs, typename... Args>
int launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl = [] { const char* e = getenv("TLS_QR_PDL"); return !(e && e[0] == '0'); }();
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, args...);
  if (e != cudaSuccess) {
    set_error("k_qr launch: %s", cudaGetErrorString(e));
    return TLS_ERR_CUDA;
  }
  return 0;
}


template <typename T, bool LOAD, int CPT, int PREC>
int qr_step_launch(T* W, const DenseView& A, int ldw, const double* dinv, int j, int RB, int bfirst, int nblk,
                   const double* wT, const double* scal, double* partP, double* G, const int* qflags, cudaStream_t st) {
  const int n = A.n;
  if constexpr (!LOAD && sizeof(T) == 4) {
    const int c0 = (j + 1) & ~3;
    const int lde = ldw < ((n + 3) & ~3) ? ldw : ((n + 3) & ~3);
    const int ngroups = (lde - c0) / 4;
    const int TG = qr_team(ngroups, CPT / 4);
    const int teams = qr_step_threads<CPT>() / TG;
    const size_t smem = teams > 1 ? (size_t)teams * ngroups * 4 * sizeof(double) : 0;
    return launch_pdl(k_qr_step_v4<CPT, PREC>, nblk, teams * TG, smem, st, reinterpret_cast<float*>(W), A.m, n, ldw,
                      j, RB, bfirst, TG, wT, scal, partP, G, qflags);
  } else {
    const int ncols = n - (j + 1);
    const int TG = qr_team(ncols, CPT);
    const int teams = qr_step_threads<CPT>() / TG;
    const size_t smem = teams > 1 ? (size_t)teams * ncols * sizeof(double) : 0;
    return launch_pdl(k_qr_step<T, LOAD, CPT, PREC>, nblk, teams * TG, smem, st, W, A.A, A.ld, dinv, A.m, n, ldw, j,
                      RB, bfirst, TG, wT, scal, partP, G, qflags);
  }
}

template <typename T, int CPT, int PREC>
int qr_t(const DenseView& A, const double* dinv, void* Wbuf, double* partP, double* wT, double* scal,
         int* qflags, double* G, cudaStream_t st, int* launches, int row_stride, int leaf) {
  const int n = A.n;
  const int64_t m = A.m;
  const int RB = qr_rows_per_cta(m, n);
  const int nb = (int)((m + RB - 1) / RB);
  T* W = static_cast<T*>(Wbuf);
  const int ldw = qr_ldw(n, PREC);
  int rc = qr_step_launch<T, true, CPT, PREC>(W, A, ldw, dinv, -1, RB, 0, nb, nullptr, nullptr, partP, G, qflags, st);
  if (rc) return rc;
  int nl = 1;
  // row_stride > 0 (the row-interleaved TSQR stack, R26): rows >= (j + 2) row_stride are zero in
  // columns j and j + 1, so the pass of column j stops there (bit-identical: they add zeros)
  auto m_act = [&](int j) -> int64_t { return row_stride > 0 ? std::min(m, (int64_t)(j + 2) * row_stride) : m; };
  // debugging aid: TLS_QR_STOP=J ends the loop after column J's update pass and, with
  // TLS_QR_DUMP=path, writes the working copy, w^T, the scalars and the partials to path
  const char* stop_e = getenv("TLS_QR_STOP");
  const int stop_j = stop_e ? atoi(stop_e) : -1;
  for (int j = 0; j < n; ++j) {
    if (stop_j >= 0 && j > stop_j) {
      const char* path = getenv("TLS_QR_DUMP");
      if (path) {
        cudaStreamSynchronize(st);
        std::vector<char> hw((size_t)m * ldw * sizeof(T));
        std::vector<double> hwt(n), hs(4 * (size_t)n), hp((size_t)nb * n);
        cudaMemcpy(hw.data(), W, hw.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(hwt.data(), wT, n * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hs.data(), scal, 4 * (size_t)n * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hp.data(), partP, (size_t)nb * n * 8, cudaMemcpyDeviceToHost);
        FILE* f = fopen(path, "wb");
        if (f) {
          const int64_t hdr[5] = {m, n, ldw, nb, (int64_t)sizeof(T)};
          fwrite(hdr, 8, 5, f);
          fwrite(hw.data(), 1, hw.size(), f);
          fwrite(hwt.data(), 8, n, f);
          fwrite(hs.data(), 8, 4 * (size_t)n, f);
          fwrite(hp.data(), 8, (size_t)nb * n, f);
          fclose(f);
        }
      }
      break;
    }
    // partials of column j were written by the pass with first row max(j - 1, 0)
    const int b0 = (int)((j > 0 ? j - 1 : 0) / RB);
    const int nbj = j == 0 ? nb : (int)((m_act(j - 1) + RB - 1) / RB);   // CTAs that wrote them
    const int nf = (n - j - 1 + 31) / 32;
    rc = launch_pdl(k_qr_fin<T, PREC>, nf > 0 ? nf : 1, kQrThreads, 0, st, (const T*)W, n, ldw, j, b0, nbj,
                    (const double*)partP, wT, scal, G, qflags, leaf, n);
    if (rc) return rc;
    ++nl;
    if (j + 1 < n) {
      const int bs = (int)(j / RB);       // CTAs whose rows are all < j would exit at once: not launched
      DenseView Aj = A;
      Aj.m = m_act(j);
      const int nbu = (int)((Aj.m + RB - 1) / RB);
      rc = qr_step_launch<T, false, CPT, PREC>(W, Aj, ldw, dinv, j, RB, bs, nbu - bs, wT, scal, partP, G, qflags, st);
      if (rc) return rc;
      ++nl;
    }
  }
  TLS_LAUNCH_CHECK();
  if (launches) *launches += nl;
  return 0;
}

template <typename T, int PREC>
int qr_dispatch(const DenseView& A, const double* dinv, void* Wbuf, double* partP, double* wT, double* scal,
                int* qflags, double* G, cudaStream_t st, int* launches, int rs, int leaf) {
  // 8 columns per thread up to n = 2048 (measured: 4 per thread is 1.2-1.3x slower at n = 1024,
  // 16 per thread with 256-thread CTAs 1.1x slower at n = 1024 and 2048)
  if (A.n <= 8 * kQrThreads) return qr_t<T, 8, PREC>(A, dinv, Wbuf, partP, wT, scal, qflags, G, st, launches, rs, leaf);
  return qr_t<T, 16, PREC>(A, dinv, Wbuf, partP, wT, scal, qflags, G, st, launches, rs, leaf);
}
}  // namespace

int qr_rows_per_cta(int64_t m, int n) {
  (void)n;
  const int64_t want = 148;   // one update-pass CTA per SM (qr_step_threads)
  int64_t rb = (m + want - 1) / want;
  if (rb < 32) rb = 32;
  return (int)rb;
}

int qr_ldw(int n, int u_f) { return u_f == TLS_FP64 ? n : (n + 3) / 4 * 4; }

size_t qr_work_bytes(int64_t m, int n, int u_f) {
  const int RB = qr_rows_per_cta(m, n);
  const int64_t nb = (m + RB - 1) / RB;
  const size_t es = (u_f == TLS_FP64) ? 8 : 4;
  return (size_t)m * qr_ldw(n, u_f) * es + (size_t)nb * n * 8 + (size_t)n * 8 + 4 * (size_t)n * 8 + 5 * 256;
}

int launch_qr(const DenseView& A, int u_f, const double* dinv, void* Wbuf, double* partP, double* wT, double* scal,
              int* qflags, double* G, cudaStream_t st, int* launches, int row_stride, int leaf) {
  if (A.n > kMaxDenseN) { set_error("QR: n > %d", kMaxDenseN); return TLS_ERR_ARG; }
  switch (u_f) {
    case TLS_FP16: return qr_dispatch<float, TLS_FP16>(A, dinv, Wbuf, partP, wT, scal, qflags, G, st, launches, row_stride, leaf);
    case TLS_BF16: return qr_dispatch<float, TLS_BF16>(A, dinv, Wbuf, partP, wT, scal, qflags, G, st, launches, row_stride, leaf);
    case TLS_FP32: return qr_dispatch<float, TLS_FP32>(A, dinv, Wbuf, partP, wT, scal, qflags, G, st, launches, row_stride, leaf);
    default: return qr_dispatch<double, TLS_FP64>(A, dinv, Wbuf, partP, wT, scal, qflags, G, st, launches, row_stride, leaf);
  }
}


// ====================================================================== blocked QR (R29, NEXT-2)
// Panels of kWyB = 128 columns: the panel is factored by the unblocked chain above restricted
// to the panel's columns (k_qr_fin + k_qr_step_v4 with n = the panel's end), then its 128
// reflectors are applied to the trailing columns at once on the tensor cores (compact WY):
//   V (m' x 128, the Householder vectors, u_f values)     k_wy_extract, k_wy_transpose
//   V^T V, V^T C (R11-style fp32 chunk sums, fp64)       launch_tc_atb (k_gram_tc, atb mode)
//   T (fp64, the WY factor), Y = fl_uf(T^T V^T C)        k_wy_T, k_wy_Y
//   C <- fl_uf(C - fl32(V Y))                             launch_qr_wy_update (tcgen05)
// A 16-bit twin W16 of the working copy feeds the tensor cores (the values are u_f values, so
// it is exact); the update writes both.  The next panel's first inner products come from a
// "virtual" update pass of column c0 - 1 with w = 0 (nothing changes, the partials of column
// c0 are accumulated), so the panel chain starts exactly as the unblocked one.
constexpr int kWyB = 128;

template <int PREC>
__global__ void k_f32_to_16(const float* __restrict__ W, int64_t ldw, uint16_t* __restrict__ W16, int64_t ld16,
                            int64_t m, int n) {
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x)
    for (int k = threadIdx.x; k < ld16; k += blockDim.x) {
      const double x = k < n ? (double)W[i * ldw + k] : 0.0;
      W16[i * ld16 + k] = PREC == TLS_FP16 ? f64_to_f16_bits(x) : f64_to_bf16_bits(x);
    }
}

// V16[i][jj] (m' x 128, i = row - c0): v_{c0+jj} (the diagonal entry v_0 from scal, below it the
// panel column as the chain left it, zero above)
template <int PREC>
__global__ void k_wy_extract(const float* __restrict__ W, int64_t ldw, const double* __restrict__ scal, int c0, int nb,
                             int64_t m, uint16_t* __restrict__ V16) {
  const int jj = threadIdx.x;
  for (int64_t i = blockIdx.x; i < m - c0; i += gridDim.x) {
    double v = 0.0;
    if (jj < nb) {
      if (i == jj) v = scal[4 * (c0 + jj) + 1];
      else if (i > jj) v = (double)W[(c0 + i) * ldw + c0 + jj];
    }
    V16[i * kWyB + jj] = PREC == TLS_FP16 ? f64_to_f16_bits(v) : f64_to_bf16_bits(v);
  }
}

// Vt16 (128 x ldv) = V16^T, 32 x 32 tiles through shared memory
__global__ void k_wy_transpose(const uint16_t* __restrict__ V16, int64_t mr, uint16_t* __restrict__ Vt16, int64_t ldv) {
  __shared__ uint16_t tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int j0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r;
    tile[r][threadIdx.x] = i < mr ? V16[i * kWyB + j0 + threadIdx.x] : (uint16_t)0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + threadIdx.x;
    if (i < ldv) Vt16[(int64_t)(j0 + r) * ldv + i] = tile[threadIdx.x][r];
  }
}

// T (128 x 128, fp64, upper): T_jj = beta_j, T[0:j, j] = -beta_j T[0:j, 0:j] VtV[0:j, j]
// (VtV symmetric: its column j is read as row j, coalesced, into shared memory per step)
__global__ void __launch_bounds__(kWyB) k_wy_T(const double* __restrict__ VtV, const double* __restrict__ scal, int c0,
                                               int nb, double* __restrict__ T) {
  extern __shared__ double Ts[];                       // [128][129], then the column vector [128]
  double* vc = Ts + kWyB * (kWyB + 1);
  const int i = threadIdx.x;
  for (int e = i; e < kWyB * (kWyB + 1); e += blockDim.x) Ts[e] = 0.0;
  // column j + 1 of VtV is loaded while step j computes (round 2 continued: the load at the top
  // of each of the 128 dependent steps was an L2 round trip on the chain)
  double vnext = nb > 0 ? VtV[i] : 0.0;
  for (int j = 0; j < nb; ++j) {
    vc[i] = vnext;
    if (j + 1 < nb) vnext = VtV[(int64_t)(j + 1) * kWyB + i];
    __syncthreads();
    const double bj = scal[4 * (c0 + j) + 3];
    if (i < j) {
      double s0 = 0.0, s1 = 0.0;                        // two chains: even and odd l, added at the end
      int l = i;
      for (; l + 1 < j; l += 2) {
        s0 = fma(Ts[i * (kWyB + 1) + l], vc[l], s0);
        s1 = fma(Ts[i * (kWyB + 1) + l + 1], vc[l + 1], s1);
      }
      if (l < j) s0 = fma(Ts[i * (kWyB + 1) + l], vc[l], s0);
      Ts[i * (kWyB + 1) + j] = -bj * (s0 + s1);
    } else if (i == j) {
      Ts[i * (kWyB + 1) + j] = bj;
    }
    __syncthreads();
  }
  for (int e = i; e < kWyB * kWyB; e += blockDim.x) T[e] = Ts[(e / kWyB) * (kWyB + 1) + e % kWyB];
}

// Y16 (128 x ldy) = fl_uf(T^T Y1) (fp64 products and sums, one rounding), Y1: 128 x ldy1.
// CTA = 32 columns k (Y1's block staged in shared memory), warp = rows p = warp, warp + 8, ...
template <int PREC>
__global__ void __launch_bounds__(256) k_wy_Y(const double* __restrict__ T, const double* __restrict__ Y1, int64_t ldy1,
                                              int nc, uint16_t* __restrict__ Y16, int64_t ldy) {
  __shared__ double ys[kWyB][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = blockIdx.x * 32 + lane;
  for (int l = warp; l < kWyB; l += 8) ys[l][lane] = k < nc ? Y1[(int64_t)l * ldy1 + k] : 0.0;
  __syncthreads();
  for (int p = warp; p < kWyB; p += 8) {
    double acc = 0.0;
    for (int l = 0; l <= p; ++l) acc = fma(__ldg(T + l * kWyB + p), ys[l][lane], acc);   // T upper: l <= p
    if (k < ldy) Y16[(int64_t)p * ldy + k] = k < nc ? (PREC == TLS_FP16 ? f64_to_f16_bits(round_uf(acc, TLS_FP16))
                                                                      : f64_to_bf16_bits(round_uf(acc, TLS_BF16)))
                                                  : (uint16_t)0;
  }
}

// R rows [c0, c1): the panel block from the chain's Gp (stride ldgp), the trailing part from W
// (final after the panel's WY update), signs as R25 (diag(R) >= 0)
__global__ void k_wy_copy_R(const double* __restrict__ Gp, int ldgp, const float* __restrict__ W, int64_t ldw,
                            const double* __restrict__ scal, int c0, int c1, int n, int trailing, double* __restrict__ G) {
  const int j = c0 + blockIdx.x;
  if (j >= c1) return;
  const double sg = scal[4 * j] < 0.0 ? -1.0 : 1.0;
  for (int k = j + threadIdx.x; k < n; k += blockDim.x) {
    if (k < c1) G[(int64_t)j * n + k] = Gp[(int64_t)j * ldgp + k];
    else if (trailing) G[(int64_t)j * n + k] = sg * (double)W[(int64_t)j * ldw + k];
  }
}

size_t qr_wy_bytes(int64_t m, int n) {
  const int64_t ld16 = (n + 63) / 64 * 64, ldv = (m + 63) / 64 * 64;
  return (size_t)m * ld16 * 2 + (size_t)m * kWyB * 2 + (size_t)kWyB * ldv * 2 + (size_t)n * n * 8 +
         (size_t)kWyB * kWyB * 8 * 2 + (size_t)kWyB * ld16 * 8 + (size_t)kWyB * ld16 * 2 + tc_atb_ws_bytes(n) +
         (size_t)n * 8 * 5 + 16 * 256;
}

// the panel passes cover <= kWyB = 128 columns: one 4-column group per thread, 16 one-warp teams
// per CTA (512 threads), 8 rows per team in flight (qr_update_v4)
constexpr int kPanelCPT = 4;

template <int CPT, int PREC>
int qr_blocked_t(const DenseView& A, const double* dinv, float* W, double* partP, double* wT, double* scal,
                 int* qflags, double* G, char* wy, cudaStream_t st, int* launches) {
  const int n = A.n;
  const int64_t m = A.m;
  const int RB = qr_rows_per_cta(m, n);
  const int nb = (int)((m + RB - 1) / RB);
  const int ldw = qr_ldw(n, PREC);
  const int64_t ld16 = (n + 63) / 64 * 64, ldv = (m + 63) / 64 * 64;
  // carve the WY buffers
  char* p = wy;
  auto take = [&](size_t bytes) { char* r = p; p += (bytes + 255) & ~(size_t)255; return r; };
  uint16_t* W16 = reinterpret_cast<uint16_t*>(take((size_t)m * ld16 * 2));
  uint16_t* V16 = reinterpret_cast<uint16_t*>(take((size_t)m * kWyB * 2));
  uint16_t* Vt16 = reinterpret_cast<uint16_t*>(take((size_t)kWyB * ldv * 2));
  double* Gp = reinterpret_cast<double*>(take((size_t)n * n * 8));
  double* VtV = reinterpret_cast<double*>(take((size_t)kWyB * kWyB * 8));
  double* T = reinterpret_cast<double*>(take((size_t)kWyB * kWyB * 8));
  double* Y1 = reinterpret_cast<double*>(take((size_t)kWyB * ld16 * 8));
  uint16_t* Y16 = reinterpret_cast<uint16_t*>(take((size_t)kWyB * ld16 * 2));
  const size_t atb_bytes = tc_atb_ws_bytes(n);
  double* atb = reinterpret_cast<double*>(take(atb_bytes));
  double* zw = reinterpret_cast<double*>(take((size_t)n * 8));
  double* zs = reinterpret_cast<double*>(take((size_t)n * 8 * 4));
  TLS_CUDA_TRY(cudaMemsetAsync(zw, 0, (size_t)n * 8, st));
  TLS_CUDA_TRY(cudaMemsetAsync(zs, 0, (size_t)n * 32, st));
  int nl = 0;
  // LOAD: W = fl_uf(A D^-1) and the partials of column 0; its 16-bit twin
  int rc = qr_step_launch<float, true, CPT, PREC>(W, A, ldw, dinv, -1, RB, 0, nb, nullptr, nullptr, partP, Gp, qflags, st);
  if (rc) return rc;
  k_f32_to_16<PREC><<<(int)std::min<int64_t>(m, 4096), 256, 0, st>>>(W, ldw, W16, ld16, m, n);
  nl += 2;
  for (int c0 = 0; c0 < n; c0 += kWyB) {
    const int c1 = std::min(n, c0 + kWyB);
    DenseView Ap = A;
    Ap.n = c1;                                        // the chain works on the panel's columns only
    if (c0 > 0) {
      // the previous panel's R rows: its block from Gp (stride c0, its end), its trailing part from W
      k_wy_copy_R<<<kWyB, 256, 0, st>>>(Gp, c0, W, ldw, scal, c0 - kWyB, c0, n, 1, G);
      // partials of column c0 over the panel (the pass of column c0 - 1 with w = 0: no change)
      const int j = c0 - 1;
      const int bs = j / RB;
      rc = qr_step_launch<float, false, kPanelCPT, PREC>(W, Ap, ldw, dinv, j, RB, bs, nb - bs, zw, zs, partP, Gp, qflags,
                                                          st);
      if (rc) return rc;
      nl += 2;
    }
    for (int j = c0; j < c1; ++j) {
      const int b0 = (j > 0 ? j - 1 : 0) / RB;
      const int nf = (c1 - j - 1 + 31) / 32;
      rc = launch_pdl(k_qr_fin<float, PREC>, nf > 0 ? nf : 1, kQrThreads, 0, st, (const float*)W, c1, ldw, j, b0, nb,
                      (const double*)partP, wT, scal, Gp, qflags, 0, j == 0 ? n : c1);
      if (rc) return rc;
      ++nl;
      if (j + 1 < c1) {
        const int bs = j / RB;
        rc = qr_step_launch<float, false, kPanelCPT, PREC>(W, Ap, ldw, dinv, j, RB, bs, nb - bs, wT, scal, partP, Gp,
                                                            qflags, st);
        if (rc) return rc;
        ++nl;
      }
    }
    if (c1 == n) {
      k_wy_copy_R<<<kWyB, 256, 0, st>>>(Gp, c1, W, ldw, scal, c0, c1, n, 0, G);
      ++nl;
      break;
    }
    const int64_t mr = m - c0;
    k_wy_extract<PREC><<<(int)std::min<int64_t>(mr, 8192), kWyB, 0, st>>>(W, ldw, scal, c0, kWyB, m, V16);
    k_wy_transpose<<<dim3((unsigned)((ldv - c0 + 31) / 32), kWyB / 32), dim3(32, 8), 0, st>>>(V16, mr, Vt16, ldv);
    TLS_LAUNCH_CHECK();
    rc = launch_tc_atb(PREC, V16, kWyB, V16, kWyB, mr, kWyB, VtV, kWyB, atb, atb_bytes, st);
    if (!rc) rc = launch_tc_atb(PREC, V16, kWyB, W16 + (int64_t)c0 * ld16 + c1, ld16, mr, n - c1, Y1, (int)ld16, atb,
                                atb_bytes, st);
    if (rc) return rc;
    const size_t tsm = (size_t)kWyB * (kWyB + 2) * 8;
    static bool attr = false;
    if (!attr) {
      TLS_CUDA_TRY(cudaFuncSetAttribute(k_wy_T, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
      attr = true;
    }
    k_wy_T<<<1, kWyB, tsm, st>>>(VtV, scal, c0, kWyB, T);
    k_wy_Y<PREC><<<(unsigned)((n - c1 + 31) / 32), 256, 0, st>>>(T, Y1, ld16, n - c1, Y16, ld16);
    TLS_LAUNCH_CHECK();
    rc = launch_qr_wy_update(PREC, Vt16, ldv, Y16, ld16, W, W16, ldw, ld16, c0, c1, m, n, st);
    if (rc) return rc;
    nl += 10;   // extract, transpose, 2 x (atb + reduce + memset), T, Y, update
  }
  TLS_LAUNCH_CHECK();
  if (launches) *launches += nl;
  return 0;
}

int launch_qr_blocked(const DenseView& A, int u_f, const double* dinv, void* Wbuf, double* partP, double* wT,
                      double* scal, int* qflags, double* G, void* wy, cudaStream_t st, int* launches) {
  if (u_f != TLS_FP16 && u_f != TLS_BF16) {
    set_error("blocked QR: u_f must be fp16 or bf16 (the tensor-core formats)");
    return TLS_ERR_UNSUPPORTED;
  }
  if (A.n > 8 * kQrThreads) { set_error("blocked QR: n > %d", 8 * kQrThreads); return TLS_ERR_UNSUPPORTED; }
  float* W = static_cast<float*>(Wbuf);
  char* wyb = static_cast<char*>(wy);
  if (u_f == TLS_FP16) return qr_blocked_t<8, TLS_FP16>(A, dinv, W, partP, wT, scal, qflags, G, wyb, st, launches);
  return qr_blocked_t<8, TLS_BF16>(A, dinv, W, partP, wT, scal, qflags, G, wyb, st, launches);
}
}  // namespace tls
