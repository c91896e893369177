// k_csr.cu — the sparse (CSR) hot path of BASELINE.json configs[2] (cfg3):
// SURVEY §8(a) rows a1 (column statistics), a2 (u_f Gram), a5/a7 (residual and
// operator passes) for A given as CSR (include/tlsrqi.h, TLS_CSR).
//
//   colstats  c_j = max_i |a_ij| (order-free integer max on the fp64 bit
//             pattern) and ||A||_F^2 (fixed per-CTA partials, fixed-order sum)
//   Gram      G = A^^T A^, A^ = fl_uf(A D^{-1}).  For
//             u_f = fp16 every A^ value is an integer multiple of 2^-24 with
//             |A^| < 2, so each product is an exact integer multiple of 2^-48
//             below 2^50 in magnitude; products are accumulated EXACTLY in a
//             two-limb fixed-point sum (int64 atomics: order-free, deterministic)
//             and G is that exact sum rounded once to fp64 (reading R19).  For
//             bf16/fp32/fp64 the (exact, for bf16/fp32) products are summed with
//             fp64 atomics (order not fixed; last-bit effects only).
//   passes    row phase: t_i = a_i . q_r (8 lanes per row), tau or (rho, gamma)
//             per-CTA partials; column phase over a CSC copy: v_j = sum_i a_ij t_i
//             (one warp per column, fixed order).  A is read once per phase.
//   CSC       built once per solve, deterministic: per-chunk column counts, a
//             column-wise prefix over chunks, and an in-order fill per chunk
//             (ascending rows within every column).
#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

constexpr int kCsrChunks = 592;        // row chunks of the CSC build (4 x 148)
constexpr int kCsrRowCTAs = 4 * 148;   // CTAs of the row phase
constexpr int kCsrT = 256;

__device__ __forceinline__ bool csr_active(const int* active) {
  return active == nullptr || (active[0] | active[1]) != 0;
}

// ----------------------------------------------------------------------------- a1
__global__ void __launch_bounds__(kCsrT) k_csr_colstats(CsrView A, double* __restrict__ colmax,
                                                        double* __restrict__ partial) {
  __shared__ double red[32];
  const int64_t e0 = A.nnz * blockIdx.x / gridDim.x, e1 = A.nnz * (blockIdx.x + 1) / gridDim.x;
  double s = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const double v = A.vals[e];
    const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(v));
    atomicMax(reinterpret_cast<unsigned long long*>(colmax) + A.colidx[e], bits);
    s = fma(v, v, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// colstats[n] = sum of the partials (fixed order); colstats[n+1 .. 2n) = 0
__global__ void __launch_bounds__(kCsrT) k_csr_colstats_fin(const double* __restrict__ partial, int G, int n,
                                                            double* __restrict__ colstats) {
  __shared__ double red[32];
  double s = 0.0;
  for (int g = threadIdx.x; g < G; g += blockDim.x) s += partial[g];
  s = block_sum(s, red);
  for (int j = threadIdx.x; j < n; j += blockDim.x) colstats[n + j] = (j == 0) ? s : 0.0;
}

int launch_csr_colstats(const CsrView& A, double* colstats, double* partials, cudaStream_t st) {
  TLS_CUDA_TRY(cudaMemsetAsync(colstats, 0, (size_t)A.n * 8, st));
  const int G = kCsrRowCTAs;
  if (A.nnz > 0) {
    k_csr_colstats<<<G, kCsrT, 0, st>>>(A, colstats, partials);
    k_csr_colstats_fin<<<1, kCsrT, 0, st>>>(partials, G, A.n, colstats);
  } else {
    TLS_CUDA_TRY(cudaMemsetAsync(colstats + A.n, 0, (size_t)A.n * 8, st));
  }
  TLS_LAUNCH_CHECK();
  return 0;
}

// ----------------------------------------------------------------------------- a2
// one warp per row (grid-stride, any order: the sums are order-free)
__global__ void __launch_bounds__(kCsrT) k_csr_gram_f16(CsrView A, const double* __restrict__ dinv,
                                                        unsigned long long* __restrict__ S, int* __restrict__ range) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const size_t nn = (size_t)A.n * A.n;
  int bad = 0;
  for (int64_t i = wid; i < A.m; i += nw) {
    const int64_t r0 = A.rowptr[i], len = A.rowptr[i + 1] - r0;
    for (int64_t a = lane; a < len; a += 32) {
      const int ja = A.colidx[r0 + a];
      const double ha = round_rne<11, -14, 15>(A.vals[r0 + a] * dinv[ja]);
      if (!isfinite(ha)) bad = 1;
      const long long Ia = __double2ll_rn(ha * 0x1p24);        // exact: A^ in Z * 2^-24
      for (int64_t b = a; b < len; ++b) {
        const int jb = A.colidx[r0 + b];
        const double hb = round_rne<11, -14, 15>(A.vals[r0 + b] * dinv[jb]);
        const long long P = Ia * __double2ll_rn(hb * 0x1p24);   // |P| < 2^50, exact
        const int lo = ja < jb ? ja : jb, hi = ja < jb ? jb : ja;
        const size_t idx = (size_t)lo * A.n + hi;
        atomicAdd(&S[idx], (unsigned long long)(P >> 25));           // two's complement limbs
        atomicAdd(&S[nn + idx], (unsigned long long)(P & ((1ll << 25) - 1)));
      }
    }
  }
  if (bad) atomicExch(range, 1);
}

// G[j][k] = G[k][j] = (S_hi * 2^25 + S_lo) * 2^-48 rounded once (both limbs exact in fp64)
__global__ void k_csr_gram_f16_fin(const unsigned long long* __restrict__ S, int n, double* __restrict__ G) {
  const size_t nn = (size_t)n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < nn; e += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / n), k = (int)(e % n);
    if (k < j) continue;
    const double hi = (double)(long long)S[e] * 0x1p25;           // exact (|S_hi| < 2^53)
    const double lo = (double)(long long)S[nn + e];               // exact (< 2^53)
    const double g = (hi + lo) * 0x1p-48;                        // one rounding, exact scaling
    G[(size_t)j * n + k] = g;
    G[(size_t)k * n + j] = g;
  }
}

template <int PREC>
__global__ void __launch_bounds__(kCsrT) k_csr_gram_f64(CsrView A, const double* __restrict__ dinv,
                                                        double* __restrict__ G, int* __restrict__ range) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int bad = 0;
  for (int64_t i = wid; i < A.m; i += nw) {
    const int64_t r0 = A.rowptr[i], len = A.rowptr[i + 1] - r0;
    for (int64_t a = lane; a < len; a += 32) {
      const int ja = A.colidx[r0 + a];
      const double ha = round_uf(A.vals[r0 + a] * dinv[ja], PREC);
      if (!isfinite(ha)) bad = 1;
      for (int64_t b = a; b < len; ++b) {
        const int jb = A.colidx[r0 + b];
        const double hb = round_uf(A.vals[r0 + b] * dinv[jb], PREC);
        const int lo = ja < jb ? ja : jb, hi = ja < jb ? jb : ja;
        atomicAdd(&G[(size_t)lo * A.n + hi], ha * hb);
      }
    }
  }
  if (bad) atomicExch(range, 1);
}

__global__ void k_mirror_upper(double* __restrict__ G, int n) {
  const size_t nn = (size_t)n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < nn; e += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / n), k = (int)(e % n);
    if (k > j) G[(size_t)k * n + j] = G[e];
  }
}

size_t csr_gram_ws_bytes(int n) { return 2 * (size_t)n * n * 8; }

int launch_csr_gram(const CsrView& A, int u_f, const double* dinv, double* G, void* ws, size_t ws_bytes,
                    int* range_flag, cudaStream_t st, int* launches, bool fixed_point_out) {
  const int n = A.n;
  const int grid = 8 * num_sms();
  int nl = 0;
  if (u_f == TLS_FP16) {
    if (ws_bytes < csr_gram_ws_bytes(n)) { set_error("csr gram: workspace too small"); return TLS_ERR_WORKSPACE; }
    unsigned long long* S = static_cast<unsigned long long*>(ws);
    TLS_CUDA_TRY(cudaMemsetAsync(S, 0, csr_gram_ws_bytes(n), st));
    if (A.m > 0) { k_csr_gram_f16<<<grid, kCsrT, 0, st>>>(A, dinv, S, range_flag); ++nl; }
    if (!fixed_point_out) { k_csr_gram_f16_fin<<<grid, 256, 0, st>>>(S, n, G); ++nl; }
  } else {
    TLS_CUDA_TRY(cudaMemsetAsync(G, 0, (size_t)n * n * 8, st));
    if (A.m > 0) {
      switch (u_f) {
        case TLS_BF16: k_csr_gram_f64<TLS_BF16><<<grid, kCsrT, 0, st>>>(A, dinv, G, range_flag); break;
        case TLS_FP32: k_csr_gram_f64<TLS_FP32><<<grid, kCsrT, 0, st>>>(A, dinv, G, range_flag); break;
        default: k_csr_gram_f64<TLS_FP64><<<grid, kCsrT, 0, st>>>(A, dinv, G, range_flag); break;
      }
      ++nl;
    }
    k_mirror_upper<<<grid, 256, 0, st>>>(G, n);
    ++nl;
  }
  TLS_LAUNCH_CHECK();
  if (launches) *launches += nl;
  return 0;
}

int launch_csr_gram_fin(const void* ws, int n, double* G, cudaStream_t st) {
  k_csr_gram_f16_fin<<<8 * num_sms(), 256, 0, st>>>(static_cast<const unsigned long long*>(ws), n, G);
  TLS_LAUNCH_CHECK();
  return 0;
}

// ----------------------------------------------------------------------------- CSC build
size_t csc_scratch_bytes(int64_t m, int n) {
  (void)m;
  return ((size_t)kCsrChunks * n + n) * sizeof(int);
}

__global__ void __launch_bounds__(kCsrT) k_csc_count(CsrView A, int* __restrict__ cnt) {
  extern __shared__ int hist[];
  const int ch = blockIdx.x;
  for (int j = threadIdx.x; j < A.n; j += blockDim.x) hist[j] = 0;
  __syncthreads();
  const int64_t i0 = A.m * ch / gridDim.x, i1 = A.m * (ch + 1) / gridDim.x;
  const int64_t e0 = A.rowptr[i0], e1 = A.rowptr[i1];
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&hist[A.colidx[e]], 1);
  __syncthreads();
  for (int j = threadIdx.x; j < A.n; j += blockDim.x) cnt[(size_t)ch * A.n + j] = hist[j];
}

// per column: running prefix over chunks (in place) and the column total
// (16 chunk counts are loaded before they are scanned: one L2 round trip per 16 chunks
// instead of one per chunk; 174 -> 39 us on cfg3)
__global__ void k_csc_prefix(int* __restrict__ cnt, int nch, int n, int* __restrict__ colcnt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int run = 0;
  int ch = 0;
  for (; ch + 16 <= nch; ch += 16) {
    int c[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) c[k] = cnt[(size_t)(ch + k) * n + j];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      cnt[(size_t)(ch + k) * n + j] = run;
      run += c[k];
    }
  }
  for (; ch < nch; ++ch) {
    const int c = cnt[(size_t)ch * n + j];
    cnt[(size_t)ch * n + j] = run;
    run += c;
  }
  colcnt[j] = run;
}

// colptr = exclusive scan of colcnt (one CTA of 1024 threads, fixed order)
__global__ void __launch_bounds__(1024) k_csc_colptr(const int* __restrict__ colcnt, int n, int64_t* __restrict__ colptr) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int per = (n + 1023) / 1024;
  const int j0 = t * per, j1 = min(n, j0 + per);
  int64_t s = 0;
  for (int j = j0; j < j1; ++j) s += colcnt[j];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {       // inclusive Hillis-Steele scan of the thread totals
    const int64_t v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = t ? part[t - 1] : 0;
  for (int j = j0; j < j1; ++j) {
    colptr[j] = run;
    run += colcnt[j];
  }
  if (t == 1023) colptr[n] = part[1023];
}

// one warp per chunk: rows in ascending order, lanes over a row's entries (distinct columns),
// so every column receives its entries in row order (deterministic CSC).  The chunk's row
// pointers are staged in shared memory and the next row's (column, value) pairs are loaded
// while the current row is scattered (322 -> 169 us on cfg3; a four-row-deep version
// measured 214 us); rows longer than 32 take the plain loop.
__global__ void __launch_bounds__(32) k_csc_fill(CsrView A, const int* __restrict__ rel, const int64_t* __restrict__ colptr,
                                                 CscView C, int rp_cap) {
  extern __shared__ int64_t off[];          // [n] column cursors, then [rp_cap] row pointers
  int64_t* rp = off + A.n;
  const int ch = blockIdx.x, lane = threadIdx.x;
  for (int j = lane; j < A.n; j += 32) off[j] = colptr[j] + rel[(size_t)ch * A.n + j];
  const int64_t i0 = A.m * ch / gridDim.x, i1 = A.m * (ch + 1) / gridDim.x;
  const int nr = (int)(i1 - i0);
  const bool staged = nr + 1 <= rp_cap;
  if (staged)
    for (int k = lane; k <= nr; k += 32) rp[k] = A.rowptr[i0 + k];
  __syncwarp();
  auto rowp = [&](int k) -> int64_t { return staged ? rp[k] : A.rowptr[i0 + k]; };
  int64_t r0 = nr > 0 ? rowp(0) : 0, r1 = nr > 0 ? rowp(1) : 0;
  int jc = 0;
  double vc = 0.0;
  if (nr > 0 && r0 + lane < r1 && r1 - r0 <= 32) { jc = A.colidx[r0 + lane]; vc = A.vals[r0 + lane]; }
  for (int k = 0; k < nr; ++k) {
    const int64_t i = i0 + k;
    const int64_t r2 = k + 1 < nr ? rowp(k + 2) : r1;
    int jn = 0;
    double vn = 0.0;
    if (k + 1 < nr && r1 + lane < r2 && r2 - r1 <= 32) { jn = A.colidx[r1 + lane]; vn = A.vals[r1 + lane]; }
    if (r1 - r0 <= 32) {
      if (r0 + lane < r1) {
        const int64_t pos = off[jc]++;
        C.rowidx[pos] = (int32_t)i;
        C.vals[pos] = vc;
      }
    } else {
      for (int64_t e = r0 + lane; e < r1; e += 32) {
        const int j = A.colidx[e];
        const int64_t pos = off[j]++;
        C.rowidx[pos] = (int32_t)i;
        C.vals[pos] = A.vals[e];
      }
    }
    __syncwarp();
    jc = jn;
    vc = vn;
    r0 = r1;
    r1 = r2;
  }
}

int launch_csc_build(const CsrView& A, CscView C, void* scratch, cudaStream_t st, int* launches) {
  int* cnt = static_cast<int*>(scratch);
  int* colcnt = cnt + (size_t)kCsrChunks * A.n;
  const size_t hsm = (size_t)A.n * sizeof(int);
  // row pointers of a chunk staged when they fit next to the column cursors (48 KB total)
  const int64_t chunk_rows = (A.m + kCsrChunks - 1) / kCsrChunks + 1;
  int rp_cap = (int)(((int64_t)48 * 1024 - (int64_t)A.n * 8) / 8);
  if (rp_cap < 0) rp_cap = 0;
  if (rp_cap > chunk_rows) rp_cap = (int)chunk_rows;
  const size_t osm = ((size_t)A.n + (size_t)rp_cap) * sizeof(int64_t);
  static size_t attr = 0;
  if (osm > 48 * 1024 && attr < osm) {
    TLS_CUDA_TRY(cudaFuncSetAttribute(k_csc_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)osm));
    attr = osm;
  }
  k_csc_count<<<kCsrChunks, kCsrT, hsm, st>>>(A, cnt);
  k_csc_prefix<<<(A.n + 255) / 256, 256, 0, st>>>(cnt, kCsrChunks, A.n, colcnt);
  k_csc_colptr<<<1, 1024, 0, st>>>(colcnt, A.n, C.colptr);
  k_csc_fill<<<kCsrChunks, 32, osm, st>>>(A, cnt, C.colptr, C, rp_cap);
  TLS_LAUNCH_CHECK();
  if (launches) *launches += 4;
  return 0;
}

// ----------------------------------------------------------------------------- a5 / a7
// Row phase: 8 lanes per row.  MODE PASS_OPERATOR: t_r = A q_r, s_r += t_r^2;
// PASS_RESIDUAL: t = b - A x, s0 += t^2, s1 += b t.  Partials: [grid][2].
template <int NRHS, int MODE>
__global__ void __launch_bounds__(kCsrT) k_csr_rows(CsrView A, const double* __restrict__ q,
                                                    const double* __restrict__ b, double* __restrict__ tbuf,
                                                    double* __restrict__ partials, const int* __restrict__ active) {
  if (!csr_active(active)) return;
  __shared__ double red[32];
  const int sub = threadIdx.x & 7;
  // the warp walks groups of 4 consecutive rows together (warp-uniform trip count:
  // the octet shuffles below need every lane of the warp)
  const int64_t w0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 4;
  const int64_t wstride = (((int64_t)gridDim.x * blockDim.x) >> 5) * 4;
  double s0 = 0.0, s1 = 0.0;
  // two row groups per trip (base, base + wstride), their loads interleaved: the chain rowptr ->
  // colidx / vals -> q of the second group overlaps the first's (round 2 continued); every row's
  // products and the s0 / s1 accumulation keep their order (group k before group k + 1)
  for (int64_t base = w0; base < A.m; base += 2 * wstride) {
    int64_t ii[2], r0[2], r1[2];
    bool valid[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ii[h] = base + h * wstride + ((threadIdx.x & 31) >> 3);
      valid[h] = ii[h] < A.m;
      r0[h] = valid[h] ? A.rowptr[ii[h]] : 0;
      r1[h] = valid[h] ? A.rowptr[ii[h] + 1] : 0;
    }
    double t[2][NRHS];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int r = 0; r < NRHS; ++r) t[h][r] = 0.0;
    // the first two nonzeros of each of the octet's rows, both groups, loads first
    {
      double a[2][2];
      int jj[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int64_t e = r0[h] + sub + 8 * k;
          const bool ok = e < r1[h];
          a[h][k] = ok ? A.vals[e] : 0.0;
          jj[h][k] = ok ? A.colidx[e] : -1;
        }
      double qq[2][2][NRHS];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int r = 0; r < NRHS; ++r) qq[h][k][r] = jj[h][k] >= 0 ? q[(size_t)r * A.n + jj[h][k]] : 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (jj[h][k] >= 0)
#pragma unroll
            for (int r = 0; r < NRHS; ++r) t[h][r] = fma(a[h][k], qq[h][k][r], t[h][r]);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
      for (int64_t e = r0[h] + sub + 16; e < r1[h]; e += 8) {     // longer rows: the rest in order
        const double a = A.vals[e];
        const int j = A.colidx[e];
#pragma unroll
        for (int r = 0; r < NRHS; ++r) t[h][r] = fma(a, q[(size_t)r * A.n + j], t[h][r]);
      }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
        t[h][r] += __shfl_xor_sync(0xffffffffu, t[h][r], 4);
        t[h][r] += __shfl_xor_sync(0xffffffffu, t[h][r], 2);
        t[h][r] += __shfl_xor_sync(0xffffffffu, t[h][r], 1);
      }
      const int64_t i = ii[h];
      if (sub == 0 && valid[h]) {
        if (MODE == PASS_RESIDUAL) {
          const double bi = b[i];
          const double ti = bi - t[h][0];
          tbuf[i] = ti;
          s0 = fma(ti, ti, s0);
          s1 = fma(bi, ti, s1);
        } else {
#pragma unroll
          for (int r = 0; r < NRHS; ++r) tbuf[(size_t)r * A.m + i] = t[h][r];
          s0 = fma(t[h][0], t[h][0], s0);
          if (NRHS == 2) s1 = fma(t[h][NRHS - 1], t[h][NRHS - 1], s1);
        }
      }
    }
  }
  s0 = block_sum(s0, red);
  s1 = block_sum(s1, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = s0;
    partials[2 * blockIdx.x + 1] = s1;
  }
}

// Column phase: one warp per column j, v_r[j] = sum_{e in col j} a_e t_r[row_e] (fixed
// order); the last CTA sums the scalar partials of the row phase (fixed order).
template <int NRHS>
__global__ void __launch_bounds__(kCsrT) k_csr_cols(int64_t m, int n, CscView C, const double* __restrict__ tbuf,
                                                    const double* __restrict__ partials, int G, double* __restrict__ out,
                                                    const int* __restrict__ active) {
  if (!csr_active(active)) return;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == gridDim.x - 1) {
    __shared__ double red[32];
    double s0 = 0.0, s1 = 0.0;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
      s0 += partials[2 * g];
      s1 += partials[2 * g + 1];
    }
    s0 = block_sum(s0, red);
    s1 = block_sum(s1, red);
    if (threadIdx.x == 0) {
      out[(size_t)NRHS * n] = s0;
      out[(size_t)NRHS * n + 1] = s1;
    }
    return;
  }
  const int j = blockIdx.x * (kCsrT / 32) + (threadIdx.x >> 5);
  if (j >= n) return;
  const int64_t e0 = C.colptr[j], e1 = C.colptr[j + 1];
  double v[NRHS];
#pragma unroll
  for (int r = 0; r < NRHS; ++r) v[r] = 0.0;
  int64_t e = e0 + lane;
  for (; e + 224 < e1; e += 256) {     // 8 independent gathers in flight per lane (round 2
    int rw[8];                         // continued: 4 before; the same order, the same bits)
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { rw[u] = C.rowidx[e + 32 * u]; a[u] = C.vals[e + 32 * u]; }
    double tv[8][NRHS];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int r = 0; r < NRHS; ++r) tv[u][r] = tbuf[(size_t)r * m + rw[u]];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int r = 0; r < NRHS; ++r) v[r] = fma(a[u], tv[u][r], v[r]);
  }
  for (; e + 96 < e1; e += 128) {      // 4 independent gathers in flight per lane
    int rw[4];
    double a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { rw[u] = C.rowidx[e + 32 * u]; a[u] = C.vals[e + 32 * u]; }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < NRHS; ++r) v[r] = fma(a[u], tbuf[(size_t)r * m + rw[u]], v[r]);
  }
  for (; e < e1; e += 32) {
    const int rw = C.rowidx[e];
    const double a = C.vals[e];
#pragma unroll
    for (int r = 0; r < NRHS; ++r) v[r] = fma(a, tbuf[(size_t)r * m + rw], v[r]);
  }
#pragma unroll
  for (int r = 0; r < NRHS; ++r) {
    const double s = warp_sum(v[r]);
    if (lane == 0) out[(size_t)r * n + j] = s;
  }
}

size_t csr_pass_partials_doubles() { return 2 * (size_t)kCsrRowCTAs; }

int launch_csr_pass(const CsrView& A, const CscView& C, int mode, int nrhs, const double* q, const double* b,
                    double* tbuf, double* partials, double* out, const int* active, cudaStream_t st) {
  const int G = kCsrRowCTAs;
  const int gc = (A.n + kCsrT / 32 - 1) / (kCsrT / 32) + 1;
  if (mode == PASS_RESIDUAL) {
    k_csr_rows<1, PASS_RESIDUAL><<<G, kCsrT, 0, st>>>(A, q, b, tbuf, partials, active);
    k_csr_cols<1><<<gc, kCsrT, 0, st>>>(A.m, A.n, C, tbuf, partials, G, out, active);
  } else if (nrhs == 1) {
    k_csr_rows<1, PASS_OPERATOR><<<G, kCsrT, 0, st>>>(A, q, b, tbuf, partials, active);
    k_csr_cols<1><<<gc, kCsrT, 0, st>>>(A.m, A.n, C, tbuf, partials, G, out, active);
  } else {
    k_csr_rows<2, PASS_OPERATOR><<<G, kCsrT, 0, st>>>(A, q, b, tbuf, partials, active);
    k_csr_cols<2><<<gc, kCsrT, 0, st>>>(A.m, A.n, C, tbuf, partials, G, out, active);
  }
  TLS_LAUNCH_CHECK();
  return 0;
}

}  // namespace tls
