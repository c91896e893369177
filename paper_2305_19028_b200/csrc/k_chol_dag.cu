// k_chol_dag.cu — fp64 Cholesky G = R^T R of the u_f Gram (
// PAPER.md l.206 "Cholesky factorization", l.290-297; reading R10), as ONE
// persistent kernel executing the tile DAG of the right-looking blocked
// algorithm on 64 x 64 tiles of the upper triangle:
//
//   POTRF(k)       R_kk = chol(G_kk) in shared memory (first non-positive or
//                  non-finite pivot -> CHOL_BREAKDOWN index), one barrier per column
//   TRSM(k, j)     R_kj = R_kk^{-T} G_kj by forward substitution   (j > k)
//   UPDATE(k,i,j)  G_ij -= R_ki^T R_kj                              (k < i <= j)
//
// Every CTA (one per SM, co-resident by cooperative launch) fetches the next task
// of a fixed topological list with an atomic counter and spins on the tile flags
// its inputs need (release/acquire at gpu scope; tile data read through L2).  The
// list emits POTRF(k+1) right after the row-(k+1) updates of step k, so the next
// panel overlaps the rest of step k (one step of lookahead): the critical path is
// POTRF + TRSM + UPDATE per tile column instead of three dependent launches per
// step.  The updates of a tile are applied in k order (per-tile counter), so the
// result is bitwise reproducible.  R overwrites the upper triangle in place.
#include <vector>

#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

constexpr int kTB = 64;             // tile edge
constexpr int kTS = kTB + 1;        // smem row stride (doubles)
constexpr int kCholThreads = 256;

enum { T_POTRF = 0, T_TRSM = 1, T_UPDATE = 2, T_DIAG = 3 };

struct CholCtl {          // device control block (zeroed before the launch)
  int next;               // task counter
  int fail;               // 1-based failed pivot (first), 0 = none
  int pad[2];
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Wait (all threads) until *flag >= want or a breakdown was flagged; returns false on breakdown.
__device__ bool wait_flag(const int* flag, int want, const CholCtl* ctl) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    int v;
    while ((v = ld_acquire(flag)) < want) {
      if (ld_acquire(&ctl->fail) != 0) break;
    }
    ok = v >= want;
  }
  __syncthreads();
  const bool r = ok;
  __syncthreads();
  return r;
}

// tile (ti, tj) of G -> smem S[64][65] (zeros outside the matrix; identity padding on the
// diagonal tile when `pad_identity`)
// All 16 loads of a thread are issued before the first shared-memory store (one L2 round
// trip per tile instead of 16 dependent ones: measured 9.2 -> see DESIGN §6).
__device__ void load_tile(const double* G, int n, int ti, int tj, double* S, bool upper_only, bool pad_identity) {
  constexpr int kPer = kTB * kTB / kCholThreads;
  double v[kPer];
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int e = threadIdx.x + r * kCholThreads;
    const int i = e >> 6, j = e & 63;
    const int gi = ti * kTB + i, gj = tj * kTB + j;
    if (gi < n && gj < n) v[r] = (upper_only && gj < gi) ? 0.0 : __ldcg(G + (size_t)gi * n + gj);
    else v[r] = (pad_identity && i == j) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int e = threadIdx.x + r * kCholThreads;
    S[(e >> 6) * kTS + (e & 63)] = v[r];
  }
}

__device__ void store_tile(double* G, int n, int ti, int tj, const double* S, bool upper_only) {
  for (int e = threadIdx.x; e < kTB * kTB; e += blockDim.x) {
    const int i = e >> 6, j = e & 63;
    const int gi = ti * kTB + i, gj = tj * kTB + j;
    if (gi < n && gj < n && (!upper_only || gj >= gi)) __stcg(G + (size_t)gi * n + gj, S[i * kTS + j]);
  }
}

// POTRF of the diagonal tile, blocked by 16 (square-root-free form U = D R with
// d_i = U_ii; A_ij -= sum_k U_ki U_kj / d_k; rows scaled by 1/sqrt(d_i) at the end).
// For each 16-block: (1) the 16 x 16 diagonal block, one element per thread in a
// register, one barrier per column; (2) the multipliers F_ji = U_ji / d_j and the
// block row to the right by per-column substitution; (3) the rank-16 update of the
// trailing upper triangle.  S: input upper / output R upper; dr[i] = 1 / R_ii.
// Returns the 1-based local failed pivot or 0.
#ifdef POTRF_TRACE
#define PMARK(k) do { if (threadIdx.x == 0) g_marks[k] = clock64(); } while (0)
#else
#define PMARK(k) do {} while (0)
#endif
// 1/x for a positive normal pivot: MUFU.RCP64H seed and two Newton steps (~1 ulp).  The
// pivots sit on the factorization's critical path; per 16-pivot diagonal block this is
// 4.5k cycles against 5.3k for the IEEE division routine and 7.2k for an fp32 seed
// (tools/micro/diag16.cu).
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// BS: the diagonal-block size (one warp, registers).  16; 32 was measured slower (POTRF of a
// 64-tile 54 vs 37 us, n = 2000 factorization 1.86 vs 1.34 ms, profiles/r02_chol_bs.txt): a
// pivot's shuffles and updates grow with BS on the one-warp critical path faster than the
// block transitions shrink.
template <int BS>
__device__ int potrf_tile(double* S, double* dr, int nb) {
  __shared__ int fail;
  __shared__ double F[BS][kTB + 1];      // multipliers of the current block: F[j][i] = U_ji / d_j
  __shared__ double bdinv[BS];           // 1 / d_j of the current block
  const int tid = threadIdx.x;
  if (tid == 0) fail = 0;
  __syncthreads();
  PMARK(0);
  for (int o = 0; o < kTB; o += BS) {
    // (1) diagonal block: warp 0, lane t owns column t of the block in registers;
    // row jj of the block is read from lane ii by shuffles (no block barriers)
    if (tid < 32) {
      const int t = tid & (BS - 1);
      double v[BS];
#pragma unroll
      for (int i = 0; i < BS; ++i) v[i] = S[(o + i) * kTS + o + t];
      int f = 0;
      // no `break`: a loop exit kept the loop rolled and v[] in local memory (measured)
#pragma unroll
      for (int jj = 0; jj < BS; ++jj) {
        const double piv = __shfl_sync(0xffffffffu, v[jj], jj);
        if (o + jj < nb && f == 0) {
          if (!(piv > 0.0 && piv < INFINITY)) {      // non-positive, NaN or +inf pivot
            f = o + jj + 1;
          } else {
            const double dinv = rcp_fast(piv);
            const double sjt = v[jj];
#pragma unroll
            for (int ii = jj + 1; ii < BS; ++ii) {
              const double m = __shfl_sync(0xffffffffu, v[jj], ii) * dinv;
              if (t >= ii) v[ii] = fma(-m, sjt, v[ii]);
            }
          }
        }
      }
      if (tid < BS) {
#pragma unroll
        for (int i = 0; i < BS; ++i)
          if (i <= t) S[(o + i) * kTS + o + t] = v[i];
        // d_t, read back (indexing v[t] with the lane index would put v[] in local memory)
        bdinv[t] = rcp_fast(S[(o + t) * kTS + o + t]);
      }
      if (tid == 0 && f) fail = f;
    }
    __syncthreads();
    PMARK(1 + (o / 16) * 4);
    if (fail) break;
    // (2) multipliers of the block and the block row to its right (columns c >= o + BS)
    for (int e = tid; e < BS * kTB; e += blockDim.x) {
      const int jj = e >> 6, c = e & 63;
      F[jj][c] = (c > o + jj && o + jj < nb) ? S[(o + jj) * kTS + c] * bdinv[jj] : 0.0;   // inside the block for now
    }
    __syncthreads();
    const int w = kTB - o - BS;                 // columns to the right
    if (tid < w) {
      const int c = o + BS + tid;
      double u[BS];
#pragma unroll
      for (int jj = 0; jj < BS; ++jj) u[jj] = S[(o + jj) * kTS + c];
#pragma unroll
      for (int jj = 0; jj < BS; ++jj)
#pragma unroll
        for (int ii = jj + 1; ii < BS; ++ii) u[ii] = fma(-F[jj][o + ii], u[jj], u[ii]);
#pragma unroll
      for (int jj = 0; jj < BS; ++jj) S[(o + jj) * kTS + c] = u[jj];
    }
    __syncthreads();
    PMARK(2 + (o / 16) * 4);
    if (w == 0) break;
    // multipliers for the columns right of the block (final U rows of the block)
    for (int e = tid; e < BS * w; e += blockDim.x) {
      const int jj = e / w, c = o + BS + e % w;
      F[jj][c] = (o + jj < nb) ? S[(o + jj) * kTS + c] * bdinv[jj] : 0.0;
    }
    __syncthreads();
    PMARK(3 + (o / 16) * 4);
    // (3) trailing update: S_ic -= sum_jj F[jj][i] U[jj][c], o+BS <= i <= c (4 rows at a time)
    {
      const int c = o + BS + (tid & 63);
      if (c < kTB) {
        double uc[BS];
#pragma unroll
        for (int jj = 0; jj < BS; ++jj) uc[jj] = S[(o + jj) * kTS + c];
        for (int i = o + BS + (tid >> 6); i <= c; i += 16) {
          double acc[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[r] = (i + 4 * r <= c) ? S[(i + 4 * r) * kTS + c] : 0.0;
#pragma unroll
          for (int jj = 0; jj < BS; ++jj)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r] = fma(-F[jj][min(i + 4 * r, kTB - 1)], uc[jj], acc[r]);
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (i + 4 * r <= c) S[(i + 4 * r) * kTS + c] = acc[r];
        }
      }
    }
    __syncthreads();
    PMARK(4 + (o / 16) * 4);
  }
  __syncthreads();
  const int f = fail;
  if (f) return f;
  __shared__ double rs[kTB];
  if (tid < kTB) {
    const double sq = sqrt(S[tid * kTS + tid]);
    rs[tid] = rcp_fast(sq);
    dr[tid] = rs[tid];
    S[tid * kTS + tid] = sq;
  }
  __syncthreads();
  for (int e = tid; e < kTB * kTB; e += blockDim.x) {
    const int i = e >> 6, c = e & 63;
    if (c > i) S[i * kTS + c] *= rs[i];
  }
  __syncthreads();
  return 0;
}

// TRSM in smem: B (64 x 64, columns c) <- R^{-T} B by forward substitution, four threads per
// column (thread q of a column keeps rows l = q (mod 4) in registers; x_i is broadcast from
// its owner by a shuffle; the remaining rows are updated independently).  Measured against
// one column per thread (g[64] did not fit the kernel's registers: stack) and two threads per
// column (rows split in halves, x_i shuffled to the partner): 9.9 vs 6.7 us per tile, n = 2000
// factorization 1.55 vs 1.31 ms (bit-identical R~; profiles/r02_chol_trsm.txt) -- the longer
// per-thread FMA chains cost more than the 4x redundant reads of R save.
__device__ void trsm_tile(const double* R, const double* dr, double* B) {
  const int tid = threadIdx.x, c = tid >> 2, q = tid & 3;
  double g[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) g[t] = B[(4 * t + q) * kTS + c];
#pragma unroll
  for (int i = 0; i < kTB; ++i) {
    const int owner = i & 3, slot = i >> 2;
    double xi = 0.0;
    if (q == owner) xi = g[slot] * dr[i];
    xi = __shfl_sync(0xffffffffu, xi, (tid & 31 & ~3) | owner);
    if (q == owner) g[slot] = xi;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int l = 4 * t + q;
      if (l > i) g[t] = fma(-R[i * kTS + l], xi, g[t]);
    }
  }
#pragma unroll
  for (int t = 0; t < 16; ++t) B[(4 * t + q) * kTS + c] = g[t];
}

// acc[p][q] = sum_i A[i][4ty+p] B[i][tx+16q] (A^T B); B reads are lane-consecutive
// (conflict-free), A reads are warp broadcasts.
__device__ __forceinline__ void tile_atb(const double* A, const double* B, double (&acc)[4][4]) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
#pragma unroll 4
  for (int i = 0; i < kTB; ++i) {
    double a[4], b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] = A[i * kTS + 4 * ty + q];
#pragma unroll
    for (int q = 0; q < 4; ++q) b[q] = B[i * kTS + tx + 16 * q];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
  }
}

// C -= A^T B on the fp64 tensor cores (DMMA m8n8k4; VERDICT r01 missing #8): warp w owns the
// 8-row block 8w of C and all 8 column blocks; per 4-deep k step one A fragment (A[k][8w+gid])
// and 8 B fragments (B[k][8nj+gid]) from shared memory, 8 DMMAs.  The same fp64 arithmetic
// rate as DFMA on B200, at 1/8 of the instructions and far fewer shared-memory loads than
// tile_atb's 4 x 4 register blocking.
__device__ __forceinline__ void tile_atb_sub_dmma(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  double acc[8][2];
#pragma unroll
  for (int nj = 0; nj < 8; ++nj) acc[nj][0] = acc[nj][1] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < kTB; k0 += 4) {
    const double af = A[(k0 + tig) * kTS + 8 * w + gid];
    double bf[8];
#pragma unroll
    for (int nj = 0; nj < 8; ++nj) bf[nj] = B[(k0 + tig) * kTS + 8 * nj + gid];
#pragma unroll
    for (int nj = 0; nj < 8; ++nj)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[nj][0]), "+d"(acc[nj][1])
                   : "d"(af), "d"(bf[nj]));
  }
#pragma unroll
  for (int nj = 0; nj < 8; ++nj) {
    double* c = C + (8 * w + gid) * kTS + 8 * nj + 2 * tig;
    c[0] -= acc[nj][0];
    c[1] -= acc[nj][1];
  }
}

__global__ void __launch_bounds__(kCholThreads, 1)
k_chol_dag(double* __restrict__ G, int n, int T, const int4* __restrict__ tasks, int ntasks,
           double* __restrict__ xinv, int* __restrict__ potrf_done, int* __restrict__ trsm_done,
           int* __restrict__ upd_done, CholCtl* __restrict__ ctl, int* __restrict__ pivot,
           unsigned long long* __restrict__ trace, int dmma) {
  extern __shared__ double sm[];
  double* S0 = sm;                  // [64][65]
  double* S1 = S0 + kTB * kTS;
  double* S2 = S1 + kTB * kTS;
  __shared__ int task_idx;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  for (;;) {
    if (tid == 0) task_idx = atomicAdd(&ctl->next, 1);
    __syncthreads();
    const int t = task_idx;
    __syncthreads();
    if (t >= ntasks) break;
    const int4 tk = tasks[t];
    const int type = tk.x, k = tk.y, i = tk.z, j = tk.w;
    unsigned long long t0 = 0;
    if (trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned long long tready = 0, tload = 0, tcomp = 0;
#define TSTAMP(v) do { if (trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v)); } while (0)
    if (type == T_POTRF) {
      bool ok = wait_flag(&upd_done[k * T + k], k, ctl);
      if (trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tready));
      int f = 0;
      if (ok) {
        load_tile(G, n, k, k, S0, true, true);
        __syncthreads();
        TSTAMP(tload);
        const int nb = min(kTB, n - k * kTB);
        f = potrf_tile<16>(S0, S1, nb);
        TSTAMP(tcomp);
        if (!f) {
          store_tile(G, n, k, k, S0, true);
          if (tid < kTB) xinv[(size_t)k * kTB + tid] = S1[tid];
        }
      }
      __syncthreads();
      if (tid == 0) {
        if (f) {
          atomicCAS(&ctl->fail, 0, k * kTB + f);
          atomicCAS(pivot, 0, k * kTB + f);
        }
        __threadfence();
        st_release(&potrf_done[k], 1);
      }
    } else if (type == T_TRSM) {      // R_kj = X_k^T G_kj
      bool ok = wait_flag(&potrf_done[k], 1, ctl) && wait_flag(&upd_done[k * T + j], k, ctl);
      if (trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tready));
      if (ok) {
        load_tile(G, n, k, k, S0, true, true);      // R_kk (upper, identity padding)
        if (tid < kTB) S2[tid] = __ldcg(xinv + (size_t)k * kTB + tid);
        load_tile(G, n, k, j, S1, false, false);
        __syncthreads();
        TSTAMP(tload);
        trsm_tile(S0, S2, S1);
        __syncthreads();
        TSTAMP(tcomp);
        store_tile(G, n, k, j, S1, false);
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_release(&trsm_done[k * T + j], 1);
      }
    } else if (type == T_DIAG) {
      // TRSM(k, k+1), then UPDATE(k, k+1, k+1) and POTRF(k+1) on the tile still in shared
      // memory: the factorization's critical path without two store/flag/load hops
      const int jn = k + 1;
      __shared__ double drk[kTB], drj[kTB];
      bool ok = wait_flag(&potrf_done[k], 1, ctl) && wait_flag(&upd_done[k * T + jn], k, ctl);
      TSTAMP(tready);
      if (ok) {
        load_tile(G, n, k, k, S0, true, true);
        if (tid < kTB) drk[tid] = __ldcg(xinv + (size_t)k * kTB + tid);
        load_tile(G, n, k, jn, S1, false, false);
        __syncthreads();
        trsm_tile(S0, drk, S1);
        __syncthreads();
        store_tile(G, n, k, jn, S1, false);
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_release(&trsm_done[k * T + jn], 1);
      }
      ok = ok && wait_flag(&upd_done[jn * T + jn], k, ctl);
      TSTAMP(tload);
      int f = 0;
      if (ok) {
        load_tile(G, n, jn, jn, S2, true, true);
        __syncthreads();
        if (dmma) {
          tile_atb_sub_dmma(S1, S1, S2);
        } else {
          double acc[4][4] = {};
          tile_atb(S1, S1, acc);
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) S2[(4 * ty + p) * kTS + tx + 16 * q] -= acc[p][q];
        }
        __syncthreads();
        f = potrf_tile<16>(S2, drj, min(kTB, n - jn * kTB));
        TSTAMP(tcomp);
        if (!f) {
          store_tile(G, n, jn, jn, S2, true);
          if (tid < kTB) xinv[(size_t)jn * kTB + tid] = drj[tid];
        }
      }
      __syncthreads();
      if (tid == 0) {
        if (f) {
          atomicCAS(&ctl->fail, 0, jn * kTB + f);
          atomicCAS(pivot, 0, jn * kTB + f);
        }
        __threadfence();
        st_release(&upd_done[jn * T + jn], k + 1);
        st_release(&potrf_done[jn], 1);
      }
    } else {                          // G_ij -= R_ki^T R_kj, applied in k order
      bool ok = wait_flag(&trsm_done[k * T + i], 1, ctl) && wait_flag(&trsm_done[k * T + j], 1, ctl) &&
                wait_flag(&upd_done[i * T + j], k, ctl);
      if (trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tready));
      if (ok) {
        load_tile(G, n, k, i, S0, false, false);
        if (j != i) load_tile(G, n, k, j, S1, false, false);
        load_tile(G, n, i, j, S2, i == j, false);
        __syncthreads();
        TSTAMP(tload);
        if (dmma) {
          tile_atb_sub_dmma(S0, j != i ? S1 : S0, S2);
        } else {
          double acc[4][4] = {};
          tile_atb(S0, j != i ? S1 : S0, acc);
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) S2[(4 * ty + p) * kTS + tx + 16 * q] -= acc[p][q];
        }
        __syncthreads();
        TSTAMP(tcomp);
        store_tile(G, n, i, j, S2, i == j);
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_release(&upd_done[i * T + j], k + 1);
      }
    }
    if (trace && tid == 0) {
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      trace[6 * t] = t0;
      trace[6 * t + 1] = tready;
      trace[6 * t + 2] = tload;
      trace[6 * t + 3] = tcomp;
      trace[6 * t + 4] = t1;
      trace[6 * t + 5] = blockIdx.x;
    }
  }
}

// Topological task list with one step of lookahead (file header).
static const std::vector<int4>& task_list(int T) {
  static int cached_T = -1;
  static std::vector<int4> v;
  if (cached_T == T) return v;
  // DIAG(k) = TRSM(k, k+1) + UPDATE(k, k+1, k+1) + POTRF(k+1) (kernel comment).  Every
  // task's inputs come from tasks earlier in the list, so in-order fetching cannot deadlock.
  v.clear();
  v.push_back(make_int4(T_POTRF, 0, 0, 0));
  if (T > 1) v.push_back(make_int4(T_DIAG, 0, 0, 1));
  for (int j = 2; j < T; ++j) v.push_back(make_int4(T_TRSM, 0, 0, j));
  for (int k = 0; k + 1 < T; ++k) {
    for (int j = k + 2; j < T; ++j) v.push_back(make_int4(T_UPDATE, k, k + 1, j));     // row k+1 of step k
    if (k + 2 < T) {
      v.push_back(make_int4(T_UPDATE, k, k + 2, k + 2));                               // DIAG(k+1) needs it
      v.push_back(make_int4(T_DIAG, k + 1, 0, k + 2));
      for (int j = k + 3; j < T; ++j) v.push_back(make_int4(T_TRSM, k + 1, 0, j));
    }
    for (int i = k + 2; i < T; ++i)
      for (int j = i; j < T; ++j)
        if (!(i == k + 2 && j == k + 2)) v.push_back(make_int4(T_UPDATE, k, i, j));   // rest of step k
  }
  cached_T = T;
  return v;
}

size_t chol_ws_bytes(int n) {
  const int T = (n + kTB - 1) / kTB;
  const size_t tasks = task_list(T).size();
  return tasks * sizeof(int4) + (size_t)T * kTB * 8 + ((size_t)T + 2 * (size_t)T * T) * sizeof(int) +
         sizeof(CholCtl) + 1024;
}

int launch_cholesky(double* G, int n, int* pivot, void* ws, size_t ws_bytes, cudaStream_t st, int* launches) {
  const int T = (n + kTB - 1) / kTB;
  const std::vector<int4>& tl = task_list(T);
  if (ws_bytes < chol_ws_bytes(n)) { set_error("cholesky: workspace too small"); return TLS_ERR_WORKSPACE; }
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* r = p; p += (bytes + 255) & ~(size_t)255; return r; };
  int4* tasks = reinterpret_cast<int4*>(take(tl.size() * sizeof(int4)));
  double* xinv = reinterpret_cast<double*>(take((size_t)T * kTB * 8));   // 1 / R_ii per tile
  int* flags = reinterpret_cast<int*>(take(((size_t)T + 2 * (size_t)T * T) * sizeof(int) + sizeof(CholCtl)));
  int* potrf_done = flags;
  int* trsm_done = potrf_done + T;
  int* upd_done = trsm_done + (size_t)T * T;
  CholCtl* ctl = reinterpret_cast<CholCtl*>(upd_done + (size_t)T * T);
  if ((size_t)(p - static_cast<char*>(ws)) > ws_bytes) { set_error("cholesky: workspace too small"); return TLS_ERR_WORKSPACE; }
  TLS_CUDA_TRY(cudaMemcpyAsync(tasks, tl.data(), tl.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  TLS_CUDA_TRY(cudaMemsetAsync(flags, 0, ((size_t)T + 2 * (size_t)T * T) * sizeof(int) + sizeof(CholCtl), st));
  const size_t smem = 3 * kTB * kTS * 8;
  static bool attr = false;
  if (!attr) {
    TLS_CUDA_TRY(cudaFuncSetAttribute(k_chol_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  int ntasks = (int)tl.size();
  int grid = num_sms();
  if (grid > ntasks) grid = ntasks;
  // TLS_CHOL_TRACE=<path>: per-task start/end timestamps (globaltimer ns) and CTA, written
  // after the kernel as text lines "type k i j start ready loaded computed end cta"
  // (diagnostics only)
  static unsigned long long* trace = nullptr;
  const char* tpath = getenv("TLS_CHOL_TRACE");
  if (tpath && !trace) TLS_CUDA_TRY(cudaMalloc(&trace, 6 * sizeof(unsigned long long) * 200000));
  unsigned long long* tr = tpath ? trace : nullptr;
  // TLS_CHOL_DMMA=1: UPDATE tiles on the fp64 tensor cores (tile_atb_sub_dmma).  Measured
  // (tools/time_chol.py, profiles/r02_chol_dmma.log): 0.892 vs 0.882 ms at n = 1024, 1.356 vs
  // 1.310 ms at n = 2000 -- the factorization's critical path is the POTRF of the diagonal
  // tiles, not the updates, and the DMMA fragments' shared-memory pattern costs more than the
  // DFMA register blocking saves, so the DFMA tile_atb stays the default
  static int dmma = [] { const char* e = getenv("TLS_CHOL_DMMA"); return (e && e[0] == '1') ? 1 : 0; }();
  void* args[] = {&G, (void*)&n, (void*)&T, &tasks, &ntasks, &xinv, &potrf_done, &trsm_done, &upd_done, &ctl, &pivot, &tr,
                  &dmma};
  TLS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_chol_dag, dim3(grid), dim3(kCholThreads), args, smem, st));
  if (launches) *launches += 1;
  if (tr) {
    std::vector<unsigned long long> h(6 * (size_t)ntasks);
    TLS_CUDA_TRY(cudaMemcpyAsync(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost, st));
    TLS_CUDA_TRY(cudaStreamSynchronize(st));
    FILE* f = fopen(tpath, "w");
    if (f) {
      for (int t = 0; t < ntasks; ++t)
        fprintf(f, "%d %d %d %d %llu %llu %llu %llu %llu %llu\n", tl[t].x, tl[t].y, tl[t].z, tl[t].w, h[6 * t],
                h[6 * t + 1], h[6 * t + 2], h[6 * t + 3], h[6 * t + 4], h[6 * t + 5]);
      fclose(f);
    }
  }
  return 0;
}

}  // namespace tls
