// k_trsv.cu — preconditioner solves with the stored-low R~ and the fused PCG /
// RQI vector kernels.
//
//   back   q = P^{-1} p  = D^{-1} (R~^{-1} p)      (Alg. 3 l.193)
//   fwd    w = P^{-T} y  = R~^{-T} (D^{-1} y)      (Alg. 3 l.191, l.197)
// Both are blocked solves over 32-row blocks inside ONE CTA per right-hand
// side (the n-vector lives in shared memory), warp-specialised by block row
// (trsv_ws below): each warp owns every kTW-th block row, accumulates its tile
// updates as soon as the mbarrier of the needed solution block fires, and
// solves its diagonal block with the fp64 inverse of R~_kk (staged by cp.async)
// — so only one tile update and one 32 x 32 solve per block row are on the
// critical path.  Tiles of R~ (back) or R~^T (fwd) are streamed from L2 in u_f
// and upcast on load.  The two right-hand sides of a batched PCG step (RHS a:
// -f, RHS b: x_k) run on two CTAs (two SMs) concurrently.
//
// The PCG recurrences of Alg. 3 (delta, alpha, omega, s, eta, beta, p;
// PAPER.md l.191-201 with the A-in-loop operator of l.324, reading R1) are
// fused into k_pcg_step around the forward solve, followed by the next
// iteration's back solve; the RQI updates of Alg. 4 (l.238-255) live in
// k_rqi_eval / k_rqi_update / k_boot_x1.  All reductions are fixed-order.
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>

#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

constexpr int kTT = 512;  // threads of the single-CTA kernels

// ---------------------------------------------------------------- 32-value row segments
template <typename T> struct SegTraits { static constexpr int NV = 32 * (int)sizeof(T) / 16; };

template <typename T>
__device__ __forceinline__ double seg_get(const uint4 (&raw)[SegTraits<T>::NV], int l);

template <> __device__ __forceinline__ double seg_get<F16s>(const uint4 (&raw)[4], int l) {
  const uint4 u = raw[l >> 3];
  const int k = (l & 7) >> 1;
  const uint32_t w = k == 0 ? u.x : k == 1 ? u.y : k == 2 ? u.z : u.w;
  const uint16_t h = (l & 1) ? (uint16_t)(w >> 16) : (uint16_t)(w & 0xffff);
  return (double)dec_f16(h);
}
template <> __device__ __forceinline__ double seg_get<B16s>(const uint4 (&raw)[4], int l) {
  const uint4 u = raw[l >> 3];
  const int k = (l & 7) >> 1;
  const uint32_t w = k == 0 ? u.x : k == 1 ? u.y : k == 2 ? u.z : u.w;
  return (double)__uint_as_float((l & 1) ? (w & 0xffff0000u) : (w << 16));
}
template <> __device__ __forceinline__ double seg_get<float>(const uint4 (&raw)[8], int l) {
  const uint4 u = raw[l >> 2];
  const int k = l & 3;
  return (double)__uint_as_float(k == 0 ? u.x : k == 1 ? u.y : k == 2 ? u.z : u.w);
}
template <> __device__ __forceinline__ double seg_get<double>(const uint4 (&raw)[16], int l) {
  const uint4 u = raw[l >> 1];
  return (l & 1) ? __hiloint2double((int)u.w, (int)u.z) : __hiloint2double((int)u.y, (int)u.x);
}

template <typename T>
__device__ __forceinline__ void seg_load(const T* p, uint4 (&raw)[SegTraits<T>::NV]) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int k = 0; k < SegTraits<T>::NV; ++k) raw[k] = __ldg(q + k);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------- warp-specialised blocked TRSV
// One CTA (kTW warps) solves one right-hand side.  The npad x npad triangle is
// cut into NB = npad/32 block rows, numbered u = 0..NB-1 in SOLVE order
// (back substitution: real block NB-1-u; forward: real block u).  Warp w owns the
// blocks u = w (mod kTW).  For each owned block, in ascending u, the warp
// accumulates acc = sum_{u' < u} M_{u,u'} x_{u'} over the 32 x 32 tiles of its
// block row, waiting on the mbarrier of x_{u'} before each tile, then solves
// x_u = D_u (y_u - acc) with the fp64 inverse D_u of the diagonal block (staged in
// the warp's shared-memory slot by cp.async while the warp accumulates) and
// publishes x_u (smem + mbarrier arrive).  Tile rows of R~ (u_f, 32 values per
// lane) are loaded from L2 through a register FIFO of depth TileDP ahead of use,
// so the loads overlap the wait for x.  The critical path per block row is one
// tile update plus one 32 x 32 solve; the other tile updates of all warps run
// concurrently with it.
constexpr int kTW = 8;   // warps of a TRSV CTA

// Built with -DTLS_TRSV_TRACE (TLS_EXTRA_NVCC; diagnostics only) and run with
// TLS_TRSV_TRACE=<path> (tls_precond_apply): per solution block u, the globaltimer when its
// owner warp starts solve() (its tile updates are done), when x_{u-1} has arrived and when x_u
// is published; written by launch_precond_apply as text lines
// "cta warp u t_solve t_arrived t_published" for RHS 0.  Compiled out by default: a global
// load per solve() on the chain measurably slowed the solves (tools/trsv_trace.py).
#ifdef TLS_TRSV_TRACE
__device__ unsigned long long* g_trsv_trace = nullptr;
#define TRSV_TRACE_PTR g_trsv_trace
#else
#define TRSV_TRACE_PTR ((unsigned long long*)nullptr)
#endif
#ifndef TLS_TRSV_RUN
#define TLS_TRSV_RUN 1
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <typename T> struct TileDP { static constexpr int v = SegTraits<T>::NV <= 4 ? 4 : (SegTraits<T>::NV <= 8 ? 2 : 1); };

struct TrsvSm {
  uint32_t phase; // parity of the barrier phase the next solve completes (one phase per solve)
  double* y;      // [npad] right-hand side in, solution out (in place)
  double* D;      // [kTW][2048] per-warp slot: inverse of the diagonal block, then its E block
  double* ys;     // [kTW][32] per-warp scratch of the block solve
  uint64_t* bar;  // [NB] x_u published
  double* red;    // [32] block_sum scratch
};
// dynamic smem of a TRSV CTA
__host__ __device__ inline size_t trsv_smem(int npad) {
  return (size_t)npad * 8 + (size_t)kTW * 2048 * 8 + (size_t)kTW * 32 * 8 + (size_t)(npad / 32) * 8 + 32 * 8;
}
__device__ __forceinline__ TrsvSm trsv_carve(int npad) {
  extern __shared__ __align__(16) double tsm[];
  TrsvSm s;
  s.phase = 0;
  s.y = tsm;
  s.D = s.y + npad;
  s.ys = s.D + kTW * 2048;
  s.red = s.ys + kTW * 32;
  s.bar = reinterpret_cast<uint64_t*>(s.red + 32);
  return s;
}

// Initialise the block barriers once per kernel (they are never re-initialised:
// each solve completes exactly one phase of every barrier).  All threads call it.
__device__ __forceinline__ void trsv_init(const TrsvSm& sm, int npad) {
  for (int i = threadIdx.x; i < (npad >> 5); i += blockDim.x) mbar_init(&sm.bar[i], 1);
  if (threadIdx.x == 0) fence_mbar_init();
  cluster_sync_all();   // the cluster's CTAs may address these barriers from now on
}

__device__ __forceinline__ void stage_dinv_warp(double* dst, const double* src, const double* esrc) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 16; ++k) cp_async16(dst + (k * 32 + lane) * 2, src + (k * 32 + lane) * 2);
#pragma unroll
  for (int k = 0; k < 16; ++k) cp_async16(dst + 1024 + (k * 32 + lane) * 2, esrc + (k * 32 + lane) * 2);
  cp_async_commit();
}

// Element e of a 16-byte chunk of u_f values.
template <typename T> __device__ __forceinline__ double chunk_get(const uint4& u, int e);
template <> __device__ __forceinline__ double chunk_get<F16s>(const uint4& u, int e) {
  // one F2F.F64.F16 (half-register select), no fp32 step
  const uint32_t w = (e >> 1) == 0 ? u.x : (e >> 1) == 1 ? u.y : (e >> 1) == 2 ? u.z : u.w;
  const uint16_t h = (e & 1) ? (uint16_t)(w >> 16) : (uint16_t)(w & 0xffff);
  double d;
  asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(h));
  return d;
}
template <> __device__ __forceinline__ double chunk_get<B16s>(const uint4& u, int e) {
  const uint32_t w = (e >> 1) == 0 ? u.x : (e >> 1) == 1 ? u.y : (e >> 1) == 2 ? u.z : u.w;
  return (double)__uint_as_float((e & 1) ? (w & 0xffff0000u) : (w << 16));
}
template <> __device__ __forceinline__ double chunk_get<float>(const uint4& u, int e) {
  return (double)__uint_as_float(e == 0 ? u.x : e == 1 ? u.y : e == 2 ? u.z : u.w);
}
template <> __device__ __forceinline__ double chunk_get<double>(const uint4& u, int e) {
  return e ? __hiloint2double((int)u.w, (int)u.z) : __hiloint2double((int)u.y, (int)u.x);
}

// BACK: solve R~ x = y with M = Rrow (upper), Dinv = DinvB.
// !BACK: solve R~^T x = y with M = RTrow (lower), Dinv = DinvF.
// Tile loads are coalesced: load k of a tile brings RPI = 32/CPR whole 32-value row
// segments (lane group g = lane/CPR reads row k*RPI + g, 16-byte chunk lane%CPR), so
// each lane accumulates, per k, a partial dot product over its chunk's columns; the
// partials of a row are combined across its CPR lanes only when the block is solved.
// All threads of the CTA must call it (after trsv_init); ends with __syncthreads().
// Look-ahead form of each block solve (k_e_blocks in k_chol.cu): the owner accumulates
// the tile updates of block u from every solution block except the last one in solve
// order, forms z_u = D_u (y_u - acc) while x_{u-1} is still being solved elsewhere, and
// once x_{u-1} arrives computes x_u = z_u - E_u x_{u-1}, E_u = D_u T_{u,u-1}: a single
// 32 x 32 product on the critical path instead of a tile update, a cross-lane row
// reduction and the diagonal solve.
template <typename T, bool BACK>
__device__ void trsv_ws(const T* __restrict__ M, const double* __restrict__ Dinv, const double* __restrict__ Eblk,
                        int npad, TrsvSm& sm) {
  constexpr int NV = SegTraits<T>::NV, DP = TileDP<T>::v;
  constexpr int CPR = NV, RPI = 32 / CPR, EPC = 16 / (int)sizeof(T);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / CPR, cpos = lane % CPR;
  const int NB = npad >> 5;
  const int C = (int)cluster_nctarank(), cr = (int)cluster_ctarank();
  const uint32_t ph = sm.phase;
  // arm every block barrier for this solve: one local arrival + the 256 bytes of the
  // solution block, written by its owner CTA with st.async (complete_tx); the cluster
  // barrier makes sure every CTA is armed (and its y filled) before anyone sends
  for (int i = threadIdx.x; i < NB; i += blockDim.x) mbar_arrive_expect_tx(&sm.bar[i], 256);
  cluster_sync_all();
  // block u (solve order) is owned by CTA u % C, warp (u / C) % kTW; its tiles are
  // (u, 0 .. u-2) -- the coupling to u-1 is the E block.  Build-time experiments (round 2,
  // TLS_EXTRA_NVCC): -DTLS_TRSV_RUN=L, -DTLS_TRSV_EPRE (tools/runs/gpu_r02_t2.sh).
#if TLS_TRSV_RUN > 1
  // experiment: runs of L consecutive blocks per CTA (CTA (u / L) % C), most hand-offs CTA-local
  constexpr int L = TLS_TRSV_RUN;
  const int first = L * (cr + C * (warp / L)) + warp % L;
#else
  const int first = cr + C * warp;
#endif
  const int ustep = C * kTW;
  if (first < NB) {
    double* Dw = sm.D + warp * 2048;
    double* Ew = Dw + 1024;
    double* ysw = sm.ys + warp * 32;
    auto real = [&](int u) { return BACK ? NB - 1 - u : u; };
    auto issue = [&](int ui, int ci, uint4 (&raw)[NV]) {
      const T* base = M + (size_t)(32 * real(ui) + grp) * npad + 32 * real(ci) + cpos * EPC;
#pragma unroll
      for (int k = 0; k < NV; ++k) raw[k] = __ldg(reinterpret_cast<const uint4*>(base + (size_t)k * RPI * npad));
    };
    auto ntiles = [](int u) { return u >= 1 ? u - 1 : 0; };
    int total = 0;
    for (int u = first; u < NB; u += ustep) total += ntiles(u);
    stage_dinv_warp(Dw, Dinv + (size_t)real(first) * 1024, Eblk + (size_t)real(first) * 1024);
    int ui = first, ci = 0;
    while (ui < NB && ntiles(ui) == 0) ui += ustep;
    uint4 raw[DP][NV];
#pragma unroll
    for (int s = 0; s < DP; ++s) {
      if (s < total) {
        issue(ui, ci, raw[s]);
        if (++ci == ntiles(ui)) {
          ci = 0;
          do { ui += ustep; } while (ui < NB && ntiles(ui) == 0);
        }
      }
    }
    const uint32_t y_base = smem_u32(sm.y), bar_base = smem_u32(sm.bar);
    int uc = first, cc = 0;
    double acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = 0.0;
    auto solve = [&]() {
      unsigned long long* trc = TRSV_TRACE_PTR;
      unsigned long long t_solve = 0, t_arr = 0;
      if (trc && lane == 0) t_solve = gtimer();
      // row sums: combine the CPR chunk partials of each row, then move row i's sum to lane i
      double mine = 0.0;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        double v = acc[k];
#pragma unroll
        for (int o = CPR / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const double t = __shfl_sync(0xffffffffu, v, (lane % RPI) * CPR);
        if (k == lane / RPI) mine = t;
        acc[k] = 0.0;
      }
      const int o = 32 * real(uc);
      ysw[lane] = sm.y[o + lane] - mine;
      cp_async_wait<0>();
      __syncwarp();
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int l = 0; l < 32; l += 2) {
        z0 = fma(Dw[l * 32 + lane], ysw[l], z0);
        z1 = fma(Dw[(l + 1) * 32 + lane], ysw[l + 1], z1);
      }
      double xv = z0 + z1;
      if (uc >= 1) {                                     // x_u = z_u - E_u x_{u-1}
#ifdef TLS_TRSV_EPRE
        // experiment: E_u's row in registers before the wait, four FMA chains after it
        double er[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) er[l] = Ew[l * 32 + lane];
        mbar_wait_cluster(&sm.bar[uc - 1], ph);
        if (trc && lane == 0) t_arr = gtimer();
        const double2* xp = reinterpret_cast<const double2*>(sm.y + 32 * real(uc - 1));
        double e[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int l = 0; l < 32; l += 4) {
          const double2 xa = xp[l >> 1], xb = xp[(l >> 1) + 1];
          e[0] = fma(er[l], xa.x, e[0]);
          e[1] = fma(er[l + 1], xa.y, e[1]);
          e[2] = fma(er[l + 2], xb.x, e[2]);
          e[3] = fma(er[l + 3], xb.y, e[3]);
        }
        xv -= (e[0] + e[1]) + (e[2] + e[3]);
#else
        mbar_wait_cluster(&sm.bar[uc - 1], ph);
        if (trc && lane == 0) t_arr = gtimer();
        const double* xp = sm.y + 32 * real(uc - 1);
        double e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int l = 0; l < 32; l += 2) {
          e0 = fma(Ew[l * 32 + lane], xp[l], e0);
          e1 = fma(Ew[(l + 1) * 32 + lane], xp[l + 1], e1);
        }
        xv -= e0 + e1;
#endif
      }
      __syncwarp();
      // publish x_u to every CTA of the cluster (including this one)
      const uint32_t ya = y_base + (uint32_t)(o + lane) * 8u, ba = bar_base + (uint32_t)uc * 8u;
#if TLS_TRSV_RUN > 1
      const int nxt = ((uc + 1) / TLS_TRSV_RUN) % C;     // experiment: the next block's owner first
      for (int k = 0; k < C; ++k) {
        const uint32_t r = (uint32_t)((nxt + k) % C);
        st_async_f64(mapa_shared(ya, r), xv, mapa_shared(ba, r));
      }
#else
      for (int r = 0; r < C; ++r) st_async_f64(mapa_shared(ya, (uint32_t)r), xv, mapa_shared(ba, (uint32_t)r));
#endif
      if (trc && lane == 0 && blockIdx.x < (unsigned)C) {
        const unsigned long long t_pub = gtimer();
        unsigned long long* e = trc + 6 * (size_t)uc;
        e[0] = cr; e[1] = warp; e[2] = uc; e[3] = t_solve; e[4] = t_arr; e[5] = t_pub;
      }
      uc += ustep;
      cc = 0;
      if (uc < NB) stage_dinv_warp(Dw, Dinv + (size_t)real(uc) * 1024, Eblk + (size_t)real(uc) * 1024);
    };
    while (uc < NB && ntiles(uc) == 0) solve();
    for (int kb = 0; kb < total; kb += DP) {
#pragma unroll
      for (int s = 0; s < DP; ++s) {
        if (kb + s < total) {
          mbar_wait_cluster(&sm.bar[cc], ph);
          double xv[EPC];
          const double2* xp = reinterpret_cast<const double2*>(sm.y + 32 * real(cc) + cpos * EPC);
#pragma unroll
          for (int e = 0; e < EPC; e += 2) {
            const double2 t = xp[e >> 1];
            xv[e] = t.x;
            xv[e + 1] = t.y;
          }
#pragma unroll
          for (int k = 0; k < NV; ++k)
#pragma unroll
            for (int e = 0; e < EPC; ++e) acc[k] = fma(chunk_get<T>(raw[s][k], e), xv[e], acc[k]);
          if (kb + s + DP < total) {
            issue(ui, ci, raw[s]);
            if (++ci == ntiles(ui)) {
              ci = 0;
              do { ui += ustep; } while (ui < NB && ntiles(ui) == 0);
            }
          }
          if (++cc == ntiles(uc)) {
            solve();
            while (uc < NB && ntiles(uc) == 0) solve();
          }
        }
      }
    }
  }
  // every solution block (also the ones other CTAs own) must be in this CTA's y
  for (int i = threadIdx.x; i < NB; i += blockDim.x) mbar_wait_cluster(&sm.bar[i], ph);
  sm.phase ^= 1u;
  __syncthreads();
}

// ---------------------------------------------------------------- explicit-inverse apply (R24)
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

// y <- W^T y (BACK = false, the forward solve R~^T x = y) or W y (BACK = true, the back
// solve R~ x = y) with W = R~^{-1} formed once in fp64 (k_trtri; npad x npad row-major,
// zero below the diagonal).  A cluster-wide GEMV: CTA c of the cluster computes the 32-row
// (32-column) chunks q = c, c + C, ... of the result, coalesced over W's rows, and stores
// them into every CTA's staging buffer through DSMEM; no block-by-block dependency chain.
// Same contract as trsv_ws: every CTA calls it with the same y and gets the same result.
template <bool BACK>
__device__ void wgemv(const double* __restrict__ W, int npad, TrsvSm& sm) {
  const int C = (int)cluster_nctarank(), cr = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NB = npad >> 5;
  double* out = sm.D;                 // [npad] result staging (the TRSV slots are unused here)
  double* part = sm.D + 2048;         // [kTW][32] column partials
  const uint32_t out_base = smem_u32(out);
  cluster_sync_all();                 // no CTA is still reading a previous result from `out`
  for (int q = cr; q < NB; q += C) {
    if (BACK) {
      // rows 32q + warp + kTW k: x_i = sum_{j >= 32q} W_ij y_j (W_ij = 0 for j < i)
      for (int k = 0; k < 32 / kTW; ++k) {
        const int i = 32 * q + warp + kTW * k;
        const double* Wi = W + (size_t)i * npad;
        double a0 = 0.0, a1 = 0.0;
        int j = 32 * q + lane;
        for (; j + 32 < npad; j += 64) {
          a0 = fma(__ldg(Wi + j), sm.y[j], a0);
          a1 = fma(__ldg(Wi + j + 32), sm.y[j + 32], a1);
        }
        if (j < npad) a0 = fma(__ldg(Wi + j), sm.y[j], a0);
        const double acc = warp_sum(a0 + a1);
        if (lane < C) st_cluster_f64(mapa_shared(out_base + (uint32_t)i * 8u, (uint32_t)lane), acc);
      }
    } else {
      // columns j = 32q + lane: x_j = sum_{i < 32q + 32} W_ij y_i, rows split over the warps
      const int j = 32 * q + lane;
      double a0 = 0.0, a1 = 0.0;
      int i = warp;
      for (; i + kTW < 32 * q + 32; i += 2 * kTW) {
        a0 = fma(__ldg(W + (size_t)i * npad + j), sm.y[i], a0);
        a1 = fma(__ldg(W + (size_t)(i + kTW) * npad + j), sm.y[i + kTW], a1);
      }
      if (i < 32 * q + 32) a0 = fma(__ldg(W + (size_t)i * npad + j), sm.y[i], a0);
      part[warp * 32 + lane] = a0 + a1;
      __syncthreads();
      if (warp == 0) {
        double acc = 0.0;
#pragma unroll
        for (int w = 0; w < kTW; ++w) acc += part[w * 32 + lane];
        for (int r = 0; r < C; ++r) st_cluster_f64(mapa_shared(out_base + (uint32_t)j * 8u, (uint32_t)r), acc);
      }
      __syncthreads();
    }
  }
  cluster_sync_all();                 // every chunk has landed in every CTA
  for (int i = tid; i < npad; i += blockDim.x) sm.y[i] = out[i];
  __syncthreads();
}

// The preconditioner solves of every kernel below: substitution with the stored R~ (the
// default, a6 as specified) or the explicit inverse when the solve provides one (pc.W).
template <typename T, bool BACK>
__device__ __forceinline__ void pre_apply(const PrecondDev& pc, TrsvSm& sm) {
  if (pc.W != nullptr) wgemv<BACK>(pc.W, pc.npad, sm);
  else if (BACK) trsv_ws<T, true>((const T*)pc.Rrow, pc.DinvB, pc.EB, pc.npad, sm);
  else trsv_ws<T, false>((const T*)pc.RTrow, pc.DinvF, pc.EF, pc.npad, sm);
}

// W = R~^{-1} by block columns (R24): W_JJ = R~_JJ^{-1} (the DinvB blocks), then for
// I = J-1 .. 0: W_IJ = -R~_II^{-1} sum_{K=I+1..J} R~_IK W_KJ.  CTA (J, c) owns 4 columns of
// block column J and keeps their strip of W in shared memory (DinvB_I staged by cp.async).  Warp w takes the blocks
// K = I+1+w, I+1+w+8, ...; lane r multiplies the 32-element segment of row 32I+r of R~_IK
// (one vector load, the next one in flight) into the strip; the 8 warp partials are summed
// in fixed order and the 32 x 32 inverse is applied.  W, WT zeroed beforehand; WT = W^T.
constexpr int kTriW = 8, kTriT = kTriW * 32;   // warps of k_trtri: warp w takes every 8th block K (16 measured slower)

template <typename T>
__global__ void __launch_bounds__(kTriT) k_trtri(PrecondDev pc, double* __restrict__ W, double* __restrict__ WT) {
  constexpr int NV = SegTraits<T>::NV;
  extern __shared__ double wsm[];
  const int npad = pc.npad;
  const int J = blockIdx.x >> 3, c0 = (blockIdx.x & 7) * 4;
  double* Wc = wsm;                          // [npad][4]
  double* Tp = Wc + (size_t)npad * 4;        // [kTriW][32][4] partials
  double* Tf = Tp + kTriW * 32 * 4;          // [32][4]
  double* Di = Tf + 32 * 4;                  // [1024] DinvB block of the current I (staged by cp.async)
  const int tid = threadIdx.x, w = tid >> 5, r = tid & 31;
  const T* R = reinterpret_cast<const T*>(pc.Rrow);
  if (tid < 128) {                           // DinvB[kb][l][i] = (R~_kk^{-1})[i][l]
    const int rr = tid >> 2, cc = tid & 3;
    const double v = pc.DinvB[(size_t)J * 1024 + (c0 + cc) * 32 + rr];
    Wc[(32 * J + rr) * 4 + cc] = v;
    W[(size_t)(32 * J + rr) * npad + 32 * J + c0 + cc] = v;
    WT[(size_t)(32 * J + c0 + cc) * npad + 32 * J + rr] = v;
  }
  __syncthreads();
  for (int I = J - 1; I >= 0; --I) {
    // the 32 x 32 inverse of block I arrives while the products are formed
#pragma unroll
    for (int k = tid; k < 512; k += kTriT) cp_async16(Di + 2 * k, pc.DinvB + (size_t)I * 1024 + 2 * k);
    cp_async_commit();
    const T* Rr = R + (size_t)(32 * I + r) * npad;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    uint4 cur[NV], nxt[NV];
    int K = I + 1 + w;
    if (K <= J) seg_load<T>(Rr + 32 * K, cur);
    for (; K <= J; K += kTriW) {
      if (K + kTriW <= J) seg_load<T>(Rr + 32 * (K + kTriW), nxt);
      const double* wk = Wc + (size_t)(32 * K) * 4;
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        const double rv = seg_get<T>(cur, l);
        const double4 wv = *reinterpret_cast<const double4*>(wk + 4 * l);
        a[0] = fma(rv, wv.x, a[0]);
        a[1] = fma(rv, wv.y, a[1]);
        a[2] = fma(rv, wv.z, a[2]);
        a[3] = fma(rv, wv.w, a[3]);
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) cur[k] = nxt[k];
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) Tp[(w * 32 + r) * 4 + cc] = a[cc];
    cp_async_wait<0>();
    __syncthreads();
    if (tid < 128) {
      const int rr = tid >> 2, cc = tid & 3;
      double t = 0.0;
#pragma unroll
      for (int h = 0; h < kTriW; ++h) t += Tp[(h * 32 + rr) * 4 + cc];
      Tf[rr * 4 + cc] = t;
    }
    __syncthreads();
    if (tid < 128) {
      const int rr = tid >> 2, cc = tid & 3;
      double s = 0.0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) s = fma(Di[l * 32 + rr], Tf[l * 4 + cc], s);
      Wc[(32 * I + rr) * 4 + cc] = -s;
      W[(size_t)(32 * I + rr) * npad + 32 * J + c0 + cc] = -s;
      WT[(size_t)(32 * J + c0 + cc) * npad + 32 * I + rr] = -s;
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------- explicit-inverse PCG (R24)
// With W = R~^{-1} the two preconditioner solves of a PCG step are products with W^T and W
// that every SM can share (the substitutions are a dependency chain on one 8-CTA cluster):
//   k_wgemv_grid  rows of WT (forward) or W (back) against the staged vectors of the active
//                 right-hand sides, one warp per row, both RHS in the same read of the row;
//   k_wpcg_*_mid  the n-vector recurrences of Alg. 3 (l.194-201), one CTA per RHS, with the
//                 same decisions, state updates and fixed-order reductions as k_pcg_step.
// One row of a GEMV against up to two vectors in shared memory, lane-strided over [j0, j1)
// (j0 a multiple of 32): lane l takes j = j0 + l + 32k and adds its products in increasing j,
// as the plain strided loop does (the same bits), but every load of a 1024-element chunk is
// issued before the chunk's FMAs -- one L2 round trip per chunk instead of one per few
// elements (measured: the explicit-inverse step's GEMVs were load-latency bound, VERDICT r01
// NEXT-3 target).
__device__ __forceinline__ void row_dot2(const double* __restrict__ Mi, int j0, int j1, const double* v0,
                                         const double* v1, bool u0, bool u1, double& a0, double& a1, int lane) {
  for (int c = j0; c < j1; c += 1024) {
    double m[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int j = c + lane + 32 * k;
      m[k] = j < j1 ? __ldg(Mi + j) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int j = c + lane + 32 * k;
      if (j < j1) {
        if (u0) a0 = fma(m[k], v0[j], a0);
        if (u1) a1 = fma(m[k], v1[j], a1);
      }
    }
  }
}

// mode 0: s = p = W^T (D^{-1} rhs), omega = 0 (pcg_init); mode 1: w = W^T y with
// y = D^{-1}(A^T t - sigma^2 q) (variant 0) or D^{-1} q (variant 1); mode 2: q = D^{-1} W p.
constexpr int kWG = 256;
__global__ void __launch_bounds__(kWG) k_wgemv_grid(PrecondDev pc, PcgVecs v, const double* __restrict__ passout,
                                                   const PcgState* __restrict__ S, int nrhs, int mode, int variant,
                                                   int all) {
  extern __shared__ double vin[];       // [2][npad]
  const int n = pc.n, npad = pc.npad, tid = threadIdx.x, lane = tid & 31;
  bool act[2];
  for (int r = 0; r < 2; ++r) act[r] = r < nrhs && (all || S->active[r] != 0);
  if (!act[0] && !act[1]) return;
  const double sig2 = S->sigma2;
  for (int r = 0; r < 2; ++r) {
    if (!act[r]) continue;
    const size_t off = (size_t)r * n;
    for (int j = tid; j < npad; j += kWG) {
      double x = 0.0;
      if (j < n) {
        if (mode == 0) x = v.rhs[off + j] * pc.dinv[j];
        else if (mode == 1) x = (variant == 0 ? passout[off + j] - sig2 * v.q[off + j] : v.q[off + j]) * pc.dinv[j];
        else x = v.p[off + j];
      }
      vin[(size_t)r * npad + j] = x;
    }
  }
  __syncthreads();
  const double* M = mode == 2 ? pc.W : pc.WT;
  const int nw = gridDim.x * (kWG / 32);
  for (int i = blockIdx.x * (kWG / 32) + (tid >> 5); i < n; i += nw) {
    const double* Mi = M + (size_t)i * npad;
    // upper rows (W) from the 32-aligned chunk of the diagonal on; lower rows (WT) up to it
    const int j0 = mode == 2 ? (i & ~31) : 0, j1 = mode == 2 ? npad : ((i | 31) + 1);
    double a0 = 0.0, a1 = 0.0;
    row_dot2(Mi, j0, j1, vin, vin + npad, act[0], act[1], a0, a1, lane);
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    if (lane < 2 && act[lane]) {
      const double a = lane == 0 ? a0 : a1;
      const size_t o = (size_t)lane * n + i;
      if (mode == 0) { v.s[o] = a; v.p[o] = a; v.omega[o] = 0.0; }
      else if (mode == 1) v.w[o] = a;
      else v.q[o] = a * pc.dinv[i];
    }
  }
}

// One PCG step on the explicit inverse as ONE cooperative kernel over every SM (R24):
//   A  w = W^T y, rows of WT spread over the grid               -> grid barrier
//   B  every CTA forms the same delta, alpha, s', eta', beta, p' (fixed-order sums)
//                                                                -> grid barrier
//   C  CTA 0 writes s, p and the state; q = D^{-1} W p' spread over the grid.
// Same decisions, updates and state as k_pcg_step.
//   0  (partials != nullptr, NEXT-3) the operator pass's per-CTA partials are reduced here in
//      k_reduce_partials' fixed order (8 row groups, then the group sums in order: the same
//      bits), column slices spread over the grid, into passout -> grid barrier.  Saves the
//      separate reduction launch of every PCG iteration on one rank.
// passout is not __restrict__: with phase 0 this kernel writes it (pout) before reading it, so
// its loads must stay coherent (no read-only-path caching across the grid barrier).
__global__ void __launch_bounds__(kWG) k_wpcg_step_coop(PrecondDev pc, PcgVecs v, const double* passout,
                                                       PcgState* __restrict__ S, int nrhs, int rule, int next_q,
                                                       int variant, int pass_nrhs, const double* __restrict__ partials,
                                                       int G, double* __restrict__ pout, const int* __restrict__ nq_dev) {
  // programmatic dependent launch (NEXT-3): wait for the operator pass, release the next pass
  // at once (it waits for this grid's completion before reading anything)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (nq_dev) next_q = *nq_dev;         // graph-captured loop (NEXT-3): decided on the device
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double wsh[];
  const int n = pc.n, npad = pc.npad, tid = threadIdx.x, lane = tid & 31;
  double* vin = wsh;                    // [2][npad]: y, later p'
  double* snb = wsh + 2 * (size_t)npad; // [2][npad]: s'
  __shared__ double red[64];
  __shared__ double s_al[2], s_be[2], s_dl[2], s_qq[2], s_eta[2], s_pp[2];
  __shared__ int s_upd[2], s_cont[2], s_brk[2];
  bool act[2];
  for (int r = 0; r < 2; ++r) act[r] = r < nrhs && S->active[r] != 0;
  if (!act[0] && !act[1]) return;       // uniform over the grid
  const double sig2 = S->sigma2;
  if (partials != nullptr) {
    // ---- 0: passout = fixed-order sum of the G partial rows (k_reduce_partials' order)
    const int W = pass_nrhs * n + 2;
    const int tx = tid & 31, grp = tid >> 5;          // 32 columns x 8 row groups per block
    double* gs = snb;                                   // [8][33] scratch (snb is free until B)
    for (int cb = blockIdx.x; cb * 32 < W; cb += gridDim.x) {
      const int w = cb * 32 + tx;
      const int g0 = G * grp / 8, g1 = G * (grp + 1) / 8;
      double acc = 0.0;
      if (w < W) {
        for (int g = g0; g < g1; g += 20) {             // the group's rows in flight, added in row order
          double v[20];
#pragma unroll
          for (int k = 0; k < 20; ++k) v[k] = g + k < g1 ? partials[(size_t)(g + k) * W + w] : 0.0;
#pragma unroll
          for (int k = 0; k < 20; ++k)
            if (g + k < g1) acc += v[k];
        }
      }
      gs[grp * 33 + tx] = acc;
      __syncthreads();
      if (grp == 0 && w < W) {
        double r = gs[tx];
        for (int k = 1; k < 8; ++k) r += gs[k * 33 + tx];
        pout[w] = r;
      }
      __syncthreads();
    }
    grid.sync();
  }
  // ---- A (the staging loads of four elements first: the shared-memory stores could alias them)
  for (int r = 0; r < 2; ++r) {
    if (!act[r]) continue;
    const size_t off = (size_t)r * n;
    for (int j0 = tid; j0 < npad; j0 += 4 * kWG) {
      double po[4], qv[4], dv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * kWG;
        const bool ok = j < n;
        po[u] = (ok && variant == 0) ? passout[off + j] : 0.0;
        qv[u] = ok ? v.q[off + j] : 0.0;
        dv[u] = ok ? pc.dinv[j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * kWG;
        if (j < npad) vin[(size_t)r * npad + j] = j < n ? (variant == 0 ? po[u] - sig2 * qv[u] : qv[u]) * dv[u] : 0.0;
      }
    }
  }
  __syncthreads();
  const int nw = gridDim.x * (kWG / 32);
  for (int i = blockIdx.x * (kWG / 32) + (tid >> 5); i < n; i += nw) {
    const double* Mi = pc.WT + (size_t)i * npad;
    double a0 = 0.0, a1 = 0.0;
    row_dot2(Mi, 0, (i | 31) + 1, vin, vin + npad, act[0], act[1], a0, a1, lane);
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    if (lane < 2 && act[lane]) v.w[(size_t)lane * n + i] = lane == 0 ? a0 : a1;
  }
  grid.sync();
  // ---- B (redundant in every CTA; both right-hand sides share each fixed-order block sum --
  // block_sum2: the same bits as one block_sum per RHS, half the barriers)
  {
    double e0 = 0.0, e1 = 0.0;
    for (int i = tid; i < n; i += kWG) {
      if (act[0]) e0 = fma(v.q[i], v.q[i], e0);
      if (act[1]) e1 = fma(v.q[n + i], v.q[n + i], e1);
    }
    double qq[2];
    block_sum2(e0, e1, red, qq[0], qq[1]);
    if (tid == 0) {
      for (int r = 0; r < 2; ++r) {
        s_upd[r] = 0;
        s_brk[r] = 0;
        s_cont[r] = 0;
        s_al[r] = 0.0;
        if (!act[r]) continue;
        s_qq[r] = qq[r];
        const double tau = variant == 0 ? passout[(size_t)pass_nrhs * n + r] : S->pp[r];
        const double delta = tau - sig2 * qq[r];                // l.194 (R1)
        s_dl[r] = delta;
        if (!isfinite(delta) || delta == 0.0) {                 // loop guard l.192 (R3)
        } else if (delta < 0.0 && rule == 0) {                  // breakdown (R3)
          s_brk[r] = 1;
        } else {
          s_al[r] = S->eta[r] / delta;                          // l.195
          s_upd[r] = 1;
        }
      }
    }
    __syncthreads();
    bool upd[2];
    double al[2];
    for (int r = 0; r < 2; ++r) { upd[r] = act[r] && s_upd[r]; al[r] = s_al[r]; }
    double es[2] = {0.0, 0.0};
    for (int i0 = tid; i0 < n; i0 += 4 * kWG) {     // four elements' loads first (stores could alias)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (!upd[r]) continue;
        const size_t off = (size_t)r * n;
        double qv[4], wv[4], pv[4], sv[4], ov[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kWG;
          const bool ok = i < n;
          qv[u] = ok ? v.q[off + i] : 0.0;
          wv[u] = ok ? v.w[off + i] : 0.0;
          pv[u] = (ok && variant != 0) ? v.p[off + i] : 0.0;
          sv[u] = ok ? v.s[off + i] : 0.0;
          ov[u] = (ok && blockIdx.x == 0) ? v.omega[off + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kWG;
          if (i >= n) continue;
          if (blockIdx.x == 0) v.omega[off + i] = fma(al[r], qv[u], ov[u]);   // l.196 (only CTA 0 reads omega)
          const double w = variant == 0 ? wv[u] : fma(-sig2, wv[u], pv[u]);    // l.197
          const double sn = fma(-al[r], w, sv[u]);           // l.198
          snb[(size_t)r * npad + i] = sn;
          es[r] = fma(sn, sn, es[r]);
        }
      }
    }
    double etan[2];
    block_sum2(es[0], es[1], red, etan[0], etan[1]);           // l.199
    if (tid == 0) {
      for (int r = 0; r < 2; ++r) {
        if (!upd[r]) continue;
        s_eta[r] = etan[r];
        if (!(etan[r] <= S->tol2 * S->eta0[r])) { s_be[r] = etan[r] / S->eta[r]; s_cont[r] = 1; }   // R3; l.200
      }
    }
    __syncthreads();
    bool cont[2];
    double be[2];
    for (int r = 0; r < 2; ++r) { cont[r] = upd[r] && s_cont[r]; be[r] = s_be[r]; }
    double ep[2] = {0.0, 0.0};
    for (int i0 = tid; i0 < npad; i0 += 4 * kWG) {  // four elements' loads first
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (!cont[r]) continue;
        const size_t off = (size_t)r * n;
        double pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kWG;
          pv[u] = i < n ? v.p[off + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kWG;
          if (i >= npad) continue;
          const double pn = i < n ? fma(be[r], pv[u], snb[(size_t)r * npad + i]) : 0.0;   // l.201
          vin[(size_t)r * npad + i] = pn;
          ep[r] = fma(pn, pn, ep[r]);
        }
      }
    }
    double ppn[2];
    block_sum2(ep[0], ep[1], red, ppn[0], ppn[1]);
    if (tid == 0) { s_pp[0] = ppn[0]; s_pp[1] = ppn[1]; }
    __syncthreads();
  }
  grid.sync();                          // every CTA has read the old q, s, p
  // ---- C
  if (blockIdx.x == 0) {
    for (int r = 0; r < 2; ++r) {
      if (!act[r]) continue;
      const size_t off = (size_t)r * n;
      if (s_upd[r])
        for (int i = tid; i < n; i += kWG) {
          v.s[off + i] = snb[(size_t)r * npad + i];
          if (s_cont[r]) v.p[off + i] = vin[(size_t)r * npad + i];
        }
      if (tid == 0) {
        S->delta_min[r] = fmin(S->delta_min[r], s_dl[r]);
        S->qq[r] = s_qq[r];
        if (!s_upd[r]) {
          S->active[r] = 0;
          if (s_brk[r]) { S->brk[r] = 1; S->brk_j[r] = S->iter[r]; }
        } else {
          S->count[r] += 1;
          S->iter[r] += 1;
          if (s_cont[r]) { S->eta[r] = s_eta[r]; S->pp[r] = s_pp[r]; }
          else S->active[r] = 0;
        }
      }
    }
  }
  if (!next_q) return;
  bool nq[2];
  for (int r = 0; r < 2; ++r) nq[r] = act[r] && s_cont[r];
  if (!nq[0] && !nq[1]) return;
  for (int i = blockIdx.x * (kWG / 32) + (tid >> 5); i < n; i += nw) {
    const double* Mi = pc.W + (size_t)i * npad;
    double a0 = 0.0, a1 = 0.0;
    row_dot2(Mi, i & ~31, npad, vin, vin + npad, nq[0], nq[1], a0, a1, lane);
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    if (lane < 2 && nq[lane]) v.q[(size_t)lane * n + i] = (lane == 0 ? a0 : a1) * pc.dinv[i];
  }
}

// pcg_init's recurrence part (k_pcg_init after its forward solve): eta_0, the state.
__global__ void __launch_bounds__(kTT) k_wpcg_init_mid(PrecondDev pc, int nrhs, PcgVecs v, PcgState* __restrict__ S) {
  __shared__ double red[32];
  const int r = blockIdx.x, n = pc.n, tid = threadIdx.x;
  if (r >= nrhs) {                      // the unused RHS slot of a 1-RHS solve
    if (tid == 0) {
      S->active[r] = 0; S->count[r] = 0; S->brk[r] = 0; S->brk_j[r] = -1; S->iter[r] = 0;
      S->eta[r] = S->eta0[r] = S->qq[r] = S->pp[r] = 0.0;
      S->delta_min[r] = __longlong_as_double(0x7ff0000000000000ll);
    }
    for (int i = tid; i < n; i += kTT) v.q[(size_t)r * n + i] = 0.0;
    return;
  }
  double e = 0.0;
  for (int i = tid; i < n; i += kTT) e = fma(v.s[(size_t)r * n + i], v.s[(size_t)r * n + i], e);
  const double eta = block_sum(e, red);
  if (tid == 0) {
    S->eta[r] = eta; S->eta0[r] = eta; S->pp[r] = eta;
    S->delta_min[r] = __longlong_as_double(0x7ff0000000000000ll);
    S->active[r] = eta > 0.0; S->count[r] = 0; S->brk[r] = 0; S->brk_j[r] = -1; S->iter[r] = 0;
  }
}

// k_pcg_step between its two solves (same decisions and updates, R3): delta, alpha, omega,
// s, eta', beta, p; q^T q of the current q is formed here (fixed order).
__global__ void __launch_bounds__(kTT) k_wpcg_step_mid(PrecondDev pc, PcgVecs v, const double* __restrict__ passout,
                                                      PcgState* __restrict__ S, int nrhs, int rule, int variant,
                                                      int pass_nrhs) {
  __shared__ double red[32];
  __shared__ double s_alpha, s_beta;
  __shared__ int s_upd, s_cont;
  const int r = blockIdx.x, n = pc.n, tid = threadIdx.x;
  if (r >= nrhs || S->active[r] == 0) return;
  const size_t off = (size_t)r * n;
  const double sig2 = S->sigma2;
  double e = 0.0;
  for (int i = tid; i < n; i += kTT) e = fma(v.q[off + i], v.q[off + i], e);
  const double qq = block_sum(e, red);
  const int iter0 = S->iter[r], count0 = S->count[r];
  const double eta_old = S->eta[r], eta0 = S->eta0[r], tol2 = S->tol2;
  if (tid == 0) {
    s_upd = 0;
    s_alpha = 0.0;
    const double tau = variant == 0 ? passout[(size_t)pass_nrhs * n + r] : S->pp[r];
    const double delta = tau - sig2 * qq;                       // l.194 (R1)
    S->delta_min[r] = fmin(S->delta_min[r], delta);
    S->qq[r] = qq;
    if (!isfinite(delta) || delta == 0.0) {                     // loop guard l.192 (R3)
      S->active[r] = 0;
    } else if (delta < 0.0 && rule == 0) {                      // breakdown (R3)
      S->active[r] = 0; S->brk[r] = 1; S->brk_j[r] = iter0;
    } else {
      s_alpha = eta_old / delta;                                // l.195
      s_upd = 1;
    }
  }
  __syncthreads();
  if (!s_upd) return;
  const double al = s_alpha;
  e = 0.0;
  for (int i = tid; i < n; i += kTT) {
    const double q = v.q[off + i];
    v.omega[off + i] = fma(al, q, v.omega[off + i]);           // l.196
    const double w = variant == 0 ? v.w[off + i] : fma(-sig2, v.w[off + i], v.p[off + i]);   // l.197
    const double sn = fma(-al, w, v.s[off + i]);               // l.198
    v.s[off + i] = sn;
    e = fma(sn, sn, e);
  }
  const double etan = block_sum(e, red);                        // l.199
  if (tid == 0) {
    s_cont = 0;
    if (!(etan <= tol2 * eta0)) { s_beta = etan / eta_old; s_cont = 1; }   // early exit (R3); l.200
  }
  __syncthreads();
  const bool cont = s_cont;
  const double be = s_beta;
  e = 0.0;
  if (cont)
    for (int i = tid; i < n; i += kTT) {
      const double pn = fma(be, v.p[off + i], v.s[off + i]);   // l.201
      v.p[off + i] = pn;
      e = fma(pn, pn, e);
    }
  const double ppn = block_sum(e, red);
  if (tid == 0) {
    S->count[r] = count0 + 1;
    S->iter[r] = iter0 + 1;
    if (cont) { S->eta[r] = etan; S->pp[r] = ppn; }
    else S->active[r] = 0;
  }
}

// ---------------------------------------------------------------- plain apply (API / tests)
// One cluster of kTC CTAs per right-hand side r.  Every CTA of a cluster holds the whole
// vector and computes the same values; only cluster rank 0 writes global memory.
constexpr int kTC = 8;   // CTAs (SMs) per solve, the portable cluster maximum (TLS_TRSV_CLUSTER overrides)
static int trsv_cluster() {
  static const int c = [] {
    const char* e = getenv("TLS_TRSV_CLUSTER");
    const int v = e ? atoi(e) : kTC;
    return (v == 1 || v == 2 || v == 4 || v == 8) ? v : kTC;
  }();
  return c;
}

template <typename T>
__global__ void __launch_bounds__(kTW * 32, 1) k_precond_apply(PrecondDev pc, int trans, double* __restrict__ Y, int ldY) {
  TrsvSm sm = trsv_carve(pc.npad);
  trsv_init(sm, pc.npad);
  const int n = pc.n, npad = pc.npad, r = blockIdx.x / (int)cluster_nctarank();
  const bool rank0 = cluster_ctarank() == 0;
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    double v = i < n ? Y[(size_t)r * ldY + i] : 0.0;
    if (trans) v *= pc.dinv[i];
    sm.y[i] = v;
  }
  if (trans) pre_apply<T, false>(pc, sm);
  else pre_apply<T, true>(pc, sm);
  if (rank0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double v = sm.y[i];
      if (!trans) v *= pc.dinv[i];
      Y[(size_t)r * ldY + i] = v;
    }
}

// ---------------------------------------------------------------- PCGTLS (Alg. 3)
// One cluster per right-hand side r (the two solves of an RQI step are independent
// until the RQI update).  Vectors in global memory have stride n (q feeds the pass
// over A directly).
template <typename T>
__global__ void __launch_bounds__(kTW * 32, 1) k_pcg_init(PrecondDev pc, int nrhs, PcgVecs v, PcgState* __restrict__ S) {
  TrsvSm sm = trsv_carve(pc.npad);
  trsv_init(sm, pc.npad);
  const int n = pc.n, npad = pc.npad, tid = threadIdx.x, r = blockIdx.x / (int)cluster_nctarank();
  const bool rank0 = cluster_ctarank() == 0;
  if (r >= nrhs) {                 // the unused RHS slot of a 1-RHS solve
    if (rank0 && tid == 0) {
      S->active[r] = 0; S->count[r] = 0; S->brk[r] = 0; S->brk_j[r] = -1; S->iter[r] = 0;
      S->eta[r] = S->eta0[r] = S->qq[r] = S->pp[r] = 0.0;
      S->delta_min[r] = __longlong_as_double(0x7ff0000000000000ll);
    }
    // the unused q slot is read by the (2-RHS) operator pass: keep it zero
    if (rank0)
      for (int i = tid; i < pc.n; i += blockDim.x) v.q[(size_t)r * pc.n + i] = 0.0;
    return;
  }
  const size_t off = (size_t)r * n;
  // l.191: s_0 = p_0 = P^{-T} f, eta_0 = ||s_0||^2, omega_0 = 0 (four elements' loads first)
  for (int i0 = tid; i0 < npad; i0 += 4 * (int)blockDim.x) {
    double rv[4], dv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      rv[u] = i < n ? v.rhs[off + i] : 0.0;
      dv[u] = i < n ? pc.dinv[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      if (i < npad) sm.y[i] = i < n ? rv[u] * dv[u] : 0.0;
    }
  }
  pre_apply<T, false>(pc, sm);
  double e = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    const double s = sm.y[i];
    if (rank0) {
      v.s[off + i] = s;
      v.p[off + i] = s;
      v.omega[off + i] = 0.0;
    }
    e = fma(s, s, e);
  }
  const double eta = block_sum(e, sm.red);
  // first q = P^{-1} p (l.193)
  pre_apply<T, true>(pc, sm);
  e = 0.0;
  for (int i0 = tid; i0 < n; i0 += 4 * (int)blockDim.x) {   // the loads of four elements first
    double yv[4], dv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      yv[u] = i < n ? sm.y[i] : 0.0;
      dv[u] = i < n ? pc.dinv[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      if (i < n) {
        const double q = yv[u] * dv[u];
        if (rank0) v.q[off + i] = q;
        e = fma(q, q, e);
      }
    }
  }
  const double qq = block_sum(e, sm.red);
  if (rank0 && tid == 0) {
    S->eta[r] = eta;
    S->eta0[r] = eta;
    S->qq[r] = qq;
    S->pp[r] = eta;            // p_0 = s_0
    S->delta_min[r] = __longlong_as_double(0x7ff0000000000000ll);
    S->active[r] = eta > 0.0;
    S->count[r] = 0;
    S->brk[r] = 0;
    S->brk_j[r] = -1;
    S->iter[r] = 0;
  }
}

// One PCGTLS iteration of RHS r after the pass t = A q_r, v_r = A^T t_r, tau_r = t_r^T t_r
// (passout = [v_0 .. v_{nrhs-1} (stride n), tau_0, tau_1]).  Every CTA of the cluster
// reads its inputs before rank 0 writes anything (cluster barriers), so the replicas
// take identical decisions.
constexpr int kVecPerThread = 16;  // npad <= kTW * 32 * 16 = 4096
// NEXT-3 (partials != nullptr): the operator pass's per-CTA partial rows are reduced here
// instead of by a k_reduce_partials launch: CTA c of RHS r's cluster sums the columns
// [c*cw, (c+1)*cw) of v_r (cw = ceil(n / C)) and CTA 0 also t_r^T t_r, in
// k_reduce_partials' fixed order (8 row groups of the G partial rows, each summed in row
// order, then the group sums in order: the same bits), and stores them into every CTA's
// staging vector through DSMEM; a cluster barrier publishes them.  passout is then unused.
__device__ __forceinline__ void step_reduce_partials(const double* __restrict__ partials, int G, int n, int pass_nrhs,
                                                     int r, double* stage, double* gs) {
  const int C = (int)cluster_nctarank(), c = (int)cluster_ctarank();
  const int tid = threadIdx.x, grp = tid >> 5, tx = tid & 31;
  const int cw = (n + C - 1) / C, c0 = c * cw, c1 = min(n, c0 + cw);
  const size_t Wp = (size_t)pass_nrhs * n + 2;
  const int g0 = G * grp / 8, g1 = G * (grp + 1) / 8;
  const double* base = partials + (size_t)r * n;
  const int cwp = cw + 1;                         // gs: [8][cw + 1], tau in the last column
  for (int cb = c0; cb < c1; cb += 64) {          // 2 column blocks of 32 per pass, 2 x 20 rows in flight
    double acc[2];
    bool ok[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) { acc[k] = 0.0; ok[k] = cb + 32 * k + tx < c1; }
    for (int g = g0; g < g1; g += 20) {
      double vv[20][2];
#pragma unroll
      for (int u = 0; u < 20; ++u)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          vv[u][k] = (ok[k] && g + u < g1) ? base[(size_t)(g + u) * Wp + cb + 32 * k + tx] : 0.0;
#pragma unroll
      for (int u = 0; u < 20; ++u)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (g + u < g1) acc[k] += vv[u][k];
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (ok[k]) gs[grp * cwp + (cb - c0) + 32 * k + tx] = acc[k];
  }
  if (c == 0 && tx == 0) {                        // tau_r = t_r^T t_r (CTA 0: c1 > c0 always)
    double a = 0.0;
    const double* tp = partials + (size_t)pass_nrhs * n + r;
    for (int g = g0; g < g1; g += 20) {           // the group's rows in flight, added in row order
      double vv[20];
#pragma unroll
      for (int u = 0; u < 20; ++u) vv[u] = g + u < g1 ? tp[(size_t)(g + u) * Wp] : 0.0;
#pragma unroll
      for (int u = 0; u < 20; ++u)
        if (g + u < g1) a += vv[u];
    }
    gs[grp * cwp + cw] = a;
  }
  __syncthreads();
  const uint32_t sb = smem_u32(stage);
  for (int j = tid; j <= c1 - c0; j += blockDim.x) {
    const bool tau = j == c1 - c0;
    if (tau && c != 0) continue;
    const int jj = tau ? cw : j;
    double t = gs[jj];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += gs[k * cwp + jj];
    const uint32_t a = sb + (uint32_t)(tau ? n : c0 + j) * 8u;
    for (int q = 0; q < C; ++q) st_cluster_f64(mapa_shared(a, (uint32_t)q), t);
  }
  cluster_sync_all();                             // every CTA's stage is complete
}

template <typename T>
__global__ void __launch_bounds__(kTW * 32, 1) k_pcg_step(PrecondDev pc, PcgVecs v, const double* __restrict__ passout,
                                                       PcgState* __restrict__ S, int nrhs, int rule, int next_q,
                                                       int variant, int pass_nrhs, const int* __restrict__ nq_dev,
                                                       const double* __restrict__ partials, int G) {
  __shared__ double s_alpha, s_beta, s_delta;
  __shared__ int s_upd, s_cont, s_brk, s_exit;
  TrsvSm sm = trsv_carve(pc.npad);
  trsv_init(sm, pc.npad);
  // programmatic dependent launch (round 2 continued): the barrier setup above overlaps the
  // predecessor's tail; wait for its results before reading anything, and let the next operator
  // pass launch now (it waits for this grid's completion before reading anything)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (nq_dev) next_q = *nq_dev;         // graph-captured loop (NEXT-3): decided on the device
  const int r = blockIdx.x / (int)cluster_nctarank();
  const bool rank0 = cluster_ctarank() == 0;
  if (r >= nrhs || S->active[r] == 0) return;
  const int n = pc.n, npad = pc.npad, tid = threadIdx.x;
  const size_t off = (size_t)r * n;
  const double sig2 = S->sigma2;
  // the reduced pass output of this RHS: [v_r (n), tau_r] in shared memory (fused) or passout
  double* stage = sm.y + trsv_smem(npad) / 8;     // after the TRSV layout (launch_pcg_step sizes it)
  const double* pv = passout + off;
  double tau_r = 0.0;
  if (partials != nullptr) {
    step_reduce_partials(partials, G, n, pass_nrhs, r, stage, sm.D);
    pv = stage;
    tau_r = stage[n];
  } else if (variant == 0) {
    tau_r = passout[(size_t)pass_nrhs * n + r];
  }
  if (tid == 0) {
    s_upd = 0;
    s_brk = 0;
    s_exit = 0;
    s_alpha = 0.0;
    // l.194: delta = p^T C p = t^T t - sigma^2 q^T q with the operator of l.324 (variant 0),
    // or p^T p - sigma^2 q^T q as printed (variant 1, the exact-R identity of l.206)
    const double tau = variant == 0 ? tau_r : S->pp[r];
    const double delta = tau - sig2 * S->qq[r];
    s_delta = delta;
    if (!isfinite(delta) || delta == 0.0) {                 // loop guard l.192 (R3)
      s_exit = 1;
    } else if (delta < 0.0 && rule == 0) {                  // breakdown (R3)
      s_exit = 1;
      s_brk = 1;
    } else {
      s_alpha = S->eta[r] / delta;                          // l.195
      s_upd = 1;
    }
  }
  const int iter0 = S->iter[r];
  const double eta_old = S->eta[r], eta0 = S->eta0[r], tol2 = S->tol2, dmin = S->delta_min[r];
  const int count0 = S->count[r];
  cluster_sync_all();   // every CTA has read S before rank 0 updates it
  if (rank0 && tid == 0) {
    S->delta_min[r] = fmin(dmin, s_delta);
    if (s_exit) {
      S->active[r] = 0;
      if (s_brk) { S->brk[r] = 1; S->brk_j[r] = iter0; }
    }
  }
  if (!s_upd) return;
  const double al = s_alpha;
  // omega += alpha q (l.196); y = D^{-1}(A^T t - sigma^2 q) for w = P^{-T}(...) (R1).  Four
  // elements per thread with all their loads issued first (the stores to omega and y could alias
  // the next element's loads for the compiler, which serialised the round trips)
  for (int i0 = tid; i0 < npad; i0 += 4 * (int)blockDim.x) {
    double qv[4], ov[4], pvv[4], dv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      const bool ok = i < n;
      qv[u] = ok ? v.q[off + i] : 0.0;
      ov[u] = (ok && rank0) ? v.omega[off + i] : 0.0;
      pvv[u] = (ok && variant == 0) ? pv[i] : 0.0;
      dv[u] = ok ? pc.dinv[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      if (i >= npad) continue;
      double yv = 0.0;
      if (i < n) {
        if (rank0) v.omega[off + i] = fma(al, qv[u], ov[u]);
        // variant 0: w = P^{-T}(A^T t - sigma^2 q); variant 1: solve P^{-T} q (l.197)
        yv = (variant == 0 ? pvv[u] - sig2 * qv[u] : qv[u]) * dv[u];
      }
      sm.y[i] = yv;
    }
  }
  pre_apply<T, false>(pc, sm);
  // s -= alpha w (l.198), eta' = ||s||^2 (l.199); kept in registers until every CTA has read s, p
  double sn[kVecPerThread], pn[kVecPerThread];
  double e = 0.0;
#pragma unroll
  for (int k = 0; k < kVecPerThread; ++k) {      // pn[] holds the old p until the update below
    const int i = tid + k * (int)blockDim.x;
    pn[k] = i < n ? v.p[off + i] : 0.0;
    sn[k] = i < n ? v.s[off + i] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < kVecPerThread; ++k) {
    const int i = tid + k * (int)blockDim.x;
    if (i < n) {
      // w = solve result (variant 0) or p - sigma^2 P^{-T} q (variant 1, l.197-198)
      const double w = variant == 0 ? sm.y[i] : fma(-sig2, sm.y[i], pn[k]);
      sn[k] = fma(-al, w, sn[k]);
      e = fma(sn[k], sn[k], e);
    }
  }
  const double etan = block_sum(e, sm.red);
  if (tid == 0) {
    s_cont = 0;
    if (!(etan <= tol2 * eta0)) {                           // early exit (R3)
      s_beta = etan / eta_old;                              // l.200
      s_cont = 1;
    }
  }
  __syncthreads();
  const bool cont = s_cont;
  const double be = s_beta;
  // p = s + beta p (l.201)
  double ppl = 0.0;
#pragma unroll
  for (int k = 0; k < kVecPerThread; ++k) {
    const int i = tid + k * (int)blockDim.x;
    pn[k] = (cont && i < n) ? fma(be, pn[k], sn[k]) : 0.0;
    if (i < npad) sm.y[i] = pn[k];
    ppl = fma(pn[k], pn[k], ppl);
  }
  const double ppn = block_sum(ppl, sm.red);
  cluster_sync_all();   // every CTA has read the old s and p
  if (rank0) {
#pragma unroll
    for (int k = 0; k < kVecPerThread; ++k) {
      const int i = tid + k * (int)blockDim.x;
      if (i < n) {
        v.s[off + i] = sn[k];
        if (cont) v.p[off + i] = pn[k];
      }
    }
    if (tid == 0) {
      S->count[r] = count0 + 1;
      S->iter[r] = iter0 + 1;
      if (cont) { S->eta[r] = etan; S->pp[r] = ppn; }
      else S->active[r] = 0;
    }
  }
  if (!cont || !next_q) return;
  // next q = P^{-1} p (l.193 of the next iteration)
  pre_apply<T, true>(pc, sm);
  e = 0.0;
  for (int i0 = tid; i0 < n; i0 += 4 * (int)blockDim.x) {   // the loads of four elements first
    double yv[4], dv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      yv[u] = i < n ? sm.y[i] : 0.0;
      dv[u] = i < n ? pc.dinv[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      if (i < n) {
        const double q = yv[u] * dv[u];
        if (rank0) v.q[off + i] = q;
        e = fma(q, q, e);
      }
    }
  }
  const double qq = block_sum(e, sm.red);
  if (rank0 && tid == 0) S->qq[r] = qq;
}

// ---------------------------------------------------------------- RQI (Alg. 4)
// passout = [v = A^T r (n), rho = r^T r, gamma = b^T r] for r = b - A x_k.
__global__ void __launch_bounds__(kTT) k_rqi_eval(int n, const double* __restrict__ passout, const double* __restrict__ x,
                                                   PcgVecs v, PcgState* __restrict__ S) {
  __shared__ double red[32];
  const int tid = threadIdx.x;
  double e = 0.0;
  for (int i = tid; i < n; i += kTT) e = fma(x[i], x[i], e);
  const double xx = block_sum(e, red);
  const double rho = passout[n], gam = passout[n + 1];
  const double sig2 = rho / (1.0 + xx);                    // l.240
  double ff = 0.0;
  for (int i = tid; i < n; i += kTT) {
    const double f = -passout[i] - sig2 * x[i];             // l.242
    v.rhs[i] = -f;                                          // RHS (a) of l.246
    v.rhs[(size_t)n + i] = x[i];                            // RHS (b) of l.252
    ff = fma(f, f, ff);
  }
  ff = block_sum(ff, red);
  if (tid == 0) {
    const double g = -gam + sig2;                           // l.244
    S->sigma2 = sig2;
    S->g = g;
    S->xx = xx;
    S->psi = sqrt((ff + g * g) / (xx + 1.0));               // Eq. psik, l.262
  }
}

// z = x + omega_a (l.248); beta = (z^T f - g)/(z^T x + 1) (l.250); x' = z + beta omega_b (l.254).
__global__ void __launch_bounds__(kTT) k_rqi_update(int n, PcgVecs v, const PcgState* __restrict__ S,
                                                     double* __restrict__ x, double* __restrict__ x_prev) {
  if (S->brk[0] | S->brk[1]) return;   // PCG breakdown: the host returns x_k (read with the next state)
  __shared__ double red[32];
  const int tid = threadIdx.x;
  double zf = 0.0, zx = 0.0;
  for (int i = tid; i < n; i += kTT) {
    const double z = x[i] + v.omega[i];
    zf = fma(z, -v.rhs[i], zf);                             // rhs_a = -f
    zx = fma(z, x[i], zx);
  }
  zf = block_sum(zf, red);
  zx = block_sum(zx, red);
  const double beta = (zf - S->g) / (zx + 1.0);
  for (int i = tid; i < n; i += kTT) {
    const double xi = x[i];
    const double z = xi + v.omega[i];
    x_prev[i] = xi;
    x[i] = fma(beta, v.omega[(size_t)n + i], z);
  }
}

// l.227-235: sigma_0^2 = r_0^T r_0/(1 + x_0^T x_0); u_0 = P^{-1} P^{-T} x_0 (R9); x_1 = x_0 + sigma_0^2 u_0.
template <typename T>
__global__ void __launch_bounds__(kTW * 32, 1) k_boot_x1(PrecondDev pc, const double* __restrict__ passout,
                                                      const double* __restrict__ x0, double* __restrict__ x1) {
  TrsvSm sm = trsv_carve(pc.npad);
  trsv_init(sm, pc.npad);
  const int n = pc.n, npad = pc.npad, tid = threadIdx.x;
  double e = 0.0;
  for (int i = tid; i < npad; i += blockDim.x) {
    const double xv = i < n ? x0[i] : 0.0;
    e = fma(xv, xv, e);
    sm.y[i] = i < n ? xv * pc.dinv[i] : 0.0;
  }
  const double xx = block_sum(e, sm.red);
  const double sig0 = passout[n] / (1.0 + xx);
  pre_apply<T, false>(pc, sm);
  pre_apply<T, true>(pc, sm);
  if (cluster_ctarank() == 0)
    for (int i = tid; i < n; i += blockDim.x) x1[i] = fma(sig0, sm.y[i] * pc.dinv[i], x0[i]);
}

// ---------------------------------------------------------------- launchers
template <typename F>
static int set_smem(F kern, size_t bytes) {
  TLS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return 0;
}

#define TLS_DISPATCH_UF(uf, ...)                          \
  switch (uf) {                                           \
    case TLS_FP16: { using T = F16s; __VA_ARGS__; } break;  \
    case TLS_BF16: { using T = B16s; __VA_ARGS__; } break;  \
    case TLS_FP32: { using T = float; __VA_ARGS__; } break; \
    default: { using T = double; __VA_ARGS__; } break;      \
  }

// kTC-CTA clusters (one per right-hand side) of the single-CTA TRSV kernels
// pdl: programmatic stream serialisation (the kernel must execute griddepcontrol.wait before it
// reads its predecessor's results)
template <typename... KArgs, typename... Args>
static int launch_cluster_pdl(void (*kern)(KArgs...), int clusters, size_t smem, cudaStream_t st, bool pdl,
                              Args... args) {
  TLS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  const int C = trsv_cluster();
  cfg.gridDim = dim3(clusters * C);
  cfg.blockDim = dim3(kTW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  TLS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
  return 0;
}

template <typename... KArgs, typename... Args>
static int launch_cluster(void (*kern)(KArgs...), int clusters, size_t smem, cudaStream_t st, Args... args) {
  return launch_cluster_pdl(kern, clusters, smem, st, false, args...);
}

int launch_precond_apply(const PrecondDev& pc, int trans, int nrhs, double* Y, int ldY, cudaStream_t st) {
  const size_t sm = trsv_smem(pc.npad);
  int rc = 0;
#ifdef TLS_TRSV_TRACE
  const char* tpath = getenv("TLS_TRSV_TRACE");
#else
  const char* tpath = nullptr;
#endif
  static unsigned long long* tbuf = nullptr;
  const int NB = pc.npad / 32;
  if (tpath) {
    if (!tbuf) TLS_CUDA_TRY(cudaMalloc(&tbuf, 6 * 8 * 256));
    TLS_CUDA_TRY(cudaMemsetAsync(tbuf, 0, 6 * 8 * 256, st));
#ifdef TLS_TRSV_TRACE
    TLS_CUDA_TRY(cudaMemcpyToSymbolAsync(g_trsv_trace, &tbuf, sizeof(tbuf), 0, cudaMemcpyHostToDevice, st));
#endif
  }
  TLS_DISPATCH_UF(pc.u_f, { rc = launch_cluster(k_precond_apply<T>, nrhs, sm, st, pc, trans, Y, ldY); });
  if (tpath && rc == 0 && NB <= 256) {
#ifdef TLS_TRSV_TRACE
    unsigned long long* none = nullptr;
    TLS_CUDA_TRY(cudaMemcpyToSymbolAsync(g_trsv_trace, &none, sizeof(none), 0, cudaMemcpyHostToDevice, st));
#endif
    std::vector<unsigned long long> h(6 * (size_t)NB);
    TLS_CUDA_TRY(cudaMemcpyAsync(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost, st));
    TLS_CUDA_TRY(cudaStreamSynchronize(st));
    FILE* f = fopen(tpath, "w");
    if (f) {
      for (int u = 0; u < NB; ++u)
        fprintf(f, "%llu %llu %llu %llu %llu %llu\n", h[6 * u], h[6 * u + 1], h[6 * u + 2], h[6 * u + 3], h[6 * u + 4],
                h[6 * u + 5]);
      fclose(f);
    }
  }
  return rc;
}

static int wgemv_grid_launch(const PrecondDev& pc, PcgVecs v, const double* passout, const PcgState* S, int nrhs,
                             int mode, int variant, int all, cudaStream_t st) {
  const size_t smem = 2 * (size_t)pc.npad * 8;
  static size_t attr = 0;
  if (attr < smem) {
    TLS_CUDA_TRY(cudaFuncSetAttribute(k_wgemv_grid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  int g = (pc.n + kWG / 32 - 1) / (kWG / 32);
  if (g > num_sms()) g = num_sms();
  k_wgemv_grid<<<g, kWG, smem, st>>>(pc, v, passout, S, nrhs, mode, variant, all);
  TLS_LAUNCH_CHECK();
  return 0;
}

int launch_pcg_init(const PrecondDev& pc, int nrhs, PcgVecs v, PcgState* S, cudaStream_t st) {
  if (pc.W != nullptr) {                 // R24: three kernels, no substitution chain
    int rc = wgemv_grid_launch(pc, v, nullptr, S, nrhs, 0, 0, 1, st);
    if (rc) return rc;
    k_wpcg_init_mid<<<2, kTT, 0, st>>>(pc, nrhs, v, S);
    TLS_LAUNCH_CHECK();
    return wgemv_grid_launch(pc, v, nullptr, S, nrhs, 2, 0, 1, st);
  }
  const size_t sm = trsv_smem(pc.npad);
  int rc = 0;
  TLS_DISPATCH_UF(pc.u_f, { rc = launch_cluster(k_pcg_init<T>, 2, sm, st, pc, nrhs, v, S); });
  return rc;
}

int launch_pcg_step(const PrecondDev& pc, PcgVecs v, const double* passout, PcgState* S, int nrhs, int rule,
                    int next_q, int variant, int pass_nrhs, cudaStream_t st, const double* partials, int G,
                    const int* nq_dev) {
  if (pc.W != nullptr) {                 // R24: one cooperative kernel over every SM
    const size_t dbl = 4 * (size_t)pc.npad > 2 * (size_t)pc.npad + 264 ? 4 * (size_t)pc.npad : 2 * (size_t)pc.npad + 264;
    const size_t smem = dbl * 8;
    static size_t attr = 0;
    if (attr < smem) {
      TLS_CUDA_TRY(cudaFuncSetAttribute(k_wpcg_step_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = smem;
    }
    int g = (pc.n + kWG / 32 - 1) / (kWG / 32);
    if (g > num_sms()) g = num_sms();
    // TLS_WSTEP_CTAS=k caps the cooperative grid (fewer CTAs: cheaper grid barriers, longer GEMVs)
    static const int cap = [] { const char* e = getenv("TLS_WSTEP_CTAS"); return e ? atoi(e) : 0; }();
    if (cap > 0 && g > cap) g = cap;
    double* pout = const_cast<double*>(passout);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(kWG);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pass_pdl() ? 2 : 1;
    TLS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_wpcg_step_coop, pc, v, passout, S, nrhs, rule, next_q, variant, pass_nrhs,
                                    partials, G, pout, nq_dev));
    return 0;
  }
  // partials: the fused reduction (step_reduce_partials) needs a staging vector after the TRSV layout
  const size_t sm = trsv_smem(pc.npad) + (partials ? ((size_t)pc.npad + 32) * 8 : 0);
  int rc = 0;
  TLS_DISPATCH_UF(pc.u_f, { rc = launch_cluster_pdl(k_pcg_step<T>, nrhs, sm, st, pass_pdl(), pc, v, passout, S, nrhs,
                                                    rule, next_q, variant, pass_nrhs, nq_dev, partials, G); });
  return rc;
}

int launch_rqi_eval(const PrecondDev& pc, const double* passout, const double* x, PcgVecs v, PcgState* S,
                    cudaStream_t st) {
  k_rqi_eval<<<1, kTT, 0, st>>>(pc.n, passout, x, v, S);
  TLS_LAUNCH_CHECK();
  return 0;
}

int launch_rqi_update(const PrecondDev& pc, PcgVecs v, const PcgState* S, double* x, double* x_prev,
                      cudaStream_t st) {
  k_rqi_update<<<1, kTT, 0, st>>>(pc.n, v, S, x, x_prev);
  TLS_LAUNCH_CHECK();
  return 0;
}

int launch_boot_x1(const PrecondDev& pc, const double* passout_r0, const double* x0, double* x1, cudaStream_t st) {
  const size_t sm = trsv_smem(pc.npad);
  int rc = 0;
  TLS_DISPATCH_UF(pc.u_f, { rc = launch_cluster(k_boot_x1<T>, 1, sm, st, pc, passout_r0, x0, x1); });
  return rc;
}

int launch_trtri(const PrecondDev& pc, double* W, double* WT, cudaStream_t st) {
  const size_t smem = (size_t)pc.npad * 4 * 8 + (kTriW + 1) * 32 * 4 * 8 + 1024 * 8;
  TLS_CUDA_TRY(cudaMemsetAsync(W, 0, (size_t)pc.npad * pc.npad * 8, st));
  TLS_CUDA_TRY(cudaMemsetAsync(WT, 0, (size_t)pc.npad * pc.npad * 8, st));
  int rc = 0;
  TLS_DISPATCH_UF(pc.u_f, {
    static size_t attr = 0;
    if (attr < smem) {
      TLS_CUDA_TRY(cudaFuncSetAttribute(k_trtri<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = smem;
    }
    k_trtri<T><<<(pc.npad / 32) * 8, kTriT, smem, st>>>(pc, W, WT);
  });
  TLS_LAUNCH_CHECK();
  return rc;
}

}  // namespace tls
