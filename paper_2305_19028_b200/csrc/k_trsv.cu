// k_trsv.cu — preconditioner solves with the stored-low R~ and the fused PCG /
// RQI vector kernels.
//
//   back   q = P^{-1} p  = D^{-1} (R~^{-1} p)      (Alg. 3 l.193)
//   fwd    w = P^{-T} y  = R~^{-T} (D^{-1} y)      (Alg. 3 l.191, l.197)
// Both are blocked column sweeps over 32-row blocks inside ONE CTA (the
// n-vectors live in shared memory): a warp solves the 32x32 diagonal block
// with the fp64 inverse of R~_kk (staged ahead by cp.async into shared
// memory), then all warps apply the block to the remaining rows, streaming
// 32-element row segments of R~ (back) or R~^T (fwd) from L2 in u_f and
// upcasting on load.  Loads of the segments are issued before the diagonal
// solve so their latency overlaps it.  Both right-hand sides of the batched
// PCG (RHS a: -f, RHS b: x_k) are solved together.
//
// The PCG recurrences of Alg. 3 (delta, alpha, omega, s, eta, beta, p;
// PAPER.md l.191-201 with the A-in-loop operator of l.324, reading R1) are
// fused into k_pcg_step around the forward solve, followed by the next
// iteration's back solve; the RQI updates of Alg. 4 (l.238-255) live in
// k_rqi_eval / k_rqi_update / k_boot_x1.  All reductions are fixed-order.
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

// Warp 0 stages the 32x32 fp64 inverse block `src` (8 KB) into `dst` (smem).
__device__ __forceinline__ void stage_dinv(double* dst, const double* src) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 16; ++k) cp_async16(dst + (k * 32 + lane) * 2, src + (k * 32 + lane) * 2);
  cp_async_commit();
}

// Row-block update y[r][i] -= sum_l M[i][c0+l] x_r[l] (x_r = y[r][c0..c0+31]) for the
// rows i = i0 + tid + k*kTT (k < MAXR) with lo <= i < hi.  For 16-bit u_f the
// 32-value row segments are loaded before the diagonal solve (PF, latency
// overlap); wide types load them in the loop.
template <typename T, int NRHS, int MAXR>
struct RowUpd {
  static constexpr int NV = SegTraits<T>::NV;
  static constexpr bool PF = MAXR * NV <= 16;
  uint4 raw[PF ? MAXR : 1][NV];
  __device__ __forceinline__ void prefetch(const T* __restrict__ M, int npad, int c0, int i0, int lo, int hi) {
    if constexpr (PF) {
#pragma unroll
      for (int k = 0; k < MAXR; ++k) {
        const int i = i0 + (int)threadIdx.x + k * kTT;
        if (i >= lo && i < hi) seg_load<T>(M + (size_t)i * npad + c0, raw[k]);
      }
    }
  }
  __device__ __forceinline__ void apply(const T* __restrict__ M, int npad, int c0, int i0, int lo, int hi, double* y) {
    double s[MAXR][NRHS];
#pragma unroll
    for (int k = 0; k < MAXR; ++k)
#pragma unroll
      for (int r = 0; r < NRHS; ++r) s[k][r] = 0.0;
    if constexpr (PF) {
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        double xv[NRHS];
#pragma unroll
        for (int r = 0; r < NRHS; ++r) xv[r] = y[r * npad + c0 + l];
#pragma unroll
        for (int k = 0; k < MAXR; ++k) {
          const int i = i0 + (int)threadIdx.x + k * kTT;
          if (i >= lo && i < hi) {
            const double a = seg_get<T>(raw[k], l);
#pragma unroll
            for (int r = 0; r < NRHS; ++r) s[k][r] = fma(a, xv[r], s[k][r]);
          }
        }
      }
    } else {
#pragma unroll 1
      for (int k = 0; k < MAXR; ++k) {
        const int i = i0 + (int)threadIdx.x + k * kTT;
        if (i >= lo && i < hi) {
          seg_load<T>(M + (size_t)i * npad + c0, raw[0]);
#pragma unroll
          for (int l = 0; l < 32; ++l) {
            const double a = seg_get<T>(raw[0], l);
#pragma unroll
            for (int r = 0; r < NRHS; ++r) s[k][r] = fma(a, y[r * npad + c0 + l], s[k][r]);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
      const int i = i0 + (int)threadIdx.x + k * kTT;
      if (i >= lo && i < hi) {
#pragma unroll
        for (int r = 0; r < NRHS; ++r) y[r * npad + i] -= s[k][r];
      }
    }
  }
};

// Warp 0: x_blk = D x_blk with the staged 32x32 block, D[l][lane] layout.
template <int NRHS>
__device__ __forceinline__ void diag_block(const double* D, int npad, int c0, double* y) {
  const int lane = threadIdx.x & 31;
  double acc[NRHS];
#pragma unroll
  for (int r = 0; r < NRHS; ++r) acc[r] = 0.0;
#pragma unroll 8
  for (int l = 0; l < 32; ++l) {
    const double dv = D[l * 32 + lane];
#pragma unroll
    for (int r = 0; r < NRHS; ++r) acc[r] = fma(dv, y[r * npad + c0 + l], acc[r]);
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < NRHS; ++r) y[r * npad + c0 + lane] = acc[r];
}

// y: smem [NRHS][npad].  Solves R~ x = y (upper, back substitution) in place.
// Rrow: R~ row-major; DinvB[kb][l][i] = (R~_kk^{-1})[i][l].  dbuf: smem 2 x 1024 doubles.
template <typename T, int NRHS, int MAXR>
__device__ void trsv_back(const T* __restrict__ Rrow, const double* __restrict__ DinvB, int npad, double* y,
                          double* dbuf) {
  const int warp = threadIdx.x >> 5;
  const int NB = npad >> 5;
  if (warp == 0) stage_dinv(dbuf + ((NB - 1) & 1) * 1024, DinvB + (size_t)(NB - 1) * 1024);
  for (int jb = NB - 1; jb >= 0; --jb) {
    const int c0 = jb * 32;
    RowUpd<T, NRHS, MAXR> upd;
    upd.prefetch(Rrow, npad, c0, 0, 0, c0);       // rows i < c0
    if (warp == 0) {
      if (jb > 0) {
        stage_dinv(dbuf + ((jb - 1) & 1) * 1024, DinvB + (size_t)(jb - 1) * 1024);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      diag_block<NRHS>(dbuf + (jb & 1) * 1024, npad, c0, y);
    }
    __syncthreads();
    if (c0 > 0) upd.apply(Rrow, npad, c0, 0, 0, c0, y);
    __syncthreads();
  }
}

// Solves R~^T x = y (lower, forward substitution) in place.
// RTrow: R~^T row-major; DinvF[kb][l][i] = (R~_kk^{-1})[l][i].
template <typename T, int NRHS, int MAXR>
__device__ void trsv_fwd(const T* __restrict__ RTrow, const double* __restrict__ DinvF, int npad, double* y,
                         double* dbuf) {
  const int warp = threadIdx.x >> 5;
  const int NB = npad >> 5;
  if (warp == 0) stage_dinv(dbuf, DinvF);
  for (int jb = 0; jb < NB; ++jb) {
    const int c0 = jb * 32, c1 = c0 + 32;
    RowUpd<T, NRHS, MAXR> upd;
    upd.prefetch(RTrow, npad, c0, c1, c1, npad);  // rows i >= c1
    if (warp == 0) {
      if (jb + 1 < NB) {
        stage_dinv(dbuf + ((jb + 1) & 1) * 1024, DinvF + (size_t)(jb + 1) * 1024);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      diag_block<NRHS>(dbuf + (jb & 1) * 1024, npad, c0, y);
    }
    __syncthreads();
    if (c1 < npad) upd.apply(RTrow, npad, c0, c1, c1, npad, y);
    __syncthreads();
  }
}

// dynamic smem of the single-CTA kernels: y [2][npad] + dbuf [2][1024] + red [32]
static size_t vec_smem(int npad) { return (size_t)(2 * npad + 2048 + 32) * 8; }

struct VecSmem {
  double* y;
  double* dbuf;
  double* red;
};
__device__ __forceinline__ VecSmem carve(int npad) {
  extern __shared__ __align__(16) double vsm[];
  return VecSmem{vsm, vsm + 2 * npad, vsm + 2 * npad + 2048};
}

// ---------------------------------------------------------------- plain apply (API / tests)
template <typename T, int NRHS, int MAXR>
__global__ void __launch_bounds__(kTT) k_precond_apply(PrecondDev pc, int trans, double* __restrict__ Y, int ldY) {
  VecSmem sm = carve(pc.npad);
  const int n = pc.n, npad = pc.npad;
  for (int r = 0; r < NRHS; ++r)
    for (int i = threadIdx.x; i < npad; i += kTT) {
      double v = i < n ? Y[(size_t)r * ldY + i] : 0.0;
      if (trans) v *= pc.dinv[i];
      sm.y[r * npad + i] = v;
    }
  __syncthreads();
  if (trans) trsv_fwd<T, NRHS, MAXR>((const T*)pc.RTrow, pc.DinvF, npad, sm.y, sm.dbuf);
  else trsv_back<T, NRHS, MAXR>((const T*)pc.Rrow, pc.DinvB, npad, sm.y, sm.dbuf);
  for (int r = 0; r < NRHS; ++r)
    for (int i = threadIdx.x; i < n; i += kTT) {
      double v = sm.y[r * npad + i];
      if (!trans) v *= pc.dinv[i];
      Y[(size_t)r * ldY + i] = v;
    }
}

// ---------------------------------------------------------------- PCGTLS (Alg. 3)
// Vectors in global memory have stride n (q feeds the pass over A directly).
template <typename T, int MAXR>
__global__ void __launch_bounds__(kTT) k_pcg_init(PrecondDev pc, int nrhs, PcgVecs v, PcgState* __restrict__ S) {
  VecSmem sm = carve(pc.npad);
  const int n = pc.n, npad = pc.npad, tid = threadIdx.x;
  // l.191: s_0 = p_0 = P^{-T} f, eta_0 = ||s_0||^2, omega_0 = 0
  for (int r = 0; r < 2; ++r)
    for (int i = tid; i < npad; i += kTT)
      sm.y[r * npad + i] = (r < nrhs && i < n) ? v.rhs[(size_t)r * n + i] * pc.dinv[i] : 0.0;
  __syncthreads();
  trsv_fwd<T, 2, MAXR>((const T*)pc.RTrow, pc.DinvF, npad, sm.y, sm.dbuf);
  double eta[2];
  for (int r = 0; r < 2; ++r) {
    double e = 0.0;
    for (int i = tid; i < n; i += kTT) {
      const double s = sm.y[r * npad + i];
      v.s[(size_t)r * n + i] = s;
      v.p[(size_t)r * n + i] = s;
      v.omega[(size_t)r * n + i] = 0.0;
      e = fma(s, s, e);
    }
    eta[r] = block_sum(e, sm.red);
  }
  // first q = P^{-1} p (l.193)
  trsv_back<T, 2, MAXR>((const T*)pc.Rrow, pc.DinvB, npad, sm.y, sm.dbuf);
  double qq[2];
  for (int r = 0; r < 2; ++r) {
    double e = 0.0;
    for (int i = tid; i < n; i += kTT) {
      const double q = sm.y[r * npad + i] * pc.dinv[i];
      v.q[(size_t)r * n + i] = q;
      e = fma(q, q, e);
    }
    qq[r] = block_sum(e, sm.red);
  }
  if (tid == 0) {
    int any = 0;
    for (int r = 0; r < 2; ++r) {
      const bool on = r < nrhs && eta[r] > 0.0;
      S->eta[r] = eta[r];
      S->eta0[r] = eta[r];
      S->qq[r] = qq[r];
      S->delta_min[r] = __longlong_as_double(0x7ff0000000000000ll);
      S->active[r] = on;
      S->count[r] = 0;
      S->brk[r] = 0;
      S->brk_j[r] = -1;
      any |= on;
    }
    S->any_active = any;
    S->nrhs = nrhs;
    S->iter = 0;
  }
}

// One PCGTLS iteration after the pass t = A q_r, v_r = A^T t_r, tau_r = t_r^T t_r
// (passout = [v_0 .. v_{nrhs-1} (stride n), tau_0, tau_1]).
template <typename T, int MAXR>
__global__ void __launch_bounds__(kTT) k_pcg_step(PrecondDev pc, PcgVecs v, const double* __restrict__ passout,
                                                   PcgState* __restrict__ S, int rule, int next_q) {
  __shared__ double s_alpha[2], s_beta[2];
  __shared__ int s_upd[2], s_cont[2];
  if (S->any_active == 0) return;
  VecSmem sm = carve(pc.npad);
  const int n = pc.n, npad = pc.npad, tid = threadIdx.x;
  const int nrhs = S->nrhs;
  const double sig2 = S->sigma2;
  if (tid == 0) {
    for (int r = 0; r < 2; ++r) {
      s_upd[r] = 0;
      s_alpha[r] = 0.0;
      if (r >= nrhs || !S->active[r]) continue;
      const double tau = passout[(size_t)nrhs * n + r];
      const double delta = tau - sig2 * S->qq[r];          // l.194 with the operator of l.324
      S->delta_min[r] = fmin(S->delta_min[r], delta);
      if (!isfinite(delta) || delta == 0.0) {               // loop guard l.192 (R3)
        S->active[r] = 0;
      } else if (delta < 0.0 && rule == 0) {                // breakdown (R3)
        S->active[r] = 0;
        S->brk[r] = 1;
        S->brk_j[r] = S->iter;
      } else {
        s_alpha[r] = S->eta[r] / delta;                     // l.195
        s_upd[r] = 1;
      }
    }
  }
  __syncthreads();
  // omega += alpha q (l.196); y = D^{-1}(A^T t - sigma^2 q) for w = P^{-T}(...) (R1)
  for (int r = 0; r < 2; ++r) {
    const bool u = s_upd[r];
    const double al = s_alpha[r];
    for (int i = tid; i < npad; i += kTT) {
      double yv = 0.0;
      if (u && i < n) {
        const double q = v.q[(size_t)r * n + i];
        v.omega[(size_t)r * n + i] = fma(al, q, v.omega[(size_t)r * n + i]);
        yv = (passout[(size_t)r * n + i] - sig2 * q) * pc.dinv[i];
      }
      sm.y[r * npad + i] = yv;
    }
  }
  __syncthreads();
  trsv_fwd<T, 2, MAXR>((const T*)pc.RTrow, pc.DinvF, npad, sm.y, sm.dbuf);
  // s -= alpha w (l.198), eta' = ||s||^2 (l.199)
  double etan[2];
  for (int r = 0; r < 2; ++r) {
    double e = 0.0;
    if (s_upd[r]) {
      const double al = s_alpha[r];
      for (int i = tid; i < n; i += kTT) {
        const double s = fma(-al, sm.y[r * npad + i], v.s[(size_t)r * n + i]);
        v.s[(size_t)r * n + i] = s;
        e = fma(s, s, e);
      }
    }
    etan[r] = block_sum(e, sm.red);
  }
  if (tid == 0) {
    for (int r = 0; r < 2; ++r) {
      s_cont[r] = 0;
      if (!s_upd[r]) continue;
      S->count[r] += 1;
      if (etan[r] <= S->tol2 * S->eta0[r]) {                // early exit (R3)
        S->active[r] = 0;
      } else {
        s_beta[r] = etan[r] / S->eta[r];                    // l.200
        S->eta[r] = etan[r];
        s_cont[r] = 1;
      }
    }
    S->iter += 1;
    S->any_active = (S->active[0] != 0) | (S->active[1] != 0);
  }
  __syncthreads();
  // p = s + beta p (l.201)
  for (int r = 0; r < 2; ++r) {
    const bool c = s_cont[r];
    const double be = s_beta[r];
    for (int i = tid; i < npad; i += kTT) {
      double pv = 0.0;
      if (c && i < n) {
        pv = fma(be, v.p[(size_t)r * n + i], v.s[(size_t)r * n + i]);
        v.p[(size_t)r * n + i] = pv;
      }
      sm.y[r * npad + i] = pv;
    }
  }
  if (!next_q || !(s_cont[0] || s_cont[1])) return;
  __syncthreads();
  // next q = P^{-1} p (l.193 of the next iteration)
  trsv_back<T, 2, MAXR>((const T*)pc.Rrow, pc.DinvB, npad, sm.y, sm.dbuf);
  double qq[2];
  for (int r = 0; r < 2; ++r) {
    double e = 0.0;
    if (s_cont[r]) {
      for (int i = tid; i < n; i += kTT) {
        const double q = sm.y[r * npad + i] * pc.dinv[i];
        v.q[(size_t)r * n + i] = q;
        e = fma(q, q, e);
      }
    }
    qq[r] = block_sum(e, sm.red);
  }
  if (tid == 0)
    for (int r = 0; r < 2; ++r)
      if (s_cont[r]) S->qq[r] = qq[r];
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
template <typename T, int MAXR>
__global__ void __launch_bounds__(kTT) k_boot_x1(PrecondDev pc, const double* __restrict__ passout,
                                                  const double* __restrict__ x0, double* __restrict__ x1) {
  VecSmem sm = carve(pc.npad);
  const int n = pc.n, npad = pc.npad, tid = threadIdx.x;
  double e = 0.0;
  for (int i = tid; i < npad; i += kTT) {
    const double xv = i < n ? x0[i] : 0.0;
    e = fma(xv, xv, e);
    sm.y[i] = i < n ? xv * pc.dinv[i] : 0.0;
  }
  const double xx = block_sum(e, sm.red);
  const double sig0 = passout[n] / (1.0 + xx);
  trsv_fwd<T, 1, MAXR>((const T*)pc.RTrow, pc.DinvF, npad, sm.y, sm.dbuf);
  trsv_back<T, 1, MAXR>((const T*)pc.Rrow, pc.DinvB, npad, sm.y, sm.dbuf);
  for (int i = tid; i < n; i += kTT) x1[i] = fma(sig0, sm.y[i] * pc.dinv[i], x0[i]);
}

// ---------------------------------------------------------------- launchers
template <typename F>
static int set_smem(F kern, size_t bytes) {
  TLS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return 0;
}

#define TLS_DISPATCH_MAXR(npad, ...)                                   \
  do {                                                                 \
    const int _rows = ((npad) + kTT - 1) / kTT;                        \
    if (_rows <= 1) { constexpr int MAXR = 1; __VA_ARGS__; }           \
    else if (_rows <= 2) { constexpr int MAXR = 2; __VA_ARGS__; }      \
    else if (_rows <= 4) { constexpr int MAXR = 4; __VA_ARGS__; }      \
    else { constexpr int MAXR = 8; __VA_ARGS__; }                      \
  } while (0)

#define TLS_DISPATCH_UF(uf, ...)                          \
  switch (uf) {                                           \
    case TLS_FP16: { using T = F16s; __VA_ARGS__; } break;  \
    case TLS_BF16: { using T = B16s; __VA_ARGS__; } break;  \
    case TLS_FP32: { using T = float; __VA_ARGS__; } break; \
    default: { using T = double; __VA_ARGS__; } break;      \
  }

int launch_precond_apply(const PrecondDev& pc, int trans, int nrhs, double* Y, int ldY, cudaStream_t st) {
  const size_t sm = vec_smem(pc.npad);
  int rc = 0;
  TLS_DISPATCH_UF(pc.u_f, TLS_DISPATCH_MAXR(pc.npad, {
    if (nrhs == 1) {
      if ((rc = set_smem(k_precond_apply<T, 1, MAXR>, sm))) return rc;
      k_precond_apply<T, 1, MAXR><<<1, kTT, sm, st>>>(pc, trans, Y, ldY);
    } else {
      if ((rc = set_smem(k_precond_apply<T, 2, MAXR>, sm))) return rc;
      k_precond_apply<T, 2, MAXR><<<1, kTT, sm, st>>>(pc, trans, Y, ldY);
    }
  }));
  TLS_LAUNCH_CHECK();
  return 0;
}

int launch_pcg_init(const PrecondDev& pc, int nrhs, PcgVecs v, PcgState* S, cudaStream_t st) {
  const size_t sm = vec_smem(pc.npad);
  int rc = 0;
  TLS_DISPATCH_UF(pc.u_f, TLS_DISPATCH_MAXR(pc.npad, {
    if ((rc = set_smem(k_pcg_init<T, MAXR>, sm))) return rc;
    k_pcg_init<T, MAXR><<<1, kTT, sm, st>>>(pc, nrhs, v, S);
  }));
  TLS_LAUNCH_CHECK();
  return 0;
}

int launch_pcg_step(const PrecondDev& pc, PcgVecs v, const double* passout, PcgState* S, int rule, int next_q,
                    cudaStream_t st) {
  const size_t sm = vec_smem(pc.npad);
  int rc = 0;
  TLS_DISPATCH_UF(pc.u_f, TLS_DISPATCH_MAXR(pc.npad, {
    if ((rc = set_smem(k_pcg_step<T, MAXR>, sm))) return rc;
    k_pcg_step<T, MAXR><<<1, kTT, sm, st>>>(pc, v, passout, S, rule, next_q);
  }));
  TLS_LAUNCH_CHECK();
  return 0;
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
  const size_t sm = vec_smem(pc.npad);
  int rc = 0;
  TLS_DISPATCH_UF(pc.u_f, TLS_DISPATCH_MAXR(pc.npad, {
    if ((rc = set_smem(k_boot_x1<T, MAXR>, sm))) return rc;
    k_boot_x1<T, MAXR><<<1, kTT, sm, st>>>(pc, passout_r0, x0, x1);
  }));
  TLS_LAUNCH_CHECK();
  return 0;
}

}  // namespace tls
