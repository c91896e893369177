// k_peer.cu — the operator pass's reduction and its all-reduce over ranks as ONE kernel over
// peer memory ("replace the C1 ncclAllReduce launch with a one-shot
// reduction ... a deterministic rank order is kept"; the partial sums are PAPER.md Alg. 3's
// t = A q, v = A^T t, tau = t^T t of a row-sharded A).
//
// Every rank r runs k_reduce_exchange on its own GPU after its operator pass:
//   1  the pass's G per-CTA partial rows are summed in k_reduce_partials' fixed order (8 row
//      groups, then the group sums in order) -> c_r, this rank's contribution (W doubles);
//   2  c_r is stored straight into slot r of EVERY rank's receive buffer (peer pointers
//      obtained with CUDA IPC, so the stores travel over NVLink / NVSwitch), then
//      a system-scope acq_rel fence and a release store of the exchange's epoch into flag (r, cta) of
//      every rank;
//   3  the CTA waits (acquire, system scope) for the same column slice of every rank and forms
//      passout = c_0 + c_1 + ... + c_{P-1} in rank order -- the same bits on every rank, and the
//      same bits as the host-shm backend's rank-ordered sum.
// Slots are double-buffered by epoch parity: a rank can be at most one exchange ahead of any
// other (it cannot finish exchange e+1 before every rank has published e+1, which each does only
// after finishing e), so exchange e+2 never overwrites a slot still being read for e.
// A wait longer than ~2^26 polls sets *err (the solve then returns TLS_ERR_NCCL).
//
// On one GPU (the test pool has one per call) the same kernel runs all P ranks as one
// cooperative launch (tls_peer_exchange_emulate): CTAs that wait for each other must be
// co-resident there, which only a cooperative launch guarantees (B200_PROFILING.md).
#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(256) k_reduce_exchange(PeerTab pt, int P, int rank0, const double* __restrict__ partials,
                                                        size_t pstride, int G, int W, int wcap,
                                                        double* __restrict__ out, size_t ostride, int epoch,
                                                        const int* __restrict__ active, int* __restrict__ err, int cpr) {
  if (active != nullptr && (active[0] | active[1]) == 0) return;   // replicated state: uniform over ranks
  // cpr CTAs per rank (<= kXchCtas; fewer in the one-GPU emulation, where all ranks' CTAs must be
  // co-resident); CTA cb takes the column blocks cb, cb + cpr, ...
  const int lr = blockIdx.x / cpr, cb = blockIdx.x % cpr;
  const int r = rank0 + lr;
  const double* part = partials + (size_t)lr * pstride;
  const size_t par = (size_t)(epoch & 1) * P * wcap;                // double buffer by epoch parity
  const int tx = threadIdx.x & 31, grp = threadIdx.x >> 5;
  __shared__ double sm[8][33];
  // ---- 1 + 2: this CTA's column blocks (32 wide, round-robin over the rank's kXchCtas CTAs)
  for (int w0 = cb * 32; w0 < W; w0 += cpr * 32) {
    const int w = w0 + tx;
    const int g0 = G * grp / 8, g1 = G * (grp + 1) / 8;
    double acc = 0.0;
    if (w < W) {
      int g = g0;
      for (; g + 8 <= g1; g += 8) {                  // 8 loads in flight, added in row order
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = part[(size_t)(g + k) * W + w];
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
      }
      for (; g < g1; ++g) acc += part[(size_t)g * W + w];
    }
    sm[grp][tx] = acc;
    __syncthreads();
    if (grp == 0 && w < W) {
      double c = sm[0][tx];
      for (int k = 1; k < 8; ++k) c += sm[k][tx];
      for (int p = 0; p < P; ++p) pt.rbuf[p][par + (size_t)r * wcap + w] = c;   // peer stores (NVLink)
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // the CTA's stores are ordered before thread 0's by the barrier above; acq_rel at system
    // scope (not the sequentially consistent __threadfence_system) publishes them with the flags
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int p = 0; p < P; ++p) st_release_sys(pt.rflag[p] + r * kXchCtas + cb, epoch);
  }
  // ---- 3: wait for this column slice from every rank, then the rank-ordered sum
  __shared__ int ok;
  if (threadIdx.x == 0) {
    int good = 1;
    for (int p = 0; p < P && good; ++p) {
      const int* f = pt.rflag[r] + p * kXchCtas + cb;
      for (long it = 0; ld_acquire_sys(f) < epoch; ++it) {
        if (it > (1L << 26)) { atomicExch(err, 1); good = 0; break; }
      }
    }
    ok = good;
  }
  __syncthreads();
  if (!ok) return;
  const double* rb = pt.rbuf[r] + par;
  if (grp == 0)
    for (int w = cb * 32 + tx; w < W; w += cpr * 32) {
      double acc = rb[w];
      for (int p = 1; p < P; ++p) acc += rb[(size_t)p * wcap + w];
      out[(size_t)lr * ostride + w] = acc;
    }
}

int launch_reduce_exchange(const PeerTab& pt, int P, int rank0, int ranks_here, const double* partials, size_t pstride,
                           int G, int W, int wcap, double* out, size_t ostride, int epoch, const int* active, int* err,
                           bool cooperative, cudaStream_t st) {
  if (P < 1 || P > kMaxPeers || W > wcap) {
    set_error("peer exchange: P = %d (max %d), W = %d > capacity %d", P, kMaxPeers, W, wcap);
    return TLS_ERR_ARG;
  }
  int cpr = kXchCtas;
  if (cooperative) {                  // every rank's CTAs co-resident on this one GPU
    int per_sm = 0;
    TLS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_reduce_exchange, 256, 0));
    const int fit = per_sm * num_sms() / ranks_here;
    if (fit < cpr) cpr = fit;
    if (cpr < 1) { set_error("peer exchange emulation: %d ranks do not fit on this GPU", ranks_here); return TLS_ERR_ARG; }
  }
  const dim3 grid(ranks_here * cpr), block(256);
  if (cooperative) {
    PeerTab t = pt;
    void* args[] = {&t, &P, &rank0, (void*)&partials, &pstride, &G, &W, &wcap, &out, &ostride, &epoch, (void*)&active, &err,
                    &cpr};
    TLS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_reduce_exchange, grid, block, args, 0, st));
  } else {
    k_reduce_exchange<<<grid, block, 0, st>>>(pt, P, rank0, partials, pstride, G, W, wcap, out, ostride, epoch, active,
                                              err, cpr);
    TLS_LAUNCH_CHECK();
  }
  return 0;
}

}  // namespace tls
