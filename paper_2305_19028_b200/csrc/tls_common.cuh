// tls_common.cuh — device helpers shared by the libtlsrqi kernels (sm_100a).
// Nothing here is shared with oracle/ (the two share no code).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include "../../include/tlsrqi.h"

namespace tls {

// ------------------------------------------------------------------ error plumbing
void set_error(const char* fmt, ...);

#define TLS_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::tls::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return TLS_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

#define TLS_LAUNCH_CHECK()                                                          \
  do {                                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess) {                                                        \
      ::tls::set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return TLS_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

// ------------------------------------------------------------------ u_f rounding
// Direct fp64 -> (p, emin, emax) round-to-nearest-even on the fp64 bit pattern
// (reading R4: gradual underflow, overflow to +-inf).  Integer arithmetic only,
// so there is no intermediate rounding (fp64 -> bf16 is NOT done through fp32).
template <int P, int EMIN, int EMAX>
__device__ __forceinline__ double round_rne(double x) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const unsigned long long sign = bits & 0x8000000000000000ull;
  const int ex = (int)((bits >> 52) & 0x7ff);
  if (ex == 0x7ff) return x;                              // inf / nan pass through
  if (ex == 0) return __longlong_as_double((long long)sign);  // |x| < 2^-1022: below every u_f
  const unsigned long long sig = (bits & 0xFFFFFFFFFFFFFull) | 0x10000000000000ull;
  const int e = ex - 1023;
  const int shift = 52 - (P - 1) + (e < EMIN ? EMIN - e : 0);
  unsigned long long q = 0;
  if (shift < 64) {
    q = sig >> shift;
    const unsigned long long rem = sig & ((1ull << shift) - 1ull);
    const unsigned long long half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (q & 1ull))) q += 1ull;
  }
  double y = scalbn((double)q, e - 52 + shift);           // exact: q <= 2^P
  const double maxf = scalbn(2.0 - scalbn(1.0, 1 - P), EMAX);
  if (y > maxf) y = __longlong_as_double(0x7ff0000000000000ll);
  return sign ? -y : y;
}

// Hardware conversions: cvt.rn.{f16,bf16,f32}.f64 round the fp64 value ONCE to
// nearest-even (no intermediate fp32 step for bf16), with gradual underflow and
// overflow to +-inf -- the same function as round_rne<> above (bit-identical on the
// parity tests' 4e5 values incl. ties, subnormals and overflow), at one F2F each.
__device__ __forceinline__ uint16_t f64_to_f16_bits(double x) {
  uint16_t h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(x));
  return h;
}
__device__ __forceinline__ uint16_t f64_to_bf16_bits(double x) {
  uint16_t h;
  asm("cvt.rn.bf16.f64 %0, %1;" : "=h"(h) : "d"(x));
  return h;
}
__device__ __forceinline__ double f16_bits_to_f64(uint16_t h) {
  double d;
  asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(h));
  return d;
}
__device__ __forceinline__ double bf16_bits_to_f64(uint16_t h) {
  return (double)__uint_as_float(((uint32_t)h) << 16);
}

__device__ __forceinline__ double round_uf(double x, int prec) {
  switch (prec) {
    case TLS_FP16: return f16_bits_to_f64(f64_to_f16_bits(x));
    case TLS_BF16: return bf16_bits_to_f64(f64_to_bf16_bits(x));
    case TLS_FP32: return (double)__double2float_rn(x);
    default: return x;
  }
}

// Storage of u_f values: fp16 and bf16 as 16-bit patterns, fp32 as float,
// fp64 as double.  Encoders take values that are already representable.
struct F16s { uint16_t v; };
struct B16s { uint16_t v; };

__device__ __forceinline__ uint16_t enc_f16(double y) {      // y exactly representable in fp16
  return __half_as_ushort(__float2half_rn((float)y));
}
__device__ __forceinline__ uint16_t enc_b16(double y) {      // y exactly representable in bf16
  return (uint16_t)(__float_as_uint((float)y) >> 16);
}
__device__ __forceinline__ float dec_f16(uint16_t h) { return __half2float(__ushort_as_half(h)); }
__device__ __forceinline__ float dec_b16(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }

// Generic encode/decode of a u_f storage type.
template <typename T> __device__ __forceinline__ T enc(double v);
template <> __device__ __forceinline__ F16s enc<F16s>(double v) { return F16s{enc_f16(v)}; }
template <> __device__ __forceinline__ B16s enc<B16s>(double v) { return B16s{enc_b16(v)}; }
template <> __device__ __forceinline__ float enc<float>(double v) { return (float)v; }
template <> __device__ __forceinline__ double enc<double>(double v) { return v; }

template <typename T> __device__ __forceinline__ double dec(T v);
template <> __device__ __forceinline__ double dec<F16s>(F16s v) { return (double)dec_f16(v.v); }
template <> __device__ __forceinline__ double dec<B16s>(B16s v) { return (double)dec_b16(v.v); }
template <> __device__ __forceinline__ double dec<float>(float v) { return (double)v; }
template <> __device__ __forceinline__ double dec<double>(double v) { return v; }

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed order): every thread gets the result.
// red: smem of >= 32 doubles.  All threads of the block must call it.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// Two block sums at once: each value goes through exactly block_sum's operations (the same
// bits), sharing its barriers.  red: smem of >= 64 doubles.  All threads of the block call it.
__device__ __forceinline__ void block_sum2(double v0, double v1, double* red, double& s0, double& s1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v0 = warp_sum(v0);
  v1 = warp_sum(v1);
  __syncthreads();
  if (lane == 0) { red[warp] = v0; red[32 + warp] = v1; }
  __syncthreads();
  if (warp == 0) {
    double t0 = lane < nw ? red[lane] : 0.0, t1 = lane < nw ? red[32 + lane] : 0.0;
    t0 = warp_sum(t0);
    t1 = warp_sum(t1);
    __syncwarp();
    if (lane == 0) { red[0] = t0; red[32] = t1; }
  }
  __syncthreads();
  s0 = red[0];
  s1 = red[32];
  __syncthreads();
}

// Transpose-reduce V (power of two <= 32) per-lane partial values across a warp.
// On return a[0] of lane l holds the warp total of value index
//   idx(l) = sum over steps s (offset o = 16, 8, ...) with nv_s = V >> s > 1 of
//            ((l & o) ? nv_s / 2 : 0),
// and lanes agreeing on those bits hold the same value.
template <int V>
__device__ __forceinline__ void warp_transpose_reduce(double (&a)[V], int lane) {
  int o = 16;
#pragma unroll
  for (int nv = V; nv > 1; nv >>= 1, o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < nv / 2; ++i) {
      const double send = upper ? a[i] : a[i + nv / 2];
      const double keep = upper ? a[i + nv / 2] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (; o > 0; o >>= 1) a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
}

template <int V>
__device__ __forceinline__ int transpose_reduce_index(int lane) {
  int idx = 0, o = 16;
#pragma unroll
  for (int nv = V; nv > 1; nv >>= 1, o >>= 1)
    if (lane & o) idx += nv / 2;
  return idx;
}

// ------------------------------------------------------------------ mbarrier / bulk copy (TMA)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
// Non-suspending wait (test_wait in a loop): for latency-critical producer/consumer
// chains inside one CTA, where the wake-up delay of a suspended try_wait dominates.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
// ------------------------------------------------------------------ thread-block clusters (DSMEM)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// shared::cta address -> shared::cluster address of the same variable in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// all threads of all CTAs of the cluster (also a CTA-wide barrier)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 8-byte remote store whose arrival is counted on the remote CTA's mbarrier (complete_tx)
__device__ __forceinline__ void st_async_f64(uint32_t remote_addr, double v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr),
               "l"(__double_as_longlong(v)), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace tls
