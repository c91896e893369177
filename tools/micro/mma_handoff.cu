// Micro-benchmark: what does a per-chunk accumulator hand-off cost the tensor pipe?
// (the Gram's K_t = 64 chunking, reading R11; DESIGN §6 "the ~1.4 ms per-chunk cost").
// One CTA per SM, one thread issues NMMA tcgen05.mma kind::f16 (M = 128, N = 128 or 256,
// K = 16) from fixed shared-memory operands (no TMA, no epilogue) and times issue -> completion
// with clock64.  Variants: accumulate throughout; restart (accumulate = 0) every `chunk` MMAs;
// rotate the TMEM buffer at each restart; commit to an mbarrier at each restart; also commit
// every 4 MMAs (the Gram's per-stage "empty" commit).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_handoff mma_handoff.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int N) {
  return (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(su32(bar)),
      "r"(ph)
      : "memory");
}

// mode bits: 1 restart every chunk, 2 rotate buffers at restart, 4 commit per chunk, 8 commit per 4 MMAs
__global__ void __launch_bounds__(128, 1) k(int nmma, int chunk, int mode, int N, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bars[3];
  __shared__ uint32_t holder;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = holder;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(N);
    const uint32_t a0 = su32(sm), b0 = su32(sm + 16384);
    const int nbuf = 512 / N;
    uint32_t nchunk_commits = 0, nstage_commits = 0;
    const long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const int c = i / chunk, kk = i % 4;
      const bool start = (mode & 1) ? (i % chunk == 0) : (i == 0);
      const uint32_t buf = (mode & 2) ? (uint32_t)(c % nbuf) : 0u;
      mma(tm + buf * N, desc(a0 + kk * 2048, 8192, 1024), desc(b0 + kk * 2048, 8192, 1024), id, start ? 0u : 1u);
      if ((mode & 8) && kk == 3) { commit(&bars[1]); ++nstage_commits; }
      if ((mode & 4) && (i % chunk == chunk - 1)) { commit(&bars[2]); ++nchunk_commits; }
    }
    commit(&bars[0]);
    wait(&bars[0], 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, nsm * sizeof(long long));
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int nmma = 16384;
  struct V { int N, chunk, mode; const char* what; } vs[] = {
      {128, 1 << 30, 0, "N=128 accumulate throughout"},
      {128, 4, 1, "N=128 restart every 4 (same buffer)"},
      {128, 4, 3, "N=128 restart every 4, rotate 4 buffers"},
      {128, 4, 7, "N=128 restart+rotate+commit per chunk"},
      {128, 4, 15, "N=128 restart+rotate+commit per chunk+per stage (Gram K_t=64)"},
      {128, 8, 15, "N=128 as Gram, K_t=128"},
      {128, 16, 15, "N=128 as Gram, K_t=256"},
      {128, 1 << 30, 8, "N=128 commit per stage only"},
      {256, 1 << 30, 0, "N=256 accumulate throughout"},
      {256, 4, 3, "N=256 restart every 4, rotate 2 buffers"},
      {256, 4, 15, "N=256 restart+rotate+commits (K_t=64)"},
  };
  for (auto& v : vs) {
    for (int rep = 0; rep < 2; ++rep) {
      k<<<nsm, 128, smem>>>(nmma, v.chunk, v.mode, v.N, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", v.what, cudaGetErrorString(e)); return 1; }
    }
    long long h[256];
    cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0, sum = 0;
    for (int i = 0; i < nsm; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    printf("%-66s cycles/MMA mean %.1f max %.1f  (ideal %d)\n", v.what, (double)sum / nsm / nmma, (double)mx / nmma,
           v.N / 2);
  }
  return 0;
}
