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

// template variant: RESTART (accumulate = 0 at each chunk start), ROT (next TMEM buffer per chunk),
// CCOMMIT (commit to an mbarrier per chunk), PRE (the chunk's buffer was zeroed instead: accumulate
// = 1 always), IL (two accumulators interleaved MMA by MMA)
template <int N, bool RESTART, bool ROT, bool CCOMMIT, bool IL>
__global__ void __launch_bounds__(128, 1) kt(int nchunks, long long* out) {
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
    constexpr uint32_t id = idesc(N);
    const uint32_t a0 = su32(sm), b0 = su32(sm + 16384);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) { ad[kk] = desc(a0 + kk * 2048, 8192, 1024); bd[kk] = desc(b0 + kk * 2048, 8192, 1024); }
    constexpr int NB = 512 / N;
    const long long t0 = clock64();
    for (int c = 0; c < nchunks; ++c) {
      const uint32_t buf = ROT ? (uint32_t)(c & (NB - 1)) : 0u;
      if (IL) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          mma(tm, ad[kk], bd[kk], id, (RESTART && kk == 0) ? 0u : 1u);
          mma(tm + N, bd[kk], ad[kk], id, (RESTART && kk == 0) ? 0u : 1u);
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma(tm + buf * N, ad[kk], bd[kk], id, (RESTART && kk == 0) ? 0u : 1u);
      }
      if (CCOMMIT) commit(&bars[2]);
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

template <int N, bool RESTART, bool ROT, bool CCOMMIT, bool IL>
void run(const char* what, int nsm, long long* d) {
  const int smem = 64 * 1024 + 1024, nchunks = 4096;
  cudaFuncSetAttribute(kt<N, RESTART, ROT, CCOMMIT, IL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) kt<N, RESTART, ROT, CCOMMIT, IL><<<nsm, 128, smem>>>(nchunks, d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: error\n", what); return; }
  long long h[256];
  cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0, sum = 0;
  for (int i = 0; i < nsm; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
  const int mmas = nchunks * 4 * (IL ? 2 : 1);
  printf("v2 %-58s cycles/MMA %.1f  per chunk %.0f  (ideal/MMA %d)\n", what, (double)sum / nsm / mmas,
         (double)sum / nsm / nchunks, N / 2);
}

// Ring variant (the Gram's TMEM ring): NB accumulators of N columns; chunk j goes to buffer
// j % NB and is committed to tfull[buf]; before chunk j >= NB the issuer waits until buffer
// j % NB is free: EPI = false -> on tfull of chunk j - NB itself (an instant epilogue);
// EPI = true -> on tempty, arrived by 8 epilogue warps after they observed tfull (and, LD = true,
// loaded the chunk's 64 columns per warp from TMEM first).  SPIN: test_wait instead of try_wait.
__device__ __forceinline__ void wait_spin(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tW2: mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W2;\n\t}" ::"r"(su32(bar)),
      "r"(ph)
      : "memory");
}
template <int N, int NB, bool EPI, bool LD, bool SPIN, bool FULL = false>
__global__ void __launch_bounds__(320, 1) kr(int nchunks, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t tfull[8], tempty[8], fin;
  __shared__ uint32_t holder;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&tfull[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su32(&tempty[i])) : "memory");
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&fin)) : "memory");
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc(N);
    const uint32_t a0 = su32(sm), b0 = su32(sm + 16384);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) { ad[kk] = desc(a0 + kk * 2048, 8192, 1024); bd[kk] = desc(b0 + kk * 2048, 8192, 1024); }
    const long long t0 = clock64();
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c % NB;
      if (c >= NB) {
        const uint32_t ph = (uint32_t)(c / NB - 1) & 1u;
        uint64_t* b = EPI ? &tempty[buf] : &tfull[buf];
        if (SPIN) wait_spin(b, ph); else wait(b, ph);
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma(tm + buf * N, ad[kk], bd[kk], id, kk == 0 ? 0u : 1u);
      commit(&tfull[buf]);
    }
    commit(&fin);
    wait(&fin, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  } else if (EPI && warp >= 2) {
    const int q = warp & 3, half = (warp - 2) >> 2;
    float acc = 0.f;
    float2 s2[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) s2[i] = make_float2(0.f, 0.f);
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c % NB;
      if (SPIN) wait_spin(&tfull[buf], (uint32_t)(c / NB) & 1u); else wait(&tfull[buf], (uint32_t)(c / NB) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (LD && N == 256 && FULL) {
        // the Gram epilogue: all 128 columns of this warp's half, 4 x (LDTM.x32, wait, 16 FADD2)
        const uint32_t ta = tm + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * N + half * 128);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t r[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
              "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
                "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
                "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
              : "r"(ta + g * 32)
              : "memory");
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 16; ++e) s2[g * 16 + e] = __fadd2_rn(s2[g * 16 + e], make_float2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])));
        }
      } else if (LD) {
        uint32_t r[32];
        const uint32_t ta = tm + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * N + half * (N / 2));
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
            "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
              "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(ta)
            : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 32; ++e) acc += __uint_as_float(r[e]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[buf])) : "memory");
    }
    for (int i = 0; i < 64; ++i) acc += s2[i].x + s2[i].y;
    if (acc == 12345.f) out[0] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
  }
}

template <int N, int NB, bool EPI, bool LD, bool SPIN, bool FULL = false>
void runr(const char* what, int nsm, long long* d) {
  const int smem = 64 * 1024 + 1024, nchunks = 4096;
  cudaFuncSetAttribute(kr<N, NB, EPI, LD, SPIN, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) kr<N, NB, EPI, LD, SPIN, FULL><<<nsm, 320, smem>>>(nchunks, d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: error\n", what); return; }
  long long h[256];
  cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long sum = 0;
  for (int i = 0; i < nsm; ++i) sum += h[i];
  printf("ring %-56s cycles per chunk %.0f  (MMA work %d)\n", what, (double)sum / nsm / nchunks, 4 * N / 2);
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
  runr<128, 4, false, false, false>("N=128 4 bufs, wait on tfull(j-4) (instant epilogue)", nsm, d);
  runr<128, 4, false, false, true>("N=128 4 bufs, wait on tfull(j-4), spin", nsm, d);
  runr<128, 4, true, false, false>("N=128 4 bufs, epilogue warps relay (no ld)", nsm, d);
  runr<128, 4, true, true, false>("N=128 4 bufs, epilogue warps ld 32 cols + relay", nsm, d);
  runr<128, 4, true, true, true>("N=128 4 bufs, epilogue ld + relay, spin", nsm, d);
  runr<128, 2, true, true, false>("N=128 2 bufs, epilogue ld + relay", nsm, d);
  runr<256, 2, true, true, false>("N=256 2 bufs, epilogue ld + relay", nsm, d);
  runr<64, 8, true, true, false>("N=64 8 bufs, epilogue ld + relay", nsm, d);
  runr<256, 2, true, true, false, true>("N=256 2 bufs, epilogue 4 LDTM + 64 FADD2 (Gram drain)", nsm, d);
  runr<256, 2, true, true, true, true>("N=256 2 bufs, Gram drain, spin waits", nsm, d);
  run<128, false, false, false, false>("N=128 acc throughout", nsm, d);
  run<128, true, false, false, false>("N=128 restart/4, same buffer", nsm, d);
  run<128, false, true, false, false>("N=128 no restart, rotate/4", nsm, d);
  run<128, true, true, false, false>("N=128 restart + rotate", nsm, d);
  run<128, true, true, true, false>("N=128 restart + rotate + commit/chunk", nsm, d);
  run<128, false, true, true, false>("N=128 rotate + commit/chunk", nsm, d);
  run<128, true, false, true, false>("N=128 restart + commit/chunk", nsm, d);
  run<128, false, false, true, false>("N=128 commit/chunk only", nsm, d);
  run<128, true, false, false, true>("N=128 2 interleaved accs, restart/4", nsm, d);
  run<128, false, false, false, true>("N=128 2 interleaved accs, no restart", nsm, d);
  run<256, false, false, false, false>("N=256 acc throughout", nsm, d);
  run<256, true, false, false, false>("N=256 restart/4, same buffer", nsm, d);
  run<256, true, true, true, false>("N=256 restart + rotate + commit/chunk", nsm, d);
  run<256, false, true, true, false>("N=256 rotate + commit/chunk", nsm, d);
  return 0;
}
