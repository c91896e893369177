// k_gram_tc.cu — the u_f Gram on the 5th-generation tensor cores (SURVEY §8(a)
// row a2; readings R10, R11), u_f in {fp16, bf16}.
//
//  1. k_round_scaled: A^ = fl_uf(A D^{-1}) (direct fp64 -> u_f RNE, reading R4)
//     written once as a row-major 16-bit matrix (HBM-bound pass).
//  2. k_gram_tc: G_IJ = A^_I^T A^_J for 128x128 tiles of the upper triangle,
//     split over K_t-row chunks.  Warp-specialised persistent-tile CTA:
//       warp 0      TMA producer: 2-D tensor loads (128B swizzle) of the two
//                   64-row x 128-column operand panels into a 4-stage ring
//       warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//                   (kind::f16, M=128 N=128 K=16, fp32 accumulators in TMEM,
//                   both operands MN-major straight from the row-major A^)
//       warps 2-9   epilogue: after every K_t rows, tcgen05.ld the fp32 chunk
//                   sum (reading R11: the tensor cores accumulate each K_t-row
//                   chunk in fp32) and add it to an fp32 Kahan-compensated
//                   register accumulator (FP32 pipe); every `super` chunks the
//                   compensated sum is flushed into this CTA's fp64 partial
//                   tile in global memory (L2).  A per-chunk fp32 -> fp64
//                   conversion (XU pipe, ~16/clk/SM) bound the previous design
//                   (ncu: XU 65% busy, tensor pipe 12%).  Four TMEM accumulators
//                   (all 512 columns) rotate so the MMA runs up to three chunks
//                   ahead of the drain (flushes included).
//  3. the split partials are summed in fixed order (k_gram_reduce_t).
#include <cuda.h>

#include <cstdio>
#include <vector>

#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

constexpr int kTcTile = 128;      // output tile edge (UMMA M = N = 128)
constexpr int kTcBK = 64;         // rows of A^ per pipeline stage
constexpr int kTcStages = 4;
constexpr int kTcAcc = 4;         // TMEM accumulators (4 x 128 columns = all 512): 3 chunks of drain slack
constexpr int kTcPanel = kTcTile * kTcBK * 2;   // 16 KB: one operand panel (2 TMA boxes of 8 KB)
constexpr int kTcThreads = 320;
constexpr size_t kTcSmem = 2 * kTcStages * kTcPanel + 1024 + 512 + 8 * 32 * 33 * 8;   // + the flush staging

// ------------------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
#define TLS_TMEM_LD32(taddr, r)                                                                                  \
  asm volatile(                                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                             \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),         \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),   \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])  \
      : "r"(taddr)                                                                                               \
      : "memory")

// fp64 reduction into a partial tile kept in L2 (evict_last): the tiles (36 MB at n = 1024) are
// re-touched every 64 chunks while ~2 GB of A^ streams through L2 (ncu without the hint: ~1.1 GB
// of partial-tile traffic each way to DRAM)
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void red_add_keep(double* p, double v, uint64_t pol) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
#define TLS_TMEM_LD16(taddr, r)                                                                                  \
  asm volatile(                                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"      \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),         \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])    \
      : "r"(taddr)                                                                                               \
      : "memory")

// TMA multicast: the box lands at the same offset in every CTA of `mask` (cluster) and each
// destination CTA's mbarrier at `bar`'s offset counts the bytes
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}

// UMMA shared-memory descriptor, 128-byte swizzle, MN-major canonical layout
// ((8 elem,8,m),(8 rows,k)) : ((1,8,LBO),(64 elem,SBO)) — what a TMA box of
// 64 columns (128 B) x 64 rows with CU_TENSOR_MAP_SWIZZLE_128B produces.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D fp32, A/B = fp16 (0) or bf16 (1), both MN-major, M = N = 128.
__host__ __device__ constexpr uint32_t idesc_f16(int fmt) {
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | (1u << 15) | (1u << 16) |
         ((uint32_t)(kTcTile >> 3) << 17) | ((uint32_t)(kTcTile >> 4) << 24);
}

// ------------------------------------------------------------------------------ 1. A^ = fl_uf(A D^-1)
template <int PREC, int kRows>
__global__ void __launch_bounds__(256, 6) k_round_scaled(const double* __restrict__ A, int64_t m, int n, int64_t ld,
                                                         const double* __restrict__ dinv, uint16_t* __restrict__ Ah, int npad,
                                                         int* __restrict__ range) {
  // Fully coalesced: a warp reads 32 consecutive column pairs of a row (512 B, one
  // 16-byte load per lane; ld even and A 16-B aligned) and writes 32 consecutive u_f
  // pairs (128 B).  Rows are spread over the grid.  Each thread issues the loads of two
  // pairs in kRows rows (kRows x 2 x 16 B) before its first conversion: beside the segmented
  // SYRK (168 registers x 320 threads) only ONE 256-thread CTA of this kernel fits an SM
  // (hence <= 40 registers: __launch_bounds__(256, 6)), and with one row (2 x 16 B) in
  // flight per thread it was latency-bound there.  Same products, same rounding.  Measured
  // (tools/time_round.py, profiles/r02f_round.log): tls_gram 2^20 x 1024 3.30 -> 3.24 ms
  // (fp16), 3.26 -> 3.18 ms (bf16); G bit-identical.
  const int pairs = npad / 2;
  const int64_t G = gridDim.x;
  int bad = 0;
  for (int64_t row0 = blockIdx.x; row0 < m; row0 += kRows * G) {
    for (int p0 = threadIdx.x; p0 < pairs; p0 += 2 * blockDim.x) {
      double2 v[kRows][2];
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const int64_t row = row0 + r * G;
        const double* src = A + row * ld;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = 2 * (p0 + u * (int)blockDim.x);
          if (row < m && c + 1 < n) v[r][u] = __ldcs(reinterpret_cast<const double2*>(src + c));   // streamed once
          else v[r][u] = make_double2(row < m && c < n ? src[c] : 0.0, 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int pp = p0 + u * (int)blockDim.x;
        if (pp >= pairs) break;
        const int c = 2 * pp;
        const double s0 = c < n ? dinv[c] : 0.0;
        const double s1 = c + 1 < n ? dinv[c + 1] : 0.0;
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          const int64_t row = row0 + r * G;
          if (row >= m) break;
          const double x0 = c < n ? v[r][u].x * s0 : 0.0;
          const double x1 = c + 1 < n ? v[r][u].y * s1 : 0.0;
          const uint16_t h0 = PREC == TLS_FP16 ? f64_to_f16_bits(x0) : f64_to_bf16_bits(x0);   // one RNE rounding
          const uint16_t h1 = PREC == TLS_FP16 ? f64_to_f16_bits(x1) : f64_to_bf16_bits(x1);
          const uint32_t lim = PREC == TLS_FP16 ? 0x7c00u : 0x7f80u;                               // inf / nan
          bad |= ((h0 & 0x7fffu) >= lim) | ((h1 & 0x7fffu) >= lim);
          reinterpret_cast<uint32_t*>(Ah + row * npad)[pp] = (uint32_t)h0 | ((uint32_t)h1 << 16);
        }
      }
    }
  }
  if (bad) atomicExch(range, 1);
}

// The same pass with the fp64 rows staged in shared memory by the bulk-copy (TMA) engine
// (TLS_ROUND=3, n even): beside the SYRK only one CTA of the register form fits an SM, with
// 16 KB of loads in flight; here the bytes in flight live in a ring of kRbStages x 8 KB of
// the shared memory the SYRK leaves free, issued by one producer lane, and cost no registers.
// A unit = (row, chunk of <= 1024 columns); same products, same single rounding, same bytes of A^.
constexpr int kRbStages = 8;
constexpr int kRbChunk = 1024;                                   // doubles per stage
constexpr int kRbThreads = 288;                                  // 8 consumer warps + the producer warp
constexpr size_t kRbSmem = (size_t)kRbStages * kRbChunk * 8 + 2 * kRbStages * 8 + 128;
template <int PREC>
__global__ void __launch_bounds__(kRbThreads, 5) k_round_bulk(const double* __restrict__ A, int64_t m, int n, int64_t ld,
                                                              const double* __restrict__ dinv, uint16_t* __restrict__ Ah,
                                                              int npad, int* __restrict__ range) {
  extern __shared__ __align__(128) unsigned char rb_raw[];
  double* ring = reinterpret_cast<double*>(rb_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(rb_raw + (size_t)kRbStages * kRbChunk * 8);
  uint64_t* empty = full + kRbStages;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nch = (n + kRbChunk - 1) / kRbChunk;
  const int64_t G = gridDim.x;
  const int64_t nrows = blockIdx.x < m ? (m - blockIdx.x + G - 1) / G : 0;
  const int64_t units = nrows * nch;
  if (tid == 0) {
    for (int i = 0; i < kRbStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 8); }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 8) {
    if (tid == 256) {
      const uint64_t pol = policy_evict_first();
      const double* src = A + (int64_t)blockIdx.x * ld;
      int st = 0, ch = 0;
      uint32_t ph = 1;                                              // parity of the previous use of the stage
      bool first = true;
      for (int64_t u = 0; u < units; ++u) {
        if (!first) mbar_wait(&empty[st], ph);
        const int cnt = n - ch * kRbChunk < kRbChunk ? n - ch * kRbChunk : kRbChunk;
        mbar_arrive_expect_tx(&full[st], (uint32_t)cnt * 8u);
        bulk_g2s(ring + (size_t)st * kRbChunk, src + ch * kRbChunk, (uint32_t)cnt * 8u, &full[st], pol);
        if (++ch == nch) { ch = 0; src += G * ld; }
        if (++st == kRbStages) { st = 0; ph ^= 1; first = false; }
      }
    }
    return;
  }
  int bad = 0;
  const int lane = tid & 31;
  uint16_t* dst = Ah + (int64_t)blockIdx.x * npad;
  int st = 0, ch = 0;
  uint32_t ph = 0;
  for (int64_t u = 0; u < units; ++u) {
    const int c0 = ch * kRbChunk;
    const int cnt = n - c0 < kRbChunk ? n - c0 : kRbChunk;                  // even (n even)
    const int outp = (npad - c0 < kRbChunk ? npad - c0 : kRbChunk) / 2;     // pairs written (zero pad included)
    mbar_wait(&full[st], ph);
    const double2* sp = reinterpret_cast<const double2*>(ring + (size_t)st * kRbChunk);
    double2 v[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int pp = tid + k * 256;
      v[k] = 2 * pp < cnt ? sp[pp] : make_double2(0.0, 0.0);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);                                 // this warp has read its part of the stage
    uint32_t* orow = reinterpret_cast<uint32_t*>(dst) + c0 / 2;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int pp = tid + k * 256;
      if (pp >= outp) break;
      const int c = c0 + 2 * pp;
      const bool in = 2 * pp < cnt;
      const double x0 = in ? v[k].x * __ldg(dinv + c) : 0.0;
      const double x1 = in ? v[k].y * __ldg(dinv + c + 1) : 0.0;
      const uint16_t h0 = PREC == TLS_FP16 ? f64_to_f16_bits(x0) : f64_to_bf16_bits(x0);   // one RNE rounding
      const uint16_t h1 = PREC == TLS_FP16 ? f64_to_f16_bits(x1) : f64_to_bf16_bits(x1);
      const uint32_t lim = PREC == TLS_FP16 ? 0x7c00u : 0x7f80u;                               // inf / nan
      bad |= ((h0 & 0x7fffu) >= lim) | ((h1 & 0x7fffu) >= lim);
      orow[pp] = (uint32_t)h0 | ((uint32_t)h1 << 16);
    }
    if (++ch == nch) { ch = 0; dst += G * npad; }
    if (++st == kRbStages) { st = 0; ph ^= 1; }
  }
  if (bad) atomicExch(range, 1);
}

// ------------------------------------------------------------------------------ 2. tcgen05 SYRK
template <int FMT, bool KAHAN>
__global__ void __launch_bounds__(kTcThreads, 1)
k_gram_tc(const __grid_constant__ CUtensorMap tmap, int64_t m, int TT, int nchunks, int nsplit, int kpc,
          int super, int epi, double* __restrict__ part, int kb0, const __grid_constant__ CUtensorMap tmapB,
          int atb) {
  // atb = 1 (the blocked QR's V^T C, k_qr_wy.cu): A = the single 128-column panel of `tmap`,
  // B = the 128-column tile blockIdx.x of `tmapB`; otherwise the upper tiles (I, J) of tmap^T tmap
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the 128B-swizzled operand panels
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* panA = smem;                                  // [stages][16 KB]
  unsigned char* panB = smem + kTcStages * kTcPanel;           // [stages][16 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * kTcStages * kTcPanel);
  uint64_t* empty = full + kTcStages;
  uint64_t* tfull = empty + kTcStages;
  uint64_t* tempty = tfull + kTcAcc;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + kTcAcc);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = blockIdx.x, I = 0;
  if (!atb) while (t >= TT - I) { t -= TT - I; ++I; }
  const int J = atb ? (int)blockIdx.x : I + t;
  const bool diag = !atb && (I == J);
  const CUtensorMap* mapB = atb ? &tmapB : &tmap;
  const int s = blockIdx.y;
  const int c0 = (int)((int64_t)nchunks * s / nsplit), c1 = (int)((int64_t)nchunks * (s + 1) / nsplit);
  const int kb_total = (int)((m + kTcBK - 1) / kTcBK);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kTcAcc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kTcAcc * kTcTile)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      if (atb) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(mapB)) : "memory");
      const uint32_t bytes = diag ? kTcPanel : 2 * kTcPanel;
      int it = 0;
      for (int c = c0; c < c1; ++c) {
        const int kb1 = min((c + 1) * kpc, kb_total);
        for (int kb = c * kpc; kb < kb1; ++kb, ++it) {
          const int st = it % kTcStages;
          const uint32_t ph = (uint32_t)(it / kTcStages) & 1u;
          if (it >= kTcStages) mbar_wait(&empty[st], ph ^ 1u);
          mbar_arrive_expect_tx(&full[st], bytes);
          const int row = (kb0 + kb) * kTcBK;      // kb0: the segment's first block (launch_gram_tc)
          unsigned char* a = panA + st * kTcPanel;
          tma_load_2d(a, &tmap, I * kTcTile, row, &full[st]);
          tma_load_2d(a + kTcPanel / 2, &tmap, I * kTcTile + 64, row, &full[st]);
          if (!diag) {
            unsigned char* b = panB + st * kTcPanel;
            tma_load_2d(b, mapB, J * kTcTile, row, &full[st]);
            tma_load_2d(b + kTcPanel / 2, mapB, J * kTcTile + 64, row, &full[st]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      const uint32_t idesc = idesc_f16(FMT);
      int it = 0;
      for (int c = c0; c < c1; ++c) {
        const int j = c - c0;
        const int buf = j % kTcAcc;
        if (j >= kTcAcc) mbar_wait(&tempty[buf], (uint32_t)(j / kTcAcc - 1) & 1u);
        tc_fence_after();
        const uint32_t dtm = tmem_base + (uint32_t)(buf * kTcTile);
        const int kb1 = min((c + 1) * kpc, kb_total);
        for (int kb = c * kpc; kb < kb1; ++kb, ++it) {
          const int st = it % kTcStages;
          const uint32_t ph = (uint32_t)(it / kTcStages) & 1u;
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(panA + st * kTcPanel);
          const uint32_t b0 = smem_u32((diag ? panA : panB) + st * kTcPanel);
#pragma unroll
          for (int kk = 0; kk < kTcBK / 16; ++kk) {
            // K = 16 rows = two 8-row groups of 1024 B (SBO); MN halves 8 KB apart (LBO)
            const uint64_t ad = sw128_desc(a0 + kk * 2048, kTcPanel / 2, 1024);
            const uint64_t bd = sw128_desc(b0 + kk * 2048, kTcPanel / 2, 1024);
            tc_mma_f16(dtm, ad, bd, idesc, (kb > c * kpc || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[st]);
        }
        tc_commit(&tfull[buf]);
      }
    }
  } else {
    // ---------------- epilogue: fp32 chunk sums -> (compensated) fp32 -> fp64 partial tile
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;       // column half: 0 -> cols 0..63, 1 -> 64..127
    double* ob = part + ((size_t)s * gridDim.x + blockIdx.x) * (kTcTile * kTcTile) + (size_t)(q * 32) * kTcTile + half * 64;
    double* stg = reinterpret_cast<double*>(smem + 2 * kTcStages * kTcPanel + 512) + (warp - 2) * 32 * 33;
    const uint64_t pol = l2_evict_last_policy();
    float2 sm[32], cm[32];                  // 64 fp32 sums (and Kahan compensations), added pairwise
#pragma unroll
    for (int i = 0; i < 32; ++i) { sm[i] = make_float2(0.f, 0.f); cm[i] = make_float2(0.f, 0.f); }
    int pending = 0;
    // flush: fire-and-forget fp64 reductions (RED.ADD.F64) into this CTA's partial tile (zeroed
    // before the launch), coalesced: 32 x 32 blocks transposed through shared memory so that a
    // warp's reduction covers 32 consecutive columns of one row.  Each element has exactly one
    // writer thread, so its adds are applied in program order (deterministic) and the epilogue
    // never waits for an L2 round trip.
    auto flush = [&]() {
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 v = sm[cb * 16 + e], w = cm[cb * 16 + e];
          stg[lane * 33 + 2 * e] = KAHAN ? (double)v.x - (double)w.x : (double)v.x;
          stg[lane * 33 + 2 * e + 1] = KAHAN ? (double)v.y - (double)w.y : (double)v.y;
          sm[cb * 16 + e] = make_float2(0.f, 0.f);
          cm[cb * 16 + e] = make_float2(0.f, 0.f);
        }
        __syncwarp();
#pragma unroll 8
        for (int r = 0; r < 32; ++r) red_add_keep(ob + (size_t)r * kTcTile + cb * 32 + lane, stg[r * 33 + lane], pol);
        __syncwarp();
      }
      pending = 0;
    };
    for (int c = c0; c < c1; ++c) {
      const int j = c - c0;
      const int buf = j % kTcAcc;
      mbar_wait(&tfull[buf], (uint32_t)(j / kTcAcc) & 1u);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kTcTile + half * 64);
      if (epi > 0) {
        TLS_TMEM_LD32(ta, r0);           // both loads in flight, one wait
        TLS_TMEM_LD32(ta + 32, r1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
      // the chunk sum is in registers: hand the TMEM buffer back before the adds
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (epi > 1) {
        if (KAHAN) {
#pragma unroll
          for (int k = 0; k < 64; ++k) {        // Kahan: |error| <= 2u sum|x| + O(super u^2)
            float& sk = (k & 1) ? sm[k >> 1].y : sm[k >> 1].x;
            float& ck = (k & 1) ? cm[k >> 1].y : cm[k >> 1].x;
            const float x = __uint_as_float(k < 32 ? r0[k] : r1[k - 32]);
            const float y = __fsub_rn(x, ck);
            const float t = __fadd_rn(sk, y);
            ck = __fsub_rn(__fsub_rn(t, sk), y);
            sk = t;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            sm[k] = __fadd2_rn(sm[k], make_float2(__uint_as_float(r0[2 * k]), __uint_as_float(r0[2 * k + 1])));
            sm[k + 16] = __fadd2_rn(sm[k + 16], make_float2(__uint_as_float(r1[2 * k]), __uint_as_float(r1[2 * k + 1])));
          }
        }
      }
      if (++pending == super) flush();
    }
    if (pending) flush();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcAcc * kTcTile) : "memory");
  }
}

// ------------------------------------------------------------------------------ ring hand-off helpers
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_geq(const int* p, int target, int* err) {
  for (long it = 0; ld_acquire(p) < target; ++it) {
    if (it > (1L << 24)) { atomicExch(err, 1); return; }
    __nanosleep(64);
  }
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------------------------ 2b. SYRK on 128 x 256 blocks
// k_gram_tc2: k_gram_tc with UMMA N = 256 -- each CTA owns the block (I, P) = tiles (I, 2P) and
// (I, 2P + 1) of the upper triangle (the lower tile of a diagonal block is computed and dropped).
// Why (tools/micro/mma_handoff.cu, profiles/r02_mma_handoff.log): with N = 128 a K_t = 64 chunk
// is 4 MMAs of 64 cycles, and the per-chunk accumulator hand-off (commit, the TMEM ring's
// barrier round trip, accumulate = 0 restart) adds ~45% to it even with an instant epilogue;
// with N = 256 a chunk is 512 cycles of MMA and the same hand-off is hidden entirely.  It also
// loads 24 KB of operand panels per tile and stage instead of 32 KB (the main loop is L2->SM
// bound).  Two TMEM accumulators of 256 columns; 8 epilogue warps, each draining 128 columns of
// its lane quarter into 128 fp32 register sums (reading R11 unchanged: fp32 chunk sums of K_t
// rows, fp32 sums of `super` chunk sums, fp64 flushes, split partials summed in fixed order).
constexpr int kT2N = 256;
constexpr int kT2PanelB = kT2N * kTcBK * 2;                 // 32 KB: 4 TMA boxes of 8 KB
constexpr int kT2Stage = kTcPanel + kT2PanelB;              // 48 KB per stage
constexpr size_t t2_smem(int stages, int ew = 8) { return (size_t)stages * kT2Stage + 1024 + 256 + (size_t)ew * 32 * 33 * 4; }   // + flush staging

__host__ __device__ constexpr uint32_t idesc_f16_n(int fmt, int N) {
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | (1u << 15) | (1u << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTcTile >> 4) << 24);
}

static int t2_blocks(int TT) {
  const int TP = (TT + 1) / 2;
  int b = 0;
  for (int I = 0; I < TT; ++I) b += TP - I / 2;
  return b;
}

// RING (k_gram_fused2's SYRK role): chunk j of split s is read from slot j % R of the split's
// L2 ring (rows (s R + slot) 64 ..) once ready[s R + slot] >= j / R + 1, and the slot is released
// (done += 1) as soon as the chunk's panels have landed in shared memory.
struct T2Ring {
  int* ready;
  int* done;
  int R;
  int* err;
  unsigned long long* prof;   // debugging: per CTA [8] ns (k_gram_fused2, TLS_FZ_PROF=1)
};

// MC (2-CTA clusters, TLS_GRAM_MC=1): the two CTAs of a cluster own blocks (2a, P) and
// (2a + 1, P) -- every block column P has 2P + 2 blocks when TT is even -- and share the
// 256-column B panel: each loads half of it with TMA multicast into both, so a stage costs the
// pair 32 + 2 x 16 KB of L2 reads instead of 2 x 48 (the diagonal pair a = P loads B only).  A
// stage is free again when BOTH CTAs' MMAs are done with it (empty barriers of count 2, commits
// multicast to the pair).
// EW: epilogue warps (8: 128 columns each, 10 warps per CTA; 16: 64 columns each, 18 warps, the
// drain of a chunk split over twice the warps at half the registers per thread).
template <int FMT, int kT2Stages, bool RING, bool MC = false, int EW = 8>
__device__ __forceinline__ void tc2_body(const CUtensorMap* tmap_p, unsigned char* smem, int bidx, int s, int64_t m,
                                         int TT, int nchunks, int nsplit, int kpc, int super, double* __restrict__ part,
                                         int kb0, T2Ring rg) {
  const CUtensorMap& tmap = *tmap_p;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kT2Stages * kT2Stage);
  uint64_t* empty = full + kT2Stages;
  uint64_t* tfull = empty + kT2Stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TP = (TT + 1) / 2;
  int I = 0, P = 0;
  if (MC) {                                   // bidx = 2 x pair + rank; pairs (P, a), a = 0..P
    int pr = bidx >> 1;
    while (pr >= P + 1) { pr -= P + 1; ++P; }
    I = 2 * pr + (bidx & 1);
  } else {
    int t = bidx;
    while (t >= TP - I / 2) { t -= TP - I / 2; ++I; }
    P = I / 2 + t;
  }
  const bool dblk = (P == I / 2);             // the block holds tile (I, I): A is a half of B
  const int ahalf = I - 2 * P;
  const int ntiles = TT * (TT + 1) / 2;
  const int c0 = (int)((int64_t)nchunks * s / nsplit), c1 = (int)((int64_t)nchunks * (s + 1) / nsplit);
  const int kb_total = (int)((m + kTcBK - 1) / kTcBK);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kT2Stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], MC ? 2 : 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], EW);
    }
    fence_mbar_init();
  }
  if (MC) cluster_sync_all();                 // the partner's barriers exist before any multicast
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(2 * kT2N)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      const uint32_t bytes = dblk ? kT2PanelB : kT2Stage;
      int it = 0;
      for (int c = c0; c < c1; ++c) {
        const int kb1 = min((c + 1) * kpc, kb_total);
        for (int kb = c * kpc; kb < kb1; ++kb, ++it) {
          const int st = it % kT2Stages;
          const uint32_t ph = (uint32_t)(it / kT2Stages) & 1u;
          if (it >= kT2Stages) {
            mbar_wait(&empty[st], ph ^ 1u);
            if (RING) {       // chunk it - S was consumed (its MMAs are done): free its ring slot
              // (relaxed: its TMA reads completed before the MMAs could start; a release here cost a
              // gpu-scope fence per chunk -- measured 3x slower when the MMA thread did it)
              const int slot = (c - c0 - kT2Stages) % rg.R;
              asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(rg.done + s * rg.R + slot) : "memory");
            }
          }
          int row = (kb0 + kb) * kTcBK;
          if (RING) {                                   // kpc == 1: chunk c is block kb
            const int j = c - c0, slot = j % rg.R;
            const unsigned long long t0 = rg.prof ? gtime() : 0;
            wait_geq(&rg.ready[s * rg.R + slot], j / rg.R + 1, rg.err);
            if (rg.prof) rg.prof[blockIdx.x * 8 + 3] += gtime() - t0;
            fence_proxy_async_global();                 // generic-proxy writes -> TMA reads
            row = (s * rg.R + slot) * kTcBK;
          }
          mbar_arrive_expect_tx(&full[st], bytes);
          unsigned char* sa = smem + st * kT2Stage;
          unsigned char* sb = sa + kTcPanel;
          if (!dblk) {
            tma_load_2d(sa, &tmap, I * kTcTile, row, &full[st]);
            tma_load_2d(sa + kTcPanel / 2, &tmap, I * kTcTile + 64, row, &full[st]);
          }
          if (MC) {
            const int rk = I & 1;                   // this CTA's half of B, multicast to the pair
#pragma unroll
            for (int q = 2 * rk; q < 2 * rk + 2; ++q)
              tma_load_2d_mc(sb + q * (kTcPanel / 2), &tmap, P * kT2N + 64 * q, row, &full[st], (uint16_t)3);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) tma_load_2d(sb + q * (kTcPanel / 2), &tmap, P * kT2N + 64 * q, row, &full[st]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread): M = 128 (tile row I), N = 256 (tiles 2P, 2P + 1)
    if (lane == 0) {
      const uint32_t idesc = idesc_f16_n(FMT, kT2N);
      // descriptors of stage 0; stage st and K step kk add (st * kT2Stage + kk * 2048) >> 4 to the
      // start-address field (smem offsets < 256 KB: no carry out of its 14 bits)
      const uint32_t b00 = smem_u32(smem + kTcPanel);
      const uint64_t bd0 = sw128_desc(b00, kTcPanel / 2, 1024);
      const uint64_t ad0 = sw128_desc(dblk ? b00 + (uint32_t)(ahalf * kTcPanel) : smem_u32(smem), kTcPanel / 2, 1024);
      int it = 0;
      int st = 0;
      uint32_t ph = 0;
      for (int c = c0; c < c1; ++c) {
        const int j = c - c0;
        const int buf = j & 1;
        if (j >= 2) mbar_wait(&tempty[buf], (uint32_t)((j >> 1) - 1) & 1u);
        tc_fence_after();
        const uint32_t dtm = tmem_base + (uint32_t)(buf * kT2N);
        const int kb1 = min((c + 1) * kpc, kb_total);
        for (int kb = c * kpc; kb < kb1; ++kb, ++it) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint64_t so = (uint64_t)((st * kT2Stage) >> 4);
#pragma unroll
          for (int kk = 0; kk < kTcBK / 16; ++kk)
            tc_mma_f16(dtm, ad0 + so + (uint64_t)(kk * 128), bd0 + so + (uint64_t)(kk * 128), idesc,
                       (kb > c * kpc || kk > 0) ? 1u : 0u);
          if (MC) tc_commit_mc(&empty[st], (uint16_t)3);
          else tc_commit(&empty[st]);
          if (++st == kT2Stages) { st = 0; ph ^= 1u; }
        }
        tc_commit(&tfull[buf]);
      }
    }
  } else {
    // ---------------- epilogue: warp (q, hq) drains TMEM lanes 32q.. and CW columns from hq CW
    constexpr int CW = kT2N / (EW / 4);                            // 128 (EW = 8) or 64 (EW = 16)
    const int q = warp & 3;
    const int hq = (warp - 2) >> 2;
    const int col0 = hq * CW;                                       // within the 256-column block
    const int J = 2 * P + col0 / kTcTile;
    const int tc0 = col0 % kTcTile;                                 // within tile J
    const bool valid = (J >= I) && (J < TT);
    const int tix = I * TT - I * (I - 1) / 2 + (J - I);          // upper-triangle index of (I, J)
    float2 sm[CW / 2];                                             // CW fp32 sums, added pairwise (FADD2)
#pragma unroll
    for (int i = 0; i < CW / 2; ++i) sm[i] = make_float2(0.f, 0.f);
    float* stg = reinterpret_cast<float*>(smem + kT2Stages * kT2Stage + 256) + (warp - 2) * 32 * 33;
    const uint64_t pol = l2_evict_last_policy();
    double* ob = part + ((size_t)s * ntiles + (valid ? tix : 0)) * (kTcTile * kTcTile) + (size_t)(q * 32) * kTcTile + tc0;
    int pending = 0;
    for (int c = c0; c < c1; ++c) {
      const int j = c - c0;
      const int buf = j & 1;
      mbar_wait(&tfull[buf], (uint32_t)(j >> 1) & 1u);
      tc_fence_after();
      if (valid) {
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kT2N + col0);
#pragma unroll
        for (int g = 0; g < CW / 16; ++g) {
          uint32_t r[16];
          TLS_TMEM_LD16(ta + g * 16, r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 8; ++e)
            sm[g * 8 + e] = __fadd2_rn(sm[g * 8 + e], make_float2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (++pending == super || c + 1 == c1) {
        if (valid) {
          // coalesced flush: 32 x 32 blocks transposed through shared memory, so that a warp's
          // fp64 reduction covers 32 consecutive columns of one row (two 128-B lines) instead of
          // one column of 32 rows (32 lines); each element still has exactly one writer thread
#pragma unroll
          for (int cb = 0; cb < CW / 32; ++cb) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              stg[lane * 33 + 2 * e] = sm[cb * 16 + e].x;
              stg[lane * 33 + 2 * e + 1] = sm[cb * 16 + e].y;
              sm[cb * 16 + e] = make_float2(0.f, 0.f);
            }
            __syncwarp();
#pragma unroll 8
            for (int r = 0; r < 32; ++r) red_add_keep(ob + (size_t)r * kTcTile + cb * 32 + lane, (double)stg[r * 33 + lane], pol);
            __syncwarp();
          }
        }
        pending = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (MC) cluster_sync_all();                 // no multicast or remote commit still targets us
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * kT2N) : "memory");
  }
}

// TLS_T2_MAXNREG (compile-time experiment): cap the SYRK's registers so that more CTAs of the
// concurrent rounding pass fit beside it (168 registers x 320 threads leave room for one)
#ifdef TLS_T2_MAXNREG
template <int FMT, int kT2Stages, bool MC = false, int EW = 8>
__global__ void __maxnreg__(TLS_T2_MAXNREG)
#else
template <int FMT, int kT2Stages, bool MC = false, int EW = 8>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
#endif
k_gram_tc2(const __grid_constant__ CUtensorMap tmap, int64_t m, int TT, int nchunks, int nsplit, int kpc, int super,
           double* __restrict__ part, int kb0) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  tc2_body<FMT, kT2Stages, false, MC, EW>(&tmap, smem, blockIdx.x, blockIdx.y, m, TT, nchunks, nsplit, kpc, super, part,
                                          kb0, T2Ring{nullptr, nullptr, 1, nullptr, nullptr});
}

// ------------------------------------------------------------------------------ 2'. fused rounding + SYRK
// k_gram_fused: steps 1 and 2 in ONE cooperative launch, with A^ never written to HBM.
// Every CTA of split s (one per upper 128-tile) also runs 4 converter warps: the 64-row blocks
// of the split are rounded cooperatively -- unit u = (row r, 64-column chunk q) of a block goes
// to CTA u mod ntiles, converter warp (u / ntiles) mod 4 -- from fp64 A (TMA bulk copies into a
// per-warp staging ring, converted in registers with the hardware cvt.rn: the same single RNE
// rounding as k_round_scaled) into a small L2-resident ring of kFzRing blocks per split, from
// which the tile's TMA producer loads its 128B-swizzled panels exactly as k_gram_tc does.
// Hand-off through two monotonic counters per ring slot (gpu-scope release/acquire, proxy
// fences for the generic-store -> TMA-load path):
//   ready[s][slot]  += 1 per converter warp and block   (consumer waits (gen+1) * ntiles * 4)
//   done[s][slot]   += 1 per tile CTA once its TMA of the block landed
//                                                       (converter waits gen * ntiles to reuse)
// All CTAs are co-resident (cooperative launch, one CTA per SM), so the spin waits progress; a
// wait that exceeds ~1 s of spinning sets *err and proceeds (the host reports TLS_ERR_CUDA).
// HBM traffic: one read of A (8 m n bytes); the ring stays in L2.  The MMA issuer and the
// epilogue (fp32 chunk sums, K_t rows per TMEM chunk, reading R11) are k_gram_tc's.
constexpr int kFzRing = 16;
constexpr int kFzConvWarps = 4;
constexpr int kFzThreads = kTcThreads + 32 * kFzConvWarps;   // 448
constexpr int kFzSlots = 2;                        // staging slots per converter warp
constexpr int kFzSeg = 1024;                       // one unit: up to 1024 fp64 of one row (8 KB)
constexpr int kFzUnit = kFzSeg * 8;
constexpr int kFzMaxN = 2048;                      // D^{-1} staged in shared memory
constexpr int kFzPub = 2;                          // units per release
constexpr size_t kFzSmem = 2 * kTcStages * kTcPanel + (size_t)kFzConvWarps * kFzSlots * kFzUnit + kFzMaxN * 8 +
                           2048 + 1024;

struct FzArgs {
  const double* A;
  int64_t ld;
  int n;
  const double* dinv;
  uint16_t* ring;       // [nsplit][kFzRing][64][npad64]
  int npad64;
  int* ready;           // [nsplit][kFzRing]
  int* done;            // [nsplit][kFzRing]
  int* err;
  int* range;
  unsigned long long* prof;   // debugging (TLS_FZ_PROF=1): per CTA [8] nanoseconds, else nullptr
};


template <int FMT>
__global__ void __launch_bounds__(kFzThreads, 1)
k_gram_fused(const __grid_constant__ CUtensorMap tmap, FzArgs fz, int64_t m, int TT, int nchunks, int nsplit,
             int kpc, int super, double* __restrict__ part) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* panA = smem;
  unsigned char* panB = smem + kTcStages * kTcPanel;
  unsigned char* stg = smem + 2 * kTcStages * kTcPanel;                          // [4 warps][32][512 B]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + (size_t)kFzConvWarps * kFzSlots * kFzUnit);
  uint64_t* empty = full + kTcStages;
  uint64_t* tfull = empty + kTcStages;
  uint64_t* tempty = tfull + kTcAcc;
  uint64_t* cbar = tempty + kTcAcc;                                              // [warps][slots]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(cbar + kFzConvWarps * kFzSlots);
  double* sdinv = reinterpret_cast<double*>(smem + 2 * kTcStages * kTcPanel +
                                            (size_t)kFzConvWarps * kFzSlots * kFzUnit + 2048);   // [kFzMaxN]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = gridDim.x;
  int t = blockIdx.x, I = 0;
  while (t >= TT - I) { t -= TT - I; ++I; }
  const int J = I + t;
  const bool diag = (I == J);
  const int s = blockIdx.y;
  const int c0 = (int)((int64_t)nchunks * s / nsplit), c1 = (int)((int64_t)nchunks * (s + 1) / nsplit);
  const int kb_total = (int)((m + kTcBK - 1) / kTcBK);
  const int kb_begin = c0 * kpc, kb_end = min(c1 * kpc, kb_total);
  const int nblk = kb_end > kb_begin ? kb_end - kb_begin : 0;
  int* ready = fz.ready + s * kFzRing;
  int* done = fz.done + s * kFzRing;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kTcStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < kTcAcc; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8); }
    for (int i = 0; i < kFzConvWarps * kFzSlots; ++i) mbar_init(&cbar[i], 1);
    fence_mbar_init();
  }
  for (int c = threadIdx.x; c < kFzMaxN; c += blockDim.x) sdinv[c] = c < fz.n ? fz.dinv[c] : 0.0;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kTcAcc * kTcTile)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp >= 10) {
    // ---------------- converters: fp64 A -> fl_uf(A D^-1) into the L2 ring.  Units are row
    // segments of up to 1024 columns (8 KB, one bulk copy); the split's units, row by row, go
    // round-robin to its ntiles x 4 converter warps.  A warp converts a unit with 16-byte lanes
    // (16 sub-chunks of 64 columns, unrolled) and releases every kFzPub units.
    const int cw = warp - 10;
    const int nseg = (fz.n + kFzSeg - 1) / kFzSeg;
    const int nconv = ntiles * kFzConvWarps;
    const int wid = blockIdx.x * kFzConvWarps + cw;          // 0..nconv-1 within the split
    const int64_t nu = (int64_t)nblk * kTcBK * nseg;            // units of the split
    unsigned char* my = stg + (size_t)cw * kFzSlots * kFzUnit;
    uint64_t* mb = cbar + cw * kFzSlots;
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int64_t u, int slot) {                     // lane 0
      const int64_t rowl = u / nseg;                            // row within the split
      const int seg = (int)(u % nseg);
      const int64_t row = (int64_t)kb_begin * kTcBK + rowl;
      uint64_t* bar = &mb[slot];
      if (row < m) {
        int cols = (int)(fz.ld - (int64_t)kFzSeg * seg);
        if (cols > kFzSeg) cols = kFzSeg;
        mbar_arrive_expect_tx(bar, (uint32_t)cols * 8);
        bulk_g2s(my + slot * kFzUnit, fz.A + row * fz.ld + (int64_t)kFzSeg * seg, (uint32_t)cols * 8, bar, pol);
      } else {
        mbar_arrive(bar);
      }
    };
    const int nmine = nu > wid ? (int)((nu - 1 - wid) / nconv + 1) : 0;
    if (lane == 0)
      for (int i = 0; i < kFzSlots && i < nmine; ++i) issue(wid + (int64_t)i * nconv, i);
    int bad = 0;
    uint32_t slot_par = 0;
    unsigned long long t_wd = 0, t_mb = 0, t_cv = 0, t_pub = 0;
    int pend[kFzPub];
    int npend = 0;
    int last_gen_waited = -1, last_l = -1;
    for (int i = 0; i < nmine; ++i) {
      const int64_t u = wid + (int64_t)i * nconv;
      const int64_t rowl = u / nseg;
      const int seg = (int)(u % nseg);
      const int l = (int)(rowl / kTcBK), r = (int)(rowl % kTcBK);
      const int slot = l % kFzRing, gen = l / kFzRing;
      unsigned long long ta = fz.prof ? gtime() : 0;
      if (l != last_l) {                        // first unit of this block: the slot must be free
        if (lane == 0 && gen > 0) wait_geq(&done[slot], gen * ntiles, fz.err);
        __syncwarp();
        last_l = l;
      }
      (void)last_gen_waited;
      if (fz.prof) { const unsigned long long tb = gtime(); t_wd += tb - ta; ta = tb; }
      const int sl = i % kFzSlots;
      mbar_wait(&mb[sl], (slot_par >> sl) & 1u);
      slot_par ^= 1u << sl;
      if (fz.prof) { const unsigned long long tb = gtime(); t_mb += tb - ta; ta = tb; }
      const bool live = (int64_t)kb_begin * kTcBK + rowl < m;
      uint16_t* dst = fz.ring + ((size_t)(s * kFzRing + slot) * kTcBK + r) * fz.npad64 + (size_t)kFzSeg * seg;
      const uint32_t src = smem_u32(my + sl * kFzUnit) + 16 * lane;
      const uint32_t dsrc = smem_u32(sdinv + kFzSeg * seg) + 16 * lane;
      const int hmax = min(kFzSeg / 64, (fz.npad64 - kFzSeg * seg) / 64);       // warp-uniform
      // branch-free in the sub-chunk loop: all loads first (the staging slot and sdinv are always
      // in bounds; columns past the copy are garbage but selected away), then convert and store
#pragma unroll
      for (int h0 = 0; h0 < kFzSeg / 64; h0 += 8) {
        double2 v[8], dv[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[h].x), "=d"(v[h].y) : "r"(src + 512 * (h0 + h)));
          asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(dv[h].x), "=d"(dv[h].y) : "r"(dsrc + 512 * (h0 + h)));
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const double x0 = live ? v[h].x * dv[h].x : 0.0;      // sdinv = 0 beyond n
          const double x1 = live ? v[h].y * dv[h].y : 0.0;
          const uint16_t b0 = FMT == 0 ? f64_to_f16_bits(x0) : f64_to_bf16_bits(x0);
          const uint16_t b1 = FMT == 0 ? f64_to_f16_bits(x1) : f64_to_bf16_bits(x1);
          const uint32_t lim = FMT == 0 ? 0x7c00u : 0x7f80u;
          if (h0 + h < hmax) {
            bad |= ((b0 & 0x7fffu) >= lim) | ((b1 & 0x7fffu) >= lim);
            *reinterpret_cast<uint32_t*>(dst + 64 * (h0 + h) + 2 * lane) = (uint32_t)b0 | ((uint32_t)b1 << 16);
          }
        }
      }
      __syncwarp();                             // the slot was read by every lane: refill it
      if (lane == 0 && i + kFzSlots < nmine) issue(u + (int64_t)kFzSlots * nconv, sl);
      if (fz.prof) { const unsigned long long tb = gtime(); t_cv += tb - ta; ta = tb; }
      pend[npend++ % kFzPub] = slot;
      if (npend == kFzPub || i + 1 == nmine) {  // release: generic stores -> TMA (async proxy)
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0)
          for (int p = 0; p < npend; ++p) atomicAdd(&ready[pend[p]], 1);
        npend = 0;
      }
      if (fz.prof) t_pub += gtime() - ta;
    }
    if (bad) atomicExch(fz.range, 1);
    if (fz.prof && lane == 0) {
      unsigned long long* pr = fz.prof + 8 * ((size_t)blockIdx.y * gridDim.x + blockIdx.x);
      atomicAdd(pr + 0, t_wd); atomicAdd(pr + 1, t_mb); atomicAdd(pr + 2, t_cv); atomicAdd(pr + 3, t_pub);
    }
  } else if (warp == 0) {
    // ---------------- TMA producer (ring -> swizzled panels)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      const uint32_t bytes = diag ? kTcPanel : 2 * kTcPanel;
      unsigned long long t_we = 0, t_wr = 0;
      for (int l = 0; l < nblk; ++l) {
        const int st = l % kTcStages;
        const uint32_t ph = (uint32_t)(l / kTcStages) & 1u;
        unsigned long long ta = fz.prof ? gtime() : 0;
        if (l >= kTcStages) mbar_wait(&empty[st], ph ^ 1u);
        if (fz.prof) { const unsigned long long tb = gtime(); t_we += tb - ta; ta = tb; }
        wait_geq(&ready[l % kFzRing], (l / kFzRing + 1) * kTcBK * ((fz.n + kFzSeg - 1) / kFzSeg), fz.err);
        if (fz.prof) t_wr += gtime() - ta;
        fence_proxy_async_global();
        mbar_arrive_expect_tx(&full[st], bytes);
        const int row = (s * kFzRing + l % kFzRing) * kTcBK;
        unsigned char* a = panA + st * kTcPanel;
        tma_load_2d(a, &tmap, I * kTcTile, row, &full[st]);
        tma_load_2d(a + kTcPanel / 2, &tmap, I * kTcTile + 64, row, &full[st]);
        if (!diag) {
          unsigned char* b = panB + st * kTcPanel;
          tma_load_2d(b, &tmap, J * kTcTile, row, &full[st]);
          tma_load_2d(b + kTcPanel / 2, &tmap, J * kTcTile + 64, row, &full[st]);
        }
      }
      if (fz.prof) {
        unsigned long long* pr = fz.prof + 8 * ((size_t)blockIdx.y * gridDim.x + blockIdx.x);
        atomicAdd(pr + 4, t_we); atomicAdd(pr + 5, t_wr);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread), k_gram_tc's loop over the split's chunks
    if (lane == 0) {
      const uint32_t idesc = idesc_f16(FMT);
      int l = 0;
      unsigned long long t_wf = 0, t_wt = 0;
      for (int c = c0; c < c1; ++c) {
        const int j = c - c0;
        const int buf = j % kTcAcc;
        unsigned long long ta = fz.prof ? gtime() : 0;
        if (j >= kTcAcc) mbar_wait(&tempty[buf], (uint32_t)(j / kTcAcc - 1) & 1u);
        if (fz.prof) t_wt += gtime() - ta;
        tc_fence_after();
        const uint32_t dtm = tmem_base + (uint32_t)(buf * kTcTile);
        const int kb1 = min((c + 1) * kpc, kb_total);
        for (int kb = c * kpc; kb < kb1; ++kb, ++l) {
          const int st = l % kTcStages;
          ta = fz.prof ? gtime() : 0;
          mbar_wait(&full[st], (uint32_t)(l / kTcStages) & 1u);
          if (fz.prof) t_wf += gtime() - ta;
          atomicAdd(&done[l % kFzRing], 1);     // the panels of block l are in shared memory
          tc_fence_after();
          const uint32_t a0 = smem_u32(panA + st * kTcPanel);
          const uint32_t b0 = smem_u32((diag ? panA : panB) + st * kTcPanel);
#pragma unroll
          for (int kk = 0; kk < kTcBK / 16; ++kk) {
            const uint64_t ad = sw128_desc(a0 + kk * 2048, kTcPanel / 2, 1024);
            const uint64_t bd = sw128_desc(b0 + kk * 2048, kTcPanel / 2, 1024);
            tc_mma_f16(dtm, ad, bd, idesc, (kb > c * kpc || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[st]);
        }
        tc_commit(&tfull[buf]);
      }
      if (fz.prof) {
        unsigned long long* pr = fz.prof + 8 * ((size_t)blockIdx.y * gridDim.x + blockIdx.x);
        atomicAdd(pr + 6, t_wf); atomicAdd(pr + 7, t_wt);
      }
    }
  } else {
    // ---------------- epilogue (warps 2-9): k_gram_tc's, draining 32 columns at a time
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    double* out = part + ((size_t)s * gridDim.x + blockIdx.x) * (kTcTile * kTcTile) + (size_t)row * kTcTile + half * 64;
    float sm[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) sm[i] = 0.f;
    int pending = 0;
    for (int c = c0; c < c1; ++c) {
      const int j = c - c0;
      const int buf = j % kTcAcc;
      mbar_wait(&tfull[buf], (uint32_t)(j / kTcAcc) & 1u);
      tc_fence_after();
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kTcTile + half * 64);
      uint32_t r0[32];
      TLS_TMEM_LD32(ta, r0);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 32; ++k) sm[k] = __fadd_rn(sm[k], __uint_as_float(r0[k]));
      TLS_TMEM_LD32(ta + 32, r0);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
#pragma unroll
      for (int k = 0; k < 32; ++k) sm[k + 32] = __fadd_rn(sm[k + 32], __uint_as_float(r0[k]));
      if (++pending == super) {
#pragma unroll
        for (int k = 0; k < 64; ++k) { atomicAdd(out + k, (double)sm[k]); sm[k] = 0.f; }
        pending = 0;
      }
    }
    if (pending) {
#pragma unroll
      for (int k = 0; k < 64; ++k) atomicAdd(out + k, (double)sm[k]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcAcc * kTcTile) : "memory");
  }
}

// ------------------------------------------------------------------------------ 2''. split-role fused Gram
// k_gram_fused2 (opt-in TLS_GRAM_FUSED=2, n > 896, K_t = 64; A^ "formed on chip,
// never stored"): ONE cooperative launch of one CTA per SM in two roles.  CTAs [0, nblk2 * nsplit) are
// k_gram_tc2's SYRK CTAs reading their panels from a per-split L2 ring of kF2R 64-row blocks
// (tc2_body<RING>); the other CTAs are converters: they stream fp64 A through shared memory with
// bulk copies (3 pieces of up to 64 KB in flight), form fl_uf(A D^-1) with the same single RNE
// rounding as k_round_scaled (so G is bit-identical to the two-kernel path with the same splits),
// and write each block into its ring slot once all nblk2 CTAs of the split have taken the previous
// generation (done counters), then publish it (ready).  Why split roles: converter warps inside
// the SYRK CTAs (k_gram_fused) were limited to 4 per SM by the epilogue's registers and ran
// latency-bound; a whole SM streams ~86 GB/s (tools/micro/conv_bw.cu, profiles/r02_conv_bw.log).
// Deadlock-free: each converter takes its units in increasing (chunk, split) order, a unit only
// waits for consumers of an earlier generation, and all CTAs are co-resident (cooperative launch).
constexpr int kF2R = 32;                 // ring blocks per split
constexpr int kF2Buf = 3;                // converter pieces in flight

template <int PREC, int prow>
__device__ __forceinline__ void conv_body(int cv, int ncv, const FzArgs& fz, int64_t m, int nchunks, int nsplit,
                                          int nblk2, unsigned char* smem) {
  const int n = fz.n, npad64 = fz.npad64, tid = threadIdx.x;
  const int64_t ld = fz.ld;
  double* buf = reinterpret_cast<double*>(smem);                              // [kF2Buf][prow * ld]
  double* sdinv = buf + (size_t)kF2Buf * prow * ld;                           // [n]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sdinv + ((n + 1) & ~1));        // [kF2Buf]
  if (tid == 0) {
    for (int i = 0; i < kF2Buf; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  for (int c = tid; c < n; c += blockDim.x) sdinv[c] = fz.dinv[c];
  __syncthreads();
  const int maxch = (nchunks + nsplit - 1) / nsplit;
  const int64_t total = (int64_t)maxch * nsplit;
  const int ppu = kTcBK / prow;                                               // pieces per 64-row unit
  const uint64_t pol = policy_evict_first();
  struct U { bool any, valid; int s, j, c0s; };
  auto unit = [&](int64_t p) -> U {
    U u{};
    const int64_t idx = cv + (p / ppu) * ncv;
    if (idx >= total) return u;
    u.any = true;
    u.s = (int)(idx % nsplit);
    u.j = (int)(idx / nsplit);
    u.c0s = (int)((int64_t)nchunks * u.s / nsplit);
    u.valid = u.j < (int)((int64_t)nchunks * (u.s + 1) / nsplit) - u.c0s;
    return u;
  };
  auto issue = [&](int64_t p) {                                               // thread 0
    const U u = unit(p);
    if (!u.any) return;
    uint64_t* b = &bar[p % kF2Buf];
    const int64_t row0 = (int64_t)(u.c0s + u.j) * kTcBK + (p % ppu) * prow;
    const int64_t rows = u.valid ? (m - row0 < prow ? (m - row0 > 0 ? m - row0 : 0) : prow) : 0;
    if (rows > 0) {
      mbar_arrive_expect_tx(b, (uint32_t)(rows * ld * 8));
      bulk_g2s(buf + (size_t)(p % kF2Buf) * prow * ld, fz.A + row0 * ld, (uint32_t)(rows * ld * 8), b, pol);
    } else {
      mbar_arrive(b);
    }
  };
  if (tid == 0)
    for (int p = 0; p < kF2Buf; ++p) issue(p);
  uint32_t* ring32 = reinterpret_cast<uint32_t*>(fz.ring);
  const int pairs = npad64 / 2;
  int bad = 0;
  unsigned long long t_ld = 0, t_dn = 0, t_cv = 0, ta = 0, tb = 0;
  const bool prof = fz.prof != nullptr && tid == 0;
  for (int64_t p = 0;; ++p) {
    const U u = unit(p);
    if (!u.any) break;
    if (prof) ta = gtime();
    mbar_wait(&bar[p % kF2Buf], (uint32_t)(p / kF2Buf) & 1u);
    if (prof) { tb = gtime(); t_ld += tb - ta; }
    const int sub = (int)(p % ppu);
    const int slot = u.j % kF2R, gen = u.j / kF2R;
    if (u.valid) {
      if (sub == 0) {                                   // the slot's previous block has been taken
        if (tid == 0 && gen > 0) wait_geq(&fz.done[u.s * kF2R + slot], gen * nblk2, fz.err);
        __syncthreads();
        if (prof) { ta = gtime(); t_dn += ta - tb; tb = ta; }
      }
      const double* src = buf + (size_t)(p % kF2Buf) * prow * ld;
      const int64_t row0 = (int64_t)(u.c0s + u.j) * kTcBK + sub * prow;
      const int64_t rows = m - row0 < prow ? (m - row0 > 0 ? m - row0 : 0) : prow;
      uint32_t* dst = ring32 + ((int64_t)(u.s * kF2R + slot) * kTcBK + sub * prow) * pairs;
      for (int cp = tid; cp < pairs; cp += blockDim.x) {
        const int c = 2 * cp;
        const double d0 = c < n ? sdinv[c] : 0.0, d1 = c + 1 < n ? sdinv[c + 1] : 0.0;
#pragma unroll
        for (int rr = 0; rr < prow; ++rr) {                     // prow independent loads in flight
          double x0 = 0.0, x1 = 0.0;
          if (rr < rows) {
            if (c + 1 < n) {
              const double2 v = *reinterpret_cast<const double2*>(src + rr * ld + c);
              x0 = v.x * d0;
              x1 = v.y * d1;
            } else if (c < n) {
              x0 = src[rr * ld + c] * d0;
            }
          }
          const uint16_t h0 = PREC == TLS_FP16 ? f64_to_f16_bits(x0) : f64_to_bf16_bits(x0);   // one RNE rounding
          const uint16_t h1 = PREC == TLS_FP16 ? f64_to_f16_bits(x1) : f64_to_bf16_bits(x1);
          const uint32_t lim = PREC == TLS_FP16 ? 0x7c00u : 0x7f80u;
          bad |= ((h0 & 0x7fffu) >= lim) | ((h1 & 0x7fffu) >= lim);
          dst[(int64_t)rr * pairs + cp] = (uint32_t)h0 | ((uint32_t)h1 << 16);
        }
      }
    }
    __syncthreads();                                    // the piece is read and its rows written
    if (prof) t_cv += gtime() - tb;
    if (tid == 0) {
      issue(p + kF2Buf);
      if (u.valid && sub == ppu - 1) {
        __threadfence();
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(fz.ready + u.s * kF2R + slot), "r"(gen + 1) : "memory");
      }
    }
  }
  if (bad) atomicExch(fz.range, 1);
  if (prof) {
    fz.prof[blockIdx.x * 8 + 0] = t_ld;
    fz.prof[blockIdx.x * 8 + 1] = t_dn;
    fz.prof[blockIdx.x * 8 + 2] = t_cv;
  }
}

template <int FMT>
__global__ void __launch_bounds__(kTcThreads, 1)
k_gram_fused2(const __grid_constant__ CUtensorMap rmap, FzArgs fz, int64_t m, int TT, int nchunks, int nsplit,
              int nblk2, int super, double* __restrict__ part, int prow) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int nsy = nblk2 * nsplit;
  if ((int)blockIdx.x < nsy)
    tc2_body<FMT, 3, true>(&rmap, smem, blockIdx.x % nblk2, blockIdx.x / nblk2, m, TT, nchunks, nsplit, 1, super, part, 0,
                           T2Ring{fz.ready, fz.done, kF2R, fz.err, fz.prof});
  else {
    constexpr int PREC = FMT == 0 ? TLS_FP16 : TLS_BF16;
    const int cv = blockIdx.x - nsy, ncv = gridDim.x - nsy;
    switch (prow) {
      case 8: conv_body<PREC, 8>(cv, ncv, fz, m, nchunks, nsplit, nblk2, smem); break;
      case 4: conv_body<PREC, 4>(cv, ncv, fz, m, nchunks, nsplit, nblk2, smem); break;
      case 2: conv_body<PREC, 2>(cv, ncv, fz, m, nchunks, nsplit, nblk2, smem); break;
      default: conv_body<PREC, 1>(cv, ncv, fz, m, nchunks, nsplit, nblk2, smem); break;
    }
  }
}

// The split-role plan: nsplit maximising throughput under the measured rates (SYRK ~0.68 us per
// 128 x 256 block and 64-row chunk at n = 1024; a converter CTA ~86 GB/s of fp64), at least 16
// converters.  Returns nsplit, or 0 when the fused path does not apply.
static int fused2_plan(int64_t m, int n, int64_t ld, int sms, int& prow) {
  const int TT = (n + kTcTile - 1) / kTcTile;
  const int nblk2 = t2_blocks(TT);
  prow = 0;
  for (int r = 8; r >= 1; r >>= 1)
    if ((int64_t)r * ld * 8 <= 65536) { prow = r; break; }
  if (prow == 0 || n > kFzMaxN) return 0;
  const int64_t nchunks = (m + kTcBK - 1) / kTcBK;
  int best = 0;
  double bt = 1e30;
  for (int s = 1; nblk2 * s + 16 <= sms && s <= nchunks; ++s) {
    const double ts = (double)((nchunks + s - 1) / s) * 0.68e-6;
    const double tc = (double)m * ld * 8 / ((double)(sms - nblk2 * s) * 86e9);
    const double t = ts > tc ? ts : tc;
    if (t < bt) { bt = t; best = s; }
  }
  return best;
}

static size_t conv_smem(int prow, int64_t ld, int n) {
  return (size_t)kF2Buf * prow * ld * 8 + (size_t)((n + 1) & ~1) * 8 + kF2Buf * 8 + 64;
}

// ------------------------------------------------------------------------------ 3. split reduction
// Split partials -> G (both triangles).  CTA (tile, 8-row chunk): every thread adds its elements'
// nsplit partials in split order (the same bits as one split at a time), with all of them in
// flight; the row-major write is coalesced and the transposed one goes through shared memory
// in 64-byte column segments.  (Round 2 continued: one CTA per tile with a strided transposed
// store took ~125 us per factorization at n = 1024.)
constexpr int kRedRows = 8;
constexpr int kRedMaxSplit = 16;
__global__ void __launch_bounds__(256) k_gram_reduce_t(const double* __restrict__ part, int ntiles, int nsplit, int TT,
                                                      int tile, int n, double* __restrict__ G) {
  __shared__ double tr[kRedRows][kTcTile + 1];
  int t = blockIdx.x, I = 0;
  while (t >= TT - I) { t -= TT - I; ++I; }
  const int J = I + t;
  const int te = tile * tile;
  const int i0 = blockIdx.y * kRedRows;
  const int cpt = tile / 32;                             // columns per lane (tile = 128: 4)
  const int ri = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = i0 + ri, gi = I * tile + i;
  for (int c = 0; c < cpt; ++c) {
    const int j = lane + 32 * c, gj = J * tile + j;
    const int e = i * tile + j;
    double v[kRedMaxSplit];
#pragma unroll
    for (int s = 0; s < kRedMaxSplit; ++s) v[s] = s < nsplit ? part[((size_t)s * ntiles + blockIdx.x) * te + e] : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < kRedMaxSplit; ++s)
      if (s < nsplit) acc += v[s];
    for (int s = kRedMaxSplit; s < nsplit; ++s) acc += part[((size_t)s * ntiles + blockIdx.x) * te + e];
    if (gi < n && gj < n) G[(size_t)gi * n + gj] = acc;
    tr[ri][j] = acc;
  }
  __syncthreads();
  // transposed: G[gj][gi] for the chunk's 8 rows i: thread = (column j, row lane pair)
  for (int k = threadIdx.x; k < tile * kRedRows; k += blockDim.x) {
    const int j = k / kRedRows, r = k % kRedRows;
    const int gj = J * tile + j, gir = I * tile + i0 + r;
    if (gj < n && gir < n) G[(size_t)gj * n + gir] = tr[r][j];
  }
}

// ------------------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Chunk sums per fp64 flush and the compensation switch (TLS_GRAM_SUPER / TLS_GRAM_KAHAN
// override the defaults for accuracy experiments, tools/gram_check.py).
static int gram_super() {
  const char* e = getenv("TLS_GRAM_SUPER");
  const int v = e ? atoi(e) : 64;
  return v < 1 ? 1 : v;
}
static int gram_kahan() {
  const char* e = getenv("TLS_GRAM_KAHAN");
  return e ? atoi(e) != 0 : 0;
}

// k_gram_tc2 (128 x 256 blocks) for n > 896 (TT >= 8 tiles: measured faster at 2^20 x 1024,
// 200000 x 2000, 65536 x 2048; slower at n = 256, where a diagonal block wastes half its work);
// TLS_GRAM_TC=128 / =256 force either kernel; TLS_GRAM_KAHAN uses the 128 x 128 kernel
static bool gram_tc2_enabled(int n) {
  const char* e = getenv("TLS_GRAM_TC");
  if (gram_kahan() || (e && atoi(e) == 128)) return false;
  if (e && atoi(e) == 256) return true;
  return (n + kTcTile - 1) / kTcTile >= 8;
}

static void tc_shape(int64_t m, int n, int K_t, int& TT, int& ntiles, int& nchunks, int& nsplit, bool tc2) {
  TT = (n + kTcTile - 1) / kTcTile;
  ntiles = TT * (TT + 1) / 2;
  nchunks = (int)((m + K_t - 1) / K_t);
  if (nchunks < 1) nchunks = 1;
  // one wave of persistent-tile CTAs (1 CTA/SM): CTAs per split * nsplit <= #SMs when possible
  nsplit = num_sms() / (tc2 ? t2_blocks(TT) : ntiles);
  if (nsplit > nchunks) nsplit = nchunks;
  if (nsplit < 1) nsplit = 1;
}
static void tc_shape(int64_t m, int n, int K_t, int& TT, int& ntiles, int& nchunks, int& nsplit) {
  tc_shape(m, n, K_t, TT, ntiles, nchunks, nsplit, false);
}

bool gram_tc_supported(int u_f, int K_t) {
  if (u_f != TLS_FP16 && u_f != TLS_BF16) return false;
  if (K_t % kTcBK != 0) return false;
  const char* e = getenv("TLS_GRAM");
  if (e && e[0] == 'c') return false;  // TLS_GRAM=cc forces the CUDA-core path
  return encode_fn() != nullptr;
}

// The fused path's ring (kFzRing 64-row blocks of A^ per split, rows of round64(n) 16-bit
// values) plus its counters; used in place of the A^ buffer of the two-kernel path.
static size_t fz_ring_bytes(int n, int nsplit) {
  const int npad64 = (n + 63) / 64 * 64;
  return (size_t)nsplit * kFzRing * kTcBK * npad64 * 2 + 2 * (size_t)nsplit * kFzRing * 4 + 256;
}

size_t gram_tc_ws_bytes(int64_t m, int n, int K_t) {
  int TT, ntiles, nchunks, nsplit;
  tc_shape(m, n, K_t < kTcBK ? kTcBK : K_t, TT, ntiles, nchunks, nsplit);
  int ns2 = 0;
  tc_shape(m, n, K_t < kTcBK ? kTcBK : K_t, TT, ntiles, nchunks, ns2, true);
  const int nsp = ns2 > nsplit ? ns2 : nsplit;                   // partials for either kernel
  const int npad = (n + 7) / 8 * 8;
  size_t ah = ((size_t)m * npad * 2 + 1023) & ~(size_t)1023;
  const size_t fz = (fz_ring_bytes(n, nsplit) + 1023) & ~(size_t)1023;
  if (fz > ah) ah = fz;
  return ah + (size_t)nsp * ntiles * kTcTile * kTcTile * 8;
}

// TLS_GRAM_FUSED=1 selects the fused kernel.  Measured (tools/time_gram_fused.py, profiles/
// r02_gram_fused.txt): bit-identical G, HBM traffic = one read of A (ncu: 2.17 GB read, 37 MB
// written at 2^18 x 1024: the ring never leaves L2), but 7.8 ms against 4.5 ms for the
// two-kernel path at 2^20 x 1024: the 4 converter warps per SM the register file leaves next to
// the 8-warp epilogue (448 threads x 128 registers) are issue/latency-bound (ncu: 0.25 eligible
// warps per scheduler, 18% issue slots busy), so the default stays k_round_scaled + k_gram_tc.
static bool gram_fused_enabled() {
  const char* e = getenv("TLS_GRAM_FUSED");
  return e && e[0] == '1';
}

int launch_gram_tc(const DenseView& A, int u_f, const double* dinv, int K_t, double* G, void* ws, size_t ws_bytes,
                   int* range_flag, cudaStream_t st, int* launches) {
  int TT, ntiles, nchunks, nsplit;
  tc_shape(A.m, A.n, K_t, TT, ntiles, nchunks, nsplit);
  const int npad = (A.n + 7) / 8 * 8;
  const size_t ah_bytes = ((size_t)A.m * npad * 2 + 1023) & ~(size_t)1023;
  if (gram_tc_ws_bytes(A.m, A.n, K_t) > ws_bytes) {
    set_error("gram_tc: workspace too small");
    return TLS_ERR_WORKSPACE;
  }
  uint16_t* Ah = static_cast<uint16_t*>(ws);
  size_t a_region = ah_bytes;
  {
    const size_t fz = (fz_ring_bytes(A.n, nsplit) + 1023) & ~(size_t)1023;
    if (fz > a_region) a_region = fz;
  }
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + a_region);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (gram_fused_enabled() && ntiles * nsplit <= sms && A.n <= kFzMaxN) {
    // ---- fused: rounding inside the tensor-core kernel, A^ only in an L2-resident ring
    const int npad64 = (A.n + 63) / 64 * 64;
    FzArgs fz;
    fz.A = A.A;
    fz.ld = A.ld;
    fz.n = A.n;
    fz.dinv = dinv;
    fz.ring = Ah;
    fz.npad64 = npad64;
    fz.ready = reinterpret_cast<int*>(reinterpret_cast<char*>(Ah) + (size_t)nsplit * kFzRing * kTcBK * npad64 * 2);
    fz.done = fz.ready + nsplit * kFzRing;
    fz.err = range_flag + 3;            // the factor's flags[4]: a ring hand-off timed out
    fz.range = range_flag;
    fz.prof = nullptr;
    const char* pe = getenv("TLS_FZ_PROF");
    if (pe && pe[0] == '1') {                  // debugging only: per-CTA wait/work times
      TLS_CUDA_TRY(cudaMalloc(&fz.prof, (size_t)ntiles * nsplit * 8 * 8));
      TLS_CUDA_TRY(cudaMemsetAsync(fz.prof, 0, (size_t)ntiles * nsplit * 8 * 8, st));
    }
    TLS_CUDA_TRY(cudaMemsetAsync(fz.ready, 0, 2 * (size_t)nsplit * kFzRing * 4, st));
    CUtensorMap rmap;
    const cuuint64_t dims[2] = {(cuuint64_t)npad64, (cuuint64_t)nsplit * kFzRing * kTcBK};
    const cuuint64_t strides[1] = {(cuuint64_t)npad64 * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)kTcBK};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&rmap, u_f == TLS_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                   2, Ah, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (ring) failed (%d)", (int)r);
      return TLS_ERR_CUDA;
    }
    TLS_CUDA_TRY(cudaMemsetAsync(part, 0, (size_t)nsplit * ntiles * kTcTile * kTcTile * 8, st));
    auto kern = u_f == TLS_FP16 ? k_gram_fused<0> : k_gram_fused<1>;
    TLS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFzSmem));
    int per_sm = 0;
    TLS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFzThreads, kFzSmem));
    if (per_sm >= 1) {
      int64_t mm = A.m;
      int tt = TT, nc = nchunks, ns = nsplit, kpc = K_t / kTcBK, sup = gram_super();
      void* args[] = {(void*)&rmap, &fz, &mm, &tt, &nc, &ns, &kpc, &sup, &part};
      TLS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(ntiles, nsplit), dim3(kFzThreads), args, kFzSmem, st));
      k_gram_reduce_t<<<dim3(ntiles, kTcTile / kRedRows), 256, 0, st>>>(part, ntiles, nsplit, TT, kTcTile, A.n, G);
      TLS_LAUNCH_CHECK();
      if (fz.prof) {
        std::vector<unsigned long long> h((size_t)ntiles * nsplit * 8);
        cudaMemcpy(h.data(), fz.prof, h.size() * 8, cudaMemcpyDeviceToHost);
        double avg[8] = {};
        for (size_t b = 0; b < (size_t)ntiles * nsplit; ++b)
          for (int k = 0; k < 8; ++k) avg[k] += h[b * 8 + k] / 1e6 / (ntiles * nsplit) / (k < 4 ? kFzConvWarps : 1);
        fprintf(stderr, "[fz] ms per CTA: conv wait_done %.3f wait_stage %.3f convert %.3f publish %.3f | "
                "producer wait_empty %.3f wait_ready %.3f | mma wait_full %.3f wait_tempty %.3f\n",
                avg[0], avg[1], avg[2], avg[3], avg[4], avg[5], avg[6], avg[7]);
        cudaFree(fz.prof);
      }
      if (launches) *launches += 2;
      return 0;
    }
  }
  // ---- the split-role fused Gram (k_gram_fused2, opt-in TLS_GRAM_FUSED=2; =1 is k_gram_fused above).
  // Measured (tools/time_gram_fused2.py, profiles/r02_gram_fused2.txt): G bit-identical to the
  // two-kernel path with the same splits, but 8.9 ms against 3.27 ms at 2^20 x 1024: sharing L2
  // with the SYRK's ~10 TB/s of panel reads, a converter SM streams ~44 GB/s instead of the 86 it
  // reaches alone (tools/micro/conv_bw.cu), and the SYRK CTAs slow down too, so not the default.
  {
    const char* fe = getenv("TLS_GRAM_FUSED");
    const bool want = fe && fe[0] == '2';
    int prow = 0;
    int ns2 = (want && gram_tc2_enabled(A.n) && K_t == kTcBK) ? fused2_plan(A.m, A.n, A.ld, sms, prow) : 0;
    const char* nse = getenv("TLS_GRAM_NSPLIT");                    // test knob: force the split count
    if (ns2 > 0 && nse && atoi(nse) > 0) {
      ns2 = atoi(nse);
      if (ns2 > (sms - 16) / t2_blocks(TT)) ns2 = (sms - 16) / t2_blocks(TT);
    }
    const int npad64 = (A.n + 63) / 64 * 64;
    const size_t ring_bytes = (size_t)ns2 * kF2R * kTcBK * npad64 * 2;
    int split2 = 0, TT2, nt2, nc2;
    tc_shape(A.m, A.n, K_t, TT2, nt2, nc2, split2, true);
    if (ns2 > 0 && ns2 <= split2 && ring_bytes + 2 * (size_t)ns2 * kF2R * 4 + 256 <= a_region) {
      const int nblk2 = t2_blocks(TT);
      FzArgs fz;
      fz.A = A.A;
      fz.ld = A.ld;
      fz.n = A.n;
      fz.dinv = dinv;
      fz.ring = Ah;
      fz.npad64 = npad64;
      fz.ready = reinterpret_cast<int*>(reinterpret_cast<char*>(Ah) + ring_bytes);
      fz.done = fz.ready + ns2 * kF2R;
      fz.err = range_flag + 3;            // the factor's flags[4]: a ring hand-off timed out
      fz.range = range_flag;
      fz.prof = nullptr;
      const char* pe = getenv("TLS_FZ_PROF");
      if (pe && pe[0] == '1') {                  // debugging only: per-CTA wait/work times
        TLS_CUDA_TRY(cudaMalloc(&fz.prof, (size_t)sms * 8 * 8));
        TLS_CUDA_TRY(cudaMemsetAsync(fz.prof, 0, (size_t)sms * 8 * 8, st));
      }
      TLS_CUDA_TRY(cudaMemsetAsync(fz.ready, 0, 2 * (size_t)ns2 * kF2R * 4, st));
      TLS_CUDA_TRY(cudaMemsetAsync(part, 0, (size_t)ns2 * ntiles * kTcTile * kTcTile * 8, st));
      CUtensorMap rmap;
      const cuuint64_t dims[2] = {(cuuint64_t)npad64, (cuuint64_t)ns2 * kF2R * kTcBK};
      const cuuint64_t strides[1] = {(cuuint64_t)npad64 * 2};
      const cuuint32_t box[2] = {64, (cuuint32_t)kTcBK};
      const cuuint32_t estr[2] = {1, 1};
      const CUresult r = encode_fn()(&rmap, u_f == TLS_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                     2, Ah, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (fused2 ring) failed (%d)", (int)r);
        return TLS_ERR_CUDA;
      }
      size_t smem2 = t2_smem(3);
      const size_t cs = conv_smem(prow, A.ld, A.n) + 1024;
      if (cs > smem2) smem2 = cs;
      auto kern = u_f == TLS_FP16 ? k_gram_fused2<0> : k_gram_fused2<1>;
      TLS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      int per_sm = 0;
      TLS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTcThreads, smem2));
      if (per_sm >= 1) {
        int64_t mm = A.m;
        int tt = TT, nc = nchunks, ns = ns2, nb = nblk2, sup = gram_super(), pr = prow;
        void* args[] = {(void*)&rmap, &fz, &mm, &tt, &nc, &ns, &nb, &sup, &part, &pr};
        TLS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(sms), dim3(kTcThreads), args, smem2, st));
        k_gram_reduce_t<<<dim3(ntiles, kTcTile / kRedRows), 256, 0, st>>>(part, ntiles, ns2, TT, kTcTile, A.n, G);
        TLS_LAUNCH_CHECK();
        if (fz.prof) {
          std::vector<unsigned long long> h((size_t)sms * 8);
          cudaMemcpy(h.data(), fz.prof, h.size() * 8, cudaMemcpyDeviceToHost);
          const int nsy = nblk2 * ns2;
          double cv[3] = {}, sy = 0;
          for (int b = 0; b < sms; ++b) {
            if (b < nsy) sy += h[b * 8 + 3] / 1e6 / nsy;
            else for (int k = 0; k < 3; ++k) cv[k] += h[b * 8 + k] / 1e6 / (sms - nsy);
          }
          fprintf(stderr, "[fused2] %d SYRK CTAs (%d splits), %d converters; ms per CTA: converter wait-load %.3f "
                  "wait-done %.3f convert %.3f | SYRK producer wait-ready %.3f\n", nsy, ns2, sms - nsy, cv[0], cv[1], cv[2], sy);
          cudaFree(fz.prof);
        }
        if (launches) *launches += 2;
        return 0;
      }
    }
  }
  // 1.+2. row segments: k_round_scaled of segment k+1 (side stream) overlaps k_gram_tc of segment
  // k (caller's stream): the rounding pass is HBM-bound, the SYRK L2/latency-bound, and both
  // fit on an SM together (registers 320 x 168 + 256 x 32, one SYRK CTA per SM).  Segment
  // boundaries are multiples of K_t rows, so every K_t chunk stays within one segment; each
  // segment's launch restarts the 64-chunk fp32 flush grouping (another member of R11's family).
  CUtensorMap tmap;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)npad, (cuuint64_t)A.m};
    const cuuint64_t strides[1] = {(cuuint64_t)npad * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)kTcBK};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&tmap, u_f == TLS_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                   2, Ah, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
      return TLS_ERR_CUDA;
    }
  }
  const char* se = getenv("TLS_GRAM_SEGS");
  int nseg = se ? atoi(se) : 8;
  const int64_t seg_unit = K_t;                                   // boundaries on chunk edges
  const int64_t units = (A.m + seg_unit - 1) / seg_unit;
  if (nseg < 1) nseg = 1;
  if (units < (int64_t)nseg * nsplit * 4) nseg = 1;               // small m: one launch
  // the side stream and the events (one set per device, made on first use)
  struct Side { int dev = -1; cudaStream_t s = nullptr; cudaEvent_t fork = nullptr, ev[16] = {}; };
  static Side side_cache[8];
  Side& sd = side_cache[dev & 7];
  if (nseg > 1 && sd.dev != dev) {
    TLS_CUDA_TRY(cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking));
    TLS_CUDA_TRY(cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming));
    for (auto& e : sd.ev) TLS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    sd.dev = dev;
  }
  if (nseg > 16) nseg = 16;
  const bool tc2 = gram_tc2_enabled(A.n);
  if (tc2) tc_shape(A.m, A.n, K_t, TT, ntiles, nchunks, nsplit, true);   // splits of the 128 x 256 blocks
  if (const char* nse = getenv("TLS_GRAM_NSPLIT"))                         // test knob: fewer splits
    if (atoi(nse) > 0 && atoi(nse) < nsplit) nsplit = atoi(nse);
  // 3 stages (144 KB) measured faster than 4 at 2^20 x 1024, alone (3.46 vs 3.52 ms incl. the
  // rounding pass) and overlapped with it (3.36 vs 4.80: with 4 stages the SYRK CTA's 226 KB of
  // shared memory leaves the concurrent rounding pass no L1); TLS_GRAM_STAGES=4 for experiments
  const char* sge = getenv("TLS_GRAM_STAGES");
  const int st2 = sge && atoi(sge) == 4 ? 4 : 3;
  // TLS_GRAM_EW=16: 16 epilogue warps of 64 columns (experiment)
  const char* ewe = getenv("TLS_GRAM_EW");
  const int ew = (ewe && atoi(ewe) == 16 && st2 == 3) ? 16 : 8;
  const size_t smem = tc2 ? t2_smem(st2, ew) : kTcSmem;
  const bool kahan = gram_kahan();
  const char* ee = getenv("TLS_GRAM_EPI");   // experiment knob: 0 sync only, 1 + TMEM loads, 2 full
  auto kfn = u_f == TLS_FP16 ? (kahan ? k_gram_tc<0, true> : k_gram_tc<0, false>)
                             : (kahan ? k_gram_tc<1, true> : k_gram_tc<1, false>);
  auto kfn2 = u_f == TLS_FP16 ? (st2 == 3 ? k_gram_tc2<0, 3> : k_gram_tc2<0, 4>) : (st2 == 3 ? k_gram_tc2<1, 3> : k_gram_tc2<1, 4>);
  // TLS_GRAM_MC=1: 2-CTA clusters sharing the B panel by TMA multicast (needs an even tile count)
  const char* mce = getenv("TLS_GRAM_MC");
  const bool mc = tc2 && mce && mce[0] == '1' && (TT % 2 == 0) && st2 == 3;
  auto kfn2mc = u_f == TLS_FP16 ? k_gram_tc2<0, 3, true> : k_gram_tc2<1, 3, true>;
  if (mc) TLS_CUDA_TRY(cudaFuncSetAttribute(kfn2mc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t2_smem(3)));
  auto kfn2ew = u_f == TLS_FP16 ? k_gram_tc2<0, 3, false, 16> : k_gram_tc2<1, 3, false, 16>;
  if (ew == 16) TLS_CUDA_TRY(cudaFuncSetAttribute(kfn2ew, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  TLS_CUDA_TRY(cudaFuncSetAttribute(tc2 ? (const void*)kfn2 : (const void*)kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  TLS_CUDA_TRY(cudaMemsetAsync(part, 0, (size_t)nsplit * ntiles * kTcTile * kTcTile * 8, st));
  const int nblk2 = t2_blocks(TT);
  // TLS_ROUND=1: round 2's one row in flight per thread (read per call: the equality test
  // switches it); default two rows.  A third form with the loads staged in shared memory by
  // cp.async was bit-identical and slower (2^20 x 1024: 4.44 vs 3.24 ms, profiles/r02f_round.log)
  const char* rve = getenv("TLS_ROUND");
  int rv = (rve && atoi(rve) == 1) ? 1 : ((rve && atoi(rve) == 3) ? 3 : 2);
  if (rv == 3 && (A.n & 1)) rv = 2;                                // bulk copies move multiples of 16 B
  if (rv == 3) {
    TLS_CUDA_TRY(cudaFuncSetAttribute(k_round_bulk<TLS_FP16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRbSmem));
    TLS_CUDA_TRY(cudaFuncSetAttribute(k_round_bulk<TLS_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRbSmem));
  }
  cudaStream_t rs = nseg > 1 ? sd.s : st;
  if (nseg > 1) {
    TLS_CUDA_TRY(cudaEventRecord(sd.fork, st));                    // D^{-1} and the memset are ready
    TLS_CUDA_TRY(cudaStreamWaitEvent(rs, sd.fork, 0));
  }
  for (int k = 0; k < nseg; ++k) {
    const int64_t r0 = units * k / nseg * seg_unit;
    int64_t r1 = units * (k + 1) / nseg * seg_unit;
    if (r1 > A.m) r1 = A.m;
    const int64_t rows = r1 - r0;
    if (rows <= 0) continue;
    int64_t g = rows;
    const int64_t gmax = (int64_t)num_sms() * (nseg > 1 ? 4 : 8);
    if (g > gmax) g = gmax;
    const double* src = A.A + r0 * A.ld;
    uint16_t* dst = Ah + r0 * npad;
    if (rv == 3) {
      const char* ge = getenv("TLS_ROUND_GRID");
      int64_t gb = (int64_t)num_sms() * (ge && atoi(ge) > 0 ? atoi(ge) : 3);   // 3 per SM measured best (r02h_round_bulk.log)
      if (gb > rows) gb = rows;
      if (u_f == TLS_FP16)
        k_round_bulk<TLS_FP16><<<(int)gb, kRbThreads, kRbSmem, rs>>>(src, rows, A.n, A.ld, dinv, dst, npad, range_flag);
      else
        k_round_bulk<TLS_BF16><<<(int)gb, kRbThreads, kRbSmem, rs>>>(src, rows, A.n, A.ld, dinv, dst, npad, range_flag);
    } else if (rv == 1) {
      if (u_f == TLS_FP16)
        k_round_scaled<TLS_FP16, 1><<<(int)g, 256, 0, rs>>>(src, rows, A.n, A.ld, dinv, dst, npad, range_flag);
      else
        k_round_scaled<TLS_BF16, 1><<<(int)g, 256, 0, rs>>>(src, rows, A.n, A.ld, dinv, dst, npad, range_flag);
    } else {
      if (u_f == TLS_FP16)
        k_round_scaled<TLS_FP16, 2><<<(int)g, 256, 0, rs>>>(src, rows, A.n, A.ld, dinv, dst, npad, range_flag);
      else
        k_round_scaled<TLS_BF16, 2><<<(int)g, 256, 0, rs>>>(src, rows, A.n, A.ld, dinv, dst, npad, range_flag);
    }
    TLS_LAUNCH_CHECK();
    if (nseg > 1) {
      TLS_CUDA_TRY(cudaEventRecord(sd.ev[k], rs));
      TLS_CUDA_TRY(cudaStreamWaitEvent(st, sd.ev[k], 0));
    }
    int TTs, nts, ncs, nss;
    tc_shape(rows, A.n, K_t, TTs, nts, ncs, nss);
    const int ns_use = nsplit < ncs ? nsplit : ncs;               // the part buffer holds nsplit splits
    if (tc2 && mc) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nblk2, ns_use);
      cfg.blockDim = dim3(kTcThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int kbs = (int)(r0 / kTcBK), kpcv = K_t / kTcBK, sup = gram_super();
      TLS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kfn2mc, tmap, rows, TT, ncs, ns_use, kpcv, sup, part, kbs));
    } else if (tc2 && ew == 16)
      kfn2ew<<<dim3(nblk2, ns_use), 64 + 32 * 16, smem, st>>>(tmap, rows, TT, ncs, ns_use, K_t / kTcBK, gram_super(), part,
                                                              (int)(r0 / kTcBK));
    else if (tc2)
      kfn2<<<dim3(nblk2, ns_use), kTcThreads, smem, st>>>(tmap, rows, TT, ncs, ns_use, K_t / kTcBK, gram_super(), part,
                                                         (int)(r0 / kTcBK));
    else
      kfn<<<dim3(ntiles, ns_use), kTcThreads, smem, st>>>(tmap, rows, TT, ncs, ns_use, K_t / kTcBK, gram_super(),
                                                          ee ? atoi(ee) : 2, part, (int)(r0 / kTcBK), tmap, 0);
    TLS_LAUNCH_CHECK();
    if (launches) *launches += 2;
  }
  k_gram_reduce_t<<<dim3(ntiles, kTcTile / kRedRows), 256, 0, st>>>(part, ntiles, nsplit, TT, kTcTile, A.n, G);
  TLS_LAUNCH_CHECK();
  if (launches) *launches += 1;
  return 0;
}

// ------------------------------------------------------------------------------ 2''. A^T B for the blocked QR
// out (128 x ldo, fp64) = A^T B where A is the 16-bit row-major m x 128 matrix at `a` (row
// stride lda elements) and B the 16-bit row-major m x nb matrix at `b` (row stride ldb), with
// k_gram_tc's accumulation (fp32 per K_t = 64-row chunk, fp32 sums of 64 chunk sums, fp64
// flushes and split sums: reading R11 / R29).  b == a, nb == 128: the Gram of the panel.
__global__ void k_atb_reduce(const double* __restrict__ part, int ntiles, int nsplit, int nb, double* __restrict__ out,
                             int ldo) {
  // grid (ntiles, 64): CTA (J, y) sums rows 2y, 2y + 1 of tile J over the splits, in split order
  const int J = blockIdx.x;
  const int te = kTcTile * kTcTile;
  const int e = blockIdx.y * 256 + threadIdx.x;
  const int i = e / kTcTile, j = e % kTcTile;
  double acc = 0.0;
  for (int s = 0; s < nsplit; ++s) acc += part[((size_t)s * ntiles + J) * te + e];
  if (J * kTcTile + j < nb) out[(size_t)i * ldo + J * kTcTile + j] = acc;
}

static int make_map16(CUtensorMap* map, int u_f, const void* base, int64_t rows, int64_t cols, int64_t ld) {
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)kTcBK};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, u_f == TLS_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (16-bit operand) failed (%d)", (int)r);
    return TLS_ERR_CUDA;
  }
  return 0;
}

size_t tc_atb_ws_bytes(int nb) {
  // nsplit * ntiles <= #SMs for every B width up to nb (nsplit = #SMs / ntiles, or 1)
  const int nt = (nb + kTcTile - 1) / kTcTile;
  const int tiles = nt > num_sms() ? nt : num_sms();
  return (size_t)tiles * kTcTile * kTcTile * 8;
}

int launch_tc_atb(int u_f, const uint16_t* a, int64_t lda, const uint16_t* b, int64_t ldb, int64_t m, int nb,
                  double* out, int ldo, double* part, size_t part_bytes, cudaStream_t st) {
  if (m <= 0) {
    TLS_CUDA_TRY(cudaMemset2DAsync(out, (size_t)ldo * 8, 0, (size_t)nb * 8, kTcTile, st));
    return 0;
  }
  const int ntiles = (nb + kTcTile - 1) / kTcTile;
  const int nchunks = (int)((m + kTcBK - 1) / kTcBK);
  int nsplit = num_sms() / ntiles;
  if (nsplit > nchunks) nsplit = nchunks;
  if (nsplit < 1) nsplit = 1;
  if ((size_t)nsplit * ntiles * kTcTile * kTcTile * 8 > part_bytes) {
    set_error("tc_atb: partials buffer too small");
    return TLS_ERR_WORKSPACE;
  }
  CUtensorMap ma, mb;
  int rc = make_map16(&ma, u_f, a, m, kTcTile, lda);
  if (!rc) rc = make_map16(&mb, u_f, b, m, nb, ldb);   // columns past nb: TMA zero fill
  if (rc) return rc;
  const size_t smem = kTcSmem;
  auto kfn = u_f == TLS_FP16 ? k_gram_tc<0, false> : k_gram_tc<1, false>;
  TLS_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  TLS_CUDA_TRY(cudaMemsetAsync(part, 0, (size_t)nsplit * ntiles * kTcTile * kTcTile * 8, st));
  kfn<<<dim3(ntiles, nsplit), kTcThreads, smem, st>>>(ma, m, 1, nchunks, nsplit, 1, gram_super(), 2, part, 0, mb, 1);
  TLS_LAUNCH_CHECK();
  k_atb_reduce<<<dim3(ntiles, kTcTile * kTcTile / 256), 256, 0, st>>>(part, ntiles, nsplit, nb, out, ldo);
  TLS_LAUNCH_CHECK();
  return 0;
}


// ------------------------------------------------------------------------------ blocked QR update
// k_qr_wy_update (reading R29, the compact-WY trailing update of the blocked Householder QR,
// SURVEY §8(f) NEXT-2 on tensor cores): C <- fl_uf(C - fl32(V Y)) for one 128 x 128 tile of the
// trailing matrix C.  V Y is one tcgen05 kind::f16 product with K = 128 (the panel's
// reflectors): A = V from Vt (128 x m', row-major: the rows of C contiguous, MN-major like the
// Gram's operands), B = Y (128 x n', row-major: MN-major), fp32 accumulator in TMEM.  The
// epilogue (4 warps, TMEM lane = row of the tile) forms the difference in fp64 (both operands
// fp32), rounds it once to u_f, and writes the fp32 working copy W and its 16-bit twin W16.
template <int FMT>
__global__ void __launch_bounds__(128, 1)
k_qr_wy_update(const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapY, float* __restrict__ W,
               uint16_t* __restrict__ W16, int64_t ldw, int64_t ld16, int64_t r0, int c0, int64_t m, int n) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* panA = smem;                         // [2 K-stages][16 KB]
  unsigned char* panB = smem + 2 * kTcPanel;          // [2][16 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 4 * kTcPanel);
  uint64_t* done = full + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M0 = blockIdx.x * kTcTile, N0 = blockIdx.y * kTcTile;   // tile origin in (rows - r0, cols - c0)
  if (threadIdx.x == 0) {
    mbar_init(full, 1);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kTcTile)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (threadIdx.x == 0) {                              // TMA: both K halves of A and B at once
    mbar_arrive_expect_tx(full, 4 * kTcPanel);
    for (int k = 0; k < 2; ++k) {
      unsigned char* a = panA + k * kTcPanel;
      tma_load_2d(a, &mapV, M0, 64 * k, full);
      tma_load_2d(a + kTcPanel / 2, &mapV, M0 + 64, 64 * k, full);
      unsigned char* b = panB + k * kTcPanel;
      tma_load_2d(b, &mapY, N0, 64 * k, full);
      tma_load_2d(b + kTcPanel / 2, &mapY, N0 + 64, 64 * k, full);
    }
  }
  if (threadIdx.x == 32) {                             // MMA: 2 x 4 steps of K = 16
    mbar_wait(full, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_f16(FMT);
    for (int k = 0; k < 2; ++k) {
      const uint32_t a0 = smem_u32(panA + k * kTcPanel), b0 = smem_u32(panB + k * kTcPanel);
#pragma unroll
      for (int kk = 0; kk < kTcBK / 16; ++kk) {
        const uint64_t ad = sw128_desc(a0 + kk * 2048, kTcPanel / 2, 1024);
        const uint64_t bd = sw128_desc(b0 + kk * 2048, kTcPanel / 2, 1024);
        tc_mma_f16(tmem, ad, bd, idesc, (k > 0 || kk > 0) ? 1u : 0u);
      }
    }
    tc_commit(done);
  }
  mbar_wait(done, 0);
  tc_fence_after();
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows M0 + 32w + lane of the tile), 32 columns
  // at a time, and transposes them through shared memory so that W and W16 are read and written
  // along rows (lane = column)
  float* stage = reinterpret_cast<float*>(panA) + warp * 32 * 33;    // the operand panels are consumed
  constexpr int prec = FMT == 0 ? TLS_FP16 : TLS_BF16;
  for (int cc = 0; cc < kTcTile / 32; ++cc) {
    uint32_t acc[32];
    TLS_TMEM_LD32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(cc * 32), acc);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 32; ++e) stage[lane * 33 + e] = __uint_as_float(acc[e]);
    __syncwarp();
    const int col = c0 + N0 + cc * 32 + lane;
    for (int r = 0; r < 32; ++r) {
      const int64_t row = r0 + M0 + warp * 32 + r;
      if (row < m && col < n) {
        const double x = round_uf((double)W[row * ldw + col] - (double)stage[r * 33 + lane], prec);
        W[row * ldw + col] = (float)x;
        W16[row * ld16 + col] = FMT == 0 ? f64_to_f16_bits(x) : f64_to_bf16_bits(x);
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcTile) : "memory");
  }
}

int launch_qr_wy_update(int u_f, const uint16_t* Vt, int64_t ldv, const uint16_t* Y, int64_t ldy, float* W,
                        uint16_t* W16, int64_t ldw, int64_t ld16, int64_t r0, int c0, int64_t m, int n, cudaStream_t st) {
  const int64_t mr = m - r0;
  const int nc = n - c0;
  if (mr <= 0 || nc <= 0) return 0;
  CUtensorMap mv, my;
  int rc = make_map16(&mv, u_f, Vt, kTcTile, mr, ldv);      // 128 rows (K) x m' columns (M)
  if (!rc) rc = make_map16(&my, u_f, Y, kTcTile, nc, ldy);   // 128 rows (K) x n' columns (N)
  if (rc) return rc;
  const size_t smem = 4 * kTcPanel + 1024 + 256;
  auto kfn = u_f == TLS_FP16 ? k_qr_wy_update<0> : k_qr_wy_update<1>;
  TLS_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)((mr + kTcTile - 1) / kTcTile), (unsigned)((nc + kTcTile - 1) / kTcTile));
  kfn<<<grid, 128, smem, st>>>(mv, my, W, W16, ldw, ld16, r0, c0, m, n);
  TLS_LAUNCH_CHECK();
  return 0;
}
}  // namespace tls
