// Micro-benchmark for a split-role fused Gram: how fast can NCV "converter" CTAs (one per SM)
// turn fp64 A (m x n row-major) into fl_uf(A D^-1) (fp16) in an L2-resident ring?  Each CTA
// walks 64-row units u = blockIdx.x, u += NCV; a unit arrives in shared memory as pieces of
// ROWS rows by cp.async.bulk (contiguous: ld == n), NBUF pieces in flight, is scaled and
// rounded by all threads (cvt.rn.f16.f64 via __double2half) and stored, coalesced, into ring
// slot u % 256 (16 MB).  Prints GB/s of fp64 read for NCV in {8 .. 148}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o conv_bw conv_bw.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int ROWS, int NBUF, int MODE>
__global__ void __launch_bounds__(256, 1) conv(const double* __restrict__ A, int64_t m, int n, const double* __restrict__ dinv,
                                              __half* __restrict__ ring, int nslots) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* buf = reinterpret_cast<double*>(sm);                       // [NBUF][ROWS * n]
  double* dsm = buf + (size_t)NBUF * ROWS * n;                        // [n]
  __shared__ uint64_t bar[NBUF];
  const int tid = threadIdx.x;
  for (int j = tid; j < n; j += blockDim.x) dsm[j] = dinv[j];
  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t units = (m + 63) / 64;
  const int per_unit = 64 / ROWS;
  const uint32_t bytes = (uint32_t)ROWS * n * 8;
  // piece sequence of this CTA: p = 0, 1, ... -> (unit blockIdx.x + (p / per_unit) * gridDim.x, sub p % per_unit)
  auto piece_row = [&](int64_t p) -> int64_t {
    const int64_t u = blockIdx.x + (p / per_unit) * gridDim.x;
    return u < units ? u * 64 + (p % per_unit) * ROWS : -1;
  };
  auto issue = [&](int64_t p) {
    const int64_t r = piece_row(p);
    if (r < 0) return;
    const int b = (int)(p % NBUF);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(buf + (size_t)b * ROWS * n)),
                 "l"(A + r * n), "r"(bytes), "r"(su32(&bar[b]))
                 : "memory");
  };
  if (tid == 0)
    for (int p = 0; p < NBUF; ++p) issue(p);
  for (int64_t p = 0;; ++p) {
    const int64_t r = piece_row(p);
    if (r < 0) break;
    const int b = (int)(p % NBUF);
    const uint32_t ph = (uint32_t)(p / NBUF) & 1u;
    asm volatile(
        "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(su32(&bar[b])),
        "r"(ph)
        : "memory");
    const double* src = buf + (size_t)b * ROWS * n;
    const int64_t u = r / 64;
    __half2* dst = reinterpret_cast<__half2*>(ring + ((size_t)(u % nslots) * 64 + (r % 64)) * n);
    if (MODE == 0) {
      for (int e = tid; e < ROWS * n / 2; e += blockDim.x) {
        const double2 v = reinterpret_cast<const double2*>(src)[e];
        const int c = (2 * e) % n;
        dst[e] = __halves2half2(__double2half(v.x * dsm[c]), __double2half(v.y * dsm[c + 1]));
      }
    } else {
      // fixed columns per thread (n / 2 pairs per row, blockDim divides them), dinv in registers
      for (int cp = tid; cp < n / 2; cp += blockDim.x) {
        const double d0 = dsm[2 * cp], d1 = dsm[2 * cp + 1];
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr) {
          const double2 v = reinterpret_cast<const double2*>(src)[rr * (n / 2) + cp];
          if (MODE == 1)
            dst[rr * (n / 2) + cp] = __halves2half2(__double2half(v.x * d0), __double2half(v.y * d1));
          else   // speed probe only (double rounding): fp64 -> fp32 -> fp16
            dst[rr * (n / 2) + cp] = __floats2half2_rn((float)(v.x * d0), (float)(v.y * d1));
        }
      }
    }
    __syncthreads();
    if (tid == 0) issue(p + NBUF);
  }
}

int main() {
  const int64_t m = 1 << 20;
  const int n = 1024;
  double* A;
  double* d;
  __half* ring;
  cudaMalloc(&A, (size_t)m * n * 8);
  cudaMalloc(&d, n * 8);
  cudaMalloc(&ring, (size_t)256 * 64 * n * 2);
  cudaMemset(A, 0, (size_t)m * n * 8);
  cudaMemset(d, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, int rows, int nbuf, int ncv) {
    const size_t smem = (size_t)nbuf * rows * n * 8 + n * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<ncv, 256, smem>>>(A, m, n, d, ring, 256);
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) kern<<<ncv, 256, smem>>>(A, m, n, d, ring, 256);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 3;
    printf("rows %d nbuf %d ncv %3d: %7.3f ms  %6.0f GB/s fp64 read  (%5.1f GB/s per CTA) %s\n", rows, nbuf, ncv, ms,
           m * n * 8 / ms / 1e6, m * n * 8 / ms / 1e6 / ncv, err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  for (int ncv : {16, 40, 148}) {
    printf("-- mode 0 (modulo, dinv from smem)\n");
    run(conv<8, 3, 0>, 8, 3, ncv);
    printf("-- mode 1 (fixed columns, dinv in registers)\n");
    run(conv<8, 3, 1>, 8, 3, ncv);
    run(conv<4, 6, 1>, 4, 6, ncv);
    printf("-- mode 2 (speed probe: via fp32)\n");
    run(conv<8, 3, 2>, 8, 3, ncv);
  }
  return 0;
}
