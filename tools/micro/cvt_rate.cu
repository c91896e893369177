// Throughput of cvt.rn.f16.f64 (F2F.F16.F64) per SM per clock, against a DMUL-only loop:
// the rounding pass fl_uf(A D^-1) needs one per entry of A (2^30 at cfg4w).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cvt_rate cvt_rate.cu && ./cvt_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, double s, int iters) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = 1.0 + threadIdx.x * 1e-3 + k;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x[k] *= s;                                              // DMUL (both modes)
      if (MODE == 1) {
        uint16_t h;
        asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(x[k]));
        acc += h;
      } else if (MODE == 2) {
        uint16_t h;
        asm volatile("cvt.rn.bf16.f64 %0, %1;" : "=h"(h) : "d"(x[k]));
        acc += h;
      } else if (MODE == 3) {
        float f;
        asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(x[k]));
        acc += __float_as_uint(f);
      }
    }
  }
  double t = acc;
  for (int k = 0; k < 8; ++k) t += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE>
float run(double* out, int blocks, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<MODE><<<blocks, 256>>>(out, 1.0000001, iters);
  cudaEventRecord(a);
  k<MODE><<<blocks, 256>>>(out, 1.0000001, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms;
}
int main() {
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, iters = 4096;
  double* out; cudaMalloc(&out, (size_t)blocks * 256 * 8);
  const double n = (double)blocks * 256 * iters * 8;
  const float t0 = run<0>(out, blocks, iters), t1 = run<1>(out, blocks, iters), t2 = run<2>(out, blocks, iters),
              t3 = run<3>(out, blocks, iters);
  printf("SMs %d, max clock %.0f MHz, %.3g elements per launch\n", sms, khz / 1e3, n);
  printf("DMUL only      %8.3f ms  %7.2f G elem/s\n", t0, n / t0 / 1e6);
  printf("+ cvt f16.f64  %8.3f ms  %7.2f G elem/s  (cvt alone: %7.2f G/s = %.2f per SM per clock at max clock)\n", t1, n / t1 / 1e6,
         n / (t1 - t0) / 1e6, n / (t1 - t0) / 1e6 * 1e9 / sms / (khz * 1e3));
  printf("+ cvt bf16.f64 %8.3f ms  %7.2f G elem/s  (cvt alone: %7.2f G/s)\n", t2, n / t2 / 1e6, n / (t2 - t0) / 1e6);
  printf("+ cvt f32.f64  %8.3f ms  %7.2f G elem/s  (cvt alone: %7.2f G/s)\n", t3, n / t3 / 1e6, n / (t3 - t0) / 1e6);
  return 0;
}
