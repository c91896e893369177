// DMMA (mma.sync m8n8k4 f64) throughput on one SM vs DFMA: FMAs per cycle per SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8 * 1024);
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    dmma<<<1, threads>>>(out, iters, cyc);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double fmas = (double)iters * 8 * 256 * (threads / 32);   // m8n8k4 = 256 FMA per warp-instruction
    printf("DMMA %4d threads, 1 SM: %.1f FMA/cycle/SM (%.2f us)\n", threads, fmas / h, h / 1.9e3);
  }
  dmma<<<148, 512>>>(out, iters, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); dmma<<<148 * 2, 512>>>(out, iters, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("DMMA all SMs: %.1f TFLOP/s\n", 2.0 * iters * 8 * 256 * 16 * 148 * 2 / (ms * 1e-3) / 1e12);
}
