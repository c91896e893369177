// Microbenchmark: fp64 DFMA dependent-chain latency, DFMA throughput per SM, fp64 div latency,
// F2F.F64.F32 throughput (clock64 on one SM).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, double a, double b, int iters, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void divlat(double* out, double a, int iters, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = 1.0 / (x + 1.5); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void tput(double* out, double a, double b, int iters, long long* cyc) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void f2f(double* out, const float* in, int iters, long long* cyc) {
  float f0 = in[threadIdx.x], f1 = f0 + 1.f, f2 = f0 + 2.f, f3 = f0 + 3.f;
  double acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    acc += (double)f0; acc += (double)f1; acc += (double)f2; acc += (double)f3;
    f0 += 1.f; f1 += 1.f; f2 += 1.f; f3 += 1.f;
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = acc; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; float* in;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 4096 * 8); cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  long long h[4];
  int it = 1 << 14;
  lat<<<1, 32>>>(out, 0.5, 0.999, it, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h[0] / (4.0 * it));
  divlat<<<1, 32>>>(out, 0.5, it, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("fp64 1/(x+c) dependent latency: %.2f cycles\n", (double)h[0] / it);
  for (int thr : {128, 256, 512, 1024}) {
    tput<<<1, thr>>>(out, 0.5, 0.999, it, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput (%4d threads, 1 SM): %.2f DFMA/cycle/SM\n", thr, 8.0 * it * thr / h[0]);
  }
  for (int thr : {256, 1024}) {
    f2f<<<1, thr>>>(out, in, it, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("F2F.F64.F32 + DADD (%4d threads): %.2f conversions/cycle/SM\n", thr, 4.0 * it * thr / h[0]);
  }
  return 0;
}
