// Per-step cost breakdown of the POTRF column loop (one CTA of 256 threads).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(const double* G, long long* cyc, double* sink) {
  __shared__ double rowj[2][64];
  __shared__ double S[64 * 65];
  const int tid = threadIdx.x, l = tid & 63, i0 = tid >> 6;
  for (int e = tid; e < 64 * 64; e += 256) S[(e >> 6) * 65 + (e & 63)] = G[e];
  double v[16];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = S[(i0 + 4 * r) * 65 + l];
  if (tid < 64) rowj[0][tid] = S[tid];
  __syncthreads();
  long long a = clock64();
  for (int j = 0; j < 64; ++j) {
    const double* rj = rowj[j & 1];
    double dinv = 1.0;
    if (MODE >= 1) { const double piv = rj[j]; dinv = 1.0 / piv; }
    if (MODE >= 2) {
      const double sjl = rj[l] * dinv;
      double mrow[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) mrow[r] = rj[i0 + 4 * r];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int i = i0 + 4 * r;
        if (i > j && l >= i) v[r] = fma(-mrow[r], sjl, v[r]);
      }
    }
    if (MODE >= 3) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (i0 + 4 * r == j + 1) rowj[(j + 1) & 1][l] = v[r];
    }
    __syncthreads();
  }
  long long b = clock64();
  double s = 0; for (int r = 0; r < 16; ++r) s += v[r];
  sink[tid] = s;
  if (tid == 0) cyc[0] = b - a;
}
int main() {
  double hG[4096]; for (int i = 0; i < 4096; ++i) hG[i] = ((i >> 6) == (i & 63)) ? 100.0 : 0.01;
  double *G, *sink; long long* cyc; cudaMalloc(&G, sizeof(hG)); cudaMalloc(&sink, 8192); cudaMalloc(&cyc, 8);
  cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  long long h;
  k<0><<<1, 256>>>(G, cyc, sink); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("sync only: %lld cyc/step\n", h / 64);
  k<1><<<1, 256>>>(G, cyc, sink); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("+div: %lld cyc/step\n", h / 64);
  k<2><<<1, 256>>>(G, cyc, sink); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("+update: %lld cyc/step\n", h / 64);
  k<3><<<1, 256>>>(G, cyc, sink); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("+publish: %lld cyc/step\n", h / 64);
}
