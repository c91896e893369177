// Microbenchmark of the Cholesky tile routines of k_chol_dag.cu on one SM (clock64 per call).
#include "../../paper_2305_19028_b200/csrc/k_chol_dag.cu"
namespace tls { void set_error(const char*, ...) {} int num_sms() { return 148; } }
using namespace tls;
__global__ void bench(const double* G, long long* cyc, double* sink) {
  extern __shared__ double sm[];
  double* S0 = sm; double* S1 = S0 + kTB * kTS; double* S2 = S1 + kTB * kTS;
  long long t[4] = {0, 0, 0, 0};
  for (int rep = 0; rep < 10; ++rep) {
    load_tile(G, 64, 0, 0, S0, true, true);
    __syncthreads();
    long long a = clock64();
    potrf_tile(S0, S2, 64);
    __syncthreads();
    long long b = clock64();
    load_tile(G, 64, 0, 0, S1, false, false);
    __syncthreads();
    long long c = clock64();
    trsm_tile(S0, S2, S1);
    __syncthreads();
    long long d = clock64();
    double acc[4][4] = {};
    tile_atb(S0, S1, acc);
    __syncthreads();
    long long e = clock64();
    t[0] += b - a; t[1] += d - c; t[2] += e - d;
    if (threadIdx.x == 0) sink[rep] = acc[0][0] + S1[5];
  }
  if (threadIdx.x == 0) { cyc[0] = t[0] / 10; cyc[1] = t[1] / 10; cyc[2] = t[2] / 10; }
}
int main() {
  double hG[64 * 64];
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) hG[i * 64 + j] = (i == j) ? 64.0 + i : 1.0 / (1 + i + j);
  double *G, *sink; long long* cyc;
  cudaMalloc(&G, sizeof(hG)); cudaMalloc(&sink, 1024); cudaMalloc(&cyc, 64);
  cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  const int smem = 3 * kTB * kTS * 8;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<<<1, 256, smem>>>(G, cyc, sink);
  long long h[3]; cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
  printf("potrf_tile %lld cycles, trsm_tile %lld cycles, tile_atb %lld cycles (%s)\n", h[0], h[1], h[2],
         cudaGetErrorString(cudaGetLastError()));
}
