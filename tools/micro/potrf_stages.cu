// Stage timing of potrf_tile (k_chol_dag.cu) via a copy with clock64 marks (TILE_TRACE).
#define POTRF_TRACE 1
#include <cstdio>
__device__ long long g_marks[64];
#include "../../paper_2305_19028_b200/csrc/k_chol_dag.cu"
namespace tls { void set_error(const char*, ...) {} int num_sms() { return 148; } }
using namespace tls;
__global__ void bench(const double* G, long long* out) {
  extern __shared__ double sm[];
  double* S0 = sm; double* S2 = S0 + 2 * kTB * kTS;
  load_tile(G, 64, 0, 0, S0, true, true);
  __syncthreads();
  potrf_tile(S0, S2, 64);
  __syncthreads();
  if (threadIdx.x == 0) for (int i = 0; i < 64; ++i) out[i] = g_marks[i];
}
int main() {
  double hG[64 * 64];
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) hG[i * 64 + j] = (i == j) ? 64.0 + i : 1.0 / (1 + i + j);
  double* G; long long* o; cudaMalloc(&G, sizeof(hG)); cudaMalloc(&o, 64 * 8);
  cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 64 * 65 * 8);
  bench<<<1, 256, 3 * 64 * 65 * 8>>>(G, o);
  long long h[64]; cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  for (int i = 1; i < 17; ++i) printf("mark %d: +%lld\n", i, h[i] - h[i - 1]);
}
