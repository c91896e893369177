// potrf_tile (blocked) vs potrf_tile2 (unblocked, one barrier per pivot): cycles and
// max |R1 - R2| / |R1| on an SPD 64x64 tile.
#include <cstdio>
#include "../../paper_2305_19028_b200/csrc/k_chol_dag.cu"
namespace tls { void set_error(const char*, ...) {} int num_sms() { return 148; } }
using namespace tls;
template <int V>
__global__ void bench(const double* G, long long* cyc, double* R, int nb) {
  extern __shared__ double sm[];
  double* S0 = sm; double* S2 = S0 + 2 * kTB * kTS;
  load_tile(G, 64, 0, 0, S0, true, true);
  __syncthreads();
  long long a = clock64();
  int f = V == 1 ? potrf_tile(S0, S2, nb) : potrf_tile2(S0, S2, nb);
  __syncthreads();
  long long b = clock64();
  if (threadIdx.x == 0) { cyc[0] = b - a; cyc[1] = f; }
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) R[e] = ((e & 63) >= (e >> 6)) ? S0[(e >> 6) * kTS + (e & 63)] : 0.0;
}
int main() {
  static double hA[64 * 64], hG[64 * 64];
  unsigned s = 1;
  for (int i = 0; i < 4096; ++i) { s = s * 1103515245u + 12345u; hA[i] = ((s >> 8) & 0xffff) / 65536.0 - 0.5; }
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) {
    double t = 0; for (int k = 0; k < 64; ++k) t += hA[k * 64 + i] * hA[k * 64 + j];
    hG[i * 64 + j] = t + (i == j ? 0.5 : 0.0);
  }
  double *G, *R; long long* c; cudaMalloc(&G, sizeof(hG)); cudaMalloc(&R, sizeof(hG)); cudaMalloc(&c, 16);
  cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  const int smem = 3 * 64 * 65 * 8;
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  static double R1[4096], R2[4096];
  long long h[2];
  for (int rep = 0; rep < 3; ++rep) {
    bench<1><<<1, 256, smem>>>(G, c, R, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(R1, R, sizeof(R1), cudaMemcpyDeviceToHost); printf("blocked:   %lld cyc (fail %lld)\n", h[0], h[1]);
    bench<2><<<1, 256, smem>>>(G, c, R, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(R2, R, sizeof(R2), cudaMemcpyDeviceToHost); printf("unblocked: %lld cyc (fail %lld)\n", h[0], h[1]);
  }
  double md = 0, mx = 0;
  for (int i = 0; i < 4096; ++i) { md = fmax(md, fabs(R1[i] - R2[i])); mx = fmax(mx, fabs(R1[i])); }
  // R^T R vs G
  double me = 0;
  for (int i = 0; i < 64; ++i) for (int j = i; j < 64; ++j) {
    double t = 0; for (int k = 0; k <= i; ++k) t += R2[k * 64 + i] * R2[k * 64 + j];
    me = fmax(me, fabs(t - hG[i * 64 + j]) / fabs(hG[i * 64 + i]));
  }
  printf("max |R1-R2| / max|R1| = %.2e   max |R2^T R2 - G| / G_ii = %.2e\n", md / mx, me);
  // breakdown on an indefinite tile
  hG[40 * 64 + 40] = -1.0; cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  bench<1><<<1, 256, smem>>>(G, c, R, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); printf("indefinite: blocked fail %lld\n", h[1]);
  bench<2><<<1, 256, smem>>>(G, c, R, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); printf("indefinite: unblocked fail %lld\n", h[1]);
}
