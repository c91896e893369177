// potrf_tile<16> / trsm_tile (k_chol_dag.cu) vs potrf_tile_reg / trsm_tile_reg (one thread per
// column, the column in registers, fully unrolled): cycles on one CTA, the difference of the
// factors, R^T R - G, the TRSM bits, breakdown pivots.  Measured (profiles/r02_chol_reg.log):
// POTRF 38.7k vs 41.5k cycles, TRSM 6.7k vs 11.6k cycles alone -- but inside k_chol_dag both
// were slower (n = 2000: 1.52 vs 1.31 ms; inlined 2.9 ms): the fully unrolled 64-step code
// (~100 KB of SASS per routine) streams through the instruction cache on every task, and
// the kernel's register budget (255) forces stack/spills around them.  Not adopted.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o /tmp/chol_reg tools/micro/chol_reg.cu
#include <cstdio>
#include "../../paper_2305_19028_b200/csrc/k_chol_dag.cu"
namespace tls { void set_error(const char*, ...) {} int num_sms() { return 148; } }
using namespace tls;
namespace tls {
// POTRF of the diagonal tile with the columns in registers (round 2 experiment, not adopted): thread t < 64
// owns column t of the tile (64 doubles, static indices in the fully unrolled pivot loop), the
// same square-root-free elimination as potrf_tile (G_ic -= U_ji U_jc / d_j, U_jj = d_j, then
// R = D^{-1/2} U) without the blocking: per pivot j every thread forms its multiplier
// m_t = U_jt / d_j from the published row j, updates its row-(j+1) entry FIRST and publishes
// it (so the next pivot's inputs are on the chain, not the rest of the update), then applies
// the rest of the rank-1 update; one 64-thread named barrier per pivot.  Row j of U is kept in
// `rowbuf` (64 x 64 scratch, written once per row: no write-after-read hazard).  The other
// threads of the CTA only join the final barrier.  Same contract as potrf_tile.
__device__ __noinline__ int potrf_tile_reg(double* S, double* dr, int nb, double* rowbuf) {
  __shared__ int fail_r;
  __shared__ double rs[kTB];
  const int t = threadIdx.x;
  if (t < kTB) {
    double g[kTB];
#pragma unroll
    for (int i = 0; i < kTB; ++i) g[i] = S[i * kTS + t];   // entries below the diagonal are never used
    rowbuf[t] = g[0];
    int f = 0;
    named_bar_sync(1, kTB);
#pragma unroll
    for (int j = 0; j < kTB; ++j) {
      const double* rj = rowbuf + j * kTB;
      const double piv = rj[j];
      if (j < nb && f == 0 && !(piv > 0.0 && piv < INFINITY)) f = j + 1;   // the same for every thread
      if (j + 1 < kTB && f == 0) {
        const double m = rj[t] * rcp_fast(piv);   // U_jt / d_j (used by t > j only)
        if (t > j) {
          g[j + 1] = fma(-rj[j + 1], m, g[j + 1]);
          rowbuf[(j + 1) * kTB + t] = g[j + 1];
        }
#pragma unroll
        for (int i = j + 2; i < kTB; ++i)
          if (i <= t) g[i] = fma(-rj[i], m, g[i]);
        named_bar_sync(1, kTB);
      }
    }
    if (t == 0) fail_r = f;
    if (f == 0) {
      const double sq = sqrt(rowbuf[t * kTB + t]);
      rs[t] = rcp_fast(sq);
      dr[t] = rs[t];
      named_bar_sync(1, kTB);
#pragma unroll
      for (int i = 0; i < kTB; ++i)
        if (i < t) S[i * kTS + t] = g[i] * rs[i];
      S[t * kTS + t] = sq;
    }
  }
  __syncthreads();
  return fail_r;
}

// TRSM with the columns in registers (round 2 experiment, not adopted): thread c < 64 owns column c of B
// and runs its forward substitution alone (R_il broadcast from shared memory); the same
// operations in the same order as trsm_tile, so the same bits, without its per-pivot shuffles.
__device__ __noinline__ void trsm_tile_reg(const double* R, const double* dr, double* B) {
  const int c = threadIdx.x;
  if (c < kTB) {
    double g[kTB];
#pragma unroll
    for (int i = 0; i < kTB; ++i) g[i] = B[i * kTS + c];
#pragma unroll
    for (int i = 0; i < kTB; ++i) {
      const double xi = g[i] * dr[i];
      g[i] = xi;
#pragma unroll
      for (int l = i + 1; l < kTB; ++l) g[l] = fma(-R[i * kTS + l], xi, g[l]);
    }
#pragma unroll
    for (int i = 0; i < kTB; ++i) B[i * kTS + c] = g[i];
  }
}

}  // namespace tls
template <int V>
__global__ void __launch_bounds__(256, 1) bench_potrf(const double* G, long long* cyc, double* R, double* dr, int nb) {
  extern __shared__ double sm[];
  double* S0 = sm; double* S1 = S0 + kTB * kTS; double* S2 = S1 + kTB * kTS;
  load_tile(G, 64, 0, 0, S0, true, true);
  __syncthreads();
  long long a = clock64();
  int f = V == 1 ? potrf_tile<16>(S0, S1, nb) : potrf_tile_reg(S0, S1, nb, S2);
  __syncthreads();
  long long b = clock64();
  if (threadIdx.x == 0) { cyc[0] = b - a; cyc[1] = f; }
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) R[e] = ((e & 63) >= (e >> 6)) ? S0[(e >> 6) * kTS + (e & 63)] : 0.0;
  if (threadIdx.x < 64) dr[threadIdx.x] = S1[threadIdx.x];
}
template <int V>
__global__ void __launch_bounds__(256, 1) bench_trsm(const double* R, const double* dr, const double* B, long long* cyc, double* X) {
  extern __shared__ double sm[];
  double* S0 = sm; double* S1 = S0 + kTB * kTS; double* S2 = S1 + kTB * kTS;
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) {
    S0[(e >> 6) * kTS + (e & 63)] = R[e];
    S1[(e >> 6) * kTS + (e & 63)] = B[e];
  }
  if (threadIdx.x < 64) S2[threadIdx.x] = dr[threadIdx.x];
  __syncthreads();
  long long a = clock64();
  if (V == 1) trsm_tile(S0, S2, S1); else trsm_tile_reg(S0, S2, S1);
  __syncthreads();
  long long b = clock64();
  if (threadIdx.x == 0) cyc[0] = b - a;
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) X[e] = S1[(e >> 6) * kTS + (e & 63)];
}
int main() {
  static double hA[64 * 64], hG[64 * 64], hB[64 * 64];
  unsigned s = 1;
  for (int i = 0; i < 4096; ++i) { s = s * 1103515245u + 12345u; hA[i] = ((s >> 8) & 0xffff) / 65536.0 - 0.5; }
  for (int i = 0; i < 4096; ++i) { s = s * 1103515245u + 12345u; hB[i] = ((s >> 8) & 0xffff) / 65536.0 - 0.5; }
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) {
    double t = 0; for (int k = 0; k < 64; ++k) t += hA[k * 64 + i] * hA[k * 64 + j];
    hG[i * 64 + j] = t + (i == j ? 0.5 : 0.0);
  }
  double *G, *R, *dr, *B, *X; long long* c;
  cudaMalloc(&G, sizeof(hG)); cudaMalloc(&R, sizeof(hG)); cudaMalloc(&B, sizeof(hG)); cudaMalloc(&X, sizeof(hG));
  cudaMalloc(&dr, 64 * 8); cudaMalloc(&c, 16);
  cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof(hB), cudaMemcpyHostToDevice);
  const int smem = 3 * 64 * 65 * 8;
  cudaFuncSetAttribute(bench_potrf<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench_potrf<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench_trsm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench_trsm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  static double R1[4096], R2[4096], X1[4096], X2[4096];
  long long h[2];
  for (int rep = 0; rep < 3; ++rep) {
    bench_potrf<1><<<1, 256, smem>>>(G, c, R, dr, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(R1, R, sizeof(R1), cudaMemcpyDeviceToHost); printf("potrf blocked16: %6lld cyc (fail %lld)\n", h[0], h[1]);
    bench_potrf<2><<<1, 256, smem>>>(G, c, R, dr, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(R2, R, sizeof(R2), cudaMemcpyDeviceToHost); printf("potrf reg:       %6lld cyc (fail %lld)\n", h[0], h[1]);
  }
  double md = 0, mx = 0;
  for (int i = 0; i < 4096; ++i) { md = fmax(md, fabs(R1[i] - R2[i])); mx = fmax(mx, fabs(R1[i])); }
  double me = 0;
  for (int i = 0; i < 64; ++i) for (int j = i; j < 64; ++j) {
    double t = 0; for (int k = 0; k <= i; ++k) t += R2[k * 64 + i] * R2[k * 64 + j];
    me = fmax(me, fabs(t - hG[i * 64 + j]) / fabs(hG[i * 64 + i]));
  }
  printf("max |R1-R2| / max|R1| = %.2e   max |R2^T R2 - G| / G_ii = %.2e\n", md / mx, me);
  // TRSM with the reg factor
  for (int rep = 0; rep < 3; ++rep) {
    bench_trsm<1><<<1, 256, smem>>>(R, dr, B, c, X); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(X1, X, sizeof(X1), cudaMemcpyDeviceToHost); printf("trsm 4/col:      %6lld cyc\n", h[0]);
    bench_trsm<2><<<1, 256, smem>>>(R, dr, B, c, X); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(X2, X, sizeof(X2), cudaMemcpyDeviceToHost); printf("trsm reg:        %6lld cyc\n", h[0]);
  }
  int same = 0;
  for (int i = 0; i < 4096; ++i) same += X1[i] == X2[i];
  printf("trsm bit-identical entries: %d / 4096\n", same);
  // breakdowns: an indefinite tile, and a padded tile (nb = 40)
  hG[40 * 64 + 40] = -1.0; cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  bench_potrf<1><<<1, 256, smem>>>(G, c, R, dr, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); printf("indefinite: blocked16 fail %lld\n", h[1]);
  bench_potrf<2><<<1, 256, smem>>>(G, c, R, dr, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); printf("indefinite: reg fail %lld\n", h[1]);
  hG[40 * 64 + 40] = NAN; cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  bench_potrf<1><<<1, 256, smem>>>(G, c, R, dr, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); printf("NaN: blocked16 fail %lld\n", h[1]);
  bench_potrf<2><<<1, 256, smem>>>(G, c, R, dr, 64); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); printf("NaN: reg fail %lld\n", h[1]);
  cudaError_t e = cudaDeviceSynchronize();
  printf("cuda: %s\n", cudaGetErrorString(e));
}
