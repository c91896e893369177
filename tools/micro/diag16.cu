// Cycle cost of potrf_tile's 16x16 diagonal-block step (k_chol_dag.cu (1)) and variants,
// one warp, 16 sequential pivots.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 diag16.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_fast(double x) {
  const double ax = fabs(x);
  if (!(ax > 1e-30 && ax < 1e30)) return 1.0 / x;
  double r = (double)__frcp_rn((float)x);
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rcp_mufu(double x) {   // MUFU.RCP64H seed + 2 Newton steps
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
template <int MODE>
__global__ void k(const double* S, long long* cyc, double* out) {
  const int tid = threadIdx.x, t = tid & 15;
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = S[i * 16 + t];
  int f = 0;
  __syncwarp();
  long long a = clock64();
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) {
    const double piv = __shfl_sync(0xffffffffu, v[jj], jj);
    bool bad = false;
    if (MODE != 3) bad = !(piv > 0.0) || !isfinite(piv);
    if (f == 0) {
      if (bad) f = jj + 1;
      else {
        double dinv;
        if (MODE == 0 || MODE == 3) dinv = rcp_fast(piv);
        else if (MODE == 1) dinv = 1.0 / piv;
        else dinv = rcp_mufu(piv);
        const double sjt = v[jj];
#pragma unroll
        for (int ii = jj + 1; ii < 16; ++ii) {
          const double m = __shfl_sync(0xffffffffu, v[jj], ii) * dinv;
          if (t >= ii) v[ii] = fma(-m, sjt, v[ii]);
        }
      }
    }
  }
  long long b = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  out[tid] = s + f;
  if (tid == 0) cyc[0] = b - a;
}
int main() {
  double h[256];
  for (int i = 0; i < 16; ++i) for (int j = 0; j < 16; ++j) h[i * 16 + j] = (i == j) ? 16.0 + i : 0.1 / (1 + i + j);
  double *S, *o; long long* c; cudaMalloc(&S, sizeof(h)); cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 8);
  cudaMemcpy(S, h, sizeof(h), cudaMemcpyHostToDevice);
  long long r;
  const char* names[] = {"rcp_fast (fp32 seed)", "IEEE div", "rcp.approx.f64 seed", "rcp_fast, no finite check"};
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 32>>>(S, c, o); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cyc\n", names[0], r);
    k<1><<<1, 32>>>(S, c, o); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cyc\n", names[1], r);
    k<2><<<1, 32>>>(S, c, o); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cyc\n", names[2], r);
    k<3><<<1, 32>>>(S, c, o); cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cyc\n", names[3], r);
  }
}
