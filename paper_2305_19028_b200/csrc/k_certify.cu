// k_certify.cu — the compensated final certificate (SURVEY §8(c) c2 step 8, §8(b)
// tls_info_t.sigma_certified): sigma = sqrt(||b - A x||^2 / (1 + ||x||^2)) with every
// residual r_i = b_i - a_i . x and the sum ||r||^2 formed by Dot2 (Ogita, Rump & Oishi:
// TwoProduct by fma, TwoSum accumulation), i.e. as accurate as in twice fp64.  One extra
// pass over A after the solve (opts.certify).  Each CTA leaves a (sum, compensation)
// pair; the pairs are combined in fixed order, all-reduced over ranks by the host, and
// ||x||^2 is a Dot2 over the replicated x.
#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
// (s, c) += a * b, Dot2 step
__device__ __forceinline__ void dot2_step(double a, double b, double& s, double& c) {
  const double p = a * b;
  const double e = fma(a, b, -p);
  double q;
  two_sum(s, p, s, q);
  c += q + e;
}
// (s, c) += (s2, c2)
__device__ __forceinline__ void dot2_merge(double& s, double& c, double s2, double c2) {
  double q;
  two_sum(s, s2, s, q);
  c += c2 + q;
}
__device__ __forceinline__ void warp_dot2(double& s, double& c) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const double s2 = __shfl_xor_sync(0xffffffffu, s, o), c2 = __shfl_xor_sync(0xffffffffu, c, o);
    // both lanes of a pair combine in the same (lower lane first) order: identical results
    const bool lower = (threadIdx.x & o) == 0;
    double a = lower ? s : s2, ac = lower ? c : c2, b = lower ? s2 : s, bc = lower ? c2 : c;
    dot2_merge(a, ac, b, bc);
    s = a;
    c = ac;
  }
}

constexpr int kCertT = 256;

// one warp per row; partials [gridDim.x][2]
template <bool CSR>
__global__ void __launch_bounds__(kCertT) k_certify(DenseView D, CsrView S, const double* __restrict__ b,
                                                    const double* __restrict__ x, double* __restrict__ part) {
  __shared__ double ws[kCertT / 32][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t m = CSR ? S.m : D.m;
  double rs = 0.0, rc = 0.0;             // Dot2 of sum r_i^2 (this warp's rows)
  for (int64_t i = blockIdx.x * (int64_t)(kCertT / 32) + warp; i < m; i += (int64_t)gridDim.x * (kCertT / 32)) {
    double s = 0.0, c = 0.0;
    if (lane == 0) s = b[i];             // the term b_i * 1
    if (CSR) {
      for (int64_t e = S.rowptr[i] + lane; e < S.rowptr[i + 1]; e += 32) dot2_step(-S.vals[e], x[S.colidx[e]], s, c);
    } else {
      const double* a = D.A + i * D.ld;
      for (int j = lane; j < D.n; j += 32) dot2_step(-a[j], x[j], s, c);
    }
    warp_dot2(s, c);
    const double r = s + c;
    if (lane == 0) dot2_step(r, r, rs, rc);
  }
  if (lane == 0) { ws[warp][0] = rs; ws[warp][1] = rc; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, c = 0.0;
    for (int w = 0; w < kCertT / 32; ++w) dot2_merge(s, c, ws[w][0], ws[w][1]);
    part[2 * blockIdx.x] = s;
    part[2 * blockIdx.x + 1] = c;
  }
}

// out[0] = sum of the rank's r_i^2 (rounded), out[1] = its compensation, out[2] = ||x||^2
__global__ void k_certify_fin(const double* __restrict__ part, int G, const double* __restrict__ x, int n,
                              double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double s = 0.0, c = 0.0;
  for (int g = 0; g < G; ++g) dot2_merge(s, c, part[2 * g], part[2 * g + 1]);
  double xs = 0.0, xc = 0.0;
  for (int j = 0; j < n; ++j) dot2_step(x[j], x[j], xs, xc);
  out[0] = s;
  out[1] = c;
  out[2] = xs + xc;
}

int certify_grid() { return num_sms(); }

int launch_certify(const DenseView* D, const CsrView* S, const double* b, const double* x, int n, double* part,
                   double* out, cudaStream_t st) {
  const int G = certify_grid();
  if (S) k_certify<true><<<G, kCertT, 0, st>>>(DenseView{}, *S, b, x, part);
  else k_certify<false><<<G, kCertT, 0, st>>>(*D, CsrView{}, b, x, part);
  TLS_LAUNCH_CHECK();
  k_certify_fin<<<1, 32, 0, st>>>(part, G, x, n, out);
  TLS_LAUNCH_CHECK();
  return 0;
}

}  // namespace tls
