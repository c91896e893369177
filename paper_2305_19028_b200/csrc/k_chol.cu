// k_chol.cu — blocked right-looking fp64 Cholesky G = R^T R (upper) and the
// stored-low preconditioner R~ = fl_uf(R)  (PAPER.md
// l.206, l.290-297; reading R10).
//
// Per 64-column block k: k_chol_diag factors the diagonal block in shared
// memory (first non-positive or non-finite pivot -> CHOL_BREAKDOWN index),
// k_chol_trsm forms the block row R_kJ = R_kk^{-T} G_kJ, k_chol_update applies
// G_IJ -= R_kI^T R_kJ to the trailing upper triangle (64x64 fp64 tiles).  All
// kernels read the breakdown flag first and exit once it is set.
// k_pack_R rounds R to u_f (reading R4) into the two layouts the triangular
// solves stream (row-major R~ and R~^T), k_diag_inv forms the fp64 inverses
// of the 32x32 diagonal blocks of R~ (exact upcast) used by the warp-level
// block solves of k_trsv.cu.
#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

constexpr int kCNB = 64;

__global__ void __launch_bounds__(256) k_chol_diag(double* __restrict__ G, int n, int k0, int* __restrict__ pivot) {
  __shared__ double S[kCNB][kCNB + 1];
  __shared__ int fail;
  if (*pivot != 0) return;
  const int nb = min(kCNB, n - k0);
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    S[i][j] = G[(size_t)(k0 + i) * n + k0 + j];
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double piv = S[j][j];
    if (!(piv > 0.0) || !isfinite(piv)) {
      if (tid == 0) { fail = 1; atomicCAS(pivot, 0, k0 + j + 1); }
      break;  // uniform: every thread read the same piv
    }
    const double r = sqrt(piv);
    __syncthreads();
    for (int l = j + 1 + tid; l < nb; l += blockDim.x) S[j][l] /= r;
    if (tid == 0) S[j][j] = r;
    __syncthreads();
    const int rem = nb - j - 1;
    for (int e = tid; e < rem * rem; e += blockDim.x) {
      const int i = j + 1 + e / rem, l = j + 1 + e % rem;
      if (l >= i) S[i][l] = fma(-S[j][i], S[j][l], S[i][l]);
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail) return;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    if (j >= i) G[(size_t)(k0 + i) * n + k0 + j] = S[i][j];
  }
}

// Block row: X = R_kk^{-T} G[k0:k0+nb, c] for c >= k0+nb; one thread per column.
__global__ void __launch_bounds__(128) k_chol_trsm(double* __restrict__ G, int n, int k0, const int* __restrict__ pivot) {
  extern __shared__ double sm[];
  if (*pivot != 0) return;
  const int nb = min(kCNB, n - k0);
  double* R = sm;                      // [nb][nb+1]
  double* X = sm + kCNB * (kCNB + 1);  // [nb][128]
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    R[i * (kCNB + 1) + j] = (j >= i) ? G[(size_t)(k0 + i) * n + k0 + j] : 0.0;
  }
  __syncthreads();
  const int c = k0 + nb + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  for (int i = 0; i < nb; ++i) {
    double acc = G[(size_t)(k0 + i) * n + c];
    for (int l = 0; l < i; ++l) acc = fma(-R[l * (kCNB + 1) + i], X[l * 128 + threadIdx.x], acc);
    const double xi = acc / R[i * (kCNB + 1) + i];
    X[i * 128 + threadIdx.x] = xi;
    G[(size_t)(k0 + i) * n + c] = xi;
  }
}

// Trailing update of the upper triangle: G[i][j] -= sum_l R[k0+l][i] R[k0+l][j], i <= j tiles.
__global__ void __launch_bounds__(256) k_chol_update(double* __restrict__ G, int n, int k0, int TT,
                                                     const int* __restrict__ pivot) {
  extern __shared__ double sm[];
  if (*pivot != 0) return;
  const int nb = min(kCNB, n - k0);
  const int base = k0 + nb;
  int t = blockIdx.x, I = 0;
  while (t >= TT - I) { t -= TT - I; ++I; }
  const int J = I + t;
  const int I0 = base + I * 64, J0 = base + J * 64;
  double* Pa = sm;              // [nb][64]
  double* Pb = sm + kCNB * 64;  // [nb][64]
  for (int e = threadIdx.x; e < nb * 64; e += blockDim.x) {
    const int l = e / 64, c = e % 64;
    Pa[l * 64 + c] = (I0 + c < n) ? G[(size_t)(k0 + l) * n + I0 + c] : 0.0;
    Pb[l * 64 + c] = (J0 + c < n) ? G[(size_t)(k0 + l) * n + J0 + c] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int l = 0; l < nb; ++l) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = Pa[l * 64 + ty * 4 + i];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = Pb[l * 64 + tx * 4 + j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = I0 + ty * 4 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = J0 + tx * 4 + j;
      if (gi < n && gj < n && gj >= gi) G[(size_t)gi * n + gj] -= acc[i][j];
    }
  }
}

int launch_cholesky(double* G, int n, int* pivot, cudaStream_t st, int* launches) {
  static bool attr = false;
  const int trsm_smem = (kCNB * (kCNB + 1) + kCNB * 128) * 8;
  const int upd_smem = 2 * kCNB * 64 * 8;
  if (!attr) {
    TLS_CUDA_TRY(cudaFuncSetAttribute(k_chol_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem));
    TLS_CUDA_TRY(cudaFuncSetAttribute(k_chol_update, cudaFuncAttributeMaxDynamicSharedMemorySize, upd_smem));
    attr = true;
  }
  int nl = 0;
  for (int k0 = 0; k0 < n; k0 += kCNB) {
    k_chol_diag<<<1, 256, 0, st>>>(G, n, k0, pivot);
    ++nl;
    const int rest = n - k0 - kCNB;
    if (rest > 0) {
      k_chol_trsm<<<(rest + 127) / 128, 128, trsm_smem, st>>>(G, n, k0, pivot);
      const int TT = (rest + 63) / 64;
      k_chol_update<<<TT * (TT + 1) / 2, 256, upd_smem, st>>>(G, n, k0, TT, pivot);
      nl += 2;
    }
  }
  TLS_LAUNCH_CHECK();
  if (launches) *launches += nl;
  return 0;
}

// --------------------------------------------------------------------------- R~ = fl_uf(R)
template <typename T>
__global__ void k_pack_R(const double* __restrict__ R, int ldR, int n, int npad, int prec, T* __restrict__ Rrow,
                         T* __restrict__ RTrow, int* __restrict__ range) {
  const int64_t tot = (int64_t)npad * npad;
  int bad = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / npad), j = (int)(e % npad);
    double v;
    if (i < n && j < n) {
      v = (j >= i) ? round_uf(R[(size_t)i * ldR + j], prec) : 0.0;
      if (!isfinite(v) || (i == j && v == 0.0)) bad = 1;
    } else {
      v = (i == j) ? 1.0 : 0.0;
    }
    const T ev = enc<T>(v);
    Rrow[(size_t)i * npad + j] = ev;
    RTrow[(size_t)j * npad + i] = ev;
  }
  if (bad) atomicExch(range, 1);
}

template <typename T>
__global__ void __launch_bounds__(32) k_diag_inv(const T* __restrict__ Rrow, int npad, double* __restrict__ DinvB,
                                                  double* __restrict__ DinvF) {
  __shared__ double S[32][33];
  __shared__ double X[32][33];
  const int kb = blockIdx.x, c = threadIdx.x;
  const int o = kb * 32;
  for (int i = 0; i < 32; ++i) S[i][c] = dec<T>(Rrow[(size_t)(o + i) * npad + o + c]);
  __syncwarp();
  // column c of R_kk^{-1}: back substitution R X = I
  for (int i = 31; i >= 0; --i) {
    double acc = (i == c) ? 1.0 : 0.0;
    for (int l = i + 1; l < 32; ++l) acc = fma(-S[i][l], X[l][c], acc);
    X[i][c] = acc / S[i][i];
  }
  __syncwarp();
  double* B = DinvB + (size_t)kb * 1024;
  double* F = DinvF + (size_t)kb * 1024;
  for (int l = 0; l < 32; ++l) {
    B[l * 32 + c] = X[c][l];  // DinvB[l][i] = X[i][l]
    F[l * 32 + c] = X[l][c];  // DinvF[l][i] = X[l][i]
  }
}

size_t precond_bytes(int n, int u_f) {
  const int npad = (n + 31) / 32 * 32;
  const size_t es = (u_f == TLS_FP64) ? 8 : (u_f == TLS_FP32 ? 4 : 2);
  return 2 * (size_t)npad * npad * es + 2 * (size_t)npad * 32 * 8 + 2 * (size_t)npad * 8 + 256;
}

template <typename T>
static int pack_t(const double* R, int ldR, PrecondDev& pc, int* range, cudaStream_t st) {
  const int64_t tot = (int64_t)pc.npad * pc.npad;
  int g = (int)((tot + 255) / 256);
  if (g > 8192) g = 8192;
  if (R != nullptr) {
    k_pack_R<T><<<g, 256, 0, st>>>(R, ldR, pc.n, pc.npad, pc.u_f, (T*)pc.Rrow, (T*)pc.RTrow, range);
    TLS_LAUNCH_CHECK();
  }
  k_diag_inv<T><<<pc.npad / 32, 32, 0, st>>>((const T*)pc.Rrow, pc.npad, pc.DinvB, pc.DinvF);
  TLS_LAUNCH_CHECK();
  return 0;
}

int launch_pack_R(const double* R, int ldR, PrecondDev& pc, int* range, cudaStream_t st, int* launches) {
  int rc;
  switch (pc.u_f) {
    case TLS_FP16: rc = pack_t<F16s>(R, ldR, pc, range, st); break;
    case TLS_BF16: rc = pack_t<B16s>(R, ldR, pc, range, st); break;
    case TLS_FP32: rc = pack_t<float>(R, ldR, pc, range, st); break;
    default: rc = pack_t<double>(R, ldR, pc, range, st); break;
  }
  if (launches) *launches += (R != nullptr) ? 2 : 1;
  return rc;
}

}  // namespace tls
