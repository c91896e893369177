// k_chol.cu — the stored-low preconditioner R~ = fl_uf(R)  (PAPER.md
// l.206, l.290-297; reading R10).
//
// The Cholesky itself is the tile-DAG kernel of k_chol_dag.cu.
// k_pack_R rounds R to u_f (reading R4) into the two layouts the triangular
// solves stream (row-major R~ and R~^T), k_diag_inv forms the fp64 inverses
// of the 32x32 diagonal blocks of R~ (exact upcast) used by the warp-level
// block solves of k_trsv.cu.
#include "tls_common.cuh"
#include "tls_kernels.h"

namespace tls {

// --------------------------------------------------------------------------- R~ = fl_uf(R)
template <typename T>
__global__ void k_pack_R(const double* __restrict__ R, int ldR, int lower, int n, int npad, int prec,
                         T* __restrict__ Rrow, T* __restrict__ RTrow, int* __restrict__ range) {
  const int64_t tot = (int64_t)npad * npad;
  int bad = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / npad), j = (int)(e % npad);
    double v;
    if (i < n && j < n) {
      v = (j >= i) ? round_uf(lower ? R[(size_t)j * ldR + i] : R[(size_t)i * ldR + j], prec) : 0.0;
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

// The coupling blocks of the look-ahead solve (k_trsv.cu): with solve order u, block x_u =
// z_u - E_u x_{u-1} where z_u = D_u (y_u - all tile updates except the last) and E_u = D_u
// T_{u,u-1}.  Back (R~ x = y, previous block in solve order = real block kb+1):
// E = R~_kk^{-1} R~_{kb,kb+1}; forward (R~^T x = y, previous = kb-1): E = R~_kk^{-T} R~_{kb-1,kb}^T.
// Stored [l][i] = E[i][l] (lane i reads consecutive words).  Computed once per R~ in fp64
// from the exact upcasts.
template <typename T>
__global__ void __launch_bounds__(32) k_e_blocks(const T* __restrict__ Rrow, int npad, const double* __restrict__ DinvB,
                                                  const double* __restrict__ DinvF, double* __restrict__ EB,
                                                  double* __restrict__ EF) {
  __shared__ double Tt[32][33];
  const int kb = blockIdx.x, i = threadIdx.x, NB = npad / 32;
  const int o = kb * 32;
  // back: E[i][j] = sum_l D_B[i][l] R[o + l][o + 32 + j],  D_B[i][l] = DinvB[kb][l][i]
  double* E = EB + (size_t)kb * 1024;
  if (kb + 1 < NB) {
    for (int l = 0; l < 32; ++l) Tt[l][i] = dec<T>(Rrow[(size_t)(o + l) * npad + o + 32 + i]);
    __syncwarp();
    for (int j = 0; j < 32; ++j) {
      double acc = 0.0;
      for (int l = 0; l < 32; ++l) acc = fma(DinvB[(size_t)kb * 1024 + l * 32 + i], Tt[l][j], acc);
      E[j * 32 + i] = acc;
    }
  } else {
    for (int j = 0; j < 32; ++j) E[j * 32 + i] = 0.0;
  }
  __syncwarp();
  // forward: E[i][j] = sum_l D_F[i][l] R[o - 32 + j][o + l],  D_F[i][l] = DinvF[kb][l][i]
  E = EF + (size_t)kb * 1024;
  if (kb > 0) {
    for (int j = 0; j < 32; ++j) Tt[j][i] = dec<T>(Rrow[(size_t)(o - 32 + j) * npad + o + i]);   // Tt[j][l]
    __syncwarp();
    for (int j = 0; j < 32; ++j) {
      double acc = 0.0;
      for (int l = 0; l < 32; ++l) acc = fma(DinvF[(size_t)kb * 1024 + l * 32 + i], Tt[j][l], acc);
      E[j * 32 + i] = acc;
    }
  } else {
    for (int j = 0; j < 32; ++j) E[j * 32 + i] = 0.0;
  }
}

size_t precond_bytes(int n, int u_f) {
  const int npad = (n + 31) / 32 * 32;
  const size_t es = (u_f == TLS_FP64) ? 8 : (u_f == TLS_FP32 ? 4 : 2);
  return 2 * (size_t)npad * npad * es + 4 * (size_t)npad * 32 * 8 + 2 * (size_t)npad * 8 + 256;
}

template <typename T>
static int pack_t(const double* R, int ldR, int lower, PrecondDev& pc, int* range, cudaStream_t st) {
  const int64_t tot = (int64_t)pc.npad * pc.npad;
  int g = (int)((tot + 255) / 256);
  if (g > 8192) g = 8192;
  if (R != nullptr) {
    k_pack_R<T><<<g, 256, 0, st>>>(R, ldR, lower, pc.n, pc.npad, pc.u_f, (T*)pc.Rrow, (T*)pc.RTrow, range);
    TLS_LAUNCH_CHECK();
  }
  k_diag_inv<T><<<pc.npad / 32, 32, 0, st>>>((const T*)pc.Rrow, pc.npad, pc.DinvB, pc.DinvF);
  k_e_blocks<T><<<pc.npad / 32, 32, 0, st>>>((const T*)pc.Rrow, pc.npad, pc.DinvB, pc.DinvF, pc.EB, pc.EF);
  TLS_LAUNCH_CHECK();
  return 0;
}

int launch_pack_R(const double* R, int ldR, int lower, PrecondDev& pc, int* range, cudaStream_t st, int* launches) {
  int rc;
  switch (pc.u_f) {
    case TLS_FP16: rc = pack_t<F16s>(R, ldR, lower, pc, range, st); break;
    case TLS_BF16: rc = pack_t<B16s>(R, ldR, lower, pc, range, st); break;
    case TLS_FP32: rc = pack_t<float>(R, ldR, lower, pc, range, st); break;
    default: rc = pack_t<double>(R, ldR, lower, pc, range, st); break;
  }
  if (launches) *launches += (R != nullptr) ? 3 : 2;
  return rc;
}

}  // namespace tls
