// K6: SIMT (CUDA-core) versions of K3/K4/K5 for the fp32-accurate FP32 mode (FFMA) and the FP64
// mode (DFMA).  C[i][j] = Σ_k A[i][k]·B[j][k] over 64×64 tiles, 256 threads, 4×4 register micro-tile,
// operands staged transposed in shared memory; the same fused epilogues as the tensor-core path.
#pragma once
#include <stdint.h>

#include "rf_common.cuh"

namespace rfk {

template <typename T>
struct SimtSigma {
  T* S;
  int64_t ld, M, N;
  int act;
  __device__ __forceinline__ void operator()(int64_t i, int64_t j, T v) const {
    if (i < M && j < N) S[i * ld + j] = act_t<T>(act, v);
  }
};

template <typename T>
struct SimtSyrk {
  T* G;
  int64_t ld, n;
  T scale;
  int full;
  __device__ __forceinline__ void operator()(int64_t i, int64_t j, T v) const {
    if (i < n && j < n && j >= i) {
      G[i * ld + j] = v * scale;
      if (full && j > i) G[j * ld + i] = v * scale;
    }
  }
};

template <typename T, typename RC>
struct SimtEq1 {
  T* Phi;
  int64_t ld, n;
  const RC* rc;
  const T* njt;          // ‖x_j‖²/τ
  T e0, e1, e2, f0, f1;
  int full;
  __device__ __forceinline__ void operator()(int64_t i, int64_t j, T g) const {
    if (i < n && j < n && j >= i) {
      const RC c = rc[i];
      T v = eq1_entry<T>(g, (T)c.a0, (T)c.a1, (T)c.a2h, (T)c.c, njt[j], i == j, (T)c.nu_diag, e0, e1, e2, f0, f1);
      Phi[i * ld + j] = v;
      if (full && j > i) Phi[j * ld + i] = v;
    }
  }
};

// grid: (tiles_n, row tiles in [row_tile0, row_tile0 + gridDim.y)); tri ⇒ skip tiles strictly below
// the diagonal (64×64 tiles: J < I).
template <typename T, class Epi>
__global__ void __launch_bounds__(256) simt_gemm_nt(const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                                                    int64_t ldb, int64_t M, int64_t N, int64_t K, int tri,
                                                    int row_tile0, Epi epi) {
  constexpr int BM = 64, BN = 64, BK = 16;
  const int bi = blockIdx.y + row_tile0, bj = blockIdx.x;
  if (tri && bj < bi) return;
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t i0 = (int64_t)bi * BM, j0 = (int64_t)bj * BN;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);

  for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int q = 0; q < (BM * BK) / 256; ++q) {
      const int e = tid + 256 * q;
      const int r = e / BK, kk = e % BK;
      const int64_t gi = i0 + r, gj = j0 + r, gk = k0 + kk;
      As[kk][r] = (gi < M && gk < K) ? A[gi * lda + gk] : T(0);
      Bs[kk][r] = (gj < N && gk < K) ? B[gj * ldb + gk] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[kk][ty + 16 * u];
        b[u] = Bs[kk][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) epi(i0 + ty + 16 * u, j0 + tx + 16 * v, acc[u][v]);
}

}  // namespace rfk
