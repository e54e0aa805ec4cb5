// K6: SIMT (CUDA-core) versions of K3/K4/K5 for the fp32-accurate FP32 mode (FFMA) and the FP64
// mode (DFMA).  C[i][j] = Σ_k A[i][k]·B[j][k] over 128×128 tiles, 256 threads, 8×8 register micro-tile,
// operands staged k-major in shared memory; the same fused epilogues as the tensor-core path.
#pragma once
#include <stdint.h>

#include <type_traits>

#include "rf_common.cuh"

namespace rfk {

template <typename T>
struct SimtSigma {
  T* S;
  int64_t ld, M, N;
  int act;
  ActRt ap;   // parametrised σ (ap.kind > 0) instead of act
  __device__ __forceinline__ void operator()(int64_t i, int64_t j, T v) const {
    if (i < M && j < N) S[i * ld + j] = ap.kind ? act_param<T>(ap, v) : act_t<T>(act, v);
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

// grid: (tiles_n, row tiles in [row_tile0, row_tile0 + gridDim.y)); tri = 1 ⇒ skip tiles strictly below the
// diagonal (J < I), tri = 2 ⇒ strictly above (J > I).  128×128 tiles, 256 threads, 8×8 register micro-tile per thread (rows ty·4 + {0..3} and 64 + ty·4 +
// {0..3}, columns likewise with tx), K-slices of 16 staged k-major in shared memory (two 16-B loads per operand per
// k give 64 FMAs), next slice prefetched into registers with 16-B global loads while the current one is consumed.
// Rows are 16-B aligned (ld·sizeof(T) a multiple of 16 B, validated at the ABI); the K tail is zero-filled.
constexpr int kSimtTile = 128;
// Batched launches (gridDim.z > 1): operands advance by zsA / zsB elements per z, and an epilogue with a `zstride`
// member advances its output the same way (rf_ridge factors several γ at once).
template <class E, class = void>
struct has_zstride : std::false_type {};
template <class E>
struct has_zstride<E, std::void_t<decltype(E::zstride)>> : std::true_type {};
template <typename T, class Epi>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 2 : 1) simt_gemm_nt(const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                                                    int64_t ldb, int64_t M, int64_t N, int64_t K, int tri,
                                                    int row_tile0, Epi epi, int64_t zsA = 0, int64_t zsB = 0) {
  if (blockIdx.z) {
    A += blockIdx.z * zsA;
    B += blockIdx.z * zsB;
    if constexpr (has_zstride<Epi>::value) epi.A += blockIdx.z * epi.zstride;
  }
  constexpr int BM = kSimtTile, BN = kSimtTile, BK = 16, PAD = 4;
  constexpr int VEC = 16 / (int)sizeof(T);                 // elements per 16-B vector
  constexpr int NV = BM * BK / VEC / 256;                  // vectors per thread per operand per slice
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  const int bi = blockIdx.y + row_tile0, bj = blockIdx.x;
  if ((tri == 1 && bj < bi) || (tri == 2 && bj > bi)) return;   // 1: upper tiles (j ≥ i), 2: lower tiles
  __shared__ __align__(16) T As[BK][BM + PAD];
  __shared__ __align__(16) T Bs[BK][BN + PAD];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t i0 = (int64_t)bi * BM, j0 = (int64_t)bj * BN;

  T ra[NV][VEC], rb[NV][VEC];
  auto gload = [&](int64_t k0) __attribute__((always_inline)) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int idx = tid + 256 * q;
      const int r = idx / (BK / VEC), c = (idx % (BK / VEC)) * VEC;
      const int64_t k = k0 + c;
      const int64_t gi = i0 + r, gj = j0 + r;
      if (gi < M && k + VEC <= K) {
        const V v = *reinterpret_cast<const V*>(A + gi * lda + k);
        const T* pv = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int e = 0; e < VEC; ++e) ra[q][e] = pv[e];
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e) ra[q][e] = (gi < M && k + e < K) ? A[gi * lda + k + e] : T(0);
      }
      if (gj < N && k + VEC <= K) {
        const V v = *reinterpret_cast<const V*>(B + gj * ldb + k);
        const T* pv = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int e = 0; e < VEC; ++e) rb[q][e] = pv[e];
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e) rb[q][e] = (gj < N && k + e < K) ? B[gj * ldb + k + e] : T(0);
      }
    }
  };
  auto sstore = [&]() __attribute__((always_inline)) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int idx = tid + 256 * q;
      const int r = idx / (BK / VEC), c = (idx % (BK / VEC)) * VEC;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        As[c + e][r] = ra[q][e];
        Bs[c + e][r] = rb[q][e];
      }
    }
  };

  // fp32: the accumulators are packed pairs (FFMA2, two FMAs per instruction, each rounded as the scalar op)
  constexpr bool kPk = sizeof(T) == 4;
  T acc[8][8];
  uint64_t acc2[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = T(0);
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc2[a][b] = 0ull;

  gload(0);
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    __syncthreads();                       // the previous slice has been consumed
    sstore();
    __syncthreads();
    if (k0 + BK < K) gload(k0 + BK);      // in flight while this slice is consumed
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[8], b[8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          a[4 * h + e] = As[kk][64 * h + 4 * ty + e];
          b[4 * h + e] = Bs[kk][64 * h + 4 * tx + e];
        }
      }
      if constexpr (kPk) {
        uint64_t b2[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) b2[w] = pk2((float)b[2 * w], (float)b[2 * w + 1]);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint64_t a2 = pk2((float)a[u], (float)a[u]);
#pragma unroll
          for (int w = 0; w < 4; ++w) acc2[u][w] = fma2(a2, b2[w], acc2[u][w]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int v = 0; v < 8; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
      }
    }
  }
  if constexpr (kPk) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        float lo, hi;
        up2(acc2[u][w], lo, hi);
        acc[u][2 * w] = (T)lo;
        acc[u][2 * w + 1] = (T)hi;
      }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v)
      epi(i0 + 64 * (u >> 2) + 4 * ty + (u & 3), j0 + 64 * (v >> 2) + 4 * tx + (v & 3), acc[u][v]);
}

}  // namespace rfk
