// NEXT-4: random-features kernel ridge regression on the Gram G, the paper's downstream use of G
// (P:757-761).  For each ridge parameter γ:  A = G_train + γ·I (fp64, lower triangle), A = L·Lᵀ by a
// blocked right-looking Cholesky (64-wide panels), α = L^{-T} L^{-1} Y, Ŷ_test = G_cross·α.  G_train and G_cross
// are read from the upper triangle of ONE Gram over the stacked samples [X_train; X_test] (include/rf.h rf_ridge).
//   k_ridge_build ...... A's lower triangle from G's upper triangle (32×32 smem transpose tiles), + γ on the diagonal
//   k_chol_diag ........ Cholesky of the 64×64 diagonal block in shared memory (one CTA), and its inverse
//   k_chol_panel ....... L_ik = A_ik·L_kk^{-T} for the row blocks below (one CTA per block, one thread per row)
//   trailing update .... A_ij −= L_ik·L_jkᵀ on the lower triangle: the K6 SIMT GEMM (k_simt.cuh) with SimtCholUpd
//   k_trsv_fwd / k_gemv_fwd, k_trsv_bwd / k_axpy_bwd ... the two triangular solves, block by block (the diagonal
//                        blocks through their inverses)
//   k_ridge_predict .... Ŷ[t] = Σ_i G[i][n_train + t]·α[i]
#pragma once
#include <stdint.h>

namespace rfk {

constexpr int kRB = 64;
constexpr int kMaxBatch = 16;   // γ values factored concurrently (blockIdx.z)
struct RidgeBatch {
  double gamma[kMaxBatch];
  int64_t sA, sL, sY, sYh;      // per-z strides of the factor, the inverses, α and Ŷ (elements)
};

__global__ void __launch_bounds__(256) k_ridge_build(const float* __restrict__ G, int64_t ldg, int64_t n,
                                                     RidgeBatch bt, double* __restrict__ A, int64_t lda) {
  __shared__ float t[32][33];
  A += blockIdx.z * bt.sA;
  const double gamma = bt.gamma[blockIdx.z];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;          // A block (bi, bj), bj ≤ bi (lower)
  if (bj > bi) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 × 8
  // read G rows j ∈ block bj, columns i ∈ block bi (coalesced along i): G[j][i] with j ≤ i is the upper triangle
  for (int r = ty; r < 32; r += 8) {
    const int64_t j = bj * 32 + r, i = bi * 32 + tx;
    t[r][tx] = (j < n && i < n) ? G[j * ldg + i] : 0.f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = bi * 32 + r, j = bj * 32 + tx;
    if (i < n && j < n) {
      double v = j <= i ? (double)t[tx][r] : 0.0;
      if (i == j) v += gamma;
      A[i * lda + j] = v;
    }
  }
}

// In-place Cholesky of the diagonal block k (rows/cols [64k, 64k + nb)) in shared memory, then its inverse
// L_kk^{-1} (column j by forward substitution on e_j, one thread per column) into Linv (64 × 64, row-major), which
// turns the block solves of k_trsv_fwd / k_trsv_bwd into parallel triangular products.
// info: first non-positive pivot (1-based).  Dynamic shared memory: kDiagSmem.
constexpr int kDiagSmem = 2 * kRB * (kRB + 1) * 8;
__global__ void __launch_bounds__(256) k_chol_diag(double* __restrict__ A, int64_t lda, int64_t n, int k,
                                                   int* __restrict__ info, double* __restrict__ Linv, RidgeBatch bt) {
  extern __shared__ double diag_smem[];
  A += blockIdx.z * bt.sA;
  Linv += blockIdx.z * bt.sL;
  double(*a)[kRB + 1] = reinterpret_cast<double(*)[kRB + 1]>(diag_smem);
  double(*x)[kRB + 1] = reinterpret_cast<double(*)[kRB + 1]>(diag_smem + kRB * (kRB + 1));
  const int64_t r0 = (int64_t)k * kRB;
  const int nb = (int)(n - r0 < kRB ? n - r0 : kRB);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;   // 16 × 16 thread grid for the updates
  for (int r = ty; r < kRB; r += 16)
    for (int c = tx; c < kRB; c += 16)
      a[r][c] = (r < nb && c <= r) ? A[(r0 + r) * lda + r0 + c] : (r == c ? 1.0 : 0.0);
  __syncthreads();
  __shared__ double pinv;
  for (int c = 0; c < nb; ++c) {
    if (tid == 0) {                             // one fp64 sqrt and division per column, broadcast through smem
      const double d = a[c][c];
      if (!(d > 0.0) && *info == 0) *info = (int)(r0 + c + 1);
      const double sd = sqrt(d);
      a[c][c] = sd;
      pinv = 1.0 / sd;
    }
    __syncthreads();
    const double inv = pinv;
    for (int r = c + 1 + tid; r < nb; r += 256) a[r][c] *= inv;
    __syncthreads();
    for (int r = c + 1 + ty; r < nb; r += 16)
      for (int q = c + 1 + tx; q <= r; q += 16) a[r][q] -= a[r][c] * a[q][c];
    __syncthreads();
  }
  for (int r = ty; r < nb; r += 16)
    for (int c = tx; c <= r; c += 16) A[(r0 + r) * lda + r0 + c] = a[r][c];
  // L^{-1}: column j = L^{-1} e_j (rows ≥ j), padded rows/columns (≥ nb) of the identity.  Four threads per column
  // split each row's inner product (t ≡ q mod 4) and combine it with two shuffles.
  {
    const int j = tid >> 2, q = tid & 3;
    for (int r = 0; r < kRB; ++r) {   // every lane takes every step (the shuffles need the whole warp)
      double sum = 0.0;
      for (int t = j + q; t < r; t += 4) sum += a[r][t] * x[t][j];
      sum += __shfl_xor_sync(0xFFFFFFFFu, sum, 1);
      sum += __shfl_xor_sync(0xFFFFFFFFu, sum, 2);
      if (q == 0) x[r][j] = r < j ? 0.0 : ((r == j ? 1.0 : 0.0) - sum) / a[r][r];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int r = ty; r < kRB; r += 16)
    for (int c = tx; c < kRB; c += 16) Linv[r * kRB + c] = x[r][c];
}

// Row block b (rows 64(k + 1 + b) ..) of panel k: X·L_kkᵀ = A_ik, one thread per row, forward over the columns.
constexpr int kPanelSmem = 2 * kRB * (kRB + 1) * 8;     // dynamic shared memory of k_chol_panel (66.5 KB)
__global__ void __launch_bounds__(kRB) k_chol_panel(double* __restrict__ A, int64_t lda, int64_t n, int k,
                                                    int64_t sA) {
  extern __shared__ double panel_smem[];
  A += blockIdx.z * sA;
  double(*L)[kRB + 1] = reinterpret_cast<double(*)[kRB + 1]>(panel_smem);
  double(*X)[kRB + 1] = reinterpret_cast<double(*)[kRB + 1]>(panel_smem + kRB * (kRB + 1));
  const int64_t r0 = (int64_t)k * kRB, rb = r0 + kRB * (1 + (int64_t)blockIdx.x);
  const int r = threadIdx.x;
  for (int c = 0; c < kRB; ++c) L[c][r] = (r <= c) ? A[(r0 + c) * lda + r0 + r] : 0.0;   // L[c][r], r ≤ c
  const bool live = rb + r < n;
  for (int c = 0; c < kRB; ++c) X[r][c] = live ? A[(rb + r) * lda + r0 + c] : 0.0;
  __syncthreads();
  for (int c = 0; c < kRB; ++c) {
    double s = X[r][c];
    for (int t = 0; t < c; ++t) s -= X[r][t] * L[c][t];
    X[r][c] = s / L[c][c];
  }
  if (live)
    for (int c = 0; c < kRB; ++c) A[(rb + r) * lda + r0 + c] = X[r][c];
}

// Trailing update A_ij −= (L·Lᵀ)_ij, j ≤ i, from the GEMM over the panel rows restricted to its lower tiles
// (tri = 2), so every thread updates row-major elements of the lower triangle.
struct SimtCholUpd {
  double* A;
  int64_t lda, r1, m;
  int64_t zstride;      // batched launches: factor z at A + z·zstride
  int64_t ncols;        // columns j < ncols only (the sub-panel updates stay inside their 256-wide panel)
  __device__ __forceinline__ void operator()(int64_t i, int64_t j, double v) const {
    if (i < m && j < ncols && j <= i) A[(r1 + i) * lda + r1 + j] -= v;
  }
};

// Forward solve of block k: z_k = L_kk^{-1} y_k as a triangular product with the inverse from k_chol_diag (one
// thread per (row, right-hand side)).
__global__ void __launch_bounds__(256) k_trsv_fwd(const double* __restrict__ Linv, int64_t n, int k,
                                                  double* __restrict__ Y, int64_t ldy, int nrhs, RidgeBatch bt) {
  __shared__ double y[4][kRB];
  Linv += blockIdx.z * bt.sL;
  Y += blockIdx.z * bt.sY;
  const int64_t r0 = (int64_t)k * kRB;
  const int nb = (int)(n - r0 < kRB ? n - r0 : kRB);
  const int r = threadIdx.x & (kRB - 1), w = threadIdx.x >> 6, rhs = blockIdx.x * 4 + w;
  if (rhs < nrhs) y[w][r] = r < nb ? Y[(r0 + r) * ldy + rhs] : 0.0;
  __syncthreads();
  if (rhs >= nrhs || r >= nb) return;
  double s = 0.0;
  for (int t = 0; t <= r; ++t) s += Linv[r * kRB + t] * y[w][t];
  Y[(r0 + r) * ldy + rhs] = s;
}

// y_i −= L[i][64k .. 64k+64)·z_k for the rows below block k (one warp per row).
__global__ void k_gemv_fwd(const double* __restrict__ A, int64_t lda, int64_t n, int k, double* __restrict__ Y,
                           int64_t ldy, int nrhs, RidgeBatch bt) {
  A += blockIdx.z * bt.sA;
  Y += blockIdx.z * bt.sY;
  const int lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)k * kRB;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = r0 + kRB + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const double l0 = A[i * lda + r0 + lane], l1 = A[i * lda + r0 + 32 + lane];
    for (int h = 0; h < nrhs; ++h) {
      double s = l0 * Y[(r0 + lane) * ldy + h] + l1 * Y[(r0 + 32 + lane) * ldy + h];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
      if (lane == 0) Y[i * ldy + h] -= s;
    }
  }
}

// Backward solve of block k: α_k = L_kk^{-T} z_k (the transpose of the inverse from k_chol_diag).
__global__ void __launch_bounds__(256) k_trsv_bwd(const double* __restrict__ Linv, int64_t n, int k,
                                                  double* __restrict__ Y, int64_t ldy, int nrhs, RidgeBatch bt) {
  __shared__ double y[4][kRB];
  Linv += blockIdx.z * bt.sL;
  Y += blockIdx.z * bt.sY;
  const int64_t r0 = (int64_t)k * kRB;
  const int nb = (int)(n - r0 < kRB ? n - r0 : kRB);
  const int r = threadIdx.x & (kRB - 1), w = threadIdx.x >> 6, rhs = blockIdx.x * 4 + w;
  if (rhs < nrhs) y[w][r] = r < nb ? Y[(r0 + r) * ldy + rhs] : 0.0;
  __syncthreads();
  if (rhs >= nrhs || r >= nb) return;
  double s = 0.0;
  for (int t = r; t < nb; ++t) s += Linv[t * kRB + r] * y[w][t];
  Y[(r0 + r) * ldy + rhs] = s;
}

// z_j −= Σ_{t < nb} L[64k + t][j]·α[64k + t] for the rows j above block k (one thread per j, coalesced along j).
__global__ void k_axpy_bwd(const double* __restrict__ A, int64_t lda, int64_t n, int k, double* __restrict__ Y,
                           int64_t ldy, int nrhs, RidgeBatch bt) {
  A += blockIdx.z * bt.sA;
  Y += blockIdx.z * bt.sY;
  const int64_t r0 = (int64_t)k * kRB;
  const int nb = (int)(n - r0 < kRB ? n - r0 : kRB);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < r0; j += (int64_t)gridDim.x * blockDim.x) {
    for (int h = 0; h < nrhs; ++h) {
      double s = 0.0;
      for (int t = 0; t < nb; ++t) s += A[(r0 + t) * lda + j] * Y[(r0 + t) * ldy + h];
      Y[j * ldy + h] -= s;
    }
  }
}

// Ŷ[t][h] = Σ_{i < n_train} G[i][n_train + t]·α[i][h] (G's upper triangle: rows of training samples, columns of test
// samples), one thread per test sample, coalesced along t.
__global__ void k_ridge_predict(const float* __restrict__ G, int64_t ldg, int64_t n_train, int64_t n_test,
                                const double* __restrict__ alpha, int64_t lda_, int nrhs, double* __restrict__ Yhat,
                                int64_t ldyh, RidgeBatch bt) {
  alpha += blockIdx.z * bt.sY;
  Yhat += blockIdx.z * bt.sYh;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_test; t += (int64_t)gridDim.x * blockDim.x) {
    for (int h = 0; h < nrhs; ++h) {
      double s = 0.0;
      for (int64_t i = 0; i < n_train; ++i) s += (double)G[i * ldg + n_train + t] * alpha[i * lda_ + h];
      Yhat[t * ldyh + h] = s;
    }
  }
}

// Copies one 32-bit word to mapped pinned host memory (status read-back that does not queue behind DMA copies).
__global__ void k_publish_u32(const int* __restrict__ src, volatile int* dst) {
  dst[0] = src[0];
  __threadfence_system();
}

}  // namespace rfk

