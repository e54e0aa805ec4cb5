// NEXT-2: centering K = P·A·P of a symmetric n × n matrix stored in its upper triangle (Eq. (2)),
// as a post-pass over A in place: (PAP)_ij = A_ij − r_i − r_j + s with r_i = (1/n)Σ_j A_ij, s = (1/n)Σ_i r_i.
//   k_center_rowsum  128 × 128 tiles of the upper triangle; entry (i, j), j > i, adds to the sums of rows i AND j
//                    (the mirror is implied), the diagonal to row i once; fp64 partials, one fp64 atomic per
//                    row / column of each tile.
//   k_center_scale   r ← r/n, s = mean(r) (one block, fixed order).
//   k_center_apply   A_ij ← A_ij − r_i − r_j + s on the stored part (UPPER: j ≥ i; FULL: all entries).
// HBM-bound: one read of the triangle for the sums, one read + write for the update.
#pragma once
#include <stdint.h>

namespace rfk {

constexpr int kCT = 128;   // centering tile

template <typename T>
__global__ void __launch_bounds__(256) k_center_rowsum(const T* __restrict__ A, int64_t ld, int64_t n,
                                                       double* __restrict__ rsum) {
  const int I = blockIdx.y, J = blockIdx.x;
  if (J < I) return;
  __shared__ double colpart[8][kCT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = (int64_t)I * kCT, j0 = (int64_t)J * kCT;
  // All 16 rows of this warp are loaded before any is reduced (16 independent loads in flight per lane); lane l
  // holds columns j0 + 4l .. 4l + 3, read as one 16-B vector where the row allows it.
  constexpr int R = kCT / 8;
  T v[R][4];
  const int64_t jl = j0 + 4 * lane;
  const bool vec = sizeof(T) == 4 && (ld & 3) == 0 && jl + 4 <= n && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int64_t i = i0 + warp + 8 * k;
    if (i < n && vec) {
      const float4 q = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(A) + i * ld + jl);
      v[k][0] = (T)q.x; v[k][1] = (T)q.y; v[k][2] = (T)q.z; v[k][3] = (T)q.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[k][u] = (i < n && jl + u < n) ? A[i * ld + jl + u] : T(0);
    }
  }
  double cacc[4] = {0.0, 0.0, 0.0, 0.0};   // this lane's 4 columns, over this warp's rows
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int64_t i = i0 + warp + 8 * k;
    double racc = 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = jl + u;
      if (i < n && j < n && j >= i) {
        const double x = (double)v[k][u];
        racc += x;
        if (j > i) cacc[u] += x;             // mirror entry (j, i) belongs to row j
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) racc += __shfl_xor_sync(0xffffffffu, racc, o);
    if (lane == 0 && i < n) atomicAdd(rsum + i, racc);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) colpart[warp][4 * lane + u] = cacc[u];
  __syncthreads();
  if (threadIdx.x < kCT) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += colpart[w][threadIdx.x];
    const int64_t j = j0 + threadIdx.x;
    if (j < n && s != 0.0) atomicAdd(rsum + j, s);
  }
}

// r ← r/n in place; out_s = mean of the new r.  One block of 1024 threads, fixed reduction order.
__global__ void __launch_bounds__(1024) k_center_scale(double* __restrict__ r, int64_t n, double* __restrict__ out_s) {
  __shared__ double sh[32];
  double s = 0.0;
  const double inv = 1.0 / (double)n;
  for (int64_t i = threadIdx.x; i < n; i += 1024) {
    const double v = r[i] * inv;
    r[i] = v;
    s += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = sh[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out_s[0] = s * inv;
  }
}

// A_ij ← A_ij − r_i − r_j + s.  grid (ceil(n/128), ceil(n/8)): block = 8 rows × 128 columns × … strided.
template <typename T>
__global__ void __launch_bounds__(256) k_center_apply(T* __restrict__ A, int64_t ld, int64_t n,
                                                      const double* __restrict__ r, const double* __restrict__ s_ptr,
                                                      int full) {
  const int64_t i = (int64_t)blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= n) return;
  const int lane = threadIdx.x & 31;
  const double s = *s_ptr;
  const double ri = r[i];
  const int64_t jb = (int64_t)blockIdx.x * kCT;
  if (!full && jb + kCT <= i) return;
  T* row = A + i * ld;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t j = jb + lane + 32 * u;
    if (j < n && (full || j >= i)) row[j] = (T)((double)row[j] - ri - r[j] + s);
  }
}

// ---------------------------------------------------------------------------------------------
// K̃ preparation (EQ6): column sums x̄ = Σ_i x_i, v̄ = Σ_i v_i (fp64), per-row u_i = A v_i and the uncentred row
// sums n·r_i = d1·x_iᵀx̄ + d2·u_iᵀv̄ + d0, then r'_i = r_i − s/2 for the epilogue.
constexpr int kMaxKv = 8;
struct KtA {
  double a[kMaxKv][kMaxKv];
};

// out[l] += Σ_{i in this block's row chunk} M[i][l]   (M: rows × cols, ld; grid (ceil(cols/256), chunks))
template <typename T>
__global__ void __launch_bounds__(256) k_colsum(const T* __restrict__ M, int64_t ld, int64_t rows, int64_t cols,
                                                double* __restrict__ out) {
  const int64_t l = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (l >= cols) return;
  const int64_t per = (rows + gridDim.y - 1) / gridDim.y;
  const int64_t i0 = (int64_t)blockIdx.y * per, i1 = i0 + per < rows ? i0 + per : rows;
  double s = 0.0;
  for (int64_t i = i0; i < i1; ++i) s += (double)M[i * ld + l];
  atomicAdd(out + l, s);
}

// One warp per row i: x_iᵀx̄ (fp64), u_i = A v_i, rr_i = d1·x_iᵀx̄ + d2·u_iᵀv̄ + d0; writes u (n × 8, f32, zero
// padded), vt (kMaxKv × nvt, f32, rows 16-B aligned) and rr (f64).
template <typename T>
__global__ void __launch_bounds__(256) k_ktilde_rows(const T* __restrict__ X, int64_t ldx, int64_t p, int64_t n,
                                                     const float* __restrict__ V, int64_t ldv, int kv, KtA A, double d0,
                                                     double d1, double d2, const double* __restrict__ xbar,
                                                     const double* __restrict__ vbar, float* __restrict__ u,
                                                     float* __restrict__ vt, int64_t nvt, double* __restrict__ rr) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  double dot = 0.0;
  for (int64_t l = lane; l < p; l += 32) dot += (double)X[i * ldx + l] * xbar[l];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if (lane < kMaxKv) {
    double ui = 0.0;
    if (lane < kv)
      for (int k = 0; k < kv; ++k) ui += A.a[lane][k] * (double)V[i * ldv + k];
    u[i * kMaxKv + lane] = (float)ui;
    vt[(int64_t)lane * nvt + i] = lane < kv ? V[i * ldv + lane] : 0.f;
    double uv = lane < kv ? ui * vbar[lane] : 0.0;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) uv += __shfl_xor_sync(0x000000ffu, uv, o);
    if (lane == 0) rr[i] = d1 * dot + d2 * uv + d0;
  }
}

// r'_i = r_i − s/2 as f32 (r already divided by n by k_center_scale, s = mean r)
__global__ void __launch_bounds__(256) k_center_fold(const double* __restrict__ r, const double* __restrict__ s_ptr,
                                                     int64_t n, float* __restrict__ rf) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i < n) rf[i] = (float)(r[i] - 0.5 * s_ptr[0]);
}

}  // namespace rfk
