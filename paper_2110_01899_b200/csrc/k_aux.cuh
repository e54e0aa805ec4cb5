// Small HBM-bound kernels of the path:
//   K1  row norms ‖x_i‖² (fp64 accumulation, one warp per row, warp-shuffle reduction)
//       + deterministic τ̂ = (1/n)Σ‖x_i‖² (Lemma 1) + per-row EQ1 coefficients
//   K2  fp32 → (tf32 hi, fp32 lo) split for the 3×TF32 operands; G1 fp32 → bf16 round-to-nearest-even (BF16 mode)
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "rf_common.cuh"

namespace rfk {

template <typename T> __device__ __forceinline__ double to_d(T v);
template <> __device__ __forceinline__ double to_d<double>(double v) { return v; }
template <> __device__ __forceinline__ double to_d<float>(float v) { return (double)v; }
template <> __device__ __forceinline__ double to_d<__nv_bfloat16>(__nv_bfloat16 v) { return (double)__bfloat162float(v); }

// One warp per row; 16-byte vector loads when the row is 16-B aligned (validated ldx), scalar tail.
template <typename T>
__global__ void __launch_bounds__(256) k_rownorm(const T* __restrict__ X, int64_t ldx, int64_t p, int64_t n,
                                                 double* __restrict__ nrm2) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const T* x = X + row * ldx;
  constexpr int V = 16 / sizeof(T);
  const int64_t pv = p / V;
  double s = 0.0;
  for (int64_t c = lane; c < pv; c += 32) {
    uint4 raw = __ldg(reinterpret_cast<const uint4*>(x) + c);
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int u = 0; u < V; ++u) {
      double d = to_d<T>(e[u]);
      s = fma(d, d, s);
    }
  }
  for (int64_t c = pv * V + lane; c < p; c += 32) {
    double d = to_d<T>(x[c]);
    s = fma(d, d, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) nrm2[row] = s;
}

// Single block, fixed summation order ⇒ bit-reproducible τ̂.  out[0] = τ̂, out[1] = #zero-norm rows; the same two
// words also go to `host` (mapped pinned memory) when non-null, so the caller reads them without a DMA copy.
__global__ void __launch_bounds__(1024) k_tau_reduce(const double* __restrict__ nrm2, int64_t n,
                                                     double* __restrict__ out, volatile double* host = nullptr) {
  __shared__ double sh[32];
  __shared__ int zc[32];
  double s = 0.0;
  int z = 0;
  for (int64_t i = threadIdx.x; i < n; i += 1024) {
    double v = nrm2[i];
    s += v;
    z += (v == 0.0);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    z += __shfl_xor_sync(0xffffffffu, z, o);
  }
  if ((threadIdx.x & 31) == 0) { sh[threadIdx.x >> 5] = s; zc[threadIdx.x >> 5] = z; }
  __syncthreads();
  if (threadIdx.x < 32) {
    s = sh[threadIdx.x];
    z = zc[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      z += __shfl_xor_sync(0xffffffffu, z, o);
    }
    if (threadIdx.x == 0) {
      out[0] = s / (double)n;
      out[1] = (double)z;
      if (host) {
        host[0] = s / (double)n;
        host[1] = (double)z;
        __threadfence_system();
      }
    }
  }
}

// Moments needed per row: A_j(α) = ⟨j,0⟩ + α⟨j+1,1⟩ + (α²/2)⟨j+2,2⟩, j = 0,1,2.
struct RowMoments {
  double kd[5][3];
  double inv_st;   // 1/√τ
  int form;        // 1 = EQ1, 2 = EQ2
};

// Per-row coefficients of the regrouped EQ1 (rf_common.cuh), fp64 arithmetic, stored as RC = RowCoef
// (f32) or RowCoefD (f64); the column side gets ‖x_j‖²/τ.
template <typename RC, typename NT>
__global__ void __launch_bounds__(256) k_row_coef(const double* __restrict__ nrm2, int64_t n, RowMoments m,
                                                  RC* __restrict__ rc, NT* __restrict__ njt_out) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= n) {   // the grid covers whole 256-column tiles: zero the padding K5 stages with each tile
    njt_out[i] = (NT)0;
    return;
  }
  const double r2 = nrm2[i];
  const double ua = sqrt(r2);                       // u_a = ‖x_i‖
  const double al = ua * m.inv_st - 1.0;            // α = u_a/√τ − 1
  const double h = 0.5 * al * al;
  const bool eq2 = m.form == 2;     // EQ2 keeps only the α-linear part of A0 and the constants of A1, A2
  const double A0 = m.kd[0][0] + al * m.kd[1][1] + (eq2 ? 0.0 : h * m.kd[2][2]);
  const double A1 = eq2 ? m.kd[1][0] : m.kd[1][0] + al * m.kd[2][1] + h * m.kd[3][2];
  const double A2 = eq2 ? m.kd[2][0] : m.kd[2][0] + al * m.kd[3][1] + h * m.kd[4][2];
  RC c;
  c.a0 = A0;
  c.a1 = A1;
  c.a2h = 0.5 * m.kd[0][2] * A2;
  c.c = ua > 0.0 ? m.inv_st / ua : 0.0;            // ν = g·c; a zero pivot row (R23): ν = 0, s = ‖x_j‖/√τ
  c.nu_diag = ua * m.inv_st;                        // ν on the diagonal (v_b = u_a)
  c.pad0 = c.pad1 = c.pad2 = 0;
  rc[i] = c;
  njt_out[i] = (NT)(r2 * m.inv_st * m.inv_st);      // ‖x_j‖²/τ
}

// hi = tf32 truncation of x, lo = x − hi (exact).  2-D: rows × cols with independent strides.
__global__ void __launch_bounds__(256) k_split_tf32(const float* __restrict__ src, int64_t lds, int64_t rows,
                                                    int64_t cols, float* __restrict__ hi, float* __restrict__ lo,
                                                    int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total; e += (int64_t)gridDim.x * 256) {
    const int64_t r = e / cols, c = e - r * cols;
    const float x = src[r * lds + c];
    const float h = tf32_hi(x);
    hi[r * ldd + c] = h;
    lo[r * ldd + c] = x - h;
  }
}

// G1 (BF16 mode): dst = bf16(src), round to nearest, ties to even (cvt.rn.bf16.f32; NaN stays NaN).  kVec: four
// columns per thread (cols, lds, ldd multiples of 4 and both bases 16-B / 8-B aligned, checked by the caller).
template <bool kVec>
__global__ void __launch_bounds__(256) k_round_bf16(const float* __restrict__ src, int64_t lds, int64_t rows,
                                                    int64_t cols, __nv_bfloat16* __restrict__ dst, int64_t ldd) {
  const int64_t cv = kVec ? cols / 4 : cols;
  const int64_t total = rows * cv;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total; e += (int64_t)gridDim.x * 256) {
    const int64_t r = e / cv, c = e - r * cv;
    if (kVec) {
      const float4 x = __ldcs(reinterpret_cast<const float4*>(src + r * lds) + c);
      __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&lo);
      o.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(dst + r * ldd)[c] = o;
    } else {
      dst[r * ldd + c] = __float2bfloat16_rn(src[r * lds + c]);
    }
  }
}

}  // namespace rfk
