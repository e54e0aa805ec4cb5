// Shared device helpers for the sm_100a kernels: activations σ (north star: tanh, erf,
// sigmoid − 1/2; Assumption 3 P:505-509), vectorised stores, the per-row EQ1 coefficient record.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/rf.h"

namespace rfk {

constexpr int kNumSMs = 148;

// ------------------------------------------------------------------------------------------
// σ.  sigmoid(x) − 1/2 is evaluated as ½·tanh(x/2) (identical function, no cancellation).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ float act_f32(int act, float x) {
  if (act == RF_ACT_TANH) return tanhf(x);
  if (act == RF_ACT_ERF) return erff(x);
  return 0.5f * tanhf(0.5f * x);
}
__device__ __forceinline__ double act_f64(int act, double x) {
  if (act == RF_ACT_TANH) return tanh(x);
  if (act == RF_ACT_ERF) return erf(x);
  return 0.5 * tanh(0.5 * x);
}
// Compile-time σ for the tensor-core K3 epilogue.
template <int kAct>
__device__ __forceinline__ float act_fixed(float x) {
  if (kAct == RF_ACT_TANH) return tanhf(x);
  if (kAct == RF_ACT_ERF) return erff(x);
  return 0.5f * tanhf(0.5f * x);
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// σ for BF16-stored Σ (K3, RF_PREC_BF16): sigmoid(x) − ½ = 1/(1 + 2^(−x·log2 e)) − ½ and
// tanh(x) = 2/(1 + 2^(−2x·log2 e)) − 1 on the MUFU pipe (one EX2 + one RCP).  Absolute error ≲ 3e-7
// (ex2/rcp.approx are within ~2 ulp), i.e. ≥ 30× below half an ulp of the bf16 value it is rounded to for
// |σ| ≥ 2^-6; both limits saturate correctly (2^+∞ → rcp → 0).  erf keeps the library erff.
template <int kAct>
__device__ __forceinline__ float act_bf16out(float x) {
  constexpr float kLog2e = 1.4426950408889634f;
  if (kAct == RF_ACT_SIGMOID_HALF) return rcp_approx(1.0f + ex2_approx(-kLog2e * x)) - 0.5f;
  if (kAct == RF_ACT_TANH) return fmaf(2.0f, rcp_approx(1.0f + ex2_approx(-2.0f * kLog2e * x)), -1.0f);
  return erff(x);
}

template <typename T> __device__ __forceinline__ T act_t(int act, T x);
template <> __device__ __forceinline__ float act_t<float>(int act, float x) { return act_f32(act, x); }
template <> __device__ __forceinline__ double act_t<double>(int act, double x) { return act_f64(act, x); }

// Truncation of an fp32 value to the tf32 grid (sign, 8-bit exponent, 10-bit mantissa): the "hi" half
// of the 3×TF32 split; lo = x − hi is exact in fp32.
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// ------------------------------------------------------------------------------------------
// EQ1 (readings R1-R4) regrouped for the epilogue (K5).  With
//   α = u_a/√τ − 1, s = u_b/√τ (= β + 1), ν = v_b/√τ:
//   Φ = A0(α)·C0(s) + ν·(A1(α)·C1(s) + ν·½⟨0,2⟩A2(α))
//   A_j(α) = ⟨j,0⟩ + α⟨j+1,1⟩ + (α²/2)⟨j+2,2⟩                     — per row (k_row_coef)
//   C0(s) = e0 + s(e1 + s e2), C1(s) = f0 + s f1                 — the β-polynomials re-expanded in s:
//   e0 = ⟨0,0⟩ − ⟨1,1⟩ + ½⟨2,2⟩, e1 = ⟨1,1⟩ − ⟨2,2⟩, e2 = ½⟨2,2⟩, f0 = ⟨0,1⟩ − ⟨1,2⟩, f1 = ⟨1,2⟩.
// Per entry, from g = x_iᵀx_j: ν = g·c_i with c_i = 1/(√τ‖x_i‖); s = √max(0, ‖x_j‖²/τ − ν²)
// (Gram–Schmidt P:1016-1018 scaled by 1/√τ).  Diagonal (R6): s = 0, ν = ‖x_i‖/√τ.
// ------------------------------------------------------------------------------------------
struct __align__(32) RowCoef {
  float a0, a1, a2h, c, nu_diag, pad0, pad1, pad2;
};
struct RowCoefD {
  double a0, a1, a2h, c, nu_diag, pad0, pad1, pad2;
};

__device__ __forceinline__ float sqrt_fast(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double sqrt_fast(double x) { return sqrt(x); }

template <typename T>
__device__ __forceinline__ T eq1_entry(T g, T a0, T a1, T a2h, T c, T njt, bool diag, T nu_diag, T e0, T e1, T e2,
                                       T f0, T f1) {
  T nu = g * c;
  T r = fma(-nu, nu, njt);
  r = r > T(0) ? r : T(0);
  T s = sqrt_fast(r);
  if (diag) {
    nu = nu_diag;
    s = T(0);
  }
  const T C0 = fma(s, fma(s, e2, e1), e0);
  const T C1 = fma(s, f1, f0);
  const T inner = fma(nu, a2h, a1 * C1);
  return fma(nu, inner, a0 * C0);
}

}  // namespace rfk
