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
template <typename T> __device__ __forceinline__ T act_t(int act, T x);
template <> __device__ __forceinline__ float act_t<float>(int act, float x) { return act_f32(act, x); }
template <> __device__ __forceinline__ double act_t<double>(int act, double x) { return act_f64(act, x); }

// Truncation of an fp32 value to the tf32 grid (sign, 8-bit exponent, 10-bit mantissa): the "hi" half
// of the 3×TF32 split; lo = x − hi is exact in fp32.
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// ------------------------------------------------------------------------------------------
// Per-row EQ1 data (DESIGN.md §5 "K1/K5"): for row i with α_i = ‖x_i‖/√τ − 1
//   a0 = A0(α_i), a1 = A1(α_i), a2h = ½⟨0,2⟩A2(α_i), c = 1/(√τ‖x_i‖), inv_ua = 1/‖x_i‖, nrm2 = ‖x_i‖²
// ------------------------------------------------------------------------------------------
struct __align__(32) RowCoef {
  float a0, a1, a2h, c, inv_ua, nrm2, nu_diag, pad;
};
struct RowCoefD {
  double a0, a1, a2h, c, inv_ua, nrm2, nu_diag, pad;
};

// β-polynomial coefficients: C0(β) = k00 + β(k11 + β k22h), C1(β) = k01 + β k12; inv_st = 1/√τ.
struct Eq1Consts {
  double k00, k11, k22h, k01, k12, inv_st;
};

template <typename T>
__device__ __forceinline__ T eq1_entry(T g, T a0, T a1, T a2h, T c, T inv_ua, T nrm2_j, bool diag, T nu_diag,
                                       T k00, T k11, T k22h, T k01, T k12, T inv_st) {
  T nu, beta;
  if (diag) {
    nu = nu_diag;                  // v_b = u_a ⇒ ν = ‖x_i‖/√τ
    beta = T(-1);                  // u_b = 0
  } else {
    T vb = g * inv_ua;             // v_b = x_iᵀx_j/‖x_i‖
    T r = nrm2_j - vb * vb;        // u_b² = ‖x_j‖² − v_b²
    r = r > T(0) ? r : T(0);
    beta = sqrt(r) * inv_st - T(1);
    nu = g * c;
  }
  T C0 = k00 + beta * (k11 + beta * k22h);
  T C1 = k01 + beta * k12;
  return a0 * C0 + nu * (a1 * C1 + nu * a2h);
}

}  // namespace rfk
