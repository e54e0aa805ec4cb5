// Shared device helpers for the sm_100a kernels: activations σ (north star: tanh, erf,
// sigmoid − 1/2; Assumption 3 P:505-509), vectorised stores, the per-row EQ1 coefficient record.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/rf.h"

// RF_DEBUG builds: device-side bounds / invariant checks on the store paths (compute-sanitizer is not available on
// this GPU pool; these asserts stand in for memcheck on the hand-written epilogues).  Release builds: no code.
#if defined(RF_DEBUG)
#include <cstdio>
#define RF_DCHECK(cond, ...)                                                                              \
  do {                                                                                                    \
    if (!(cond)) {                                                                                        \
      printf("[rf debug] check failed: %s (block %d thread %d) ", #cond, (int)blockIdx.x, (int)threadIdx.x); \
      printf(__VA_ARGS__);                                                                                \
      printf("\n");                                                                                      \
      __trap();                                                                                           \
    }                                                                                                     \
  } while (0)
#else
#define RF_DCHECK(cond, ...) \
  do {                       \
  } while (0)
#endif

namespace rfk {

// ------------------------------------------------------------------------------------------
// σ.  sigmoid(x) − 1/2 is evaluated as ½·tanh(x/2) (identical function, no cancellation).
// ------------------------------------------------------------------------------------------
// NEXT-3 (Table 2): ReLU, |t|, sign, 1_{t>0}, cos, sin, t, t², e^{−t²/2}.
template <typename T>
__device__ __forceinline__ T act_table2(int act, T x) {
  switch (act) {
    case RF_ACT_RELU: return x > T(0) ? x : T(0);
    case RF_ACT_ABS: return x < T(0) ? -x : x;
    case RF_ACT_SIGN: return x > T(0) ? T(1) : (x < T(0) ? T(-1) : T(0));
    case RF_ACT_STEP: return x > T(0) ? T(1) : T(0);
    case RF_ACT_COS: return cos(x);
    case RF_ACT_SIN: return sin(x);
    case RF_ACT_IDENT: return x;
    case RF_ACT_QUAD: return x * x;
    default: return exp(T(-0.5) * x * x);   // RF_ACT_BUMP
  }
}
// Parametrised Table-2 rows, registered at run time (rf_act_leaky_relu / rf_act_quadratic):
// kind 1: a₊·max(0, t) + a₋·max(0, −t) with (a0, a1) = (a₊, a₋);  kind 2: a₂t² + a₁t + a₀.  kind 0: a fixed rf_act.
struct ActRt {
  int kind;
  double a0, a1, a2;
};
template <typename T>
__device__ __forceinline__ T act_param(const ActRt& p, T x) {
  if (p.kind == 1) return T(p.a0) * (x > T(0) ? x : T(0)) + T(p.a1) * (x < T(0) ? -x : T(0));
  return fma(fma(T(p.a2), x, T(p.a1)), x, T(p.a0));
}

__device__ __forceinline__ float act_f32(int act, float x) {
  if (act == RF_ACT_TANH) return tanhf(x);
  if (act == RF_ACT_ERF) return erff(x);
  if (act == RF_ACT_SIGMOID_HALF) return 0.5f * tanhf(0.5f * x);
  return act_table2<float>(act, x);
}
__device__ __forceinline__ double act_f64(int act, double x) {
  if (act == RF_ACT_TANH) return tanh(x);
  if (act == RF_ACT_ERF) return erf(x);
  if (act == RF_ACT_SIGMOID_HALF) return 0.5 * tanh(0.5 * x);
  return act_table2<double>(act, x);
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

// Packed fp32 pairs (sm_100 FFMA2 / FMUL2: two fp32 lanes per instruction, each rounded as the scalar op).
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// Two off-diagonal EQ1 entries at once (same row i, columns j, j+1): the arithmetic of eq1_entry below,
// op for op, on fp32 pairs.  kOdd: σ odd ⇒ ⟨k,d⟩ = 0 for k + d even ⇒ A0 = A2 = 0 and Φ = ν·A1·C1(s).
template <bool kOdd>
__device__ __forceinline__ void eq1_pair(float g0, float g1, float nj0, float nj1, uint64_t c2, uint64_t a0_2,
                                         uint64_t a1_2, uint64_t a2h_2, uint64_t e0_2, uint64_t e1_2, uint64_t e2_2,
                                         uint64_t f0_2, uint64_t f1_2, float& out0, float& out1) {
  const uint64_t nu = mul2(pk2(g0, g1), c2);
  const uint64_t r = sub2(pk2(nj0, nj1), mul2(nu, nu));
  float r0, r1;
  up2(r, r0, r1);
  const uint64_t s = pk2(sqrt_fast(fabsf(r0)), sqrt_fast(fabsf(r1)));
  const uint64_t C1 = fma2(s, f1_2, f0_2);
  uint64_t o;
  if (kOdd) {
    o = mul2(nu, mul2(a1_2, C1));
  } else {
    const uint64_t C0 = fma2(s, fma2(s, e2_2, e1_2), e0_2);
    const uint64_t inner = fma2(nu, a2h_2, mul2(a1_2, C1));
    o = fma2(nu, inner, mul2(a0_2, C0));
  }
  up2(o, out0, out1);
}

// Odd σ, off the diagonal, with the row constants folded: Φ = ν·A1·(f0 + f1·s) = g·(P + Q·s), P = c·A1·f0,
// Q = c·A1·f1 (ν = g·c); one packed multiply fewer per pair than eq1_pair<true>.
__device__ __forceinline__ void eq1_pair_odd(float g0, float g1, float nj0, float nj1, uint64_t c2, uint64_t p2,
                                             uint64_t q2, float& out0, float& out1) {
  const uint64_t g = pk2(g0, g1);
  const uint64_t nu = mul2(g, c2);
  const uint64_t r = sub2(pk2(nj0, nj1), mul2(nu, nu));
  float r0, r1;
  up2(r, r0, r1);
  const uint64_t s = pk2(sqrt_fast(fabsf(r0)), sqrt_fast(fabsf(r1)));
  up2(mul2(g, fma2(s, q2, p2)), out0, out1);
}

template <typename T>
__device__ __forceinline__ T eq1_entry(T g, T a0, T a1, T a2h, T c, T njt, bool diag, T nu_diag, T e0, T e1, T e2,
                                       T f0, T f1) {
  T nu = g * c;
  // r = ‖x_j‖²/τ − ν² ≥ 0 by Cauchy–Schwarz; a rounding-negative r (near-parallel rows) is taken by magnitude:
  // |r| and max(r, 0) are equally close to the exact value (≤ the rounding of r), and |·| folds into MUFU.SQRT's
  // operand (two FMNMX fewer per entry pair in K5)
  const T r = fma(-nu, nu, njt);
  T s = sqrt_fast(r < T(0) ? -r : r);
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
