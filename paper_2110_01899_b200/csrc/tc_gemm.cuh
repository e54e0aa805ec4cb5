// Warp-specialised persistent tcgen05 GEMM for sm_100a, shared by the three tensor-core kernels:
//   K3  Σᵀ = σ(X·Wᵀ)          rectangular tiles, σ in the epilogue          (Σ = σ(WX))
//   K4  G  = ΣᵀΣ / m          upper-triangular tiles, scale in the epilogue  (Eq. def_Gram)
//   K5  Φ  = EQ1(XᵀX, …)      upper-triangular tiles, EQ1 in the epilogue
// D[i][j] = Σ_k A[i][k]·B[j][k]; A (rows i) and B (rows j) are both K-major in HBM, so
// both UMMA operands are K-major 128-B-swizzled smem tiles written by TMA.
//
// Tile 128 (M) × 256 (N), K-block = one 128-byte swizzle row (64 bf16 / 32 fp32).
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (one thread), w2 TMEM allocator,
// w3 idle, w4..w7 epilogue (warp w4+q owns TMEM lanes / tile rows 32q..32q+31).
// Pipelines: smem ring (full/empty mbarriers, STAGES deep) TMA→MMA; TMEM double-buffered accumulator
// (2 × 256 fp32 columns = all 512 columns) MMA→epilogue, so tile t+1's MMAs overlap tile t's epilogue.
// 3×TF32 (kSplit = 3): each stage holds A_hi, A_lo, B_hi, B_lo; per K-step three MMAs
// lo·hi, hi·lo, hi·hi accumulate into the same TMEM accumulator (small terms first).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "ptx_sm100.cuh"
#include "rf_common.cuh"

namespace rfk {

template <int kFmt /*1 = bf16 (kind::f16), 2 = tf32*/, int kSplit /*1 or 3*/>
struct TcCfg {
  static constexpr int BM = 128, BN = 256;
  static constexpr int ESZ = kFmt == 1 ? 2 : 4;
  static constexpr int BK = 128 / ESZ;          // elements per K-block (one 128-B swizzle row)
  static constexpr int UK = 32 / ESZ;           // K per tcgen05.mma (16 bf16 / 8 tf32) = 32 bytes
  static constexpr int NOPS = kSplit == 3 ? 2 : 1;
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = NOPS * (A_BYTES + B_BYTES);
  static constexpr int STAGES = kSplit == 3 ? 2 : 4;
  static constexpr int TMEM_COLS = 512;
  static constexpr size_t SMEM_BYTES = 1024 /*align slack*/ + (size_t)STAGES * STAGE_BYTES + 256 /*barriers*/;
  static constexpr uint32_t IDESC = ptx::idesc_f32acc(kFmt, BM, BN);
};

// Tile scheduler.  Rectangular: row tiles [row_tile0, row_tile1) × all column tiles.
// Triangular (tri = 1): row tile I covers rows [128 I, 128 I + 128) and needs the column tiles
// J ≥ floor(I/2) (tile columns are 256 wide), i.e. every tile holding some entry j ≥ i.
struct Sched {
  int tri;
  int tiles_n;
  int row_tile0, row_tile1;
  int num_tiles;

  // Σ_{r < I} floor(r/2)
  __host__ __device__ static long long half_sum(long long I) {
    long long q = I >> 1;
    return (I & 1) ? q * q : q * (q - 1);
  }
  __host__ __device__ long long prefix(long long I) const {  // tiles in rows [0, I)
    return I * (long long)tiles_n - half_sum(I);
  }
  __host__ __device__ void tile(int t, int& ti, int& tj) const {
    if (!tri) {
      ti = row_tile0 + t / tiles_n;
      tj = t % tiles_n;
      return;
    }
    const long long base = prefix(row_tile0);
    long long target = base + t;
    int lo = row_tile0, hi = row_tile1 - 1;   // largest I with prefix(I) <= target
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (prefix(mid) <= target) lo = mid; else hi = mid - 1;
    }
    ti = lo;
    tj = (lo >> 1) + (int)(target - prefix(lo));
  }
  static Sched rect(int row_tile0, int row_tile1, int tiles_n) {
    Sched s;
    s.tri = 0; s.tiles_n = tiles_n; s.row_tile0 = row_tile0; s.row_tile1 = row_tile1;
    s.num_tiles = (row_tile1 - row_tile0) * tiles_n;
    return s;
  }
  static Sched triangle(int row_tile0, int row_tile1, int tiles_n) {
    Sched s;
    s.tri = 1; s.tiles_n = tiles_n; s.row_tile0 = row_tile0; s.row_tile1 = row_tile1;
    s.num_tiles = (int)(s.prefix(row_tile1) - s.prefix(row_tile0));
    return s;
  }
};

// ------------------------------------------------------------------------------------------
// Epilogues.  operator()(row, col0, r[32]) receives row `row` (global) and accumulator columns
// [col0, col0+32) as raw fp32 bits; `chunk_needed(row_lo, row_hi, col0)` lets triangular epilogues
// skip 32-column chunks entirely below the diagonal for the warp's 32 rows (warp-uniform).
// ------------------------------------------------------------------------------------------

// K3: Σᵀ[i][k] = σ(z), z = x_iᵀw_k.  kOut: 0 = bf16, 1 = fp32, 2 = fp32 hi/lo split (3×TF32).
template <int kOut>
struct EpiSigma {
  void* out0;
  void* out1;
  int64_t ld;       // elements
  int64_t M, N;     // n rows (samples), m_local columns (features)
  int act;
  __device__ __forceinline__ bool chunk_needed(int64_t, int64_t, int64_t col0) const { return col0 < N; }
  __device__ __forceinline__ void operator()(int64_t row, int64_t col0, const uint32_t (&r)[32]) const {
    if (row >= M) return;
    float s[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) s[e] = act_f32(act, __uint_as_float(r[e]));
    const bool full = col0 + 32 <= N;
    if (kOut == 0) {
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(out0) + row * ld + col0;
      if (full) {
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint32_t w[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(s[v * 8 + 2 * h], s[v * 8 + 2 * h + 1]);
            w[h] = *reinterpret_cast<uint32_t*>(&b2);
          }
          d4[v] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      } else {
        for (int e = 0; e < 32; ++e)
          if (col0 + e < N) dst[e] = __float2bfloat16_rn(s[e]);
      }
    } else {
      float* d0 = reinterpret_cast<float*>(out0) + row * ld + col0;
      float* d1 = kOut == 2 ? reinterpret_cast<float*>(out1) + row * ld + col0 : nullptr;
      if (full) {
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          float4 a = make_float4(s[4 * v], s[4 * v + 1], s[4 * v + 2], s[4 * v + 3]);
          if (kOut == 2) {
            float4 h = make_float4(tf32_hi(a.x), tf32_hi(a.y), tf32_hi(a.z), tf32_hi(a.w));
            float4 l = make_float4(a.x - h.x, a.y - h.y, a.z - h.z, a.w - h.w);
            reinterpret_cast<float4*>(d0)[v] = h;
            reinterpret_cast<float4*>(d1)[v] = l;
          } else {
            reinterpret_cast<float4*>(d0)[v] = a;
          }
        }
      } else {
        for (int e = 0; e < 32; ++e) {
          if (col0 + e < N) {
            if (kOut == 2) {
              float h = tf32_hi(s[e]);
              d0[e] = h;
              d1[e] = s[e] - h;
            } else {
              d0[e] = s[e];
            }
          }
        }
      }
    }
  }
};

// K4: G[i][j] = scale · Σᵀ_iᵀΣᵀ_j for j ≥ i (and the mirror for FULL).
struct EpiSyrk {
  float* G;
  int64_t ld, n;
  float scale;
  int full;
  __device__ __forceinline__ bool chunk_needed(int64_t row_lo, int64_t, int64_t col0) const {
    return col0 < n && col0 + 31 >= row_lo;
  }
  __device__ __forceinline__ void operator()(int64_t row, int64_t col0, const uint32_t (&r)[32]) const {
    if (row >= n) return;
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]) * scale;
    float* dst = G + row * ld + col0;
    if (col0 >= row && col0 + 32 <= n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(dst)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (col0 + e >= row && col0 + e < n) dst[e] = v[e];
    }
    if (full) {
      // mirror: for fixed e the warp's 32 lanes write 32 consecutive floats of row col0+e (coalesced)
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (col0 + e > row && col0 + e < n) G[(col0 + e) * ld + row] = v[e];
    }
  }
};

// K5: Φ[i][j] = EQ1 with x_i as pivot (DESIGN.md §4 R6), j ≥ i.
struct EpiEq1 {
  float* Phi;
  int64_t ld, n;
  const RowCoef* rc;     // per row
  const float* nrm2;     // ‖x_j‖² per column
  float k00, k11, k22h, k01, k12, inv_st;
  int full;
  __device__ __forceinline__ bool chunk_needed(int64_t row_lo, int64_t, int64_t col0) const {
    return col0 < n && col0 + 31 >= row_lo;
  }
  __device__ __forceinline__ void operator()(int64_t row, int64_t col0, const uint32_t (&r)[32]) const {
    if (row >= n) return;
    const RowCoef c = rc[row];
    float v[32];
    float nj[32];
    if (col0 + 32 <= n) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 t = __ldg(reinterpret_cast<const float4*>(nrm2 + col0) + q);
        nj[4 * q] = t.x; nj[4 * q + 1] = t.y; nj[4 * q + 2] = t.z; nj[4 * q + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) nj[e] = (col0 + e < n) ? __ldg(nrm2 + col0 + e) : 1.f;
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const float g = __uint_as_float(r[e]);
      v[e] = eq1_entry<float>(g, c.a0, c.a1, c.a2h, c.c, c.inv_ua, nj[e], col0 + e == row, c.nu_diag, k00, k11,
                              k22h, k01, k12, inv_st);
    }
    float* dst = Phi + row * ld + col0;
    if (col0 >= row && col0 + 32 <= n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(dst)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (col0 + e >= row && col0 + e < n) dst[e] = v[e];
    }
    if (full) {
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (col0 + e > row && col0 + e < n) Phi[(col0 + e) * ld + row] = v[e];
    }
  }
};

// ------------------------------------------------------------------------------------------
// The kernel.
// ------------------------------------------------------------------------------------------
template <class Cfg, class Epi>
__global__ void __launch_bounds__(256, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA_lo, const __grid_constant__ CUtensorMap tmB_lo,
                   const Sched sched, const int num_kb, const Epi epi) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  constexpr int STAGES = Cfg::STAGES, NOPS = Cfg::NOPS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                             // [STAGES][NOPS][A_BYTES]
  uint8_t* sB = smem + (size_t)STAGES * NOPS * Cfg::A_BYTES;       // [STAGES][NOPS][B_BYTES]
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)STAGES * NOPS * Cfg::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if (NOPS == 2) {
      ptx::prefetch_tmap(&tmA_lo);
      ptx::prefetch_tmap(&tmB_lo);
    }
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 4);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol = ptx::policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < sched.num_tiles; t += gridDim.x) {
        int ti, tj;
        sched.tile(t, ti, tj);
        const int ra = ti * Cfg::BM, rb = tj * Cfg::BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          const int k = kb * Cfg::BK;
          uint8_t* a = sA + (size_t)(stage * NOPS) * Cfg::A_BYTES;
          uint8_t* b = sB + (size_t)(stage * NOPS) * Cfg::B_BYTES;
          ptx::tma_load_2d(a, &tmA, &full[stage], k, ra, pol);
          ptx::tma_load_2d(b, &tmB, &full[stage], k, rb, pol);
          if (NOPS == 2) {
            ptx::tma_load_2d(a + Cfg::A_BYTES, &tmA_lo, &full[stage], k, ra, pol);
            ptx::tma_load_2d(b + Cfg::B_BYTES, &tmB_lo, &full[stage], k, rb, pol);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer (single thread) =====
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < sched.num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + acc * Cfg::BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint8_t* a = sA + (size_t)(stage * NOPS) * Cfg::A_BYTES;
          const uint8_t* b = sB + (size_t)(stage * NOPS) * Cfg::B_BYTES;
          const uint64_t ad = ptx::sdesc_k128(ptx::smem_u32(a));
          const uint64_t bd = ptx::sdesc_k128(ptx::smem_u32(b));
#pragma unroll
          for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
            const uint64_t off = (uint64_t)((k * 32) >> 4);   // +32 B along K inside the swizzle row
            const uint32_t accum = (kb | k) != 0;
            if (NOPS == 2) {
              const uint64_t adl = ptx::sdesc_k128(ptx::smem_u32(a + Cfg::A_BYTES));
              const uint64_t bdl = ptx::sdesc_k128(ptx::smem_u32(b + Cfg::B_BYTES));
              ptx::mma_tf32(d, adl + off, bd + off, Cfg::IDESC, accum);
              ptx::mma_tf32(d, ad + off, bdl + off, Cfg::IDESC, 1u);
              ptx::mma_tf32(d, ad + off, bd + off, Cfg::IDESC, 1u);
            } else if (Cfg::ESZ == 2) {
              ptx::mma_bf16(d, ad + off, bd + off, Cfg::IDESC, accum);
            } else {
              ptx::mma_tf32(d, ad + off, bd + off, Cfg::IDESC, accum);
            }
          }
          ptx::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ===== Epilogue: TMEM → registers → fused op → global =====
    const uint32_t q = warp - 4;   // == warp % 4: TMEM lane quarter this warp may access
    int it = 0;
    for (int t = blockIdx.x; t < sched.num_tiles; t += gridDim.x, ++it) {
      int ti, tj;
      sched.tile(t, ti, tj);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int64_t row_lo = (int64_t)ti * Cfg::BM + q * 32;
      const int64_t row = row_lo + lane;
#pragma unroll 1
      for (int c = 0; c < Cfg::BN / 32; ++c) {
        const int64_t col0 = (int64_t)tj * Cfg::BN + c * 32;
        if (!epi.chunk_needed(row_lo, row_lo + 31, col0)) continue;
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * Cfg::BN + c * 32, r);
        ptx::tmem_ld_wait();
        epi(row, col0, r);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
#endif
}

}  // namespace rfk
