// Part of the single translation unit api.cu: includes, error and tracing helpers, device queries, TMA
// descriptors, launch helpers, workspace plans and the host-side launchers shared by the ABI entry points.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rf.h"
#include "k_aux.cuh"
#include "k_center.cuh"
#include "k_comm.cuh"
#include "k_simt.cuh"
#include "k_ridge.cuh"
#include "rf_common.cuh"
#include "tc_gemm.cuh"

// The context (include/rf.h): device, options, the hybrids' side stream, and the G5 exchange resources.
struct rf_ctx {
  int device = 0;
  int64_t opts[RF_OPT_COUNT];
  cudaStream_t side = nullptr;            // concurrent tail kernel of the K3 / K4 multicast + pair hybrids
  // collective (G5)
  int rank = 0, world = 1, mode = 0;      // mode: 0 none, 1 NCCL, 2 peers
  uint32_t epoch = 0;                     // collective rf_gram calls made on this context
  // NCCL
  void* comm = nullptr;
  bool own_comm = false;
  cudaStream_t comm_stream = nullptr;
  uint32_t* sync = nullptr;               // device: per-chunk counters of finished K4 (pair tile, epilogue warp)s,
                                          // monotone across calls (NCCL and peers)
  uint32_t sync_target[rfk::kMaxChunks] = {};   // host: the counter values the calls so far reach (wrap-safe GEQ)
  cudaEvent_t ev_start = nullptr, ev_done = nullptr, ev_sig = nullptr;
  bool comm_pending = false;              // ev_done recorded by an earlier call (its reduce-scatters read the send buffer)
  // peers: comm_stream sends chunk c's arrival flags once the chunk counter says its stores are done; red_stream sums
  // chunk c once every source's flag for it is up — both overlap the rest of K4
  cudaStream_t red_stream = nullptr;
  // peers: [world × recv_cap floats][flags: arrived[kMaxChunks][RF_MAX_PEERS], freed[RF_MAX_PEERS]] in one cudaMalloc
  void* stage = nullptr;
  size_t stage_bytes = 0;
  int64_t recv_cap = 0;
  float* peer[RF_MAX_PEERS] = {};
  uint32_t* peer_flags[RF_MAX_PEERS] = {};
  void* opened[RF_MAX_PEERS] = {};
  bool connected = false;
};

namespace rfh {
int compute_moments(rf_act act, double tau, int nodes, rf_moments_t* out);
// parametrised Table-2 activations (moments.cpp): id ≥ RF_ACT_PARAM_BASE → kind 1 (leaky ReLU) / 2 (quadratic)
int register_param_act(int kind, const double a[3]);
bool param_act(int id, int* kind, double a[3]);
int solve_ternary_thresholds(double d1, double d2, double tau, int sign2, double* s_minus, double* s_plus,
                             double* resid);
}

namespace {

thread_local std::string g_err;
thread_local int32_t g_launches = 0;

rf_status fail(rf_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}
rf_status ok() {
  g_err.clear();
  return RF_OK;
}

#define RF_CUDA_CHECK(expr)                                                                     \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess) return fail(RF_E_CUDA, "%s: %s (%s)", #expr, cudaGetErrorName(_e),   \
                                       cudaGetErrorString(_e));                                 \
  } while (0)

// ---------------------------------------------------------------- launch tracing (rf_profile_*)
// When enabled, every kernel launch is bracketed by two CUDA events recorded on its stream; the
// records are read back (and the events recycled) by rf_profile_read.
struct ProfRec {
  char name[32];
  cudaEvent_t a, b;
};
std::mutex g_pmu;
bool g_prof_on = false;
std::vector<ProfRec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t pool_get() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  bool on = false;
  ProfRec r{};
  cudaStream_t st;
  ProfScope(const char* name, cudaStream_t s) : st(s) {
    std::lock_guard<std::mutex> lk(g_pmu);
    if (!g_prof_on) return;
    on = true;
    std::snprintf(r.name, sizeof(r.name), "%s", name);
    r.a = pool_get();
    r.b = pool_get();
    cudaEventRecord(r.a, st);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(r.b, st);
    std::lock_guard<std::mutex> lk(g_pmu);
    g_recs.push_back(r);
  }
};

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
inline size_t align256(size_t a) { return (a + 255) & ~size_t(255); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

size_t esize_of(rf_prec prec) {
  switch (prec) {
    case RF_PREC_FP64: return 8;
    case RF_PREC_BF16: return 2;
    default: return 4;
  }
}
const char* prec_name(rf_prec p) {
  switch (p) {
    case RF_PREC_FP64: return "FP64";
    case RF_PREC_FP32: return "FP32";
    case RF_PREC_3XTF32: return "3XTF32";
    case RF_PREC_TF32: return "TF32";
    case RF_PREC_BF16: return "BF16";
  }
  return "?";
}
bool valid_prec(int p) { return p >= RF_PREC_FP64 && p <= RF_PREC_BF16; }
bool valid_act(int a) {
  int kind;
  double p[3];
  return (a >= RF_ACT_TANH && a <= RF_ACT_BUMP) || rfh::param_act(a, &kind, p);
}
// device-side description of σ for the runtime-σ epilogues (kind 0: a fixed rf_act)
rfk::ActRt act_rt(int a) {
  rfk::ActRt r{0, 0.0, 0.0, 0.0};
  double p[3];
  int kind = 0;
  if (rfh::param_act(a, &kind, p)) {
    r.kind = kind;
    r.a0 = p[0];
    r.a1 = p[1];
    r.a2 = p[2];
  }
  return r;
}
bool valid_out(int o) { return o >= RF_OUT_UPPER && o <= RF_OUT_PACKED_TILES; }
int64_t tri_tiles(int64_t n) {
  const int64_t T = (n + 255) / 256;
  return T * (T + 1) / 2;
}
// RF_OUT_PACKED_TRI: validation of the packed buffer + its TMA view ((tiles·256) × 256 rows of 256 floats)
rf_status packed_out_setup(const char* fn, const void* ptr, int64_t n, rf_prec prec, int64_t* tri_T) {
  if (prec == RF_PREC_FP64 || prec == RF_PREC_FP32)
    return fail(RF_E_INVALID, "%s: RF_OUT_PACKED_TRI needs a tensor-core precision (BF16, TF32, 3XTF32)", fn);
  if (!ptr) return fail(RF_E_INVALID, "%s: output is NULL", fn);
  if (reinterpret_cast<uintptr_t>(ptr) & 15) return fail(RF_E_INVALID, "%s: packed output is not 16-byte aligned", fn);
  *tri_T = (n + 255) / 256;
  return RF_OK;
}

// ---------------------------------------------------------------- device / driver
struct DevInfo {
  int sms = 0;
  int major = 0, minor = 0;
};
DevInfo dev_info(int dev) {
  static std::mutex mu;
  static DevInfo cache[64];
  static bool have[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && have[dev]) return cache[dev];
  DevInfo d;
  cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (dev >= 0 && dev < 64) {
    cache[dev] = d;
    have[dev] = true;
  }
  return d;
}

rf_status check_device(DevInfo* out) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(RF_E_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  DevInfo d = dev_info(dev);
  if (d.major != 10 || d.minor != 0)
    return fail(RF_E_UNSUPPORTED, "device %d is sm_%d%d; this library runs only on sm_100 (B200)", dev, d.major,
                d.minor);
  if (out) *out = d;
  return RF_OK;
}

typedef CUresult (*PFN_encode_tiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encode_tiled encode_fn() {
  static PFN_encode_tiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encode_tiled>(p);
  });
  return fn;
}

// Row-major matrix rows × kext (ld elements), box box_rows × (128 B of K), 128-B swizzle, OOB → 0.
// es: element size in bytes (1 = fp8 codes as UINT8, 2 = bf16, 4 = fp32).
rf_status make_tmap_es(CUtensorMap* m, const void* ptr, int es, int64_t rows, int64_t kext, int64_t ld,
                       int box_rows) {
  PFN_encode_tiled enc = encode_fn();
  if (!enc) return fail(RF_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)kext, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / es), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                         : (es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  CUresult r = enc(m, dt, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(RF_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return RF_OK;
}
rf_status make_tmap(CUtensorMap* m, const void* ptr, bool bf16, int64_t rows, int64_t kext, int64_t ld,
                    int box_rows) {
  return make_tmap_es(m, ptr, bf16 ? 2 : 4, rows, kext, ld, box_rows);
}

// fp32 n_rows × n_cols output map for the epilogue's TMA stores: box 32 × 32, 128-B swizzle (half: box 16 × 32,
// 64-B swizzle — the 2-KB staging buffers of EpiCtx<…, kHalf>).
// Returns false (no error) when the rows are not 16-B aligned; the epilogue then stores directly.
bool make_tmap_out(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, bool half = false) {
  PFN_encode_tiled enc = encode_fn();
  if (!enc || (reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * 4) % 16)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {half ? 16u : 32u, 32};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, half ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- context and options (include/rf.h)
constexpr int64_t kOptDefault[RF_OPT_COUNT] = {1, 1, 0, 111, 120, 24, 8, -1, 0, 4, 0, 8, 0, 3, 1, 1, 1, 1};
thread_local rf_ctx* g_ctx = nullptr;     // the context of the call in progress on this thread
int64_t opt(rf_opt o) { return g_ctx ? g_ctx->opts[o] : kOptDefault[o]; }

rf_status ctx_init(rf_ctx* c, int device) {
  c->device = device;
  for (int i = 0; i < RF_OPT_COUNT; ++i) c->opts[i] = kOptDefault[i];
  int prev = 0;
  RF_CUDA_CHECK(cudaGetDevice(&prev));
  RF_CUDA_CHECK(cudaSetDevice(device));
  cudaError_t e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(RF_E_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
  return RF_OK;
}

// This thread's default context of `device` (ctx = NULL in a call): per thread, so unrelated threads never share a
// side stream.
rf_ctx* default_ctx(int device) {
  static thread_local rf_ctx* dflt[64] = {};
  if (device < 0 || device >= 64) return nullptr;
  if (!dflt[device]) {
    int major = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    rf_ctx* c = new rf_ctx();
    if (ctx_init(c, device) != RF_OK) {
      delete c;
      return nullptr;
    }
    dflt[device] = c;
  }
  return dflt[device];
}

// Entry guard of every compute call: resolves NULL to the default context, makes the context's device current for
// the call (restored on exit) and publishes the options to the launchers.
struct CtxScope {
  rf_status status = RF_OK;
  rf_ctx* prev = nullptr;
  int prev_dev = -1;
  explicit CtxScope(rf_ctx* c) {
    prev = g_ctx;
    g_ctx = nullptr;
    int dev = 0;
    if (!c) {
      // the default context; without a usable device the call runs its argument validation on the default options
      // and then fails in check_device (RF_E_CUDA / RF_E_UNSUPPORTED) — never a CPU fallback
      if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return;
      }
      c = default_ctx(dev);
      if (!c) return;
    } else if (cudaGetDevice(&dev) != cudaSuccess) {
      status = fail(RF_E_CUDA, "cudaGetDevice failed");
      return;
    }
    if (c->device != dev) {
      prev_dev = dev;
      if (cudaSetDevice(c->device) != cudaSuccess) {
        status = fail(RF_E_CUDA, "cudaSetDevice(%d) failed", c->device);
        return;
      }
    }
    g_ctx = c;
  }
  ~CtxScope() {
    g_ctx = prev;
    if (prev_dev >= 0) cudaSetDevice(prev_dev);
  }
};
#define RF_CTX_ENTER(ctx)            \
  CtxScope ctx_scope_(ctx);          \
  if (ctx_scope_.status) return ctx_scope_.status

// Row tiles per L2 raster group (tc_gemm.cuh Sched) of kernel K3, K4, K5 (measured best).
#ifndef K4_DYN_GM
#define K4_DYN_GM 4   // super rows (512) per raster group of the K4 unit queue (A/B builds: -DK4_DYN_GM=k)
#endif
int raster_gm(int def, int kernel = 0) {
  (void)kernel;
  return def;
}

template <class Cfg, class Epi>
rf_status launch_tc(const char* name, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& alo,
                    const CUtensorMap& blo, const CUtensorMap& out, const rfk::Sched& s, const Epi& epi, int sms,
                    cudaStream_t st) {
  if (s.num_tiles <= 0) return RF_OK;
  ProfScope ps(name, st);
  auto kern = rfk::tc_gemm_kernel<Cfg, Epi>;
  RF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM_BYTES));
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Cfg::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_cl = sms / Cfg::CL;
  if (Cfg::CL > 2) {   // clusters of 4 must fit inside a GPC: ask the occupancy calculator
    cfg.gridDim = dim3(Cfg::CL * max_cl);
    int q = 0;
    RF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    if (cudaOccupancyMaxActiveClusters(&q, kern, &cfg) == cudaSuccess && q > 0) max_cl = std::min(max_cl, q);
    cudaGetLastError();
  }
  const int clusters = std::max(1, std::min(s.num_tiles, max_cl));
  cfg.gridDim = dim3(Cfg::CL * clusters);
  if (opt(RF_OPT_VERBOSE))
    std::fprintf(stderr, "[rf] %s: %d clusters of %d CTAs (%d SMs), %d tiles\n", name, clusters, Cfg::CL,
                 clusters * Cfg::CL, s.num_tiles);
  RF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a, b, alo, blo, out, s, epi));
  ++g_launches;
  return RF_OK;
}

template <typename T, class Epi>
rf_status launch_simt(const char* name, const T* A, int64_t lda, const T* B, int64_t ldb, int64_t M, int64_t N,
                      int64_t K, int tri, int row_tile0, int row_tile1, const Epi& epi, cudaStream_t st, int zcount = 1,
                      int64_t zsA = 0, int64_t zsB = 0) {
  const int tn = (int)((N + rfk::kSimtTile - 1) / rfk::kSimtTile);
  if (row_tile1 <= row_tile0 || tn == 0) return RF_OK;
  ProfScope ps(name, st);
  dim3 grid(tn, row_tile1 - row_tile0, zcount);
  rfk::simt_gemm_nt<T, Epi><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, tri, row_tile0, epi, zsA, zsB);
  RF_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  return RF_OK;
}

rf_status launch_split(const float* src, int64_t lds, int64_t rows, int64_t cols, float* hi, float* lo, int64_t ldd,
                       int sms, cudaStream_t st) {
  const int64_t total = rows * cols;
  int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
  if (grid < 1) grid = 1;
  ProfScope ps("K2_split_tf32", st);
  rfk::k_split_tf32<<<grid, 256, 0, st>>>(src, lds, rows, cols, hi, lo, ldd);
  RF_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  return RF_OK;
}

rf_status launch_round_bf16(const float* src, int64_t lds, int64_t rows, int64_t cols, void* dst, int64_t ldd,
                            int sms, cudaStream_t st) {
  const bool vec = cols % 4 == 0 && lds % 4 == 0 && ldd % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) & 7) == 0;
  const int64_t total = rows * (vec ? cols / 4 : cols);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8));
  ProfScope ps("G1_round_bf16", st);
  if (vec)
    rfk::k_round_bf16<true><<<grid, 256, 0, st>>>(src, lds, rows, cols, (__nv_bfloat16*)dst, ldd);
  else
    rfk::k_round_bf16<false><<<grid, 256, 0, st>>>(src, lds, rows, cols, (__nv_bfloat16*)dst, ldd);
  RF_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  return RF_OK;
}

rf_status launch_rownorm(const void* X, rf_prec prec, int64_t ldx, int64_t p, int64_t n, double* nrm2,
                         cudaStream_t st) {
  const int grid = (int)((n + 7) / 8);
  ProfScope ps("K1_rownorm", st);
  if (prec == RF_PREC_FP64)
    rfk::k_rownorm<double><<<grid, 256, 0, st>>>((const double*)X, ldx, p, n, nrm2);
  else if (prec == RF_PREC_BF16)
    rfk::k_rownorm<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)X, ldx, p, n, nrm2);
  else
    rfk::k_rownorm<float><<<grid, 256, 0, st>>>((const float*)X, ldx, p, n, nrm2);
  RF_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  return RF_OK;
}

// ---------------------------------------------------------------- workspace plans
// Leading dimension (elements) whose row stride is an ODD number of 128-byte lines.  Σᵀ rows are read
// by TMA as 128-row × 128-B boxes at one K offset; with a power-of-two stride (m = 65536 bf16 → 128 KB)
// every row of a box, and every row of every box in flight, shares address bits [7, 17) and lands in
// the same L2 sets — measured on configs[3] K4: 1.2 TB of DRAM reads per launch for 8.6 GB of Σᵀ.
int64_t odd_line_ld(int64_t cols, int64_t es) {
  int64_t lines = (cols * es + 127) / 128;
  if ((lines & 1) == 0) ++lines;
  return lines * 128 / es;
}

struct GramPlan {
  int64_t ldS, ldp;
  size_t off_s0, off_s1, off_xhi, off_xlo, off_whi, off_wlo, off_prog, off_cen, total;
};
GramPlan gram_plan(int64_t p, int64_t n, int64_t m_local, rf_prec prec) {
  GramPlan g{};
  const size_t es = (prec == RF_PREC_FP64) ? 8 : (prec == RF_PREC_BF16 ? 2 : 4);
  g.ldS = odd_line_ld(std::max<int64_t>(m_local, 1), (int64_t)es);
  g.ldp = odd_line_ld(p, 4);
  size_t off = 0;
  g.off_s0 = off;
  off = align256(off + (size_t)n * g.ldS * es);
  g.off_s1 = off;
  if (prec == RF_PREC_3XTF32) {
    off = align256(off + (size_t)n * g.ldS * 4);
    g.off_xhi = off; off = align256(off + (size_t)n * g.ldp * 4);
    g.off_xlo = off; off = align256(off + (size_t)n * g.ldp * 4);
    g.off_whi = off; off = align256(off + (size_t)m_local * g.ldp * 4);
    g.off_wlo = off; off = align256(off + (size_t)m_local * g.ldp * 4);
  }
  g.off_prog = off; off = align256(off + 2048);      // K4 lockstep progress words, start flag, unit queue
  g.off_cen = off; off = align256(off + (size_t)(n + 2) * 8);   // centering row sums + s (NEXT-2)
  g.total = off;
  return g;
}

struct PhiPlan {
  int64_t ldp;
  size_t off_nrm2, off_tau, off_rc, off_nrm2o, off_xhi, off_xlo, off_cen, off_queue, total;
};
PhiPlan phi_plan(int64_t p, int64_t n, rf_prec prec) {
  PhiPlan g{};
  g.ldp = odd_line_ld(p, 4);
  size_t off = 0;
  g.off_nrm2 = off; off = align256(off + (size_t)n * 8);
  g.off_tau = off; off = align256(off + 16);
  g.off_rc = off; off = align256(off + (size_t)n * (prec == RF_PREC_FP64 ? sizeof(rfk::RowCoefD) : sizeof(rfk::RowCoef)));
  g.off_nrm2o = off; off = align256(off + (size_t)round_up(n, 256) * 8);   // ‖x_j‖²/τ, padded to whole tiles (K5)
  if (prec == RF_PREC_3XTF32) {
    g.off_xhi = off; off = align256(off + (size_t)n * g.ldp * 4);
    g.off_xlo = off; off = align256(off + (size_t)n * g.ldp * 4);
  }
  g.off_cen = off; off = align256(off + (size_t)(n + 2) * 8);
  g.off_queue = off; off = align256(off + 4);   // K5's dynamic segment counter (A residency)
  g.total = off;
  return g;
}

struct GramTcArgs {
  const void* X; int64_t ldx; const void* W; int64_t ldw;
  int64_t p, n, m_local, m_total;
  rf_act act; int full; float* G; int64_t ldg;
  char* w; GramPlan pl; int sms; cudaStream_t st;
  const rfk::PackDev* pack;   // non-null: K4 writes the G5 packed tiles (send buffer or the owners' staging buffers)
  int64_t tri_T = 0;          // > 0: RF_OUT_PACKED_TRI (G is the packed triangle)
};

constexpr int kPackGm = 8;  // row tiles per G5 chunk group (chunks are runs of 8-row-tile groups, rf_tile_map)

// Hybrid K4 (bf16 / tf32 / fp8 SYRK, 256×512 pair tiles): 4-CTA clusters with B multicast on the first super
// rows and, concurrently on a second stream, pair clusters on the remaining row tiles.  Clusters of 4 must sit in
// one GPC, so only 33 fit (132 SMs); the pair kernel takes the 16 SMs left over.  The pair kernel is released
// only after the multicast kernel has started (a flag its first CTA writes, awaited by a stream-memory wait), so
// the multicast kernel always gets its clusters.  The work split follows the per-SM rates measured for the two
// kernels (f = 0.90 at 33 clusters; a ±2 % change costs 2–18 %).  prog: 1 KB of zeroed-per-call progress words.
typedef CUresult (*PFN_wait32h)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_wait32h wait32_h() {
  static PFN_wait32h fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_wait32h>(p);
  });
  return fn;
}
// The call's context owns the side stream (one per context: separate contexts never couple their streams).
static cudaStream_t side_stream() { return g_ctx ? g_ctx->side : nullptr; }

// How many 4-CTA clusters of kernel <Cm, Epi> can be co-resident (clusters must sit inside one GPC).
template <class Cm, class Epi>
rf_status max_clusters(int sms, int* mcl) {
  *mcl = 0;
  auto kern = rfk::tc_gemm_kernel<Cm, Epi>;
  RF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cm::SMEM_BYTES));
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(Cm::THREADS);
  cfg.dynamicSmemBytes = Cm::SMEM_BYTES;
  cfg.gridDim = dim3((sms / Cm::CL) * Cm::CL);   // a whole number of clusters (148 is not a multiple of 8)
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Cm::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaOccupancyMaxActiveClusters(mcl, kern, &cfg) != cudaSuccess) *mcl = 0;
  cudaGetLastError();
  return RF_OK;
}

// Launch the multicast kernel <Cm> (schedule sm, 4·mcl SMs) on st and, concurrently on the side stream, the pair
// kernel <Cp> (schedule sp, tail_sms SMs) once the multicast kernel has started (sm.started = flag, zeroed by
// the caller on st before this call).  One trace record `name` brackets both (fork → join); the parts are traced
// as `name`_mc / `name`_tail.  tBm / tBp: the B-operand "lo" maps of the two kernels (the multicast kernel of
// 256-wide tiles reads B through a 64-row box).
template <class Cm, class Cp, class Epi>
rf_status launch_hybrid_pair(const char* name, const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tBm,
                             const CUtensorMap& tBp, const CUtensorMap& tO, const rfk::Sched& sm, const rfk::Sched& sp,
                             const Epi& e, uint32_t* flag, int mc_sms, int tail_sms, cudaStream_t st,
                             const CUtensorMap* tAm = nullptr) {
  PFN_wait32h wfn = wait32_h();
  cudaStream_t st2 = side_stream();
  rf_status s;
  ProfScope whole(name, st);
  char nm_mc[32], nm_tail[32];
  std::snprintf(nm_mc, sizeof(nm_mc), "%s_mc", name);
  std::snprintf(nm_tail, sizeof(nm_tail), "%s_tail", name);
  struct Events {   // released on every return path
    cudaEvent_t e[2] = {nullptr, nullptr};
    ~Events() {
      for (cudaEvent_t x : e)
        if (x) cudaEventDestroy(x);
    }
  } evs;
  RF_CUDA_CHECK(cudaEventCreateWithFlags(&evs.e[0], cudaEventDisableTiming));
  RF_CUDA_CHECK(cudaEventCreateWithFlags(&evs.e[1], cudaEventDisableTiming));
  cudaEvent_t ev0 = evs.e[0], ev1 = evs.e[1];
  RF_CUDA_CHECK(cudaEventRecord(ev0, st));   // inputs ready and the progress words / start flag zeroed
  if ((s = launch_tc<Cm>(nm_mc, tA, tB, tAm ? *tAm : tA, tBm, tO, sm, e, mc_sms, st))) return s;
  // the pair kernel: on the side stream, after ev0 and once the multicast kernel has started
  RF_CUDA_CHECK(cudaStreamWaitEvent(st2, ev0, 0));
  CUresult r = wfn((CUstream)st2, (CUdeviceptr)(uintptr_t)flag, 1u, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(RF_E_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  s = launch_tc<Cp>(nm_tail, tA, tB, tA, tBp, tO, sp, e, tail_sms, st2);
  RF_CUDA_CHECK(cudaEventRecord(ev1, st2));
  RF_CUDA_CHECK(cudaStreamWaitEvent(st, ev1, 0));
  return s;
}

template <int kFmt, int kMcCl, class Epi>
rf_status launch_k4_hybrid_cl(const char* name, const CUtensorMap& tS, const CUtensorMap& tSh, const CUtensorMap& tO,
                              int64_t n, int kb, const Epi& e, uint32_t* prog, int lockw, int lockks, int sms,
                              cudaStream_t st, bool* used) {
  *used = false;
  const int T = (int)((n + 255) / 256), T2 = (int)((n + 511) / 512);
  if (opt(RF_OPT_K4_HYBRID) == 0 || T < 64 || !wait32_h() || !side_stream()) return RF_OK;
  using Cm = rfk::TcCfg<kFmt, 1, 512, -1, kMcCl>;
  using Cp = rfk::TcCfg<kFmt, 1, 512>;
  int mcl = 0;
  rf_status s;
  if ((s = max_clusters<Cm, Epi>(sms, &mcl))) return s;
  const int left = sms - kMcCl * mcl;
  if (mcl <= 0 || left < 2) return RF_OK;
  // work share of the multicast kernel from the per-SM rate ratio r (measured ≈ 1.11: less L2 traffic per flop
  // buys clock under the power cap for bf16 and bandwidth for fp8); env RF_HYB_FPCT overrides
  const double rate = opt(RF_OPT_K4_SPLIT_R100) / 100.0;
  const double f = ((double)kMcCl * mcl * rate) / ((double)kMcCl * mcl * rate + (left & ~1));
  double total = 0;
  for (int I = 0; I < T; ++I) total += T2 - I / 2;
  double acc = 0;
  int S1 = 0;
  while (S1 < T2 && acc < f * total) {
    for (int I = 2 * S1; I < std::min(T, 2 * S1 + 2); ++I) acc += T2 - I / 2;
    ++S1;
  }
  if (2 * S1 >= T) return RF_OK;
  RF_CUDA_CHECK(cudaMemsetAsync(prog, 0, 2048, st));
  // multicast kernel: super rows of 512; CL 4 walks 512-wide column tiles, CL 8 1024-wide super columns
  rfk::Sched sm = kMcCl == 8 ? rfk::Sched::make(1, 512, 0, S1, (int)((n + 1023) / 1024), kb, 0, raster_gm(4, 4))
                             : rfk::Sched::make(1, 256, 0, S1, T2, kb, 0, raster_gm(4, 4));
  // tail raster: with 8 pair clusters in flight, groups of 4 row tiles × 2 column tiles re-read the fewest Σᵀ panels
  // (4·32 + 2·64 MB per 8 tiles vs 8·32 + 64 for groups of 8); measured ≈ 0.8 % on the whole K4 (scripts/gpu_tailgm.sh)
  rfk::Sched sp = rfk::Sched::make(1, 512, 2 * S1, T, T2, kb, 0, 4);
  if (kMcCl == 4 && opt(RF_OPT_K4_DYNAMIC)) {
    // Dynamic units (tc_gemm.cuh TileSeq): no static split — both kernels pull 512 × 512 units of ONE raster over the
    // whole triangle from a shared counter (prog[256]); the multicast cluster computes a unit with its two pairs,
    // a pair cluster as two 256 × 512 tiles.  The pair kernel's SMs follow the raster front (L2 reuse) and both
    // kernels end together whatever their per-SM rates on this box.
    sm = rfk::Sched::make(1, 256, 0, T2, T2, kb, 0, raster_gm(K4_DYN_GM, 4));
    sp = sm;
    sm.queue = sp.queue = prog + 256;
    sp.nsub = 2;
    sm.sub_rows = sp.sub_rows = T;
  }
  if (lockw > 0) {
    sm.prog = prog;
    sp.prog = prog + 128;
    sm.lock_w = sp.lock_w = lockw;
    sm.lock_ks = sp.lock_ks = lockks;
  }
  sm.started = prog + 255;
  // evict_last on the operand loads keeps the Σᵀ panel slices of a wave in L2 a little longer: 196.6 → 195.0 ms
  // over 6 interleaved pairs (5 of 6 faster; scripts/gpu_k4pol2.sh); evict_first on G's stores showed nothing
  sm.load_pol = sp.load_pol = 1;
  sm.store_pol = sp.store_pol = 0;
  if ((s = launch_hybrid_pair<Cm, Cp>(name, tS, tS, tS, tS, tO, sm, sp, e, prog + 255, sms, left & ~1, st, &tSh)))
    return s;
  *used = true;
  return RF_OK;
}

// Hybrid K4 with 4-CTA (B shared) or, RF_K4_CL8=1, 8-CTA clusters (2 × 2 pairs sharing both A and B).
template <int kFmt, class Epi>
rf_status launch_k4_hybrid(const char* name, const CUtensorMap& tS, const CUtensorMap& tSh, const CUtensorMap& tO,
                           int64_t n, int kb, const Epi& e, uint32_t* prog, int lockw, int lockks, int sms,
                           cudaStream_t st, bool* used) {
  if (opt(RF_OPT_K4_CL8))
    return launch_k4_hybrid_cl<kFmt, 8>(name, tS, tSh, tO, n, kb, e, prog, lockw, lockks, sms, st, used);
  return launch_k4_hybrid_cl<kFmt, 4>(name, tS, tSh, tO, n, kb, e, prog, lockw, lockks, sms, st, used);
}

// Hybrid K3 (bf16 / tf32 GEMM + σ, 256×256 pair tiles, rectangular): 4-CTA clusters that share each B tile (two
// 64-row halves, one loaded by each pair and multicast to both) on the first super rows, pair clusters on the
// rest on the SMs the GPC packing leaves.  K3 is L2 → SM bandwidth bound with 256-wide tiles (64 B per SM-clock at
// full rate against the ≈ 6.3 KB/clk chip limit); the multicast cuts that to 48 B (configs[3]: 9.57 → 7.97 ms on
// 132 SMs alone).
template <class Cm, class Cp, class Epi>
rf_status launch_k3_hybrid(const char* name, const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tBh,
                           int64_t n, int64_t m, int kb, const Epi& e, uint32_t* prog, int sms, cudaStream_t st,
                           bool* used) {
  *used = false;
  const int T = (int)((n + 255) / 256), T2 = (int)((n + 511) / 512), tn = (int)((m + 255) / 256);
  if (opt(RF_OPT_K3_HYBRID) == 0 || T < 32 || !wait32_h() || !side_stream()) return RF_OK;
  int mcl = 0;
  rf_status s;
  if ((s = max_clusters<Cm, Epi>(sms, &mcl))) return s;
  const int left = sms - 4 * mcl;
  if (mcl <= 0 || left < 2) return RF_OK;
  const double rate = opt(RF_OPT_K3_SPLIT_R100) / 100.0;   // per-SM rate, multicast vs pair kernel
  const double f = (4.0 * mcl * rate) / (4.0 * mcl * rate + (left & ~1));
  const int S1 = std::min(T2, (int)std::lround(f * T / 2.0));   // rows are uniform: split by row count
  if (S1 <= 0 || 2 * S1 >= T) return RF_OK;
  RF_CUDA_CHECK(cudaMemsetAsync(prog, 0, 1024, st));
  rfk::Sched sm = rfk::Sched::make(0, 256, 0, S1, tn, kb, 0, raster_gm(4, 3));
  rfk::Sched sp = rfk::Sched::make(0, 256, 2 * S1, T, tn, kb, 0, raster_gm(8, 3));
  // evict_last on the operand loads (X and W are re-read by every tile of a row / column): 8.04 → 6.94 ms
  // (5 interleaved pairs, scripts/gpu_k3pol.sh)
  sm.load_pol = sp.load_pol = 1;
  sm.started = prog + 255;
  if ((s = launch_hybrid_pair<Cm, Cp>(name, tA, tB, tBh, tA, tA, sm, sp, e, prog + 255, sms, left & ~1, st)))
    return s;
  *used = true;
  return RF_OK;
}

// kOut: Σ storage (0 bf16, 1 fp32, 2 fp32 hi/lo).  K3 always uses 256-wide pair tiles (σ epilogue
// overlapped via two TMEM slots); K4 uses kBN4 (512: one slot, a third less L2 traffic per flop than 256).
template <int kFmt, int kSplit, int kBN4, int kOut>
rf_status gram_tc(const GramTcArgs& g, int kchunk4) {
  if (kBN4 == 512) kchunk4 = 0;   // K-chunked accumulation needs the second TMEM slot (256-wide tiles only)
  using C3 = rfk::TcCfg<kFmt, kSplit, 256, 0>;     // K3 stores Σᵀ from registers: no staging buffers
  using C4 = rfk::TcCfg<kFmt, kSplit, kBN4>;
  const bool bf = kFmt == 1;
  rf_status s;
  CUtensorMap tA, tB, tAl, tBl, tO;
  void* S0 = g.w + g.pl.off_s0;
  void* S1 = g.w + g.pl.off_s1;
  const void* XA = g.X;
  const void* WB = g.W;
  int64_t ldxa = g.ldx, ldwb = g.ldw;
  if (kSplit == 3) {
    float* Xh = (float*)(g.w + g.pl.off_xhi);
    float* Xl = (float*)(g.w + g.pl.off_xlo);
    float* Wh = (float*)(g.w + g.pl.off_whi);
    float* Wl = (float*)(g.w + g.pl.off_wlo);
    if ((s = launch_split((const float*)g.X, g.ldx, g.n, g.p, Xh, Xl, g.pl.ldp, g.sms, g.st))) return s;
    if ((s = launch_split((const float*)g.W, g.ldw, g.m_local, g.p, Wh, Wl, g.pl.ldp, g.sms, g.st))) return s;
    if ((s = make_tmap(&tAl, Xl, false, g.n, g.p, g.pl.ldp, 128))) return s;
    if ((s = make_tmap(&tBl, Wl, false, g.m_local, g.p, g.pl.ldp, 128))) return s;
    XA = Xh; WB = Wh; ldxa = ldwb = g.pl.ldp;
  }
  if ((s = make_tmap(&tA, XA, bf, g.n, g.p, ldxa, 128))) return s;
  if ((s = make_tmap(&tB, WB, bf, g.m_local, g.p, ldwb, 128))) return s;
  if (kSplit != 3) { tAl = tA; tBl = tB; }
  const int kb3 = (int)((g.p + C3::BK - 1) / C3::BK);
  rfk::Sched s3 = rfk::Sched::make(0, 256, 0, (int)((g.n + 255) / 256), (int)((g.m_local + 255) / 256), kb3, 0,
                                   raster_gm(8, 3));
  s3.load_pol = 1;
  // K3 = the pair kernel, or (bf16 / tf32, large n) the multicast + pair hybrid (launch_k3_hybrid)
  auto run_k3 = [&](const auto& e3) -> rf_status {
    using E3 = std::decay_t<decltype(e3)>;
    if constexpr (kSplit == 1) {
      if (opt(RF_OPT_K3_HYBRID)) {
        using C3m = rfk::TcCfg<kFmt, kSplit, 256, 0, 4>;
        CUtensorMap tBh;   // W with a 64-row box: the multicast kernel's half B tiles
        rf_status r;
        if ((r = make_tmap(&tBh, WB, bf, g.m_local, g.p, ldwb, 64))) return r;
        bool used = false;
        if ((r = launch_k3_hybrid<C3m, C3, E3>("K3_gemm_sigma", tA, tB, tBh, g.n, g.m_local, kb3, e3,
                                               (uint32_t*)(g.w + g.pl.off_prog), g.sms, g.st, &used)))
          return r;
        if (used) return RF_OK;
      }
    }
    return launch_tc<C3>("K3_gemm_sigma", tA, tB, tAl, tBl, tA, s3, e3, g.sms, g.st);
  };
  if (g.act == RF_ACT_TANH) {
    s = run_k3(rfk::EpiSigma<kOut, RF_ACT_TANH>{S0, S1, g.pl.ldS, g.n, g.m_local, (int)g.act, act_rt(g.act)});
  } else if (g.act == RF_ACT_ERF) {
    s = run_k3(rfk::EpiSigma<kOut, RF_ACT_ERF>{S0, S1, g.pl.ldS, g.n, g.m_local, (int)g.act, act_rt(g.act)});
  } else if (g.act == RF_ACT_SIGMOID_HALF) {
    s = run_k3(rfk::EpiSigma<kOut, RF_ACT_SIGMOID_HALF>{S0, S1, g.pl.ldS, g.n, g.m_local, (int)g.act,
                                                        act_rt(g.act)});
  } else {   // NEXT-3 Table-2 activations: one instantiation, σ chosen at run time
    s = run_k3(rfk::EpiSigma<kOut, -1>{S0, S1, g.pl.ldS, g.n, g.m_local, (int)g.act, act_rt(g.act)});
  }
  if (s) return s;

  if ((s = make_tmap(&tA, S0, bf, g.n, g.m_local, g.pl.ldS, 128))) return s;
  tB = tA;
  if (kSplit == 3) {
    if ((s = make_tmap(&tAl, S1, false, g.n, g.m_local, g.pl.ldS, 128))) return s;
    tBl = tAl;
  } else {
    tAl = tA; tBl = tA;
  }
  const bool tma_out = g.tri_T > 0 ? make_tmap_out(&tO, g.G, tri_tiles(g.n) * 256, 256, 256)
                                   : make_tmap_out(&tO, g.G, g.n, g.n, g.ldg);
  if (!tma_out) tO = tA;
  const int kb4 = (int)((g.m_local + C4::BK - 1) / C4::BK);
  const rfk::Sched s4 =
      rfk::Sched::make(1, kBN4, 0, (int)((g.n + 255) / 256), (int)((g.n + kBN4 - 1) / kBN4), kb4, kchunk4,
                       raster_gm(8, 4));
  rfk::Sched s4l = s4;
  s4l.load_pol = 1;   // as the hybrid (evict_last operands)
  const int lockw = (int)opt(RF_OPT_LOCK_W);
  if (lockw > 0) {
    s4l.prog = (uint32_t*)(g.w + g.pl.off_prog);
    s4l.lock_w = lockw;
    s4l.lock_ks = std::max(1, (int)opt(RF_OPT_LOCK_KS));
    RF_CUDA_CHECK(cudaMemsetAsync(s4l.prog, 0, 1024, g.st));
  }
  if (g.pack) {   // G5: every upper 256-tile of the partial into its exchange slot (canonical ownership, no schedule index)
    // the NCCL chunk counters expect 2 CTAs × EPI_WARPS arrivals per pair tile (abi_ctx.cuh kPackArrivals)
    static_assert(C4::EPI_WARPS == 8, "kPackArrivals = 2 × 8 epilogue warps (the hybrid's kernels have 8 as well)");
    rfk::EpiSyrkPacked e4{(float)(1.0 / (double)g.m_total), *g.pack};
    if constexpr (kBN4 == 512 && kSplit == 1) {
      if (lockw > 0) {
        bool used = false;
        CUtensorMap tSh;
        if ((s = make_tmap(&tSh, S0, bf, g.n, g.m_local, g.pl.ldS, 64))) return s;
        if ((s = launch_k4_hybrid<kFmt>("K4_syrk_packed", tA, tSh, tA, g.n, kb4, e4, s4l.prog, lockw, s4l.lock_ks,
                                         g.sms, g.st, &used)))
          return s;
        if (used) return ok();
      }
    }
    if ((s = launch_tc<C4>("K4_syrk_packed", tA, tB, tAl, tBl, tA, s4l, e4, g.sms, g.st))) return s;
    return ok();
  }
  if constexpr (kBN4 == 512 && kSplit == 1) {
    if (lockw > 0) {
      rfk::EpiSyrk eh{g.G, g.ldg, g.n, (float)(1.0 / (double)g.m_total), g.full, tma_out ? 1 : 0, g.tri_T};
      bool used = false;
      CUtensorMap tSh;   // Σᵀ with a 64-row box (the 8-CTA multicast kernel's A halves)
      if ((s = make_tmap(&tSh, S0, bf, g.n, g.m_local, g.pl.ldS, 64))) return s;
      if ((s = launch_k4_hybrid<kFmt>("K4_syrk", tA, tSh, tO, g.n, kb4, eh, s4l.prog, lockw, s4l.lock_ks, g.sms, g.st,
                                       &used)))
        return s;
      if (used) return ok();
    }
  }
  rfk::EpiSyrk e4{g.G, g.ldg, g.n, (float)(1.0 / (double)g.m_total), g.full, tma_out ? 1 : 0, g.tri_T};
  if ((s = launch_tc<C4>("K4_syrk", tA, tB, tAl, tBl, tO, s4l, e4, g.sms, g.st))) return s;
  return ok();
}

rf_status gram_tc_dispatch(const GramTcArgs& ga, rf_prec prec) {
  if (prec == RF_PREC_BF16) return gram_tc<1, 1, 512, 0>(ga, 0);
  if (prec == RF_PREC_TF32) return gram_tc<2, 1, 512, 1>(ga, 0);
  // 3×TF32: chunks of RF_OPT_KCHUNK K-blocks (default 4 = 128 features) bound the truncating tensor-pipe
  // accumulation to ≈ 2.6e-6 relative (DESIGN.md §6 finding 4)
  return gram_tc<2, 3, 256, 2>(ga, (int)opt(RF_OPT_KCHUNK));
}

// SMs the tensor-core kernels may use (RF_OPT_MAX_SMS; CTA pairs need an even count)
int usable_sms(int sms) {
  const int64_t m = opt(RF_OPT_MAX_SMS);
  return m > 0 ? std::max(2, std::min(sms, (int)m) & ~1) : sms;
}

struct K5Args {
  const void* X; int64_t ldx, p, n; rf_prec prec;
  float* Phi; int64_t ldphi; int full;
  const rfk::RowCoef* rc; const float* nj;
  float e0, e1, e2, f0, f1;
  int64_t row_begin, row_end;
  char* w; PhiPlan pl; int sms; cudaStream_t st;
  int64_t tri_T;   // > 0: RF_OUT_PACKED_TRI
};

#ifndef K5_STG
#define K5_STG 2
#endif
// One K5 launch over row tiles [rt0, rt1) of the triangle (tA: X or its hi part; tAl: the lo part in 3×TF32).
template <class C, class E>
rf_status k5_go(const CUtensorMap& tA, const CUtensorMap& tAl, const CUtensorMap& tO, const E& e, int64_t p, int rt0,
                int rt1, int tn, int sms, cudaStream_t st) {
  rfk::Sched sc = rfk::Sched::make(1, 256, rt0, rt1, tn, (int)((p + C::BK - 1) / C::BK), 0, raster_gm(16, 5));
  sc.load_pol = 1;    // evict_last operands (X is re-read by every tile of a row / column)
  sc.store_pol = 1;   // evict_first on the streamed Φ stores
  return launch_tc<C>("K5_xtx_eq1", tA, tA, tAl, tAl, tO, sc, e, sms, st);
}

// K5 with A-panel residency (TcCfg kAres): segment schedule, column blocks of kSegLen tiles (tc_gemm.cuh Sched),
// segments pulled from a device counter in schedule order (TileSeq's unit ring): a segment holds up to 16 tiles
// (≈ 60 µs at configs[4]), so a static round-robin could leave a cluster one segment behind in the last wave —
// ≈ 5 % of a rank's launch at R = 8.
constexpr int kSegLen = 16;
template <class C, class E>
rf_status k5_go_ares(const CUtensorMap& tA, const CUtensorMap& tO, const E& e, int64_t p, int rt0, int rt1, int tn,
                     uint32_t* queue, int sms, cudaStream_t st) {
  rfk::Sched sc = rfk::Sched::make(1, 256, rt0, rt1, tn, (int)((p + C::BK - 1) / C::BK), 0, 1);
  sc.seg_len = kSegLen;
  sc.num_tiles = (int)sc.seg_prefix((tn + kSegLen - 1) / kSegLen);
  sc.load_pol = 1;
  sc.store_pol = 1;
  if (queue && opt(RF_OPT_K5_DYNAMIC)) {
    RF_CUDA_CHECK(cudaMemsetAsync(queue, 0, 4, st));
    sc.queue = queue;
  }
  return launch_tc<C>("K5_xtx_eq1", tA, tA, tA, tA, tO, sc, e, sms, st);
}

// Φ4+Φ5: tensor-core XᵀX with the EQ1 epilogue over the row range's triangle pair tiles (256 × 256)
template <bool kOdd>
rf_status launch_k5(const K5Args& a) {
  const void* X = a.X;
  const int64_t ldx = a.ldx, p = a.p, n = a.n, ldphi = a.ldphi, row_begin = a.row_begin, row_end = a.row_end;
  const rf_prec prec = a.prec;
  float* Phi = a.Phi;
  const int full = a.full;
  const rfk::RowCoef* rc = a.rc;
  const float* nj = a.nj;
  const float e0 = a.e0, e1 = a.e1, e2 = a.e2, f0 = a.f0, f1 = a.f1;
  char* w = a.w;
  const PhiPlan& pl = a.pl;
  cudaStream_t st = a.st;
  struct { int sms; } dev{a.sms};
  rf_status s;
  CUtensorMap tA, tAl, tO;
  const bool tma_out = (a.tri_T > 0 ? make_tmap_out(&tO, Phi, tri_tiles(n) * 256, 256, 256)
                                    : make_tmap_out(&tO, Phi, n, n, ldphi));
  rfk::EpiEq1<kOdd> e{Phi, ldphi, n, rc, nj, e0, e1, e2, f0, f1, full, tma_out ? 1 : 0, a.tri_T};
  const int rt0 = (int)(row_begin / 256), rt1 = (int)((row_end + 255) / 256), tn = (int)((n + 255) / 256);
  if (prec == RF_PREC_BF16 || prec == RF_PREC_TF32) {
    const bool bf = prec == RF_PREC_BF16;
    if ((s = make_tmap(&tA, X, bf, n, p, ldx, 128))) return s;
    if (!tma_out) tO = tA;
    // Short K (p ≤ 512): the EQ1 epilogue, latency-bound at two warps per SM sub-partition, sets the pace, and 16
    // epilogue warps (four per TMEM lane quarter; one 4-KB staging buffer each, which keeps five operand stages;
    // 96 registers) help: configs[4] 11.3 → 9.54 ms (12 warps: 9.94).  Long K: the MMA sets it and the 8-warp
    // kernel stays ahead (configs[3] shape, p = 1024: 3.63 vs 3.78 ms).  DESIGN.md §7.
    // Since the 8-warp kernel got its interior fast path (round 2) it is ahead at every p measured (configs[4]
    // without residency: bf16 11.1 vs 13.2 ms, TF32 16.7 vs 17.3 ms; profiles/r02/k5_fast/k5_wide_vs_8.log), so
    // auto (−1) means 8 warps; 1 keeps the 16-warp kernel as an option.
    const bool wide = opt(RF_OPT_K5_WIDE) > 0;
    // A-panel residency: K = p of 5 … 8 K-blocks (the producer may run at most STAGES = 4 K-blocks ahead of the MMA,
    // which keeps the aempty parity wait exact, tc_gemm.cuh)
    const int kb5 = (int)((p + 63) / 64);
    const int ares = (int)opt(RF_OPT_K5_ARES);
    if (bf && ares > 0 && kb5 > 4 && kb5 <= 8) {
      uint32_t* q5 = (uint32_t*)(w + a.pl.off_queue);
      if (ares == 2) {   // 2-KB staging buffers: the store map with 16 × 32 boxes and 64-B swizzle
        CUtensorMap tOh;
        const bool okh = a.tri_T > 0 ? make_tmap_out(&tOh, Phi, tri_tiles(n) * 256, 256, 256, true)
                                     : make_tmap_out(&tOh, Phi, n, n, ldphi, true);
        if (!okh) tOh = tA;
        if ((s = k5_go_ares<rfk::TcCfg<1, 1, 256, 1, 2, 16, 1>>(tA, tOh, e, p, rt0, rt1, tn, q5, dev.sms, st))) return s;
      } else if (ares == 3) {
        if ((s = k5_go_ares<rfk::TcCfg<1, 1, 256, 1, 2, 12, 1>>(tA, tO, e, p, rt0, rt1, tn, q5, dev.sms, st))) return s;
      } else if ((s = k5_go_ares<rfk::TcCfg<1, 1, 256, 1, 2, 8, 1>>(tA, tO, e, p, rt0, rt1, tn, q5, dev.sms, st))) {
        return s;
      }
    } else if (bf && wide) {
      if ((s = k5_go<rfk::TcCfg<1, 1, 256, 1, 2, 16>>(tA, tA, tO, e, p, rt0, rt1, tn, dev.sms, st))) return s;
    } else if (bf) {
      if ((s = k5_go<rfk::TcCfg<1, 1, 256, K5_STG>>(tA, tA, tO, e, p, rt0, rt1, tn, dev.sms, st))) return s;
    } else if (wide) {
      if ((s = k5_go<rfk::TcCfg<2, 1, 256, 1, 2, 16>>(tA, tA, tO, e, p, rt0, rt1, tn, dev.sms, st))) return s;
    } else {
      if ((s = k5_go<rfk::TcCfg<2, 1, 256, K5_STG>>(tA, tA, tO, e, p, rt0, rt1, tn, dev.sms, st))) return s;
    }
  } else {   // 3×TF32: never K-chunked (EQ1 is nonlinear in g); 8 warps keep three 64-KB operand stages
    float* Xh = (float*)(w + pl.off_xhi);
    float* Xl = (float*)(w + pl.off_xlo);
    if ((s = launch_split((const float*)X, ldx, n, p, Xh, Xl, pl.ldp, dev.sms, st))) return s;
    if ((s = make_tmap(&tA, Xh, false, n, p, pl.ldp, 128))) return s;
    if ((s = make_tmap(&tAl, Xl, false, n, p, pl.ldp, 128))) return s;
    if (!tma_out) tO = tA;
    if ((s = k5_go<rfk::TcCfg<2, 3, 256>>(tA, tAl, tO, e, p, rt0, rt1, tn, dev.sms, st))) return s;
  }
  return ok();
}

// NEXT-2: K = P·A·P in place for a symmetric n × n matrix stored in its upper triangle (FULL: all entries
// stored).  cen = (n + 2) doubles of workspace: r[0..n), s.
template <typename T>
rf_status center_pass(T* A, int64_t ld, int64_t n, int full, double* cen, cudaStream_t st) {
  double* r = cen;
  double* sp = cen + n;
  RF_CUDA_CHECK(cudaMemsetAsync(r, 0, (size_t)n * 8, st));
  const unsigned nt = (unsigned)((n + rfk::kCT - 1) / rfk::kCT);
  {
    ProfScope ps("KC_center_rowsum", st);
    rfk::k_center_rowsum<T><<<dim3(nt, nt), 256, 0, st>>>(A, ld, n, r);
    RF_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
  }
  {
    ProfScope ps("KC_center_scale", st);
    rfk::k_center_scale<<<1, 1024, 0, st>>>(r, n, sp);
    RF_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
  }
  {
    ProfScope ps("KC_center_apply", st);
    rfk::k_center_apply<T><<<dim3(nt, (unsigned)((n + 7) / 8)), 256, 0, st>>>(A, ld, n, r, sp, full);
    RF_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
  }
  return RF_OK;
}

rf_status validate_output(const char* name, const void* ptr, int64_t ld, int64_t cols, size_t es) {
  if (!ptr) return fail(RF_E_INVALID, "%s is NULL", name);
  if ((reinterpret_cast<uintptr_t>(ptr) % es) != 0) return fail(RF_E_INVALID, "%s is not %zu-byte aligned", name, es);
  if (ld < cols) return fail(RF_E_INVALID, "ld of %s (%lld) < %lld", name, (long long)ld, (long long)cols);
  return RF_OK;
}

rf_status validate_matrix(const char* name, const void* ptr, int64_t ld, int64_t cols, size_t es) {
  if (!ptr) return fail(RF_E_INVALID, "%s is NULL", name);
  if (!aligned16(ptr)) return fail(RF_E_INVALID, "%s is not 16-byte aligned", name);
  if (ld < cols) return fail(RF_E_INVALID, "ld of %s (%lld) < %lld", name, (long long)ld, (long long)cols);
  if ((ld * (int64_t)es) % 16 != 0)
    return fail(RF_E_INVALID, "ld of %s × element size (%lld B) is not a multiple of 16 B (TMA requirement)", name,
                (long long)(ld * (int64_t)es));
  return RF_OK;
}

}  // namespace
