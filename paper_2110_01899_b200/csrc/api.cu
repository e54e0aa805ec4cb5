// C ABI (include/rf.h): validation, workspace planning, TMA descriptor creation and kernel dispatch.
// Every compute step of the path runs in this library's kernels; there is no CPU fallback.
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
#include "k_simt.cuh"
#include "k_ridge.cuh"
#include "rf_common.cuh"
#include "tc_gemm.cuh"

namespace rfh {
int compute_moments(rf_act act, double tau, int nodes, rf_moments_t* out);
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
bool valid_act(int a) { return a >= RF_ACT_TANH && a <= RF_ACT_BUMP; }
bool valid_out(int o) { return o >= RF_OUT_UPPER && o <= RF_OUT_PACKED_TRI; }
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

// fp32 n_rows × n_cols output map for the epilogue's TMA stores: box 32 × 32, 128-B swizzle.
// Returns false (no error) when the rows are not 16-B aligned; the epilogue then stores directly.
bool make_tmap_out(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld) {
  PFN_encode_tiled enc = encode_fn();
  if (!enc || (reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * 4) % 16)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Row tiles per L2 raster group (tc_gemm.cuh Sched).  Env RF_GM<k> (kernel k = 3, 4, 5) or RF_GM overrides
// (experiments).
int raster_gm(int def, int kernel = 0) {
  char name[16];
  std::snprintf(name, sizeof(name), "RF_GM%d", kernel);
  const char* e = kernel ? std::getenv(name) : nullptr;
  if (!(e && *e && std::atoi(e) > 0)) e = std::getenv("RF_GM");
  if (e && *e && std::atoi(e) > 0) return std::atoi(e);
  return def;
}

int env_int(const char* name, int def) {
  const char* e = std::getenv(name);
  if (e && *e) return std::atoi(e);
  return def;
}

// K-blocks per accumulation chunk (0 = whole K in one chunk).  Env RF_KCHUNK overrides (experiments).
int kchunk_for(rf_prec prec, int def) {
  const char* e = std::getenv("RF_KCHUNK");
  if (e && *e) return std::atoi(e);
  (void)prec;
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
  if (env_int("RF_DEBUG_LAUNCH", 0))
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
  g.off_prog = off; off = align256(off + 1024);      // K4 lockstep progress words (≤ 256 clusters)
  g.off_cen = off; off = align256(off + (size_t)(n + 2) * 8);   // centering row sums + s (NEXT-2)
  g.total = off;
  return g;
}

struct PhiPlan {
  int64_t ldp;
  size_t off_nrm2, off_tau, off_rc, off_nrm2o, off_xhi, off_xlo, off_cen, total;
};
PhiPlan phi_plan(int64_t p, int64_t n, rf_prec prec) {
  PhiPlan g{};
  g.ldp = odd_line_ld(p, 4);
  size_t off = 0;
  g.off_nrm2 = off; off = align256(off + (size_t)n * 8);
  g.off_tau = off; off = align256(off + 16);
  g.off_rc = off; off = align256(off + (size_t)n * (prec == RF_PREC_FP64 ? sizeof(rfk::RowCoefD) : sizeof(rfk::RowCoef)));
  g.off_nrm2o = off; off = align256(off + (size_t)n * 8);
  if (prec == RF_PREC_3XTF32) {
    g.off_xhi = off; off = align256(off + (size_t)n * g.ldp * 4);
    g.off_xlo = off; off = align256(off + (size_t)n * g.ldp * 4);
  }
  g.off_cen = off; off = align256(off + (size_t)(n + 2) * 8);
  g.total = off;
  return g;
}

struct PackArgs {
  float* send;
  uint32_t* sync;
  const rfk::PackDev* dev;
  int world, nchunks;
};

struct GramTcArgs {
  const void* X; int64_t ldx; const void* W; int64_t ldw;
  int64_t p, n, m_local, m_total;
  rf_act act; int full; float* G; int64_t ldg;
  char* w; GramPlan pl; int sms; cudaStream_t st;
  const PackArgs* pack;     // non-null: K4 writes packed tiles (rf_gram_packed)
  int64_t tri_T = 0;        // > 0: RF_OUT_PACKED_TRI (G is the packed triangle)
};

constexpr int kPackGm = 8;  // raster group of rf_gram_packed's K4 (chunks are runs of groups)

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
static cudaStream_t side_stream() {
  static std::mutex mu;
  static cudaStream_t s[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && !s[dev]) cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking);
  return (dev >= 0 && dev < 64) ? s[dev] : nullptr;
}

// How many 4-CTA clusters of kernel <Cm, Epi> can be co-resident (clusters must sit inside one GPC).
template <class Cm, class Epi>
rf_status max_clusters(int sms, int* mcl) {
  *mcl = 0;
  auto kern = rfk::tc_gemm_kernel<Cm, Epi>;
  RF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cm::SMEM_BYTES));
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(Cm::THREADS);
  cfg.dynamicSmemBytes = Cm::SMEM_BYTES;
  cfg.gridDim = dim3(sms);
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
  if (env_int("RF_K4_HYBRID", 1) == 0 || T < 64 || !wait32_h() || !side_stream()) return RF_OK;
  using Cm = rfk::TcCfg<kFmt, 1, 512, -1, kMcCl>;
  using Cp = rfk::TcCfg<kFmt, 1, 512>;
  int mcl = 0;
  rf_status s;
  if ((s = max_clusters<Cm, Epi>(sms, &mcl))) return s;
  const int left = sms - kMcCl * mcl;
  if (mcl <= 0 || left < 2) return RF_OK;
  // work share of the multicast kernel from the per-SM rate ratio r (measured ≈ 1.11: less L2 traffic per flop
  // buys clock under the power cap for bf16 and bandwidth for fp8); env RF_HYB_FPCT overrides
  const double rate = env_int("RF_HYB_R100", 111) / 100.0;
  double f = ((double)kMcCl * mcl * rate) / ((double)kMcCl * mcl * rate + (left & ~1));
  if (env_int("RF_HYB_FPCT", 0) > 0) f = std::min(1.0, env_int("RF_HYB_FPCT", 0) / 100.0);
  double total = 0;
  for (int I = 0; I < T; ++I) total += T2 - I / 2;
  double acc = 0;
  int S1 = 0;
  while (S1 < T2 && acc < f * total) {
    for (int I = 2 * S1; I < std::min(T, 2 * S1 + 2); ++I) acc += T2 - I / 2;
    ++S1;
  }
  if (2 * S1 >= T) return RF_OK;
  RF_CUDA_CHECK(cudaMemsetAsync(prog, 0, 1024, st));
  // multicast kernel: super rows of 512; CL 4 walks 512-wide column tiles, CL 8 1024-wide super columns
  rfk::Sched sm = kMcCl == 8 ? rfk::Sched::make(1, 512, 0, S1, (int)((n + 1023) / 1024), kb, 0, raster_gm(4, 4))
                             : rfk::Sched::make(1, 256, 0, S1, T2, kb, 0, raster_gm(4, 4));
  // tail raster: with 8 pair clusters in flight, groups of 4 row tiles × 2 column tiles re-read the fewest Σᵀ panels
  // (4·32 + 2·64 MB per 8 tiles vs 8·32 + 64 for groups of 8); measured ≈ 0.8 % on the whole K4 (scripts/gpu_tailgm.sh)
  rfk::Sched sp = rfk::Sched::make(1, 512, 2 * S1, T, T2, kb, 0, env_int("RF_TAIL_GM", 4));
  if (lockw > 0) {
    sm.prog = prog;
    sp.prog = prog + 128;
    sm.lock_w = sp.lock_w = lockw;
    sm.lock_ks = sp.lock_ks = lockks;
  }
  sm.started = prog + 255;
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
  if (env_int("RF_K4_CL8", 0))
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
  if (env_int("RF_K3_HYBRID", 1) == 0 || T < 32 || !wait32_h() || !side_stream()) return RF_OK;
  int mcl = 0;
  rf_status s;
  if ((s = max_clusters<Cm, Epi>(sms, &mcl))) return s;
  const int left = sms - 4 * mcl;
  if (mcl <= 0 || left < 2) return RF_OK;
  const double rate = env_int("RF_HYB3_R100", 120) / 100.0;   // per-SM rate, multicast vs pair kernel
  const double f = (4.0 * mcl * rate) / (4.0 * mcl * rate + (left & ~1));
  const int S1 = std::min(T2, (int)std::lround(f * T / 2.0));   // rows are uniform: split by row count
  if (S1 <= 0 || 2 * S1 >= T) return RF_OK;
  RF_CUDA_CHECK(cudaMemsetAsync(prog, 0, 1024, st));
  rfk::Sched sm = rfk::Sched::make(0, 256, 0, S1, tn, kb, 0, raster_gm(4, 3));
  rfk::Sched sp = rfk::Sched::make(0, 256, 2 * S1, T, tn, kb, 0, raster_gm(8, 3));
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
  const rfk::Sched s3 = rfk::Sched::make(0, 256, 0, (int)((g.n + 255) / 256), (int)((g.m_local + 255) / 256), kb3, 0,
                                         raster_gm(8, 3));
  // K3 = the pair kernel, or (bf16 / tf32, large n) the multicast + pair hybrid (launch_k3_hybrid)
  auto run_k3 = [&](const auto& e3) -> rf_status {
    using E3 = std::decay_t<decltype(e3)>;
    if constexpr (kSplit == 1) {
      if (env_int("RF_K3_MC", 1)) {
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
    s = run_k3(rfk::EpiSigma<kOut, RF_ACT_TANH>{S0, S1, g.pl.ldS, g.n, g.m_local, (int)g.act});
  } else if (g.act == RF_ACT_ERF) {
    s = run_k3(rfk::EpiSigma<kOut, RF_ACT_ERF>{S0, S1, g.pl.ldS, g.n, g.m_local, (int)g.act});
  } else if (g.act == RF_ACT_SIGMOID_HALF) {
    s = run_k3(rfk::EpiSigma<kOut, RF_ACT_SIGMOID_HALF>{S0, S1, g.pl.ldS, g.n, g.m_local, (int)g.act});
  } else {   // NEXT-3 Table-2 activations: one instantiation, σ chosen at run time
    s = run_k3(rfk::EpiSigma<kOut, -1>{S0, S1, g.pl.ldS, g.n, g.m_local, (int)g.act});
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
  const int lockw = env_int("RF_LOCKW", 24);
  if (lockw > 0) {
    s4l.prog = (uint32_t*)(g.w + g.pl.off_prog);
    s4l.lock_w = lockw;
    s4l.lock_ks = std::max(1, env_int("RF_LOCKKS", 8));
    RF_CUDA_CHECK(cudaMemsetAsync(s4l.prog, 0, 1024, g.st));
  }
  if constexpr (kBN4 == 512 && kSplit == 1) {
  if (!g.pack && lockw > 0 && env_int("RF_K4_MC", 0) == 0) {
    rfk::EpiSyrk eh{g.G, g.ldg, g.n, (float)(1.0 / (double)g.m_total), g.full, tma_out ? 1 : 0, g.tri_T};
    bool used = false;
    CUtensorMap tSh;   // Σᵀ with a 64-row box (the 8-CTA multicast kernel's A halves)
    if ((s = make_tmap(&tSh, S0, bf, g.n, g.m_local, g.pl.ldS, 64))) return s;
    if ((s = launch_k4_hybrid<kFmt>("K4_syrk", tA, tSh, tO, g.n, kb4, eh, s4l.prog, lockw, s4l.lock_ks, g.sms, g.st,
                                     &used)))
      return s;
    if (used) return ok();
  }
  if (!g.pack && env_int("RF_K4_MC", 0)) {
    // 4-CTA clusters with B multicast: the scheduler walks 512-row super tiles (super-row I2 covers row tiles
    // 2·I2 and 2·I2 + 1; both need column tiles J ≥ I2 of width 512).
    using C4m = rfk::TcCfg<kFmt, kSplit, 512, -1, 4>;
    rfk::Sched sm = rfk::Sched::make(1, 256, 0, (int)((g.n + 511) / 512), (int)((g.n + 511) / 512), kb4, kchunk4,
                                     raster_gm(4, 4));
    sm.prog = s4l.prog;
    sm.lock_w = s4l.lock_w;
    sm.lock_ks = s4l.lock_ks;
    rfk::EpiSyrk em{g.G, g.ldg, g.n, (float)(1.0 / (double)g.m_total), g.full, tma_out ? 1 : 0, g.tri_T};
    if ((s = launch_tc<C4m>("K4_syrk", tA, tB, tAl, tBl, tO, sm, em, g.sms, g.st))) return s;
    return ok();
  }
  }
  if (g.pack) {
    rfk::Sched sp = rfk::Sched::make(1, kBN4, 0, (int)((g.n + 255) / 256), (int)((g.n + kBN4 - 1) / kBN4), kb4,
                                     kchunk4, kPackGm);
    sp.prog = s4l.prog;
    sp.lock_w = s4l.lock_w;
    sp.lock_ks = s4l.lock_ks;
    rfk::EpiSyrkPacked e4{g.pack->send, g.pack->sync, (float)(1.0 / (double)g.m_total), g.pack->world,
                          g.pack->nchunks, kBN4, *g.pack->dev};
    if ((s = launch_tc<C4>("K4_syrk_packed", tA, tB, tAl, tBl, tA, sp, e4, g.sms, g.st))) return s;
    return ok();
  }
  rfk::EpiSyrk e4{g.G, g.ldg, g.n, (float)(1.0 / (double)g.m_total), g.full, tma_out ? 1 : 0, g.tri_T};
  if ((s = launch_tc<C4>("K4_syrk", tA, tB, tAl, tBl, tO, s4l, e4, g.sms, g.st))) return s;
  return ok();
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
  sc.load_pol = env_int("RF_K5_LOADPOL", 1);
  sc.store_pol = env_int("RF_K5_STOREPOL", 1);
  return launch_tc<C>("K5_xtx_eq1", tA, tA, tAl, tAl, tO, sc, e, sms, st);
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
  const bool tma_out = a.tri_T > 0 ? make_tmap_out(&tO, Phi, tri_tiles(n) * 256, 256, 256)
                                   : make_tmap_out(&tO, Phi, n, n, ldphi);
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
    const bool wide = env_int("RF_K5_WIDE", p <= 512 ? 1 : 0) != 0;
    if (bf && wide) {
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

// =================================================================================================
extern "C" {

const char* rf_last_error(void) { return g_err.c_str(); }
const char* rf_version(void) { return "rf_b200 0.1 (sm_100a: tcgen05/TMA/TMEM; SIMT fp32/fp64)"; }

rf_status rf_packed_tri_elems(int64_t n, int64_t* elems) {
  if (!elems || n <= 0 || n > ((int64_t)1 << 31)) return fail(RF_E_INVALID, "rf_packed_tri_elems: need n in (0, 2^31]");
  *elems = tri_tiles(n) * 65536;
  return ok();
}
int32_t rf_last_launch_count(void) { return g_launches; }

rf_status rf_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_pmu);
  g_prof_on = on != 0;
  return ok();
}

rf_status rf_profile_read(int32_t max_records, char* names, float* ms, int32_t* count) {
  if (!count || (max_records > 0 && (!names || !ms))) return fail(RF_E_INVALID, "rf_profile_read: NULL output");
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_pmu);
    recs.swap(g_recs);
  }
  int32_t k = 0;
  rf_status st = RF_OK;
  for (auto& r : recs) {
    float t = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess && st == RF_OK) st = fail(RF_E_CUDA, "rf_profile_read: %s", cudaGetErrorString(e));
    if (k < max_records) {
      std::snprintf(names + 32 * k, 32, "%s", r.name);
      ms[k] = t;
    }
    ++k;
  }
  {
    std::lock_guard<std::mutex> lk(g_pmu);
    for (auto& r : recs) {
      g_pool.push_back(r.a);
      g_pool.push_back(r.b);
    }
  }
  *count = k;
  return st == RF_OK ? ok() : st;
}

int rf_device_supported(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    return 0;
  }
  DevInfo d = dev_info(device);
  return (d.major == 10 && d.minor == 0) ? 1 : 0;
}

rf_status rf_moments(rf_act act, double tau, int32_t nodes, rf_moments_t* out) {
  if (!out) return fail(RF_E_INVALID, "rf_moments: out is NULL");
  if (!valid_act(act)) return fail(RF_E_INVALID, "rf_moments: unknown activation %d", (int)act);
  if (!(tau > 0.0) || !std::isfinite(tau)) return fail(RF_E_INVALID, "rf_moments: tau must be finite and > 0");
  if (nodes < 0 || nodes == 1 || nodes > 1024) return fail(RF_E_INVALID, "rf_moments: nodes must be 0 or in [2, 1024]");
  int r = rfh::compute_moments(act, tau, nodes, out);
  if (r == 1) return fail(RF_E_NONFINITE, "rf_moments: sigma non-finite at a quadrature node");
  if (r == 2) return fail(RF_E_INVALID, "rf_moments: Golub-Welsch eigen-solver did not converge");
  return ok();
}

rf_status rf_tau_workspace_size(int64_t n, size_t* bytes) {
  if (!bytes) return fail(RF_E_INVALID, "bytes is NULL");
  if (n <= 0) return fail(RF_E_INVALID, "n must be > 0");
  *bytes = align256((size_t)n * 8) + 256;
  return ok();
}

// τ̂ (Lemma 1) reduced on the device and handed to the host through a mapped pinned mailbox: the kernel stores the
// two words over the host link itself and the host waits on an event, so the hand-off does not queue behind bulk
// copies on the copy engines (a 16-byte cudaMemcpyAsync would wait for any multi-GB D2H in flight).
struct HostMailbox {
  volatile double* h = nullptr;
  cudaEvent_t ev = nullptr;
  int dev = -1;
};
static thread_local HostMailbox t_mailbox;

static rf_status host_mailbox(HostMailbox** out) {
  int dev = 0;
  RF_CUDA_CHECK(cudaGetDevice(&dev));
  HostMailbox& mb = t_mailbox;
  if (mb.dev != dev) {
    void* p = nullptr;
    RF_CUDA_CHECK(cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    RF_CUDA_CHECK(cudaEventCreateWithFlags(&mb.ev, cudaEventDisableTiming));
    mb.h = (volatile double*)p;
    mb.dev = dev;
  }
  *out = &mb;
  return RF_OK;
}

static rf_status tau_reduce_to_host(const double* nrm2, int64_t n, double* out_dev, cudaStream_t st, double h[2]) {
  HostMailbox* pmb = nullptr;
  rf_status s0;
  if ((s0 = host_mailbox(&pmb))) return s0;
  HostMailbox& mb = *pmb;
  mb.h[0] = mb.h[1] = -1.0;
  {
    ProfScope ps("K1_tau_reduce", st);
    rfk::k_tau_reduce<<<1, 1024, 0, st>>>(nrm2, n, out_dev, mb.h);
  }
  RF_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  RF_CUDA_CHECK(cudaEventRecord(mb.ev, st));
  RF_CUDA_CHECK(cudaEventSynchronize(mb.ev));
  h[0] = mb.h[0];
  h[1] = mb.h[1];
  return RF_OK;
}

rf_status rf_estimate_tau(const void* X, rf_dtype x_dt, int64_t ldx, int64_t p, int64_t n, double* tau_out, void* ws,
                          size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (p <= 0 || n <= 0) return fail(RF_E_INVALID, "rf_estimate_tau: p, n must be > 0");
  if (!tau_out) return fail(RF_E_INVALID, "rf_estimate_tau: tau_out is NULL");
  if (x_dt < RF_DT_F64 || x_dt > RF_DT_BF16) return fail(RF_E_INVALID, "rf_estimate_tau: bad dtype");
  const rf_prec pr = x_dt == RF_DT_F64 ? RF_PREC_FP64 : (x_dt == RF_DT_BF16 ? RF_PREC_BF16 : RF_PREC_FP32);
  rf_status s = validate_matrix("X", X, ldx, p, esize_of(pr));
  if (s) return s;
  size_t need;
  rf_tau_workspace_size(n, &need);
  if (!ws || ws_bytes < need || !aligned16(ws))
    return fail(RF_E_WORKSPACE, "rf_estimate_tau: workspace needs %zu bytes (16-B aligned)", need);
  if ((s = check_device(nullptr))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  double* nrm2 = (double*)ws;
  double* out = (double*)((char*)ws + align256((size_t)n * 8));
  if ((s = launch_rownorm(X, pr, ldx, p, n, nrm2, st))) return s;
  double h[2];
  if ((s = tau_reduce_to_host(nrm2, n, out, st, h))) return s;
  *tau_out = h[0];
  return ok();
}

rf_status rf_gram_workspace_size(int64_t p, int64_t n, int64_t m_local, rf_prec prec, size_t* bytes) {
  if (!bytes) return fail(RF_E_INVALID, "bytes is NULL");
  if (p <= 0 || n <= 0 || m_local <= 0) return fail(RF_E_INVALID, "p, n, m_local must be > 0");
  if (!valid_prec(prec)) return fail(RF_E_INVALID, "unknown precision %d", (int)prec);
  *bytes = gram_plan(p, n, m_local, prec).total;
  return ok();
}

static rf_status rf_gram_core(const void* X, int64_t ldx, const void* W, int64_t ldw, int64_t p, int64_t n,
                              int64_t m_local, int64_t m_total, rf_act act, rf_prec prec, rf_out out, void* G,
                              int64_t ldg, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (p <= 0 || n <= 0 || m_local <= 0) return fail(RF_E_INVALID, "rf_gram: p, n, m_local must be > 0");
  if (m_total < m_local) return fail(RF_E_INVALID, "rf_gram: m_total (%lld) < m_local (%lld)", (long long)m_total,
                                     (long long)m_local);
  if (n > (int64_t)1 << 31 || m_local > (int64_t)1 << 31 || p > (int64_t)1 << 31)
    return fail(RF_E_INVALID, "rf_gram: sizes must be < 2^31");
  if (!valid_act(act)) return fail(RF_E_INVALID, "rf_gram: unknown activation %d", (int)act);
  if (!valid_prec(prec)) return fail(RF_E_INVALID, "rf_gram: unknown precision %d", (int)prec);
  if (!valid_out(out)) return fail(RF_E_INVALID, "rf_gram: unknown output mode %d", (int)out);
  const size_t es = esize_of(prec);
  rf_status s;
  if ((s = validate_matrix("X", X, ldx, p, es))) return s;
  if ((s = validate_matrix("W", W, ldw, p, es))) return s;
  int64_t tri_T = 0;
  if (out == RF_OUT_PACKED_TRI) {
    if ((s = packed_out_setup("rf_gram", G, n, prec, &tri_T))) return s;
  } else if ((s = validate_output("G", G, ldg, n, prec == RF_PREC_FP64 ? 8 : 4))) {
    return s;
  }
  const GramPlan pl = gram_plan(p, n, m_local, prec);
  if (!ws || ws_bytes < pl.total || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(RF_E_WORKSPACE, "rf_gram: workspace needs %zu bytes, 256-B aligned (got %zu)", pl.total, ws_bytes);
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  const int full = (int)out & 1;

  if (prec == RF_PREC_FP64 || prec == RF_PREC_FP32) {
    if (prec == RF_PREC_FP64) {
      double* S = (double*)(w + pl.off_s0);
      rfk::SimtSigma<double> e1{S, pl.ldS, n, m_local, (int)act};
      if ((s = launch_simt<double>("K6_simt_gemm_sigma", (const double*)X, ldx, (const double*)W, ldw, n, m_local, p, 0, 0,
                                   (int)((n + rfk::kSimtTile - 1) / rfk::kSimtTile), e1, st)))
        return s;
      rfk::SimtSyrk<double> e2{(double*)G, ldg, n, 1.0 / (double)m_total, full};
      if ((s = launch_simt<double>("K6_simt_syrk", S, pl.ldS, S, pl.ldS, n, n, m_local, 1, 0, (int)((n + rfk::kSimtTile - 1) / rfk::kSimtTile), e2, st)))
        return s;
    } else {
      float* S = (float*)(w + pl.off_s0);
      rfk::SimtSigma<float> e1{S, pl.ldS, n, m_local, (int)act};
      if ((s = launch_simt<float>("K6_simt_gemm_sigma", (const float*)X, ldx, (const float*)W, ldw, n, m_local, p, 0, 0,
                                  (int)((n + rfk::kSimtTile - 1) / rfk::kSimtTile), e1, st)))
        return s;
      rfk::SimtSyrk<float> e2{(float*)G, ldg, n, (float)(1.0 / (double)m_total), full};
      if ((s = launch_simt<float>("K6_simt_syrk", S, pl.ldS, S, pl.ldS, n, n, m_local, 1, 0, (int)((n + rfk::kSimtTile - 1) / rfk::kSimtTile), e2, st)))
        return s;
    }
    return ok();
  }

  // Tensor-core path: [K2 split] → K3 (pair tiles 256×256, σ epilogue) → K4 (triangle, SYRK epilogue)
  GramTcArgs ga{X, ldx, W, ldw, p, n, m_local, m_total, act, full, (float*)G, ldg, w, pl, dev.sms, st, nullptr, tri_T};
  if (prec == RF_PREC_BF16) return gram_tc<1, 1, 512, 0>(ga, kchunk_for(prec, 0));
  if (prec == RF_PREC_TF32) return gram_tc<2, 1, 512, 1>(ga, kchunk_for(prec, 0));
  // 3×TF32: chunks of 4 K-blocks (128 features) bound the truncating tensor-pipe accumulation to
  // ≈ 2.6e-6 relative (scripts/accum_experiment.py).
  return gram_tc<2, 3, 256, 2>(ga, kchunk_for(prec, 4));
  return ok();
}

rf_status rf_gram(const void* X, int64_t ldx, const void* W, int64_t ldw, int64_t p, int64_t n, int64_t m_local,
                  int64_t m_total, rf_act act, rf_prec prec, rf_out out, void* G, int64_t ldg, void* ws,
                  size_t ws_bytes, void* stream) {
  rf_status s = rf_gram_core(X, ldx, W, ldw, p, n, m_local, m_total, act, prec, out, G, ldg, ws, ws_bytes, stream);
  if (s || !((int)out & RF_OUT_CENTER)) return s;
  // NEXT-2: K = P·G·P (Eq. (2)).  Centering is linear, so each rank may center its own partial G.
  const int32_t launches = g_launches;
  double* cen = (double*)((char*)ws + gram_plan(p, n, m_local, prec).off_cen);
  s = prec == RF_PREC_FP64 ? center_pass<double>((double*)G, ldg, n, (int)out & 1, cen, (cudaStream_t)stream)
                           : center_pass<float>((float*)G, ldg, n, (int)out & 1, cen, (cudaStream_t)stream);
  g_launches += launches;
  return s ? s : ok();
}

rf_status rf_debug_gemm_workspace_size(int64_t M, int64_t N, int64_t K, rf_prec prec, size_t* bytes) {
  if (!bytes) return fail(RF_E_INVALID, "bytes is NULL");
  if (M <= 0 || N <= 0 || K <= 0) return fail(RF_E_INVALID, "M, N, K must be > 0");
  const int64_t ldk = round_up(K, 32);
  *bytes = prec == RF_PREC_3XTF32 ? align256((size_t)(M + N) * ldk * 4 * 2) + 256 : 256;
  return ok();
}

rf_status rf_debug_gemm_nt(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                           rf_prec prec, int32_t kchunk, float* C, int64_t ldc, void* ws, size_t ws_bytes,
                           void* stream) {
  g_launches = 0;
  if (M <= 0 || N <= 0 || K <= 0) return fail(RF_E_INVALID, "rf_debug_gemm_nt: M, N, K must be > 0");
  if (prec != RF_PREC_BF16 && prec != RF_PREC_TF32 && prec != RF_PREC_3XTF32)
    return fail(RF_E_INVALID, "rf_debug_gemm_nt: tensor-core precisions only (BF16, TF32, 3XTF32)");
  const size_t es = esize_of(prec);
  rf_status s;
  if ((s = validate_matrix("A", A, lda, K, es))) return s;
  if ((s = validate_matrix("B", B, ldb, K, es))) return s;
  if ((s = validate_output("C", C, ldc, N, 4))) return s;
  size_t need = 0;
  rf_debug_gemm_workspace_size(M, N, K, prec, &need);
  if (ws_bytes < need || (need > 256 && (!ws || (reinterpret_cast<uintptr_t>(ws) & 255))))
    return fail(RF_E_WORKSPACE, "rf_debug_gemm_nt: workspace needs %zu bytes", need);
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  rfk::EpiRaw e{C, ldc, M, N};
  CUtensorMap tA, tB, tAl, tBl;
  const int rt = (int)((M + 255) / 256), tn = (int)((N + 255) / 256);
  if (prec == RF_PREC_3XTF32) {
    using Cf = rfk::TcCfg<2, 3, 256>;
    const int64_t ldk = round_up(K, 32);
    float* Ah = (float*)ws;
    float* Al = Ah + M * ldk;
    float* Bh = Al + M * ldk;
    float* Bl = Bh + N * ldk;
    if ((s = launch_split((const float*)A, lda, M, K, Ah, Al, ldk, dev.sms, st))) return s;
    if ((s = launch_split((const float*)B, ldb, N, K, Bh, Bl, ldk, dev.sms, st))) return s;
    if ((s = make_tmap(&tA, Ah, false, M, K, ldk, 128))) return s;
    if ((s = make_tmap(&tAl, Al, false, M, K, ldk, 128))) return s;
    if ((s = make_tmap(&tB, Bh, false, N, K, ldk, 128))) return s;
    if ((s = make_tmap(&tBl, Bl, false, N, K, ldk, 128))) return s;
    const rfk::Sched sc = rfk::Sched::make(0, 256, 0, rt, tn, (int)((K + Cf::BK - 1) / Cf::BK), kchunk);
    if ((s = launch_tc<Cf>("KD_gemm_nt", tA, tB, tAl, tBl, tA, sc, e, dev.sms, st))) return s;
  } else {
    const bool bf = prec == RF_PREC_BF16;
    if ((s = make_tmap(&tA, A, bf, M, K, lda, 128))) return s;
    if ((s = make_tmap(&tB, B, bf, N, K, ldb, 128))) return s;
    if (bf) {
      using Cf = rfk::TcCfg<1, 1, 256>;
      const rfk::Sched sc = rfk::Sched::make(0, 256, 0, rt, tn, (int)((K + Cf::BK - 1) / Cf::BK), kchunk);
      if ((s = launch_tc<Cf>("KD_gemm_nt", tA, tB, tA, tB, tA, sc, e, dev.sms, st))) return s;
    } else {
      using Cf = rfk::TcCfg<2, 1, 256>;
      const rfk::Sched sc = rfk::Sched::make(0, 256, 0, rt, tn, (int)((K + Cf::BK - 1) / Cf::BK), kchunk);
      if ((s = launch_tc<Cf>("KD_gemm_nt", tA, tB, tA, tB, tA, sc, e, dev.sms, st))) return s;
    }
  }
  return ok();
}

rf_status rf_phi_workspace_size(int64_t p, int64_t n, rf_prec prec, size_t* bytes) {
  if (!bytes) return fail(RF_E_INVALID, "bytes is NULL");
  if (p <= 0 || n <= 0) return fail(RF_E_INVALID, "p, n must be > 0");
  if (!valid_prec(prec)) return fail(RF_E_INVALID, "unknown precision %d", (int)prec);
  *bytes = phi_plan(p, n, prec).total;
  return ok();
}

}  // extern "C"

// ------------------------------------------------------------------------------------------------
// NEXT-2: Theorem 1's K̃ (EQ6) on the tensor cores, centred in the same pass.
namespace {
struct KtPlan {
  int64_t ldp;
  size_t off_xbar, off_vbar, off_rr, off_s, off_u, off_vt, off_rf, off_xhi, off_xlo, total;
};
KtPlan kt_plan(int64_t p, int64_t n, rf_prec prec) {
  KtPlan k{};
  k.ldp = odd_line_ld(p, 4);
  size_t off = 0;
  k.off_xbar = off; off = align256(off + (size_t)p * 8);
  k.off_vbar = off; off = align256(off + 8 * 8);
  k.off_rr = off; off = align256(off + (size_t)n * 8);
  k.off_s = off; off = align256(off + 16);
  k.off_u = off; off = align256(off + (size_t)n * 8 * 4);
  k.off_vt = off; off = align256(off + (size_t)round_up(n, 32) * 8 * 4);
  k.off_rf = off; off = align256(off + (size_t)n * 4);
  if (prec == RF_PREC_3XTF32) {
    k.off_xhi = off; off = align256(off + (size_t)n * k.ldp * 4);
    k.off_xlo = off; off = align256(off + (size_t)n * k.ldp * 4);
  }
  k.total = off;
  return k;
}
}  // namespace

extern "C" {

rf_status rf_ktilde_workspace_size(int64_t p, int64_t n, rf_prec prec, size_t* bytes) {
  if (!bytes) return fail(RF_E_INVALID, "bytes is NULL");
  if (p <= 0 || n <= 0) return fail(RF_E_INVALID, "p, n must be > 0");
  *bytes = kt_plan(p, n, prec).total;
  return ok();
}

rf_status rf_ktilde(const void* X, int64_t ldx, int64_t p, int64_t n, const float* V, int64_t ldv, int32_t kv,
                    const double* A, double d0, double d1, double d2, rf_prec prec, rf_out out, float* Kt, int64_t ldk,
                    void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (p <= 0 || n <= 0) return fail(RF_E_INVALID, "rf_ktilde: p, n must be > 0");
  if (n >= (int64_t(1) << 31) || p >= (int64_t(1) << 31)) return fail(RF_E_INVALID, "rf_ktilde: sizes must be < 2^31");
  if (kv < 0 || kv > rfk::kMaxKv) return fail(RF_E_INVALID, "rf_ktilde: kv must be in [0, %d]", rfk::kMaxKv);
  if (kv > 0 && (!V || !A || ldv < kv || (reinterpret_cast<uintptr_t>(V) & 3)))
    return fail(RF_E_INVALID, "rf_ktilde: V (device f32 n × kv, ldv >= kv) and A (host kv × kv) are required");
  if (prec != RF_PREC_BF16 && prec != RF_PREC_TF32 && prec != RF_PREC_3XTF32)
    return fail(RF_E_INVALID, "rf_ktilde: tensor-core precisions only (BF16 with bf16 X; TF32 / 3XTF32 with f32 X)");
  if (out != RF_OUT_UPPER && out != RF_OUT_FULL)
    return fail(RF_E_INVALID, "rf_ktilde: out must be UPPER or FULL (K̃ is always centred, EQ6)");
  if (!std::isfinite(d0) || !std::isfinite(d1) || !std::isfinite(d2)) return fail(RF_E_INVALID, "rf_ktilde: d0, d1, d2 must be finite");
  const size_t es = esize_of(prec);
  rf_status s;
  if ((s = validate_matrix("X", X, ldx, p, es))) return s;
  if ((s = validate_output("Kt", Kt, ldk, n, 4))) return s;
  const KtPlan pl = kt_plan(p, n, prec);
  if (!ws || ws_bytes < pl.total || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(RF_E_WORKSPACE, "rf_ktilde: workspace needs %zu bytes, 256-B aligned (got %zu)", pl.total, ws_bytes);
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  double* xbar = (double*)(w + pl.off_xbar);
  double* vbar = (double*)(w + pl.off_vbar);
  double* rr = (double*)(w + pl.off_rr);
  double* sp = (double*)(w + pl.off_s);
  float* u = (float*)(w + pl.off_u);
  float* vt = (float*)(w + pl.off_vt);
  float* rf = (float*)(w + pl.off_rf);
  rfk::KtA Ak{};
  for (int a = 0; a < kv; ++a)
    for (int b = 0; b < kv; ++b) Ak.a[a][b] = A[a * kv + b];
  RF_CUDA_CHECK(cudaMemsetAsync(xbar, 0, (size_t)p * 8, st));
  RF_CUDA_CHECK(cudaMemsetAsync(vbar, 0, 8 * 8, st));
  const unsigned chunks = (unsigned)std::min<int64_t>(std::max<int64_t>(n / 512, 1), 256);
  {
    ProfScope ps("KT_prep", st);
    if (prec == RF_PREC_BF16)
      rfk::k_colsum<__nv_bfloat16><<<dim3((unsigned)((p + 255) / 256), chunks), 256, 0, st>>>(
          (const __nv_bfloat16*)X, ldx, n, p, xbar);
    else
      rfk::k_colsum<float><<<dim3((unsigned)((p + 255) / 256), chunks), 256, 0, st>>>((const float*)X, ldx, n, p, xbar);
    if (kv > 0) rfk::k_colsum<float><<<dim3(1, chunks), 256, 0, st>>>(V, ldv, n, kv, vbar);
    const unsigned rg = (unsigned)((n + 7) / 8);
    const float* Vp = kv > 0 ? V : nullptr;   // never read when kv = 0
    if (prec == RF_PREC_BF16)
      rfk::k_ktilde_rows<__nv_bfloat16><<<rg, 256, 0, st>>>((const __nv_bfloat16*)X, ldx, p, n, Vp,
                                                            ldv, kv, Ak, d0, d1, d2, xbar, vbar, u, vt, round_up(n, 32), rr);
    else
      rfk::k_ktilde_rows<float><<<rg, 256, 0, st>>>((const float*)X, ldx, p, n, Vp, ldv, kv, Ak, d0,
                                                    d1, d2, xbar, vbar, u, vt, round_up(n, 32), rr);
    rfk::k_center_scale<<<1, 1024, 0, st>>>(rr, n, sp);
    rfk::k_center_fold<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rr, sp, n, rf);
    RF_CUDA_CHECK(cudaGetLastError());
    g_launches += 5 + (kv > 0);
  }
  CUtensorMap tA, tAl, tO;
  const bool tma_out = make_tmap_out(&tO, Kt, n, n, ldk);
  rfk::EpiKtilde e{Kt, ldk, n, u, vt, round_up(n, 32), rf, (float)d0, (float)d1, (float)d2, kv, (int)out & 1,
                   tma_out ? 1 : 0};
  const int tn = (int)((n + 255) / 256);
  if (prec == RF_PREC_BF16 || prec == RF_PREC_TF32) {
    const bool bf = prec == RF_PREC_BF16;
    if ((s = make_tmap(&tA, X, bf, n, p, ldx, 128))) return s;
    if (!tma_out) tO = tA;
    // 16 epilogue warps: K̃'s epilogue (a rank-8 product per entry) is latency-bound at two warps per SM
    // sub-partition even at p = 1024 (n = 65536: 8 / 12 / 16 warps 6.87 / 4.72 / 4.22 ms; n = 131072, p = 512:
    // 26.7 / 18.2 / 15.5 ms)
    if (bf) {
      using C = rfk::TcCfg<1, 1, 256, 1, 2, 16>;
      const rfk::Sched sc = rfk::Sched::make(1, 256, 0, tn, tn, (int)((p + C::BK - 1) / C::BK), 0, raster_gm(16, 5));
      if ((s = launch_tc<C>("KT_ktilde", tA, tA, tA, tA, tO, sc, e, dev.sms, st))) return s;
    } else {
      using C = rfk::TcCfg<2, 1, 256, 1, 2, 16>;
      const rfk::Sched sc = rfk::Sched::make(1, 256, 0, tn, tn, (int)((p + C::BK - 1) / C::BK), 0, raster_gm(16, 5));
      if ((s = launch_tc<C>("KT_ktilde", tA, tA, tA, tA, tO, sc, e, dev.sms, st))) return s;
    }
  } else {
    using C = rfk::TcCfg<2, 3, 256>;
    float* Xh = (float*)(w + pl.off_xhi);
    float* Xl = (float*)(w + pl.off_xlo);
    if ((s = launch_split((const float*)X, ldx, n, p, Xh, Xl, pl.ldp, dev.sms, st))) return s;
    if ((s = make_tmap(&tA, Xh, false, n, p, pl.ldp, 128))) return s;
    if ((s = make_tmap(&tAl, Xl, false, n, p, pl.ldp, 128))) return s;
    if (!tma_out) tO = tA;
    const rfk::Sched sc = rfk::Sched::make(1, 256, 0, tn, tn, (int)((p + C::BK - 1) / C::BK), 0, raster_gm(16, 5));
    if ((s = launch_tc<C>("KT_ktilde", tA, tA, tAl, tAl, tO, sc, e, dev.sms, st))) return s;
  }
  return ok();
}

}  // extern "C"

// ------------------------------------------------------------------------------------------------
// NEXT-1: Ternary Random Features (Eq. (3)-(5), Corollary 1, Algorithm 1).
namespace {
struct TerPlan {
  int64_t ldS;   // bytes per Σ^terᵀ row
  size_t off_s, off_prog, off_cen, total;
};
TerPlan ter_plan(int64_t n, int64_t m_local) {
  TerPlan t{};
  t.ldS = odd_line_ld(std::max<int64_t>(m_local, 1), 1);
  size_t off = 0;
  t.off_s = off; off = align256(off + (size_t)n * t.ldS);
  t.off_prog = off; off = align256(off + 1024);
  t.off_cen = off; off = align256(off + (size_t)(n + 2) * 8);
  t.total = off;
  return t;
}

rf_status ter_validate(const char* fn, const void* X, int64_t ldx, const void* T, int64_t ldt, int64_t p, int64_t n,
                       int64_t m_local, double eps, double s_minus, double s_plus) {
  if (p <= 0 || n <= 0 || m_local <= 0) return fail(RF_E_INVALID, "%s: p, n, m_local must be > 0", fn);
  if (p >= (int64_t(1) << 31) || n >= (int64_t(1) << 31) || m_local >= (int64_t(1) << 31))
    return fail(RF_E_INVALID, "%s: sizes must be < 2^31", fn);
  if (!(eps >= 0.0 && eps < 1.0)) return fail(RF_E_INVALID, "%s: eps must be in [0, 1) (Eq. (4))", fn);
  if (!(s_minus <= s_plus) || !std::isfinite(s_minus) || !std::isfinite(s_plus))
    return fail(RF_E_INVALID, "%s: need finite thresholds s_minus <= s_plus (Eq. (5))", fn);
  rf_status s;
  if ((s = validate_matrix("X", X, ldx, p, 2))) return s;
  if ((s = validate_matrix("T", T, ldt, p, 2))) return s;
  return RF_OK;
}

// K3^ter into `feat` (bytes, ld multiple of 16): σ^ter(c·XTᵀ) as fp8 codes.
rf_status launch_k3_ter(const void* X, int64_t ldx, const void* T, int64_t ldt, int64_t p, int64_t n, int64_t m_local,
                        double eps, double s_minus, double s_plus, uint8_t* feat, int64_t ldf, int sms,
                        cudaStream_t st, uint32_t* prog = nullptr) {
  using C3 = rfk::TcCfg<1, 1, 256, 0>;
  CUtensorMap tA, tB;
  rf_status s;
  if ((s = make_tmap(&tA, X, true, n, p, ldx, 128))) return s;
  if ((s = make_tmap(&tB, T, true, m_local, p, ldt, 128))) return s;
  const double inv_c = std::sqrt(1.0 - eps);   // t± = s± / c, c = (1 − ε)^{-1/2}
  rfk::EpiSigmaTer e{feat, ldf, n, m_local, (float)(s_minus * inv_c), (float)(s_plus * inv_c)};
  const int kb = (int)((p + C3::BK - 1) / C3::BK);
  if (prog && env_int("RF_K3_MC", 1)) {   // multicast + pair hybrid (workspace progress words available)
    using C3m = rfk::TcCfg<1, 1, 256, 0, 4>;
    CUtensorMap tBh;
    if ((s = make_tmap(&tBh, T, true, m_local, p, ldt, 64))) return s;
    bool used = false;
    if ((s = launch_k3_hybrid<C3m, C3>("K3_ter_features", tA, tB, tBh, n, m_local, kb, e, prog, sms, st, &used)))
      return s;
    if (used) return RF_OK;
  }
  const rfk::Sched sc =
      rfk::Sched::make(0, 256, 0, (int)((n + 255) / 256), (int)((m_local + 255) / 256), kb, 0, raster_gm(8, 3));
  return launch_tc<C3>("K3_ter_features", tA, tB, tA, tB, tA, sc, e, sms, st);
}
}  // namespace

extern "C" {

rf_status rf_trf_thresholds(double d1, double d2, double tau, int32_t sign2, double* s_minus, double* s_plus) {
  if (!s_minus || !s_plus) return fail(RF_E_INVALID, "rf_trf_thresholds: NULL output");
  if (!(tau > 0) || !std::isfinite(tau) || !(d1 >= 0) || !(d2 >= 0) || !std::isfinite(d1) || !std::isfinite(d2))
    return fail(RF_E_INVALID, "rf_trf_thresholds: need tau > 0 and finite d1, d2 >= 0");
  double r = 0;
  if (rfh::solve_ternary_thresholds(d1, d2, tau, sign2, s_minus, s_plus, &r))
    return fail(RF_E_INVALID, "rf_trf_thresholds: no ternary thresholds reproduce d1=%g, d2=%g at tau=%g "
                "(residual %.3e; sqrt(tau d1) <= 2 phi(0) and 2 tau sqrt(d2) <= 2 phi(1) are required)", d1, d2, tau, r);
  return ok();
}

rf_status rf_trf_thresholds_for(rf_act act, double tau, double* s_minus, double* s_plus) {
  if (!valid_act(act)) return fail(RF_E_INVALID, "rf_trf_thresholds_for: unknown activation %d", (int)act);
  rf_moments_t m;
  rf_status s = rf_moments(act, tau, 0, &m);
  if (s) return s;
  return rf_trf_thresholds(m.d1, m.d2, tau, m.kd[0][2] < 0 ? -1 : 1, s_minus, s_plus);
}

rf_status rf_gram_ter_workspace_size(int64_t p, int64_t n, int64_t m_local, size_t* bytes) {
  if (!bytes) return fail(RF_E_INVALID, "bytes is NULL");
  if (p <= 0 || n <= 0 || m_local <= 0) return fail(RF_E_INVALID, "p, n, m_local must be > 0");
  *bytes = ter_plan(n, m_local).total;
  return ok();
}

rf_status rf_ter_features(const void* X, int64_t ldx, const void* T, int64_t ldt, int64_t p, int64_t n,
                          int64_t m_local, double eps, double s_minus, double s_plus, void* features, int64_t ldf,
                          void* stream) {
  g_launches = 0;
  rf_status s;
  if ((s = ter_validate("rf_ter_features", X, ldx, T, ldt, p, n, m_local, eps, s_minus, s_plus))) return s;
  if (!features || !aligned16(features) || ldf < m_local || (ldf % 16) != 0)
    return fail(RF_E_INVALID, "rf_ter_features: features must be 16-B aligned with ldf >= m_local, ldf %% 16 == 0");
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  if ((s = launch_k3_ter(X, ldx, T, ldt, p, n, m_local, eps, s_minus, s_plus, (uint8_t*)features, ldf, dev.sms,
                         (cudaStream_t)stream)))
    return s;
  return ok();
}

rf_status rf_gram_ter(const void* X, int64_t ldx, const void* T, int64_t ldt, int64_t p, int64_t n, int64_t m_local,
                      int64_t m_total, double eps, double s_minus, double s_plus, rf_out out, float* G, int64_t ldg,
                      void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  rf_status s;
  if ((s = ter_validate("rf_gram_ter", X, ldx, T, ldt, p, n, m_local, eps, s_minus, s_plus))) return s;
  if (m_total < m_local) return fail(RF_E_INVALID, "rf_gram_ter: m_total < m_local");
  if (m_local > (int64_t(1) << 24))
    return fail(RF_E_INVALID, "rf_gram_ter: m_local > 2^24 (fp32 accumulation of ±1 products is exact below that)");
  if (!valid_out(out)) return fail(RF_E_INVALID, "rf_gram_ter: unknown output mode %d", (int)out);
  int64_t tri_T = 0;
  if (out == RF_OUT_PACKED_TRI) {
    if ((s = packed_out_setup("rf_gram_ter", G, n, RF_PREC_BF16, &tri_T))) return s;
  } else if ((s = validate_output("G", G, ldg, n, 4))) {
    return s;
  }
  const TerPlan pl = ter_plan(n, m_local);
  if (!ws || ws_bytes < pl.total || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(RF_E_WORKSPACE, "rf_gram_ter: workspace needs %zu bytes, 256-B aligned (got %zu)", pl.total, ws_bytes);
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  uint8_t* S = (uint8_t*)(w + pl.off_s);
  // K3^ter: Σ^terᵀ = σ^ter(c·X Tᵀ) as fp8 codes
  if ((s = launch_k3_ter(X, ldx, T, ldt, p, n, m_local, eps, s_minus, s_plus, S, pl.ldS, dev.sms, st,
                         (uint32_t*)(w + pl.off_prog))))
    return s;
  // K4^ter: G^ter = Σ^terᵀΣ^ter / m on the fp8 tensor path (kind::f8f6f4): ±1·±1 products and their sums
  // (|sum| ≤ m_local ≤ 2^24) are exact in the fp32 accumulator, so m·G^ter is an exact integer count.
  using C4 = rfk::TcCfg<3, 1, 512>;
  CUtensorMap tA, tO;
  if ((s = make_tmap_es(&tA, S, 1, n, m_local, pl.ldS, 128))) return s;
  const bool tma_out = tri_T > 0 ? make_tmap_out(&tO, G, tri_tiles(n) * 256, 256, 256) : make_tmap_out(&tO, G, n, n, ldg);
  if (!tma_out) tO = tA;
  const int kb4 = (int)((m_local + C4::BK - 1) / C4::BK);
  rfk::Sched s4 = rfk::Sched::make(1, 512, 0, (int)((n + 255) / 256), (int)((n + 511) / 512), kb4, 0, raster_gm(8, 4));
  const int lockw = env_int("RF_LOCKW", 24);
  if (lockw > 0) {
    s4.prog = (uint32_t*)(w + pl.off_prog);
    s4.lock_w = lockw;
    s4.lock_ks = std::max(1, env_int("RF_LOCKKS", 8));
    RF_CUDA_CHECK(cudaMemsetAsync(s4.prog, 0, 1024, st));
  }
  rfk::EpiSyrk e4{G, ldg, n, (float)(1.0 / (double)m_total), (int)out & 1, tma_out ? 1 : 0, tri_T};
  bool hyb = false;
  if (lockw > 0 && env_int("RF_K4TER_MC", 0) == 0) {
    CUtensorMap tSh;   // Σ^terᵀ with a 64-row box (the 8-CTA multicast kernel's A halves)
    if ((s = make_tmap_es(&tSh, S, 1, n, m_local, pl.ldS, 64))) return s;
    if ((s = launch_k4_hybrid<3>("K4_ter_syrk", tA, tSh, tO, n, kb4, e4, s4.prog, lockw, s4.lock_ks, dev.sms, st,
                                 &hyb)))
      return s;
  }
  if (hyb) {
  } else if (env_int("RF_K4TER_MC", 0)) {
    // 4-CTA clusters, B multicast (DESIGN.md §6 finding 3): the fp8 SYRK runs at full clock and is L2-bound,
    // so a third less L2 → SM traffic matters more than the SMs the GPC packing of 4-clusters leaves idle.
    using C4m = rfk::TcCfg<3, 1, 512, -1, 4>;
    rfk::Sched sm = rfk::Sched::make(1, 256, 0, (int)((n + 511) / 512), (int)((n + 511) / 512), kb4, 0, raster_gm(4, 4));
    sm.prog = s4.prog;
    sm.lock_w = s4.lock_w;
    sm.lock_ks = s4.lock_ks;
    if ((s = launch_tc<C4m>("K4_ter_syrk", tA, tA, tA, tA, tO, sm, e4, dev.sms, st))) return s;
  } else if ((s = launch_tc<C4>("K4_ter_syrk", tA, tA, tA, tA, tO, s4, e4, dev.sms, st))) {
    return s;
  }
  if ((int)out & RF_OUT_CENTER)
    if ((s = center_pass<float>(G, ldg, n, (int)out & 1, (double*)(w + pl.off_cen), st))) return s;
  return ok();
}

}  // extern "C"

// ------------------------------------------------------------------------------------------------
// G5: packed triangle tiles + chunk completion (include/rf.h).
namespace {
int pack_bn(rf_prec prec) { return prec == RF_PREC_3XTF32 ? 256 : 512; }

rf_status build_pack_plan(int64_t n, int32_t world, int32_t nchunks, rf_prec prec, rf_pack_plan_t* pl,
                          rfk::PackDev* dv) {
  if (n <= 0 || n >= (int64_t(1) << 31)) return fail(RF_E_INVALID, "rf_pack_plan: n must be in (0, 2^31)");
  if (world <= 0 || world > 4096) return fail(RF_E_INVALID, "rf_pack_plan: world must be in [1, 4096]");
  if (nchunks <= 0) return fail(RF_E_INVALID, "rf_pack_plan: nchunks must be > 0");
  if (prec != RF_PREC_BF16 && prec != RF_PREC_TF32 && prec != RF_PREC_3XTF32)
    return fail(RF_E_INVALID, "rf_pack_plan: packed output needs a tensor-core precision (BF16, TF32, 3XTF32)");
  const int bn = pack_bn(prec), tpp = bn / 256;
  const int tiles_m = (int)((n + 255) / 256), tiles_n = (int)((n + bn - 1) / bn);
  const rfk::Sched sc = rfk::Sched::make(1, bn, 0, tiles_m, tiles_n, 1, 0, kPackGm);
  std::vector<int64_t> gcnt;   // pair tiles per raster group
  for (int I0 = 0; I0 < tiles_m; I0 += kPackGm) gcnt.push_back(sc.group(I0).cnt);
  const int G = (int)gcnt.size();
  const int C = std::min<int>(std::min<int>(nchunks, RF_PACK_MAX_CHUNKS), G);
  std::memset(pl, 0, sizeof(*pl));
  pl->n = n;
  pl->world = world;
  pl->nchunks = C;
  pl->prec = (int32_t)prec;
  pl->tiles_per_pair = tpp;
  pl->pair_tiles = sc.num_tiles;
  const int64_t total = sc.num_tiles;
  int g = 0;
  int64_t acc = 0;
  std::vector<int> gfirst(C + 1, G);
  for (int c = 0; c < C; ++c) {
    gfirst[c] = g;
    pl->chunk_tile0[c] = acc;
    const int64_t target = (total * (c + 1) + C - 1) / C;
    do {
      acc += gcnt[g++];
    } while (g < G - (C - 1 - c) && acc < target);
    if (c == C - 1)
      while (g < G) acc += gcnt[g++];
  }
  pl->chunk_tile0[C] = acc;
  int64_t soff = 0, roff = 0;
  for (int c = 0; c < C; ++c) {
    const int64_t nt = (pl->chunk_tile0[c + 1] - pl->chunk_tile0[c]) * tpp;
    pl->chunk_slots[c] = (nt + world - 1) / world;
    pl->chunk_send_off[c] = soff;
    pl->chunk_recv_off[c] = roff;
    soff += pl->chunk_slots[c] * world * (int64_t)(RF_PACK_TILE * RF_PACK_TILE);
    roff += pl->chunk_slots[c] * (int64_t)(RF_PACK_TILE * RF_PACK_TILE);
  }
  pl->chunk_send_off[C] = soff;
  pl->chunk_recv_off[C] = roff;
  pl->send_elems = soff;
  pl->recv_elems = roff;
  if (dv) {
    std::memset(dv, 0, sizeof(*dv));
    for (int c = 0; c <= C; ++c) {
      dv->tile0[c] = pl->chunk_tile0[c];
      dv->soff[c] = pl->chunk_send_off[c];
      dv->roff[c] = pl->chunk_recv_off[c];
      dv->rt0[c] = std::min(gfirst[c] * kPackGm, tiles_m);
      if (c < C) dv->slots[c] = pl->chunk_slots[c];
    }
  }
  return RF_OK;
}

bool same_plan(const rf_pack_plan_t* a, const rf_pack_plan_t* b) {
  return a->n == b->n && a->world == b->world && a->nchunks == b->nchunks && a->prec == b->prec &&
         a->send_elems == b->send_elems &&
         std::memcmp(a->chunk_tile0, b->chunk_tile0, sizeof(a->chunk_tile0)) == 0 &&
         std::memcmp(a->chunk_slots, b->chunk_slots, sizeof(a->chunk_slots)) == 0;
}

typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_wait32 wait32_fn() {
  static PFN_wait32 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_wait32>(p);
  });
  return fn;
}
}  // namespace

extern "C" {

rf_status rf_pack_plan(int64_t n, int32_t world, int32_t nchunks, rf_prec prec, rf_pack_plan_t* out) {
  if (!out) return fail(RF_E_INVALID, "rf_pack_plan: out is NULL");
  rf_status s = build_pack_plan(n, world, nchunks, prec, out, nullptr);
  return s ? s : ok();
}

rf_status rf_pack_tile_map(const rf_pack_plan_t* plan, int32_t rank, int32_t* rc) {
  if (!plan || !rc) return fail(RF_E_INVALID, "rf_pack_tile_map: NULL argument");
  rf_pack_plan_t chk;
  rf_status s = build_pack_plan(plan->n, plan->world, plan->nchunks, (rf_prec)plan->prec, &chk, nullptr);
  if (s) return s;
  if (!same_plan(plan, &chk)) return fail(RF_E_INVALID, "rf_pack_tile_map: plan was not made by rf_pack_plan");
  if (rank < 0 || rank >= plan->world) return fail(RF_E_INVALID, "rf_pack_tile_map: rank out of range");
  const int bn = pack_bn((rf_prec)plan->prec), tpp = plan->tiles_per_pair;
  const int tiles_m = (int)((plan->n + 255) / 256), tiles_n = (int)((plan->n + bn - 1) / bn);
  const rfk::Sched sc = rfk::Sched::make(1, bn, 0, tiles_m, tiles_n, 1, 0, kPackGm);
  // schedule index → (ti, tj), walking groups in order (the kernels' TileCursor)
  std::vector<int32_t> ti_of(sc.num_tiles), tj_of(sc.num_tiles);
  {
    long long base = 0;
    for (int I0 = 0; I0 < tiles_m; I0 += kPackGm) {
      const rfk::Sched::Group gr = sc.group(I0);
      for (long long u = 0; u < gr.cnt; ++u) {
        int ti, tj;
        sc.in_group(gr, u, ti, tj);
        ti_of[base + u] = ti;
        tj_of[base + u] = tj;
      }
      base += gr.cnt;
    }
  }
  int64_t k = 0;
  for (int c = 0; c < plan->nchunks; ++c) {
    const int64_t nt = (plan->chunk_tile0[c + 1] - plan->chunk_tile0[c]) * tpp;
    for (int64_t slot = 0; slot < plan->chunk_slots[c]; ++slot, ++k) {
      const int64_t u = slot * plan->world + rank;
      if (u < nt) {
        const int64_t pt = plan->chunk_tile0[c] + u / tpp;
        rc[2 * k] = ti_of[pt];
        rc[2 * k + 1] = tj_of[pt] * tpp + (int32_t)(u % tpp);
      } else {
        rc[2 * k] = rc[2 * k + 1] = -1;
      }
    }
  }
  return ok();
}

rf_status rf_gram_packed(const void* X, int64_t ldx, const void* W, int64_t ldw, int64_t p, int64_t n,
                         int64_t m_local, int64_t m_total, rf_act act, rf_prec prec, const rf_pack_plan_t* plan,
                         int32_t max_sms, float* send, uint32_t* chunk_sync, uint32_t epoch, void* ws,
                         size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (p <= 0 || n <= 0 || m_local <= 0 || m_total < m_local)
    return fail(RF_E_INVALID, "rf_gram_packed: need p, n, m_local > 0 and m_total >= m_local");
  if (p >= (int64_t(1) << 31) || n >= (int64_t(1) << 31) || m_local >= (int64_t(1) << 31))
    return fail(RF_E_INVALID, "rf_gram_packed: sizes must be < 2^31");
  if (!valid_act(act)) return fail(RF_E_INVALID, "rf_gram_packed: unknown activation %d", (int)act);
  if (!plan) return fail(RF_E_INVALID, "rf_gram_packed: plan is NULL");
  if (plan->prec != (int32_t)prec || plan->n != n)
    return fail(RF_E_INVALID, "rf_gram_packed: plan was made for another n or precision");
  rf_pack_plan_t chk;
  rfk::PackDev dv;
  rf_status s = build_pack_plan(n, plan->world, plan->nchunks, prec, &chk, &dv);
  if (s) return s;
  if (!same_plan(plan, &chk)) return fail(RF_E_INVALID, "rf_gram_packed: plan was not made by rf_pack_plan");
  if (!send || (reinterpret_cast<uintptr_t>(send) & 15)) return fail(RF_E_INVALID, "rf_gram_packed: send must be 16-B aligned");
  if (!chunk_sync || (reinterpret_cast<uintptr_t>(chunk_sync) & 3))
    return fail(RF_E_INVALID, "rf_gram_packed: chunk_sync must be a 4-B aligned device array");
  if (epoch == 0) return fail(RF_E_INVALID, "rf_gram_packed: epoch is 1-based");
  const size_t es = esize_of(prec);
  if ((s = validate_matrix("X", X, ldx, p, es))) return s;
  if ((s = validate_matrix("W", W, ldw, p, es))) return s;
  const GramPlan pl = gram_plan(p, n, m_local, prec);
  if (!ws || ws_bytes < pl.total || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(RF_E_WORKSPACE, "rf_gram_packed: workspace needs %zu bytes, 256-B aligned (got %zu)", pl.total,
                ws_bytes);
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  const int sms = max_sms > 0 ? std::max(2, std::min(dev.sms, (int)max_sms)) : dev.sms;
  PackArgs pa{send, chunk_sync, &dv, plan->world, plan->nchunks};
  GramTcArgs ga{X, ldx, W, ldw, p, n, m_local, m_total, act, 0, nullptr, n, (char*)ws, pl, sms,
                (cudaStream_t)stream, &pa};
  if (prec == RF_PREC_BF16) return gram_tc<1, 1, 512, 0>(ga, kchunk_for(prec, 0));
  if (prec == RF_PREC_TF32) return gram_tc<2, 1, 512, 1>(ga, kchunk_for(prec, 0));
  return gram_tc<2, 3, 256, 2>(ga, kchunk_for(prec, 4));
}

rf_status rf_stream_wait_chunk(const rf_pack_plan_t* plan, const uint32_t* chunk_sync, int32_t chunk,
                               uint32_t epoch, void* stream) {
  if (!plan || !chunk_sync) return fail(RF_E_INVALID, "rf_stream_wait_chunk: NULL argument");
  if (chunk < 0 || chunk >= plan->nchunks) return fail(RF_E_INVALID, "rf_stream_wait_chunk: chunk out of range");
  if (epoch == 0) return fail(RF_E_INVALID, "rf_stream_wait_chunk: epoch is 1-based");
  PFN_wait32 fn = wait32_fn();
  if (!fn) return fail(RF_E_CUDA, "cuStreamWaitValue32 entry point unavailable");
  const uint32_t per = 16u * (uint32_t)(plan->chunk_tile0[chunk + 1] - plan->chunk_tile0[chunk]);
  const uint32_t target = per * epoch;   // uint32 wrap; the wait compares wrap-safe (GEQ)
  CUresult r = fn((CUstream)stream, (CUdeviceptr)(uintptr_t)(chunk_sync + chunk), target, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(RF_E_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  return ok();
}

}  // extern "C"

// ------------------------------------------------------------------------------------------------
// Fused G5 over peer memory (include/rf.h): K4's epilogue stores each tile straight into its owner's staging buffer.
extern "C" {

rf_status rf_ipc_handle(const void* dptr, uint8_t* handle64) {
  if (!dptr || !handle64) return fail(RF_E_INVALID, "rf_ipc_handle: NULL argument");
  cudaIpcMemHandle_t h;
  RF_CUDA_CHECK(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, 64);
  return ok();
}

rf_status rf_ipc_open(const uint8_t* handle64, void** dptr) {
  if (!dptr || !handle64) return fail(RF_E_INVALID, "rf_ipc_open: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  RF_CUDA_CHECK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return ok();
}

rf_status rf_ipc_close(void* dptr) {
  if (!dptr) return fail(RF_E_INVALID, "rf_ipc_close: NULL argument");
  RF_CUDA_CHECK(cudaIpcCloseMemHandle(dptr));
  return ok();
}

rf_status rf_gram_packed_p2p(const void* X, int64_t ldx, const void* W, int64_t ldw, int64_t p, int64_t n,
                             int64_t m_local, int64_t m_total, rf_act act, rf_prec prec, const rf_pack_plan_t* plan,
                             int32_t rank, float* const* staging, int32_t max_sms, void* ws, size_t ws_bytes,
                             void* stream) {
  g_launches = 0;
  if (p <= 0 || n <= 0 || m_local <= 0 || m_total < m_local)
    return fail(RF_E_INVALID, "rf_gram_packed_p2p: need p, n, m_local > 0 and m_total >= m_local");
  if (!valid_act(act)) return fail(RF_E_INVALID, "rf_gram_packed_p2p: unknown activation %d", (int)act);
  if (!plan || !staging) return fail(RF_E_INVALID, "rf_gram_packed_p2p: NULL plan or staging array");
  if (prec != RF_PREC_BF16 && prec != RF_PREC_TF32)
    return fail(RF_E_INVALID, "rf_gram_packed_p2p: BF16 or TF32 only (3XTF32's K-chunked accumulation would "
                "read back remote tiles)");
  if (plan->prec != (int32_t)prec || plan->n != n)
    return fail(RF_E_INVALID, "rf_gram_packed_p2p: plan was made for another n or precision");
  if (plan->world > rfk::kMaxP2P) return fail(RF_E_INVALID, "rf_gram_packed_p2p: world > %d", rfk::kMaxP2P);
  if (rank < 0 || rank >= plan->world) return fail(RF_E_INVALID, "rf_gram_packed_p2p: rank out of range");
  rf_pack_plan_t chk;
  rfk::PackDev dv;
  rf_status s = build_pack_plan(n, plan->world, plan->nchunks, prec, &chk, &dv);
  if (s) return s;
  if (!same_plan(plan, &chk)) return fail(RF_E_INVALID, "rf_gram_packed_p2p: plan was not made by rf_pack_plan");
  for (int r = 0; r < plan->world; ++r) {
    if (!staging[r] || (reinterpret_cast<uintptr_t>(staging[r]) & 15))
      return fail(RF_E_INVALID, "rf_gram_packed_p2p: staging[%d] must be a 16-B aligned device pointer", r);
    dv.peer[r] = staging[r];
  }
  dv.p2p = 1;
  dv.self = rank;
  dv.recv_elems = plan->recv_elems;
  const size_t es = esize_of(prec);
  if ((s = validate_matrix("X", X, ldx, p, es))) return s;
  if ((s = validate_matrix("W", W, ldw, p, es))) return s;
  const GramPlan pl = gram_plan(p, n, m_local, prec);
  if (!ws || ws_bytes < pl.total || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(RF_E_WORKSPACE, "rf_gram_packed_p2p: workspace needs %zu bytes, 256-B aligned (got %zu)", pl.total,
                ws_bytes);
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  const int sms = max_sms > 0 ? std::max(2, std::min(dev.sms, (int)max_sms)) : dev.sms;
  PackArgs pa{nullptr, nullptr, &dv, plan->world, plan->nchunks};
  GramTcArgs ga{X, ldx, W, ldw, p, n, m_local, m_total, act, 0, nullptr, n, (char*)ws, pl, sms,
                (cudaStream_t)stream, &pa};
  if (prec == RF_PREC_BF16) return gram_tc<1, 1, 512, 0>(ga, 0);
  return gram_tc<2, 1, 512, 1>(ga, 0);
}

rf_status rf_pack_reduce(const rf_pack_plan_t* plan, const float* staging_self, float* recv, void* stream) {
  if (!plan || !staging_self || !recv) return fail(RF_E_INVALID, "rf_pack_reduce: NULL argument");
  if ((reinterpret_cast<uintptr_t>(staging_self) & 15) || (reinterpret_cast<uintptr_t>(recv) & 15))
    return fail(RF_E_INVALID, "rf_pack_reduce: buffers must be 16-B aligned");
  DevInfo dev;
  rf_status s;
  if ((s = check_device(&dev))) return s;
  const int64_t recv4 = plan->recv_elems / 4;
  const int grid = (int)std::min<int64_t>((recv4 + 255) / 256, (int64_t)dev.sms * 8);
  ProfScope ps("G5_pack_reduce", (cudaStream_t)stream);
  rfk::k_pack_reduce<<<std::max(grid, 1), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(staging_self), recv4, plan->world, reinterpret_cast<float4*>(recv));
  RF_CUDA_CHECK(cudaGetLastError());
  g_launches = 1;
  return ok();
}

}  // extern "C"


extern "C" {

rf_status rf_phi_row_split(int64_t n, int32_t world, int32_t rank, int64_t* row_begin, int64_t* row_end) {
  if (n <= 0 || world <= 0 || rank < 0 || rank >= world || !row_begin || !row_end)
    return fail(RF_E_INVALID, "rf_phi_row_split: bad arguments");
  // rows of 256 (the pair tile); boundary b_r = smallest tile boundary with triangle area above ≥ r/world
  const int64_t T = (n + 255) / 256;
  auto area_before = [&](int64_t tile) -> double {   // entries j ≥ i in rows [0, 256·tile)
    const double r = std::min<int64_t>(tile * 256, n);
    return r * (double)n - r * (r - 1) / 2.0;
  };
  const double total = area_before(T);
  auto boundary = [&](int32_t r) -> int64_t {
    if (r <= 0) return 0;
    if (r >= world) return T;
    const double target = total * r / world;
    int64_t lo = 0, hi = T;
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (area_before(mid) < target) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  *row_begin = std::min<int64_t>(boundary(rank) * 256, n);
  *row_end = std::min<int64_t>(boundary(rank + 1) * 256, n);
  return ok();
}

// form: 1 = EQ1 (P:1040, 18 terms), 2 = EQ2 (P:1082, 6 terms) — same epilogue, other coefficients.
static rf_status rf_phi_core(const void* X, int64_t ldx, int64_t p, int64_t n, rf_act act, double tau,
                             const rf_moments_t* mom, rf_prec prec, rf_out out, int64_t row_begin, int64_t row_end,
                             void* Phi, int64_t ldphi, void* ws, size_t ws_bytes, void* stream, int form = 1) {
  g_launches = 0;
  if (p <= 0 || n <= 0) return fail(RF_E_INVALID, "rf_phi_closed_form: p, n must be > 0");
  if (n > (int64_t)1 << 31 || p > (int64_t)1 << 31) return fail(RF_E_INVALID, "rf_phi_closed_form: sizes must be < 2^31");
  if (!valid_act(act)) return fail(RF_E_INVALID, "rf_phi_closed_form: unknown activation %d", (int)act);
  if (!valid_prec(prec)) return fail(RF_E_INVALID, "rf_phi_closed_form: unknown precision %d", (int)prec);
  if (!valid_out(out)) return fail(RF_E_INVALID, "rf_phi_closed_form: unknown output mode %d", (int)out);
  if (row_begin < 0 || row_end > n || row_begin > row_end || (row_begin % 256) != 0 ||
      (row_end != n && (row_end % 256) != 0))
    return fail(RF_E_INVALID, "rf_phi_closed_form: row range [%lld, %lld) must satisfy 0 <= begin <= end <= n, "
                "begin %% 256 == 0, end == n or end %% 256 == 0", (long long)row_begin, (long long)row_end);
  if (!std::isfinite(tau)) return fail(RF_E_INVALID, "rf_phi_closed_form: tau is not finite");
  const size_t es = esize_of(prec);
  rf_status s;
  if ((s = validate_matrix("X", X, ldx, p, es))) return s;
  int64_t tri_T = 0;
  if (out == RF_OUT_PACKED_TRI) {
    if ((s = packed_out_setup("rf_phi_closed_form", Phi, n, prec, &tri_T))) return s;
  } else if ((s = validate_output("Phi", Phi, ldphi, n, prec == RF_PREC_FP64 ? 8 : 4))) {
    return s;
  }
  const PhiPlan pl = phi_plan(p, n, prec);
  if (!ws || ws_bytes < pl.total || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(RF_E_WORKSPACE, "rf_phi_closed_form: workspace needs %zu bytes, 256-B aligned (got %zu)", pl.total,
                ws_bytes);
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  double* nrm2 = (double*)(w + pl.off_nrm2);
  double* tau_dev = (double*)(w + pl.off_tau);

  // Φ1: row norms (all n rows: columns j of every row block need ‖x_j‖²)
  if ((s = launch_rownorm(X, prec, ldx, p, n, nrm2, st))) return s;
  if (!(tau > 0.0)) {   // Lemma 1 τ̂
    double h[2];
    if ((s = tau_reduce_to_host(nrm2, n, tau_dev, st, h))) return s;
    if (h[1] != 0.0)
      return fail(RF_E_INVALID, "rf_phi_closed_form: %lld sample(s) with zero norm (v_b undefined, P:1017)",
                  (long long)h[1]);
    tau = h[0];
    if (!(tau > 0.0)) return fail(RF_E_INVALID, "rf_phi_closed_form: estimated tau is not > 0");
  }
  // Φ2: moments
  rf_moments_t mloc;
  if (mom) {
    if (std::fabs(mom->tau - tau) > 1e-12 * std::fabs(tau))
      return fail(RF_E_INVALID, "rf_phi_closed_form: mom->tau (%.17g) != tau used (%.17g)", mom->tau, tau);
    mloc = *mom;
  } else {
    rf_status ms = rf_moments(act, tau, 0, &mloc);
    if (ms) return ms;
  }
  // Φ3: per-row coefficients
  rfk::RowMoments rm;
  std::memcpy(rm.kd, mloc.kd, sizeof(rm.kd));
  rm.inv_st = 1.0 / std::sqrt(tau);
  rm.form = form;
  const int cgrid = (int)((n + 255) / 256);
  // C0(s), C1(s) coefficients of the regrouped EQ1 (rf_common.cuh), s = u_b/√τ.  EQ2 in the same
  // shape: A0 = ⟨0,0⟩ + α⟨1,1⟩, C0 = ⟨0,0⟩ + β⟨1,1⟩, A1·C1 = ⟨1,0⟩⟨0,1⟩, A2 = ⟨2,0⟩ (k_row_coef, form 2).
  const double e0 = form == 2 ? mloc.kd[0][0] - mloc.kd[1][1] : mloc.kd[0][0] - mloc.kd[1][1] + 0.5 * mloc.kd[2][2];
  const double e1 = form == 2 ? mloc.kd[1][1] : mloc.kd[1][1] - mloc.kd[2][2];
  const double e2 = form == 2 ? 0.0 : 0.5 * mloc.kd[2][2];
  const double f0 = form == 2 ? mloc.kd[0][1] : mloc.kd[0][1] - mloc.kd[1][2];
  const double f1 = form == 2 ? 0.0 : mloc.kd[1][2];
  const int full = (int)out & 1;
  if (prec == RF_PREC_FP64) {
    rfk::RowCoefD* rc = (rfk::RowCoefD*)(w + pl.off_rc);
    double* nj = (double*)(w + pl.off_nrm2o);
    {
      ProfScope ps("K1_row_coef", st);
      rfk::k_row_coef<rfk::RowCoefD, double><<<cgrid, 256, 0, st>>>(nrm2, n, rm, rc, nj);
    }
    RF_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
    rfk::SimtEq1<double, rfk::RowCoefD> e{(double*)Phi, ldphi, n, rc, nj, e0, e1, e2, f0, f1, full};
    return (s = launch_simt<double>("K6_simt_xtx_eq1", (const double*)X, ldx, (const double*)X, ldx, n, n, p, 1, (int)(row_begin / rfk::kSimtTile),
                                    (int)((row_end + rfk::kSimtTile - 1) / rfk::kSimtTile), e, st))
               ? s
               : ok();
  }
  rfk::RowCoef* rc = (rfk::RowCoef*)(w + pl.off_rc);
  float* nj = (float*)(w + pl.off_nrm2o);
  {
    ProfScope ps("K1_row_coef", st);
    rfk::k_row_coef<rfk::RowCoef, float><<<cgrid, 256, 0, st>>>(nrm2, n, rm, rc, nj);
  }
  RF_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  if (row_end <= row_begin) return ok();
  if (prec == RF_PREC_FP32) {
    rfk::SimtEq1<float, rfk::RowCoef> e{(float*)Phi, ldphi, n, rc, nj, (float)e0, (float)e1, (float)e2, (float)f0,
                                        (float)f1, full};
    return (s = launch_simt<float>("K6_simt_xtx_eq1", (const float*)X, ldx, (const float*)X, ldx, n, n, p, 1, (int)(row_begin / rfk::kSimtTile),
                                   (int)((row_end + rfk::kSimtTile - 1) / rfk::kSimtTile), e, st))
               ? s
               : ok();
  }
  // σ odd (tanh, erf, sigmoid − ½: all north-star activations) ⇒ ⟨k,d⟩ = 0 for k + d even ⇒ A0 = A2 = 0;
  // the general form stays available (RF_EQ1_GENERAL=1, tested) for non-odd σ.
  const bool odd_act = act == RF_ACT_TANH || act == RF_ACT_ERF || act == RF_ACT_SIGMOID_HALF || act == RF_ACT_SIGN ||
                       act == RF_ACT_SIN || act == RF_ACT_IDENT;
  K5Args ka{X, ldx, p, n, prec, (float*)Phi, ldphi, full, rc, nj, (float)e0, (float)e1, (float)e2, (float)f0,
            (float)f1, row_begin, row_end, w, pl, dev.sms, st, tri_T};
  if (odd_act && env_int("RF_EQ1_GENERAL", 0) == 0) return launch_k5<true>(ka);
  return launch_k5<false>(ka);
}

static rf_status phi_entry(const void* X, int64_t ldx, int64_t p, int64_t n, rf_act act, double tau,
                           const rf_moments_t* mom, rf_prec prec, rf_out out, int64_t row_begin, int64_t row_end,
                           void* Phi, int64_t ldphi, void* ws, size_t ws_bytes, void* stream, int form) {
  if (((int)out & RF_OUT_CENTER) && !(row_begin == 0 && row_end == n))
    return fail(RF_E_INVALID, "rf_phi_closed_form: centering (RF_OUT_*_CENTERED) needs the full row range [0, n)");
  rf_status s = rf_phi_core(X, ldx, p, n, act, tau, mom, prec, out, row_begin, row_end, Phi, ldphi, ws, ws_bytes,
                            stream, form);
  if (s || !((int)out & RF_OUT_CENTER)) return s;
  const int32_t launches = g_launches;
  double* cen = (double*)((char*)ws + phi_plan(p, n, prec).off_cen);
  s = prec == RF_PREC_FP64 ? center_pass<double>((double*)Phi, ldphi, n, (int)out & 1, cen, (cudaStream_t)stream)
                           : center_pass<float>((float*)Phi, ldphi, n, (int)out & 1, cen, (cudaStream_t)stream);
  g_launches += launches;
  return s ? s : ok();
}

rf_status rf_phi_closed_form(const void* X, int64_t ldx, int64_t p, int64_t n, rf_act act, double tau,
                             const rf_moments_t* mom, rf_prec prec, rf_out out, int64_t row_begin, int64_t row_end,
                             void* Phi, int64_t ldphi, void* ws, size_t ws_bytes, void* stream) {
  return phi_entry(X, ldx, p, n, act, tau, mom, prec, out, row_begin, row_end, Phi, ldphi, ws, ws_bytes, stream, 1);
}

rf_status rf_phi_eq2(const void* X, int64_t ldx, int64_t p, int64_t n, rf_act act, double tau,
                     const rf_moments_t* mom, rf_prec prec, rf_out out, int64_t row_begin, int64_t row_end,
                     void* Phi, int64_t ldphi, void* ws, size_t ws_bytes, void* stream) {
  return phi_entry(X, ldx, p, n, act, tau, mom, prec, out, row_begin, row_end, Phi, ldphi, ws, ws_bytes, stream, 2);
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------------------------
// NEXT-4: random-features kernel ridge regression on G, include/rf.h rf_ridge.
namespace {
int64_t ridge_lda(int64_t n) { return (n + 7) / 8 * 8; }
}  // namespace

extern "C" {

// Workspace: [status word, 256 B][per γ of a batch: the fp64 factor (n × lda) | the diagonal-block inverses].
static size_t ridge_per_gamma(int64_t n) {
  const size_t nblk = (size_t)((n + rfk::kRB - 1) / rfk::kRB);
  return align256((size_t)n * ridge_lda(n) * 8) + align256(nblk * rfk::kRB * rfk::kRB * 8);
}

rf_status rf_ridge_workspace_size(int64_t n_train, size_t* bytes) {
  if (!bytes) return fail(RF_E_INVALID, "bytes is NULL");
  if (n_train <= 0 || n_train > ((int64_t)1 << 31)) return fail(RF_E_INVALID, "rf_ridge: n_train must be in (0, 2^31]");
  *bytes = 256 + ridge_per_gamma(n_train);
  return ok();
}

rf_status rf_ridge(const float* G, int64_t ldg, int64_t n_train, int64_t n_test, const double* gammas,
                   int32_t n_gamma, const double* Y, int64_t ldy, int32_t nrhs, double* alpha, double* Yhat,
                   void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (!G || !Y || !alpha || !gammas) return fail(RF_E_INVALID, "rf_ridge: G, Y, alpha and gammas are required");
  if (n_train <= 0 || n_test < 0 || nrhs <= 0 || n_gamma <= 0)
    return fail(RF_E_INVALID, "rf_ridge: need n_train > 0, n_test >= 0, nrhs > 0, n_gamma > 0");
  if (n_test > 0 && !Yhat) return fail(RF_E_INVALID, "rf_ridge: Yhat is required when n_test > 0");
  if (ldg < n_train + n_test) return fail(RF_E_INVALID, "rf_ridge: ldg (%lld) < n_train + n_test", (long long)ldg);
  if (ldy < nrhs) return fail(RF_E_INVALID, "rf_ridge: ldy < nrhs");
  if ((reinterpret_cast<uintptr_t>(G) & 3) || (reinterpret_cast<uintptr_t>(Y) & 7) ||
      (reinterpret_cast<uintptr_t>(alpha) & 7) || (Yhat && (reinterpret_cast<uintptr_t>(Yhat) & 7)))
    return fail(RF_E_INVALID, "rf_ridge: misaligned pointer (G 4 B, Y / alpha / Yhat 8 B)");
  for (int g = 0; g < n_gamma; ++g)
    if (!(gammas[g] > 0.0) || !std::isfinite(gammas[g]))
      return fail(RF_E_INVALID, "rf_ridge: gamma[%d] = %g must be finite and > 0", g, gammas[g]);
  size_t need = 0;
  rf_status s;
  if ((s = rf_ridge_workspace_size(n_train, &need))) return s;
  if (!ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(RF_E_WORKSPACE, "rf_ridge: workspace needs %zu bytes, 256-B aligned (got %zu)", need, ws_bytes);
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = n_train, lda = ridge_lda(n);
  const size_t per = ridge_per_gamma(n);
  const int batch = (int)std::min<size_t>({(size_t)n_gamma, (size_t)rfk::kMaxBatch, (ws_bytes - 256) / per});
  int* info = (int*)ws;
  double* A = (double*)((char*)ws + 256);                                   // factor of batch member z at A + z·sA
  const int64_t sA = (int64_t)(per / 8);
  double* Linv = A + align256((size_t)n * lda * 8) / 8;                     // inverses of member z at Linv + z·sA
  RF_CUDA_CHECK(cudaMemsetAsync(info, 0, sizeof(int), st));
  RF_CUDA_CHECK(cudaFuncSetAttribute(rfk::k_chol_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, rfk::kPanelSmem));
  RF_CUDA_CHECK(cudaFuncSetAttribute(rfk::k_chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, rfk::kDiagSmem));
  const int nblk = (int)((n + rfk::kRB - 1) / rfk::kRB);
  auto check = [&]() -> rf_status {
    RF_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
    return RF_OK;
  };
  for (int g0 = 0; g0 < n_gamma; g0 += batch) {
    const int nz = std::min(batch, n_gamma - g0);
    rfk::RidgeBatch bt{};
    for (int z = 0; z < nz; ++z) bt.gamma[z] = gammas[g0 + z];
    bt.sA = sA;
    bt.sL = sA;
    bt.sY = n * nrhs;
    bt.sYh = n_test * nrhs;
    double* al = alpha + (int64_t)g0 * n * nrhs;
    {
      ProfScope ps("KR_build", st);
      const unsigned nt = (unsigned)((n + 31) / 32);
      rfk::k_ridge_build<<<dim3(nt, nt, nz), 256, 0, st>>>(G, ldg, n, bt, A, lda);
    }
    if ((s = check())) return s;
    // two-level blocking: 64-column sub-panels inside 256-wide panels; the sub-panel updates stay inside the
    // panel, and one K = 256 update per panel carries the trailing matrix (4× the arithmetic per byte of C)
    constexpr int kOuter = 4 * rfk::kRB;
    for (int k = 0; k < nblk; ++k) {
      {
        ProfScope ps("KR_chol_diag", st);
        rfk::k_chol_diag<<<dim3(1, 1, nz), 256, rfk::kDiagSmem, st>>>(A, lda, n, k, info,
                                                                     Linv + (int64_t)k * rfk::kRB * rfk::kRB, bt);
      }
      if ((s = check())) return s;
      const int64_t r0 = (int64_t)k * rfk::kRB, r1 = r0 + rfk::kRB, m = n - r1;
      if (m <= 0) continue;
      {
        ProfScope ps("KR_chol_panel", st);
        rfk::k_chol_panel<<<dim3((unsigned)((m + rfk::kRB - 1) / rfk::kRB), 1, nz), rfk::kRB, rfk::kPanelSmem, st>>>(
            A, lda, n, k, sA);
      }
      if ((s = check())) return s;
      const int64_t c0 = r0 / kOuter * kOuter, c1 = std::min<int64_t>(c0 + kOuter, n);   // this 256-wide panel
      const double* Pn = A + r1 * lda + r0;                  // sub-panel rows r1.., columns r0 .. r0 + 64
      if (r1 < c1) {   // inside the panel: columns r1 .. c1
        if ((s = launch_simt<double>("KR_chol_update", Pn, lda, Pn, lda, m, c1 - r1, rfk::kRB, 2, 0,
                                     (int)((m + rfk::kSimtTile - 1) / rfk::kSimtTile),
                                     rfk::SimtCholUpd{A, lda, r1, m, sA, c1 - r1}, st, nz, sA, sA)))
          return s;
      }
      if (r1 == c1 && c1 < n) {   // panel done: the trailing matrix from columns c0 .. c1 (K = 256)
        const int64_t mt = n - c1;
        const double* Po = A + c1 * lda + c0;
        if ((s = launch_simt<double>("KR_chol_update", Po, lda, Po, lda, mt, mt, c1 - c0, 2, 0,
                                     (int)((mt + rfk::kSimtTile - 1) / rfk::kSimtTile),
                                     rfk::SimtCholUpd{A, lda, c1, mt, sA, mt}, st, nz, sA, sA)))
          return s;
      }
    }
    // α = L^{-T} L^{-1} Y, in place in alpha (row-major n × nrhs per γ)
    for (int z = 0; z < nz; ++z)
      RF_CUDA_CHECK(cudaMemcpy2DAsync(al + (int64_t)z * n * nrhs, (size_t)nrhs * 8, Y, (size_t)ldy * 8,
                                      (size_t)nrhs * 8, (size_t)n, cudaMemcpyDeviceToDevice, st));
    const unsigned rw = (unsigned)((nrhs + 3) / 4);   // 4 right-hand sides per CTA of the block solves
    for (int k = 0; k < nblk; ++k) {
      {
        ProfScope ps("KR_trsv", st);
        rfk::k_trsv_fwd<<<dim3(rw, 1, nz), 256, 0, st>>>(Linv + (int64_t)k * rfk::kRB * rfk::kRB, n, k, al, nrhs,
                                                         nrhs, bt);
      }
      if ((s = check())) return s;
      const int64_t below = n - (int64_t)(k + 1) * rfk::kRB;
      if (below > 0) {
        {
          ProfScope ps("KR_gemv", st);
          const unsigned gb = (unsigned)std::min<int64_t>((below + 7) / 8, (int64_t)dev.sms * 8);
          rfk::k_gemv_fwd<<<dim3(gb, 1, nz), 256, 0, st>>>(A, lda, n, k, al, nrhs, nrhs, bt);
        }
        if ((s = check())) return s;
      }
    }
    for (int k = nblk - 1; k >= 0; --k) {
      {
        ProfScope ps("KR_trsv", st);
        rfk::k_trsv_bwd<<<dim3(rw, 1, nz), 256, 0, st>>>(Linv + (int64_t)k * rfk::kRB * rfk::kRB, n, k, al, nrhs,
                                                         nrhs, bt);
      }
      if ((s = check())) return s;
      const int64_t r0 = (int64_t)k * rfk::kRB;
      if (r0 > 0) {
        {
          ProfScope ps("KR_gemv", st);
          const unsigned gb = (unsigned)std::min<int64_t>((r0 + 255) / 256, (int64_t)dev.sms * 4);
          rfk::k_axpy_bwd<<<dim3(gb, 1, nz), 256, 0, st>>>(A, lda, n, k, al, nrhs, nrhs, bt);
        }
        if ((s = check())) return s;
      }
    }
    if (n_test > 0) {
      {
        ProfScope ps("KR_predict", st);
        const unsigned gb = (unsigned)std::min<int64_t>((n_test + 127) / 128, (int64_t)dev.sms * 8);
        rfk::k_ridge_predict<<<dim3(gb, 1, nz), 128, 0, st>>>(G, ldg, n_train, n_test, al, nrhs, nrhs,
                                                               Yhat + (int64_t)g0 * n_test * nrhs, nrhs, bt);
      }
      if ((s = check())) return s;
    }
  }
  // factorisation status (one host sync, through the mapped mailbox)
  HostMailbox* mb = nullptr;
  if ((s = host_mailbox(&mb))) return s;
  volatile int* hi = reinterpret_cast<volatile int*>(mb->h);
  hi[0] = -1;
  rfk::k_publish_u32<<<1, 1, 0, st>>>(info, hi);
  if ((s = check())) return s;
  RF_CUDA_CHECK(cudaEventRecord(mb->ev, st));
  RF_CUDA_CHECK(cudaEventSynchronize(mb->ev));
  if (hi[0] != 0)
    return fail(RF_E_NONFINITE, "rf_ridge: G_train + gamma*I is not positive definite (pivot %d)", (int)hi[0]);
  return ok();
}

}  // extern "C"

