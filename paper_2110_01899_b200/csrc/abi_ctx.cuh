// Part of the single translation unit api.cu: the context (rf_ctx_*), its tuning options, and the multi-GPU G —
// step G5 of SURVEY.md §8(a): canonical tile ownership (rf_tile_map), the peer-memory exchange (product path) and the
// NCCL exchange (baseline), both inside one collective rf_gram call (include/rf.h "G5").  G is a sum over the m
// features (Eq. def_Gram), so each rank's partial over its W rows is summed tile by tile across ranks.
#pragma once
#include <dlfcn.h>

namespace {

// ------------------------------------------------------------------------------- G5 plan: a function of (n, world)
constexpr int kPackArrivals = 2 * 8;   // chunk-counter arrivals per K4 pair tile: 2 CTAs × 8 epilogue warps

struct G5Plan {
  int T = 0, C = 0, world = 1;
  int crow[rfk::kMaxChunks + 1] = {};       // first row tile of chunk c
  int64_t tiles[rfk::kMaxChunks] = {};      // upper 256-tiles (I, J ≥ I) with I in chunk c
  int64_t slots[rfk::kMaxChunks] = {};      // ⌈tiles / world⌉: receive slots per rank in chunk c
  int64_t soff[rfk::kMaxChunks + 1] = {}, roff[rfk::kMaxChunks + 1] = {};
  int64_t send_elems = 0, recv_elems = 0;
};

inline int64_t tri_rows_area(int64_t r, int64_t T) { return r * T - r * (r - 1) / 2; }   // tiles in rows [0, r)

rf_status build_g5_plan(int64_t n, int32_t world, G5Plan* pl) {
  if (n <= 0 || n >= (int64_t(1) << 31)) return fail(RF_E_INVALID, "G5: n must be in (0, 2^31)");
  if (world < 1 || world > 4096) return fail(RF_E_INVALID, "G5: world must be in [1, 4096]");
  *pl = G5Plan();
  const int T = (int)((n + 255) / 256);
  const int G = (T + kPackGm - 1) / kPackGm;
  const int C = std::min(rfk::kMaxChunks, G);
  pl->T = T;
  pl->C = C;
  pl->world = world;
  const double total = (double)tri_rows_area(T, T);
  int g = 0;
  for (int c = 0; c < C; ++c) {
    pl->crow[c] = std::min(g * kPackGm, T);
    int ge = g + 1;
    if (c == C - 1) {
      ge = G;
    } else {
      const double target = total * (c + 1) / C;
      while (ge < G - (C - 1 - c) && (double)tri_rows_area(std::min(ge * kPackGm, T), T) < target) ++ge;
    }
    g = ge;
  }
  pl->crow[C] = T;
  int64_t so = 0, ro = 0;
  for (int c = 0; c < C; ++c) {
    pl->tiles[c] = tri_rows_area(pl->crow[c + 1], T) - tri_rows_area(pl->crow[c], T);
    pl->slots[c] = (pl->tiles[c] + world - 1) / world;
    pl->soff[c] = so;
    pl->roff[c] = ro;
    so += pl->slots[c] * world * (int64_t)(RF_PACK_TILE * RF_PACK_TILE);
    ro += pl->slots[c] * (int64_t)(RF_PACK_TILE * RF_PACK_TILE);
  }
  pl->soff[C] = so;
  pl->roff[C] = ro;
  pl->send_elems = so;
  pl->recv_elems = ro;
  return RF_OK;
}

// K4 pair tiles whose row tile lies in chunk c (BN = 512: row tile I needs column tiles J2 ≥ I/2 of ⌈n/512⌉; BN = 256:
// J ≥ I) — the counter target of chunk c is kPackArrivals times this, per call.
int64_t chunk_pair_tiles(const G5Plan& pl, int c, int64_t n, int bn) {
  const int64_t tn = (n + bn - 1) / bn;
  int64_t k = 0;
  for (int I = pl.crow[c]; I < pl.crow[c + 1]; ++I) k += tn - (bn == 512 ? I / 2 : I);
  return k;
}

// ------------------------------------------------------------------------------- NCCL, taken from the process
struct NcclId {
  char internal[128];
};
struct NcclApi {
  bool ok = false;
  int (*get_unique_id)(NcclId*) = nullptr;
  int (*comm_init_rank)(void**, int, NcclId, int) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*comm_get_async_error)(void*, int*) = nullptr;
  int (*reduce_scatter)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
};
constexpr int kNcclFloat32 = 7, kNcclSum = 0, kNcclSuccess = 0, kNcclInProgress = 7;

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the NCCL torch already loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return;
    api.get_unique_id = (int (*)(NcclId*))dlsym(h, "ncclGetUniqueId");
    api.comm_init_rank = (int (*)(void**, int, NcclId, int))dlsym(h, "ncclCommInitRank");
    api.comm_destroy = (int (*)(void*))dlsym(h, "ncclCommDestroy");
    api.comm_get_async_error = (int (*)(void*, int*))dlsym(h, "ncclCommGetAsyncError");
    api.reduce_scatter =
        (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclReduceScatter");
    api.error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_get_async_error &&
             api.reduce_scatter && api.error_string;
  });
  return api;
}

rf_status nccl_fail(const char* what, int r) {
  return fail(RF_E_NCCL, "%s: %s (%d)", what, nccl().error_string ? nccl().error_string(r) : "?", r);
}

// ------------------------------------------------------------------------------- attach helpers
rf_status create_g5_streams(rf_ctx* c, bool peers);

rf_status attach_nccl_common(rf_ctx* c, int32_t rank, int32_t world) {
  rf_status s;
  if ((s = create_g5_streams(c, false))) return s;
  c->rank = rank;
  c->world = world;
  c->mode = 1;
  c->epoch = 0;
  return RF_OK;
}

rf_status check_attachable(const rf_ctx* c, int32_t rank, int32_t world, const char* fn) {
  if (!c) return fail(RF_E_INVALID, "%s: ctx is NULL (collectives need an explicit context)", fn);
  if (c->mode != 0) return fail(RF_E_INVALID, "%s: a collective is already attached to this context", fn);
  if (world < 1 || rank < 0 || rank >= world) return fail(RF_E_INVALID, "%s: need 0 <= rank < world", fn);
  return RF_OK;
}

struct DeviceGuard {   // make `dev` current for a set-up call
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// The flags after the staging slots: arrived[chunk][source] (source's tiles of that chunk have landed here),
// freed[source] (that owner has summed the previous call out of its staging buffer).  Values are call epochs.
constexpr int kFlagWords = (rfk::kMaxChunks + 1) * RF_MAX_PEERS;
uint32_t* flags_of(void* base, int world, int64_t recv_cap) {
  return (uint32_t*)((char*)base + (size_t)world * recv_cap * 4);
}
inline uint32_t* arrived_flag(uint32_t* flags, int chunk, int src) { return flags + chunk * RF_MAX_PEERS + src; }
inline uint32_t* freed_flag(uint32_t* flags, int src) { return flags + rfk::kMaxChunks * RF_MAX_PEERS + src; }

// Per-chunk counter targets of this call: each chunk's counter grows by kPackArrivals per K4 pair tile of the chunk;
// the running sums (not epoch × tiles) stay right when n changes between calls on one context.
void advance_sync_targets(rf_ctx* c, const G5Plan& pl, int64_t n, int bn) {
  for (int k = 0; k < pl.C; ++k) c->sync_target[k] += (uint32_t)(kPackArrivals * chunk_pair_tiles(pl, k, n, bn));
}

rf_status create_g5_streams(rf_ctx* c, bool peers) {
  RF_CUDA_CHECK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  RF_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
  RF_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  if (peers) {
    // the per-chunk flags and sums run beside K4, whose CTAs take the SM's maximum shared-memory carveout: ask for
    // the same carveout so the block scheduler can place them next to a K4 CTA (with the default preference the
    // one-thread flag kernel waited for K4 to end, and every chunk's sum with it)
    RF_CUDA_CHECK(cudaFuncSetAttribute(rfk::k_pack_reduce, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       (int)cudaSharedmemCarveoutMaxShared));
    RF_CUDA_CHECK(cudaFuncSetAttribute(rfk::k_signal, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       (int)cudaSharedmemCarveoutMaxShared));
    RF_CUDA_CHECK(cudaStreamCreateWithFlags(&c->red_stream, cudaStreamNonBlocking));
    RF_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_sig, cudaEventDisableTiming));
  }
  void* p = nullptr;
  RF_CUDA_CHECK(cudaMalloc(&p, rfk::kMaxChunks * sizeof(uint32_t)));
  RF_CUDA_CHECK(cudaMemset(p, 0, rfk::kMaxChunks * sizeof(uint32_t)));
  c->sync = (uint32_t*)p;
  for (int k = 0; k < rfk::kMaxChunks; ++k) c->sync_target[k] = 0;
  return RF_OK;
}

rf_status signal(const char* name, uint32_t* const* dst, int count, uint32_t value, cudaStream_t st) {
  if (count <= 0) return RF_OK;
  rfk::SignalArgs a{};
  for (int i = 0; i < count; ++i) a.dst[i] = dst[i];
  a.count = count;
  a.value = value;
  ProfScope ps(name, st);
  rfk::k_signal<<<1, 1, 0, st>>>(a);
  RF_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  return RF_OK;
}

rf_status stream_wait_geq(cudaStream_t st, const uint32_t* addr, uint32_t value) {
  PFN_wait32h fn = wait32_h();
  if (!fn) return fail(RF_E_CUDA, "cuStreamWaitValue32 entry point unavailable");
  CUresult r = fn((CUstream)st, (CUdeviceptr)(uintptr_t)addr, value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(RF_E_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  return RF_OK;
}

// ------------------------------------------------------------------------------- the collective rf_gram
rf_status gram_collective(const void* X, int64_t ldx, const void* W, int64_t ldw, int64_t p, int64_t n, int64_t m_local,
                          int64_t m_total, rf_act act, rf_prec prec, float* recv, void* ws, size_t ws_bytes,
                          cudaStream_t st) {
  g_launches = 0;
  rf_ctx* c = g_ctx;
  if (!c || c->mode == 0)
    return fail(RF_E_INVALID, "rf_gram: RF_OUT_PACKED_TILES needs a context with a collective attached "
                "(rf_ctx_init_nccl / rf_ctx_attach_nccl / rf_ctx_attach_peers)");
  if (p <= 0 || n <= 0 || m_local <= 0 || m_total < m_local)
    return fail(RF_E_INVALID, "rf_gram: need p, n, m_local > 0 and m_total >= m_local");
  if (p >= (int64_t(1) << 31) || n >= (int64_t(1) << 31) || m_local >= (int64_t(1) << 31))
    return fail(RF_E_INVALID, "rf_gram: sizes must be < 2^31");
  if (!valid_act(act)) return fail(RF_E_INVALID, "rf_gram: unknown activation %d", (int)act);
  const bool peers = c->mode == 2;
  if (!(prec == RF_PREC_BF16 || prec == RF_PREC_TF32 || (prec == RF_PREC_3XTF32 && !peers)))
    return fail(RF_E_INVALID, "rf_gram: RF_OUT_PACKED_TILES takes BF16 or TF32 (3XTF32 on NCCL only: its K-chunked "
                "accumulation would read tiles back over NVLink)");
  if (!recv || (reinterpret_cast<uintptr_t>(recv) & 15)) return fail(RF_E_INVALID, "rf_gram: G (recv) must be 16-B aligned");
  const size_t es = esize_of(prec);
  rf_status s;
  if ((s = validate_matrix("X", X, ldx, p, es))) return s;
  if ((s = validate_matrix("W", W, ldw, p, es))) return s;
  G5Plan pl;
  if ((s = build_g5_plan(n, c->world, &pl))) return s;
  const GramPlan gp = gram_plan(p, n, m_local, prec);
  const size_t off_send = align256(gp.total);
  const size_t need = peers ? gp.total : off_send + (size_t)pl.send_elems * 4;
  if (!ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(RF_E_WORKSPACE, "rf_gram: workspace needs %zu bytes, 256-B aligned (got %zu; rf_workspace_size)", need,
                ws_bytes);
  DevInfo dev;
  if ((s = check_device(&dev))) return s;
  rfk::PackDev dv;
  std::memset(&dv, 0, sizeof(dv));
  dv.T = pl.T;
  dv.nchunks = pl.C;
  dv.world = c->world;
  dv.self = c->rank;
  for (int k = 0; k <= pl.C; ++k) {
    dv.crow[k] = pl.crow[k];
    dv.soff[k] = pl.soff[k];
    dv.roff[k] = pl.roff[k];
    if (k < pl.C) dv.slots[k] = pl.slots[k];
  }
  dv.recv_elems = pl.recv_elems;
  char* w = (char*)ws;
  int32_t launches = 0;

  if (!peers) {   // ---------------- NCCL: packed send buffer, per-chunk counters, chunked reduce-scatter on comm stream
    const NcclApi& api = nccl();
    if (!api.ok) return fail(RF_E_NCCL, "rf_gram: NCCL symbols not found in the process");
    int aerr = 0;
    int r = api.comm_get_async_error(c->comm, &aerr);
    if (r != kNcclSuccess) return nccl_fail("ncclCommGetAsyncError", r);
    if (aerr != kNcclSuccess && aerr != kNcclInProgress) return nccl_fail("NCCL communicator async error", aerr);
    if (c->comm_pending) RF_CUDA_CHECK(cudaStreamWaitEvent(st, c->ev_done, 0));   // earlier RS still read `send`
    const uint32_t epoch = ++c->epoch;
    dv.p2p = 0;
    dv.send = (float*)(w + off_send);
    dv.sync = c->sync;
    const int sms = std::max(2, (usable_sms(dev.sms) - (int)opt(RF_OPT_COMM_SMS)) & ~1);
    RF_CUDA_CHECK(cudaEventRecord(c->ev_start, st));
    GramTcArgs ga{X, ldx, W, ldw, p, n, m_local, m_total, act, 0, nullptr, n, w, gp, sms, st, &dv, 0};
    if ((s = gram_tc_dispatch(ga, prec))) return s;
    launches = g_launches;
    RF_CUDA_CHECK(cudaStreamWaitEvent(c->comm_stream, c->ev_start, 0));
    advance_sync_targets(c, pl, n, prec == RF_PREC_3XTF32 ? 256 : 512);
    (void)epoch;
    for (int k = 0; k < pl.C; ++k) {
      if ((s = stream_wait_geq(c->comm_stream, c->sync + k, c->sync_target[k]))) return s;   // wrap-safe GEQ
      r = api.reduce_scatter(dv.send + pl.soff[k], recv + pl.roff[k], (size_t)pl.slots[k] * RF_PACK_TILE * RF_PACK_TILE,
                             kNcclFloat32, kNcclSum, c->comm, c->comm_stream);
      if (r != kNcclSuccess) return nccl_fail("ncclReduceScatter", r);
    }
    RF_CUDA_CHECK(cudaEventRecord(c->ev_done, c->comm_stream));
    RF_CUDA_CHECK(cudaStreamWaitEvent(st, c->ev_done, 0));
    c->comm_pending = true;
    g_launches = launches;
    return ok();
  }

  // ---------------- PEERS: K4 stores into the owners' staging buffers; device epoch flags order the owner-side sum.
  // Chunk-pipelined: K4 bumps the chunk counter after each pair tile's stores (system-scope fence first); on the
  // comm stream, chunk c's arrival flag goes to every owner once its counter is complete; on the reduce stream, chunk
  // c is summed once every source's flag for it is up.  Chunks complete in raster order, so the owner-side sum of
  // chunk c runs beside K4's later chunks and only the last chunk's sum is left after K4.
  if (!c->connected) return fail(RF_E_INVALID, "rf_gram: peers attached but not connected (rf_ctx_open_peers)");
  if (pl.recv_elems > c->recv_cap)
    return fail(RF_E_INVALID, "rf_gram: n = %lld exceeds the n_max the peers were attached for", (long long)n);
  const int R = c->world, me = c->rank;
  uint32_t* mine = flags_of(c->stage, R, c->recv_cap);
  const int phases = (int)opt(RF_OPT_G5_PHASES);
  // both halves in one call: the sums run on the reduce stream beside K4 (RF_OPT_G5_PIPE = 0: after K4, on the
  // caller's stream — the round-2 first cut, kept for A/B runs)
  const bool piped = phases == 3 && opt(RF_OPT_G5_PIPE) != 0;
  uint32_t* dst[RF_MAX_PEERS];
  if (phases & 1) {
    const uint32_t epoch = ++c->epoch;
    for (int o = 0; o < R; ++o)   // owner o has summed the previous call's tiles out of its staging buffer
      if (o != me && (s = stream_wait_geq(st, freed_flag(mine, o), epoch - 1))) return s;
    RF_CUDA_CHECK(cudaEventRecord(c->ev_start, st));
    dv.p2p = 1;
    dv.sync = c->sync;
    for (int o = 0; o < R; ++o) dv.peer[o] = c->peer[o];
    GramTcArgs ga{X, ldx, W, ldw, p, n, m_local, m_total, act, 0, nullptr, n, w, gp, usable_sms(dev.sms), st, &dv, 0};
    if ((s = gram_tc_dispatch(ga, prec))) return s;
    launches = g_launches;
    advance_sync_targets(c, pl, n, 512);
    RF_CUDA_CHECK(cudaStreamWaitEvent(c->comm_stream, c->ev_start, 0));
    for (int k = 0; k < pl.C; ++k) {   // chunk k's stores have landed (fenced) → arrived[k][me] at every owner
      if ((s = stream_wait_geq(c->comm_stream, c->sync + k, c->sync_target[k]))) return s;
      for (int o = 0; o < R; ++o) dst[o] = arrived_flag(c->peer_flags[o], k, me);
      g_launches = 0;
      if ((s = signal("G5_signal_arrived", dst, R, epoch, c->comm_stream))) return s;
      launches += g_launches;
    }
    RF_CUDA_CHECK(cudaEventRecord(c->ev_sig, c->comm_stream));
    if (!piped) RF_CUDA_CHECK(cudaStreamWaitEvent(st, c->ev_sig, 0));
  }
  if (!(phases & 2)) {
    g_launches = launches;
    return ok();
  }
  const uint32_t epoch = c->epoch;
  cudaStream_t rs = st;
  if (piped) {   // after st's earlier work (readers of recv), not after K4
    rs = c->red_stream;
    RF_CUDA_CHECK(cudaStreamWaitEvent(rs, c->ev_start, 0));
  }
  const int64_t stride4 = pl.recv_elems / 4;
  for (int k = 0; k < pl.C; ++k) {
    for (int q = 0; q < R; ++q)   // every source's tiles of chunk k have landed in my staging buffer
      if ((s = stream_wait_geq(rs, arrived_flag(mine, k, q), epoch))) return s;
    const int64_t off4 = pl.roff[k] / 4, cnt4 = (pl.roff[k + 1] - pl.roff[k]) / 4;
    if (cnt4 <= 0) continue;
    constexpr int kT = rfk::kReduceThreads;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cnt4 + kT - 1) / kT, (int64_t)dev.sms * 8));
    ProfScope ps("G5_pack_reduce", rs);
    rfk::k_pack_reduce<<<grid, kT, 0, rs>>>(reinterpret_cast<const float4*>(c->stage), stride4, off4, cnt4, R,
                                              reinterpret_cast<float4*>(recv));
    RF_CUDA_CHECK(cudaGetLastError());
    ++launches;
  }
  int k = 0;
  for (int q = 0; q < R; ++q)
    if (q != me) dst[k++] = freed_flag(c->peer_flags[q], me);                        // freed[me] at every source
  g_launches = 0;
  if ((s = signal("G5_signal_freed", dst, k, epoch, rs))) return s;
  launches += g_launches;
  if (piped) {
    RF_CUDA_CHECK(cudaEventRecord(c->ev_done, rs));
    RF_CUDA_CHECK(cudaStreamWaitEvent(st, c->ev_done, 0));
    RF_CUDA_CHECK(cudaStreamWaitEvent(st, c->ev_sig, 0));
  }
  g_launches = launches;
  return ok();
}

}  // namespace

extern "C" {

rf_status rf_ctx_create(int device, rf_ctx** out) {
  if (!out) return fail(RF_E_INVALID, "rf_ctx_create: out is NULL");
  *out = nullptr;
  if (!rf_device_supported(device))
    return fail(RF_E_UNSUPPORTED, "rf_ctx_create: device %d is not an sm_100 (B200) device", device);
  rf_ctx* c = new rf_ctx();
  rf_status s = ctx_init(c, device);
  if (s) {
    delete c;
    return s;
  }
  *out = c;
  return ok();
}

void rf_ctx_destroy(rf_ctx* c) {
  if (!c) return;
  DeviceGuard dg(c->device);
  if (c->comm && c->own_comm && nccl().ok) nccl().comm_destroy(c->comm);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->ev_sig) cudaEventDestroy(c->ev_sig);
  if (c->red_stream) cudaStreamDestroy(c->red_stream);
  if (c->sync) cudaFree(c->sync);
  for (int r = 0; r < RF_MAX_PEERS; ++r)
    if (c->opened[r]) cudaIpcCloseMemHandle(c->opened[r]);
  if (c->stage) cudaFree(c->stage);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
}

rf_status rf_ctx_set_option(rf_ctx* c, rf_opt o, int64_t v) {
  if (!c) return fail(RF_E_INVALID, "rf_ctx_set_option: ctx is NULL");
  if ((int)o < 0 || (int)o >= RF_OPT_COUNT) return fail(RF_E_INVALID, "rf_ctx_set_option: unknown option %d", (int)o);
  bool okv = true;
  switch (o) {
    case RF_OPT_K3_HYBRID: case RF_OPT_K4_HYBRID: case RF_OPT_K4_CL8: case RF_OPT_EQ1_GENERAL: case RF_OPT_VERBOSE:
      okv = v == 0 || v == 1; break;
    case RF_OPT_K4_SPLIT_R100: case RF_OPT_K3_SPLIT_R100: okv = v >= 50 && v <= 400; break;
    case RF_OPT_LOCK_W: case RF_OPT_KCHUNK: case RF_OPT_MAX_SMS: okv = v >= 0 && v < (1 << 20); break;
    case RF_OPT_LOCK_KS: okv = v >= 1 && v < (1 << 20); break;
    case RF_OPT_K5_WIDE: okv = v >= -1 && v <= 1; break;
    case RF_OPT_COMM_SMS: okv = v >= 0 && v <= 64; break;
    case RF_OPT_G5_PHASES: okv = v >= 1 && v <= 3; break;
    case RF_OPT_K4_DYNAMIC: case RF_OPT_K5_DYNAMIC: case RF_OPT_G5_PIPE: okv = v == 0 || v == 1; break;
    case RF_OPT_K5_ARES: okv = v >= 0 && v <= 3; break;
    default: break;
  }
  if (!okv) return fail(RF_E_INVALID, "rf_ctx_set_option: value %lld out of range for option %d", (long long)v, (int)o);
  c->opts[o] = v;
  return ok();
}

rf_status rf_ctx_get_option(const rf_ctx* c, rf_opt o, int64_t* v) {
  if (!c || !v) return fail(RF_E_INVALID, "rf_ctx_get_option: NULL argument");
  if ((int)o < 0 || (int)o >= RF_OPT_COUNT) return fail(RF_E_INVALID, "rf_ctx_get_option: unknown option %d", (int)o);
  *v = c->opts[o];
  return ok();
}

rf_status rf_tile_map(int64_t n, int32_t tile, int32_t world, int32_t rank, int64_t* tiles_owned, int64_t* ij) {
  if (tile != RF_PACK_TILE) return fail(RF_E_INVALID, "rf_tile_map: tile must be %d", RF_PACK_TILE);
  if (!tiles_owned) return fail(RF_E_INVALID, "rf_tile_map: tiles_owned is NULL");
  G5Plan pl;
  rf_status s = build_g5_plan(n, world, &pl);
  if (s) return s;
  if (rank < 0 || rank >= world) return fail(RF_E_INVALID, "rf_tile_map: rank out of range");
  *tiles_owned = pl.recv_elems / (RF_PACK_TILE * RF_PACK_TILE);
  if (!ij) return ok();
  int64_t k = 0;
  for (int c = 0; c < pl.C; ++c) {
    // walk the chunk's tiles row-major; tile u belongs to rank u mod world
    int I = pl.crow[c], J = I;
    int64_t u = 0;
    for (int64_t slot = 0; slot < pl.slots[c]; ++slot, ++k) {
      const int64_t want = slot * world + rank;
      if (want >= pl.tiles[c]) {
        ij[2 * k] = ij[2 * k + 1] = -1;
        continue;
      }
      while (u < want) {   // advance (I, J) by want − u tiles
        const int64_t left = pl.T - J;            // tiles remaining in row I from J
        if (want - u < left) {
          J += (int)(want - u);
          u = want;
        } else {
          u += left;
          ++I;
          J = I;
        }
      }
      ij[2 * k] = I;
      ij[2 * k + 1] = J;
    }
  }
  return ok();
}

rf_status rf_nccl_get_unique_id(uint8_t id128[128]) {
  if (!id128) return fail(RF_E_INVALID, "rf_nccl_get_unique_id: NULL output");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(RF_E_NCCL, "rf_nccl_get_unique_id: NCCL (libnccl.so.2) not available in this process");
  NcclId id;
  int r = api.get_unique_id(&id);
  if (r != kNcclSuccess) return nccl_fail("ncclGetUniqueId", r);
  std::memcpy(id128, id.internal, 128);
  return ok();
}

rf_status rf_ctx_init_nccl(rf_ctx* c, const uint8_t id128[128], int32_t rank, int32_t world) {
  rf_status s;
  if ((s = check_attachable(c, rank, world, "rf_ctx_init_nccl"))) return s;
  if (!id128) return fail(RF_E_INVALID, "rf_ctx_init_nccl: id is NULL");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(RF_E_NCCL, "rf_ctx_init_nccl: NCCL (libnccl.so.2) not available in this process");
  DeviceGuard dg(c->device);
  NcclId id;
  std::memcpy(id.internal, id128, 128);
  void* comm = nullptr;
  int r = api.comm_init_rank(&comm, world, id, rank);
  if (r != kNcclSuccess) return nccl_fail("ncclCommInitRank", r);
  c->comm = comm;
  c->own_comm = true;
  if ((s = attach_nccl_common(c, rank, world))) return s;
  return ok();
}

rf_status rf_ctx_attach_nccl(rf_ctx* c, void* comm, int32_t rank, int32_t world) {
  rf_status s;
  if ((s = check_attachable(c, rank, world, "rf_ctx_attach_nccl"))) return s;
  if (!comm) return fail(RF_E_INVALID, "rf_ctx_attach_nccl: comm is NULL");
  if (!nccl().ok) return fail(RF_E_NCCL, "rf_ctx_attach_nccl: NCCL (libnccl.so.2) not available in this process");
  DeviceGuard dg(c->device);
  c->comm = comm;
  c->own_comm = false;
  if ((s = attach_nccl_common(c, rank, world))) return s;
  return ok();
}

rf_status rf_ctx_attach_peers(rf_ctx* c, int32_t rank, int32_t world, int64_t n_max) {
  rf_status s;
  if ((s = check_attachable(c, rank, world, "rf_ctx_attach_peers"))) return s;
  if (world > RF_MAX_PEERS) return fail(RF_E_INVALID, "rf_ctx_attach_peers: world > %d", RF_MAX_PEERS);
  G5Plan pl;
  if ((s = build_g5_plan(n_max, world, &pl))) return s;
  DeviceGuard dg(c->device);
  // room for the receive slots of any n ≤ n_max (padding differs by at most one slot per chunk and owner)
  c->recv_cap = pl.recv_elems + (int64_t)rfk::kMaxChunks * RF_PACK_TILE * RF_PACK_TILE;
  c->stage_bytes = (size_t)world * c->recv_cap * 4 + kFlagWords * sizeof(uint32_t);
  void* p = nullptr;
  RF_CUDA_CHECK(cudaMalloc(&p, c->stage_bytes));   // its own allocation: the IPC handle names exactly this buffer
  RF_CUDA_CHECK(cudaMemset(p, 0, c->stage_bytes));
  c->stage = p;
  if ((s = create_g5_streams(c, true))) return s;
  c->rank = rank;
  c->world = world;
  c->mode = 2;
  c->epoch = 0;
  c->peer[rank] = (float*)p;
  c->peer_flags[rank] = flags_of(p, world, c->recv_cap);
  c->connected = world == 1;
  return ok();
}

rf_status rf_ctx_peer_handle(const rf_ctx* c, uint8_t handle64[64]) {
  if (!c || !handle64) return fail(RF_E_INVALID, "rf_ctx_peer_handle: NULL argument");
  if (c->mode != 2) return fail(RF_E_INVALID, "rf_ctx_peer_handle: no peers attached (rf_ctx_attach_peers)");
  DeviceGuard dg(c->device);
  cudaIpcMemHandle_t h;
  RF_CUDA_CHECK(cudaIpcGetMemHandle(&h, c->stage));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, 64);
  return ok();
}

rf_status rf_ctx_peer_base(const rf_ctx* c, void** base) {
  if (!c || !base) return fail(RF_E_INVALID, "rf_ctx_peer_base: NULL argument");
  if (c->mode != 2) return fail(RF_E_INVALID, "rf_ctx_peer_base: no peers attached (rf_ctx_attach_peers)");
  *base = c->stage;
  return ok();
}

rf_status rf_ctx_connect_peers(rf_ctx* c, void* const* bases) {
  if (!c || !bases) return fail(RF_E_INVALID, "rf_ctx_connect_peers: NULL argument");
  if (c->mode != 2) return fail(RF_E_INVALID, "rf_ctx_connect_peers: no peers attached (rf_ctx_attach_peers)");
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    if (!bases[r] || (reinterpret_cast<uintptr_t>(bases[r]) & 255))
      return fail(RF_E_INVALID, "rf_ctx_connect_peers: base of rank %d is not a staging allocation", r);
  }
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    c->peer[r] = (float*)bases[r];
    c->peer_flags[r] = flags_of(bases[r], c->world, c->recv_cap);
  }
  c->connected = true;
  return ok();
}

rf_status rf_ctx_open_peers(rf_ctx* c, const uint8_t* handles64) {
  if (!c || !handles64) return fail(RF_E_INVALID, "rf_ctx_open_peers: NULL argument");
  if (c->mode != 2) return fail(RF_E_INVALID, "rf_ctx_open_peers: no peers attached (rf_ctx_attach_peers)");
  DeviceGuard dg(c->device);
  void* bases[RF_MAX_PEERS] = {};
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) {
      bases[r] = c->stage;
      continue;
    }
    if (!c->opened[r]) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles64 + 64 * r, 64);
      RF_CUDA_CHECK(cudaIpcOpenMemHandle(&c->opened[r], h, cudaIpcMemLazyEnablePeerAccess));
    }
    bases[r] = c->opened[r];
  }
  return rf_ctx_connect_peers(c, bases);
}

rf_status rf_ctx_collective(const rf_ctx* c, int32_t* rank, int32_t* world, int32_t* mode) {
  if (!c) return fail(RF_E_INVALID, "rf_ctx_collective: ctx is NULL");
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (mode) *mode = c->mode;
  return ok();
}

rf_status rf_workspace_size(const rf_ctx* c, int32_t op, int64_t p, int64_t n, int64_t m_local, rf_prec prec,
                            rf_out out, size_t* bytes) {
  if (!bytes) return fail(RF_E_INVALID, "rf_workspace_size: bytes is NULL");
  if (!valid_prec(prec)) return fail(RF_E_INVALID, "rf_workspace_size: unknown precision %d", (int)prec);
  if (p <= 0 || n <= 0) return fail(RF_E_INVALID, "rf_workspace_size: p, n must be > 0");
  if (op == 1) {
    *bytes = phi_plan(p, n, prec).total;
    return ok();
  }
  if (op != 0) return fail(RF_E_INVALID, "rf_workspace_size: op must be 0 (rf_gram) or 1 (rf_phi_closed_form)");
  if (m_local <= 0) return fail(RF_E_INVALID, "rf_workspace_size: m_local must be > 0");
  const size_t base = gram_plan(p, n, m_local, prec).total;
  if (out == RF_OUT_PACKED_TILES && c && c->mode == 1) {
    G5Plan pl;
    rf_status s = build_g5_plan(n, c->world, &pl);
    if (s) return s;
    *bytes = align256(base) + (size_t)pl.send_elems * 4;
  } else {
    *bytes = base;
  }
  return ok();
}

}  // extern "C"
