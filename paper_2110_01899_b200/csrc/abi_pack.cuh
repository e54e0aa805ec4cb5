// Part of the single translation unit api.cu.
#pragma once

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
