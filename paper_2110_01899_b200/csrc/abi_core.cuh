// Part of the single translation unit api.cu: packed-triangle size, tracing, moments, τ̂, rf_gram, the
// mainloop test hook and Φ's workspace size (include/rf.h).
#pragma once

namespace {
rf_status gram_collective(const void* X, int64_t ldx, const void* W, int64_t ldw, int64_t p, int64_t n, int64_t m_local,
                          int64_t m_total, rf_act act, rf_prec prec, float* recv, void* ws, size_t ws_bytes,
                          cudaStream_t st);
}

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
  return rf_profile_timeline(max_records, names, nullptr, ms, count);
}

rf_status rf_profile_timeline(int32_t max_records, char* names, float* start_ms, float* ms, int32_t* count) {
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
      if (start_ms) {   // relative to the first record pushed; shifted to the earliest start below
        float t0 = 0.f;
        if (e == cudaSuccess && cudaEventElapsedTime(&t0, recs[0].a, r.a) != cudaSuccess) t0 = 0.f;
        start_ms[k] = t0;
      }
    }
    ++k;
  }
  if (start_ms && k > 0) {   // records are pushed when a launch scope closes, not in start order
    const int32_t kk = std::min(k, max_records);
    float mn = 0.f;
    for (int32_t i = 0; i < kk; ++i) mn = std::min(mn, start_ms[i]);
    for (int32_t i = 0; i < kk; ++i) start_ms[i] -= mn;
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

rf_status rf_act_leaky_relu(double a_plus, double a_minus, rf_act* act) {
  if (!act) return fail(RF_E_INVALID, "rf_act_leaky_relu: act is NULL");
  if (!std::isfinite(a_plus) || !std::isfinite(a_minus))
    return fail(RF_E_INVALID, "rf_act_leaky_relu: coefficients must be finite");
  const double a[3] = {a_plus, a_minus, 0.0};
  const int id = rfh::register_param_act(1, a);
  if (id < 0) return fail(RF_E_INVALID, "rf_act_leaky_relu: more than %d parametrised activations", RF_ACT_PARAM_MAX);
  *act = (rf_act)id;
  return ok();
}

rf_status rf_act_quadratic(double a0, double a1, double a2, rf_act* act) {
  if (!act) return fail(RF_E_INVALID, "rf_act_quadratic: act is NULL");
  if (!std::isfinite(a0) || !std::isfinite(a1) || !std::isfinite(a2))
    return fail(RF_E_INVALID, "rf_act_quadratic: coefficients must be finite");
  const double a[3] = {a0, a1, a2};
  const int id = rfh::register_param_act(2, a);
  if (id < 0) return fail(RF_E_INVALID, "rf_act_quadratic: more than %d parametrised activations", RF_ACT_PARAM_MAX);
  *act = (rf_act)id;
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

rf_status rf_estimate_tau(rf_ctx* ctx, const void* X, rf_dtype x_dt, int64_t ldx, int64_t p, int64_t n, double* tau_out,
                          void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  RF_CTX_ENTER(ctx);
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

rf_status rf_round_bf16(rf_ctx* ctx, const float* src, int64_t lds, int64_t rows, int64_t cols, void* dst, int64_t ldd,
                        void* stream) {
  g_launches = 0;
  RF_CTX_ENTER(ctx);
  if (rows < 0 || cols < 0) return fail(RF_E_INVALID, "rf_round_bf16: rows, cols must be >= 0");
  if (rows == 0 || cols == 0) return ok();
  if (!src || !dst) return fail(RF_E_INVALID, "rf_round_bf16: NULL buffer");
  if (lds < cols || ldd < cols) return fail(RF_E_INVALID, "rf_round_bf16: leading dimensions must be >= cols");
  if ((reinterpret_cast<uintptr_t>(src) & 3) || (reinterpret_cast<uintptr_t>(dst) & 1))
    return fail(RF_E_INVALID, "rf_round_bf16: src must be 4-B and dst 2-B aligned");
  DevInfo dev;
  rf_status s;
  if ((s = check_device(&dev))) return s;
  return launch_round_bf16(src, lds, rows, cols, dst, ldd, dev.sms, (cudaStream_t)stream);
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
  if (!valid_out(out) || out == RF_OUT_PACKED_TILES)
    return fail(RF_E_INVALID, "rf_gram: unknown output mode %d", (int)out);
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
      rfk::SimtSigma<double> e1{S, pl.ldS, n, m_local, (int)act, act_rt(act)};
      if ((s = launch_simt<double>("K6_simt_gemm_sigma", (const double*)X, ldx, (const double*)W, ldw, n, m_local, p, 0, 0,
                                   (int)((n + rfk::kSimtTile - 1) / rfk::kSimtTile), e1, st)))
        return s;
      rfk::SimtSyrk<double> e2{(double*)G, ldg, n, 1.0 / (double)m_total, full};
      if ((s = launch_simt<double>("K6_simt_syrk", S, pl.ldS, S, pl.ldS, n, n, m_local, 1, 0, (int)((n + rfk::kSimtTile - 1) / rfk::kSimtTile), e2, st)))
        return s;
    } else {
      float* S = (float*)(w + pl.off_s0);
      rfk::SimtSigma<float> e1{S, pl.ldS, n, m_local, (int)act, act_rt(act)};
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
  GramTcArgs ga{X, ldx, W, ldw, p, n, m_local, m_total, act, full, (float*)G, ldg, w, pl, usable_sms(dev.sms), st,
                nullptr, tri_T};
  return gram_tc_dispatch(ga, prec);
}

rf_status rf_gram(rf_ctx* ctx, const void* X, int64_t ldx, const void* W, int64_t ldw, int64_t p, int64_t n,
                  int64_t m_local, int64_t m_total, rf_act act, rf_prec prec, rf_out out, void* G, int64_t ldg, void* ws,
                  size_t ws_bytes, void* stream) {
  RF_CTX_ENTER(ctx);
  if (out == RF_OUT_PACKED_TILES)   // G5: the collective (abi_ctx.cuh)
    return gram_collective(X, ldx, W, ldw, p, n, m_local, m_total, act, prec, (float*)G, ws, ws_bytes,
                           (cudaStream_t)stream);
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

rf_status rf_debug_gemm_nt(rf_ctx* ctx, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N,
                           int64_t K, rf_prec prec, int32_t kchunk, float* C, int64_t ldc, void* ws, size_t ws_bytes,
                           void* stream) {
  g_launches = 0;
  RF_CTX_ENTER(ctx);
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
