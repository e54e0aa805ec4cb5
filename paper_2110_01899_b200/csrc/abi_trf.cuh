// Part of the single translation unit api.cu.
#pragma once

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
  t.off_prog = off; off = align256(off + 2048);   // lockstep words, start flag, unit queue
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
  if (prog && opt(RF_OPT_K3_HYBRID)) {   // multicast + pair hybrid (workspace progress words available)
    using C3m = rfk::TcCfg<1, 1, 256, 0, 4>;
    CUtensorMap tBh;
    if ((s = make_tmap(&tBh, T, true, m_local, p, ldt, 64))) return s;
    bool used = false;
    if ((s = launch_k3_hybrid<C3m, C3>("K3_ter_features", tA, tB, tBh, n, m_local, kb, e, prog, sms, st, &used)))
      return s;
    if (used) return RF_OK;
  }
  rfk::Sched sc =
      rfk::Sched::make(0, 256, 0, (int)((n + 255) / 256), (int)((m_local + 255) / 256), kb, 0, raster_gm(8, 3));
  sc.load_pol = 1;
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

rf_status rf_ter_features(rf_ctx* ctx, const void* X, int64_t ldx, const void* T, int64_t ldt, int64_t p, int64_t n,
                          int64_t m_local, double eps, double s_minus, double s_plus, void* features, int64_t ldf,
                          void* stream) {
  g_launches = 0;
  RF_CTX_ENTER(ctx);
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

rf_status rf_gram_ter(rf_ctx* ctx, const void* X, int64_t ldx, const void* T, int64_t ldt, int64_t p, int64_t n,
                      int64_t m_local, int64_t m_total, double eps, double s_minus, double s_plus, rf_out out, float* G,
                      int64_t ldg, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  RF_CTX_ENTER(ctx);
  rf_status s;
  if ((s = ter_validate("rf_gram_ter", X, ldx, T, ldt, p, n, m_local, eps, s_minus, s_plus))) return s;
  if (m_total < m_local) return fail(RF_E_INVALID, "rf_gram_ter: m_total < m_local");
  if (m_local > (int64_t(1) << 24))
    return fail(RF_E_INVALID, "rf_gram_ter: m_local > 2^24 (fp32 accumulation of ±1 products is exact below that)");
  if (!valid_out(out) || out == RF_OUT_PACKED_TILES)
    return fail(RF_E_INVALID, "rf_gram_ter: unsupported output mode %d", (int)out);
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
  const int lockw = (int)opt(RF_OPT_LOCK_W);
  if (lockw > 0) {
    s4.prog = (uint32_t*)(w + pl.off_prog);
    s4.lock_w = lockw;
    s4.lock_ks = std::max(1, (int)opt(RF_OPT_LOCK_KS));
    RF_CUDA_CHECK(cudaMemsetAsync(s4.prog, 0, 1024, st));
  }
  rfk::EpiSyrk e4{G, ldg, n, (float)(1.0 / (double)m_total), (int)out & 1, tma_out ? 1 : 0, tri_T};
  bool hyb = false;
  if (lockw > 0) {
    CUtensorMap tSh;   // Σ^terᵀ with a 64-row box (the 8-CTA multicast kernel's A halves)
    if ((s = make_tmap_es(&tSh, S, 1, n, m_local, pl.ldS, 64))) return s;
    if ((s = launch_k4_hybrid<3>("K4_ter_syrk", tA, tSh, tO, n, kb4, e4, s4.prog, lockw, s4.lock_ks, dev.sms, st,
                                 &hyb)))
      return s;
  }
  if (!hyb && (s = launch_tc<C4>("K4_ter_syrk", tA, tA, tA, tA, tO, s4, e4, dev.sms, st))) return s;
  if ((int)out & RF_OUT_CENTER)
    if ((s = center_pass<float>(G, ldg, n, (int)out & 1, (double*)(w + pl.off_cen), st))) return s;
  return ok();
}

}  // extern "C"
