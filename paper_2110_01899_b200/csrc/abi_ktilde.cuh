// Part of the single translation unit api.cu.
#pragma once

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

rf_status rf_ktilde(rf_ctx* ctx, const void* X, int64_t ldx, int64_t p, int64_t n, const float* V, int64_t ldv,
                    int32_t kv, const double* A, double d0, double d1, double d2, rf_prec prec, rf_out out, float* Kt,
                    int64_t ldk, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  RF_CTX_ENTER(ctx);
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
      rfk::Sched sc = rfk::Sched::make(1, 256, 0, tn, tn, (int)((p + C::BK - 1) / C::BK), 0, raster_gm(16, 5));
      sc.load_pol = 1;   // evict_last operands (4.18 → 4.14 ms)
      if ((s = launch_tc<C>("KT_ktilde", tA, tA, tA, tA, tO, sc, e, dev.sms, st))) return s;
    } else {
      using C = rfk::TcCfg<2, 1, 256, 1, 2, 16>;
      rfk::Sched sc = rfk::Sched::make(1, 256, 0, tn, tn, (int)((p + C::BK - 1) / C::BK), 0, raster_gm(16, 5));
      sc.load_pol = 1;   // evict_last operands (4.18 → 4.14 ms)
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
    rfk::Sched sc = rfk::Sched::make(1, 256, 0, tn, tn, (int)((p + C::BK - 1) / C::BK), 0, raster_gm(16, 5));
      sc.load_pol = 1;   // evict_last operands (4.18 → 4.14 ms)
    if ((s = launch_tc<C>("KT_ktilde", tA, tA, tAl, tAl, tO, sc, e, dev.sms, st))) return s;
  }
  return ok();
}

}  // extern "C"
