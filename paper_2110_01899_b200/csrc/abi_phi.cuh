// Part of the single translation unit api.cu: Φ by EQ1 / EQ2 and the row split (include/rf.h).
#pragma once

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
  if (!valid_out(out) || out == RF_OUT_PACKED_TILES)
    return fail(RF_E_INVALID, "rf_phi_closed_form: unsupported output mode %d", (int)out);
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
            (float)f1, row_begin, row_end, w, pl, usable_sms(dev.sms), st, tri_T};
  if (odd_act && opt(RF_OPT_EQ1_GENERAL) == 0) return launch_k5<true>(ka);
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

rf_status rf_phi_closed_form(rf_ctx* ctx, const void* X, int64_t ldx, int64_t p, int64_t n, rf_act act, double tau,
                             const rf_moments_t* mom, rf_prec prec, rf_out out, int64_t row_begin, int64_t row_end,
                             void* Phi, int64_t ldphi, void* ws, size_t ws_bytes, void* stream) {
  RF_CTX_ENTER(ctx);
  return phi_entry(X, ldx, p, n, act, tau, mom, prec, out, row_begin, row_end, Phi, ldphi, ws, ws_bytes, stream, 1);
}

rf_status rf_phi_eq2(rf_ctx* ctx, const void* X, int64_t ldx, int64_t p, int64_t n, rf_act act, double tau,
                     const rf_moments_t* mom, rf_prec prec, rf_out out, int64_t row_begin, int64_t row_end,
                     void* Phi, int64_t ldphi, void* ws, size_t ws_bytes, void* stream) {
  RF_CTX_ENTER(ctx);
  return phi_entry(X, ldx, p, n, act, tau, mom, prec, out, row_begin, row_end, Phi, ldphi, ws, ws_bytes, stream, 2);
}

}  // extern "C"
