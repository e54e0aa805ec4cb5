// Part of the single translation unit api.cu.
#pragma once

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

rf_status rf_ridge(rf_ctx* ctx, const float* G, int64_t ldg, int64_t n_train, int64_t n_test, const double* gammas,
                   int32_t n_gamma, const double* Y, int64_t ldy, int32_t nrhs, double* alpha, double* Yhat,
                   void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  RF_CTX_ENTER(ctx);
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
