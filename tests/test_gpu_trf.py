"""GPU parity of NEXT-1, Ternary Random Features (include/rf.h): σ^ter features and G^ter vs the fp64 oracle.

Where floating point decides an integer (σ^ter of a projection), the two sides may disagree only inside the band
where the exact projection is within the GPU's fp32 rounding of a threshold: every decision outside that band must
match the oracle exactly (bit-exact codes), the band must be tiny, and G^ter must equal — bit for bit — the exact
integer SYRK of the GPU's own features scaled by fp32(1/m) (the fp8 tensor-core SYRK is exact).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import trf  # noqa: E402
import paper_2110_01899_b200 as rf  # noqa: E402
import synthetic  # noqa: E402

pytestmark = pytest.mark.gpu

CODE = {0x38: 1.0, 0xB8: -1.0, 0x00: 0.0}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    assert rf.rf_device_supported(0), "device 0 is not sm_100"
    torch.cuda.set_device(0)
    yield


def _decode(codes: np.ndarray) -> np.ndarray:
    out = np.full(codes.shape, np.nan)
    for k, v in CODE.items():
        out[codes == k] = v
    assert not np.isnan(out).any(), "a feature byte is not an E4M3 code of −1, 0 or +1"
    return out


def _band(Xb: np.ndarray, eps: float, s_minus: float, s_plus: float) -> np.ndarray:
    """Per-row half-width of the band in which fp32 accumulation + the fp32 thresholds may flip a decision: the
    accumulator is rounded once per K = 16 MMA (products of bf16 and ±1 are exact), each time by ≤ 2^-23 of a
    partial sum bounded by Σ_l|x_il| (scripts/accum_experiment.py: truncation), scaled by c, plus the rounding
    of t± = s±/c to fp32."""
    p = Xb.shape[1]
    c = (1 - eps) ** -0.5
    return c * (math.ceil(p / 16) + 2) * 2.0 ** -23 * np.sum(np.abs(Xb), axis=1) + \
        2.0 ** -22 * max(abs(s_minus), abs(s_plus))


def _inputs(n, p, m, eps, cfg=0, seed_rows=None):
    X = synthetic.make_X(cfg, n=n, p=p) if seed_rows is None else synthetic.make_X(cfg, rows=seed_rows)
    T = synthetic.make_T(cfg, eps, m=m, p=p)
    Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
    Td = torch.tensor(T, device="cuda").to(torch.bfloat16)
    return Xd, Td, Xd.double().cpu().numpy(), T


def _check_features(Xd, Td, Xb, T, eps, sm, sp):
    codes = rf.rf_ter_features(Xd, Td, eps, sm, sp)
    torch.cuda.synchronize()
    S_gpu = _decode(codes.cpu().numpy())
    S_ref = trf.ternary_features(Xb, T, eps, sm, sp)
    margin = trf.decision_margin(Xb, T, eps, sm, sp)
    band = _band(Xb, eps, sm, sp)[:, None]
    diff = S_gpu != S_ref
    outside = diff & (margin > band)
    assert not outside.any(), f"{int(outside.sum())} decisions differ outside the rounding band"
    frac_band = float(np.mean(margin <= band))
    print(f"[parity] σ^ter n={Xb.shape[0]} m={T.shape[0]} eps={eps}: {int(diff.sum())} flips inside the band "
          f"(band holds {frac_band:.2e} of the entries)")
    assert frac_band < 1e-2
    return S_gpu, S_ref


@pytest.mark.parametrize("n,p,m,eps", [(600, 200, 700, 0.0), (513, 64, 1030, 0.5), (1024, 784, 512, 0.9),
                                       (300, 1000, 257, 0.9)])
def test_ter_features_decisions(n, p, m, eps):
    Xd, Td, Xb, T = _inputs(n, p, m, eps)
    tau = oracle.tau_hat(Xb)
    sm, sp = rf.rf_trf_thresholds_for("tanh", tau)
    _check_features(Xd, Td, Xb, T, eps, sm, sp)


@pytest.mark.parametrize("n,p,m,eps,out", [(600, 128, 700, 0.9, "upper"), (1000, 256, 1500, 0.5, "full"),
                                           (257, 64, 40000, 0.0, "upper")])
def test_gram_ter_exact_and_matches_oracle(n, p, m, eps, out):
    Xd, Td, Xb, T = _inputs(n, p, m, eps, cfg=1)
    tau = oracle.tau_hat(Xb)
    mo = oracle.moments("erf", tau)
    sm, sp = rf.rf_trf_thresholds(mo["d1"], mo["d2"], tau, 1)
    S_gpu, S_ref = _check_features(Xd, Td, Xb, T, eps, sm, sp)
    G = torch.full((n, n), -7.25, dtype=torch.float32, device="cuda")
    rf.rf_gram_ter(Xd, Td, eps, sm, sp, out=out, G=G)
    torch.cuda.synchronize()
    Gc = G.cpu().numpy()
    cnt = S_gpu @ S_gpu.T                                   # exact integers
    exp = (cnt.astype(np.float32) * np.float32(1.0 / m)).astype(np.float32)
    I, J = np.triu_indices(n)
    assert np.array_equal(Gc[I, J], exp[I, J]), "fp8 SYRK must be exact: G^ter = fp32(count)·fp32(1/m)"
    if out == "upper":
        L = np.tril_indices(n, -1)
        assert np.all(Gc[L] == -7.25)
    else:
        assert np.array_equal(Gc, Gc.T)
    ref = trf.gram_ter(Xb, T, eps, sm, sp)
    e = float(np.linalg.norm(Gc[I, J] - ref[I, J]) / np.linalg.norm(ref[I, J]))
    print(f"[parity] G^ter n={n} m={m} eps={eps}: rel-Frobenius vs oracle {e:.3e} (band flips only)")
    flips = (S_gpu != S_ref)
    # each flip changes a count by at most 2 per partner row: bound |ΔG_ij| ≤ (flips_i + flips_j)·2/m
    fr = flips.sum(axis=1)
    assert np.all(np.abs(Gc[I, J] - ref[I, J]) <= (fr[I] + fr[J]) * 2.0 / m + 1e-6)


def test_ter_full_size_sampled():
    """configs[3] sizes (p = 1024, n = m = 65536), ε = 0.9: G^ter on the full problem; σ^ter decisions and G^ter
    on a sampled principal submatrix S × S against the oracle (tile-boundary rows included)."""
    cfg = synthetic.CONFIGS[3]
    eps = 0.9
    n, p, m = cfg.n, cfg.p, cfg.m
    X = torch.tensor(synthetic.make_X(cfg), device="cuda").to(torch.bfloat16)
    T = torch.tensor(synthetic.make_T(cfg, eps), device="cuda").to(torch.bfloat16)
    tau = rf.rf_estimate_tau(X)
    sm, sp = rf.rf_trf_thresholds_for(cfg.act, tau)
    G = rf.rf_gram_ter(X, T, eps, sm, sp)
    S = synthetic.sample_indices(n, count=384, tile_stride=512)
    Xs = X[torch.tensor(S, device="cuda")].contiguous()
    codes = rf.rf_ter_features(Xs, T, eps, sm, sp)
    torch.cuda.synchronize()
    Xb = Xs.double().cpu().numpy()
    Tn = T.double().cpu().numpy()
    S_gpu = _decode(codes.cpu().numpy())
    S_ref = trf.ternary_features(Xb, Tn, eps, sm, sp)
    margin = trf.decision_margin(Xb, Tn, eps, sm, sp)
    assert not ((S_gpu != S_ref) & (margin > _band(Xb, eps, sm, sp)[:, None])).any()
    Gs = G[torch.tensor(S, device="cuda")][:, torch.tensor(S, device="cuda")].cpu().numpy()
    cnt = S_gpu @ S_gpu.T
    exp = (cnt.astype(np.float32) * np.float32(1.0 / m)).astype(np.float32)
    I, J = np.triu_indices(len(S))
    assert np.array_equal(Gs[I, J], exp[I, J])
    ref = (S_ref @ S_ref.T) / m
    e = float(np.linalg.norm(Gs[I, J] - ref[I, J]) / np.linalg.norm(ref[I, J]))
    print(f"[parity] G^ter configs[3] sizes eps=0.9 sampled |S|={len(S)}: rel-Frobenius {e:.3e}")
    assert e < 1e-5


def test_ter_rejects_bad_arguments():
    Xd, Td, _, _ = _inputs(64, 32, 64, 0.5)
    with pytest.raises(rf.RFError):
        rf.rf_ter_features(Xd, Td, 1.0, -0.5, 0.5)          # ε must be < 1
    with pytest.raises(rf.RFError):
        rf.rf_ter_features(Xd, Td, 0.5, 0.5, -0.5)          # s− > s+
    with pytest.raises(rf.RFError):
        rf.rf_gram_ter(Xd, Td, 0.5, -0.5, 0.5, m_total=10)  # m_total < m_local


def test_gram_ter_k3_multicast_hybrid_bit_exact():
    """At n ≥ 32 row tiles K3^ter runs as the multicast + pair hybrid; its fp8 feature codes and hence G^ter are
    the pair kernel's bit for bit (same accumulation order, same σ^ter decision)."""
    n, p, m, eps = 8448 + 77, 128, 1024 + 40, 0.9
    Xd, Td, Xb, T = _inputs(n, p, m, eps, cfg=1)
    sm, sp = rf.rf_trf_thresholds_for("tanh", 1.0)
    res = []
    ctx = rf.Context(0)
    for mc in (1, 0):
        ctx.set_option("k3_hybrid", mc)
        rf.rf_profile_read()
        rf.rf_profile_enable(True)
        G = rf.rf_gram_ter(Xd, Td, eps, sm, sp, out="upper", ctx=ctx)
        torch.cuda.synchronize()
        rf.rf_profile_enable(False)
        names = {nm for nm, _ in rf.rf_profile_read()}
        assert ("K3_ter_features_mc" in names) == bool(mc), f"k3_hybrid={mc}: {sorted(names)}"
        res.append(G)
    assert torch.equal(res[0], res[1])
    assert float(res[0].diagonal().min()) > 0.0


def test_gram_ter_k4_hybrid_bit_exact():
    """At n ≥ 64 row tiles K4^ter (the exact fp8 SYRK) runs as the multicast + pair hybrid with the unit queue; G^ter
    equals the pair kernel's bit for bit (integer sums, exact in fp32 either way), and the hybrid did run."""
    n, p, m, eps = 16384 + 77, 64, 512, 0.9
    Xd, Td, Xb, T = _inputs(n, p, m, eps, cfg=1)
    sm, sp = rf.rf_trf_thresholds_for("tanh", 1.0)
    res = []
    ctx = rf.Context(0)
    for hyb in (1, 0):
        ctx.set_option("k4_hybrid", hyb)
        rf.rf_profile_read()
        rf.rf_profile_enable(True)
        G = rf.rf_gram_ter(Xd, Td, eps, sm, sp, out="upper", ctx=ctx)
        torch.cuda.synchronize()
        rf.rf_profile_enable(False)
        names = {nm for nm, _ in rf.rf_profile_read()}
        assert ("K4_ter_syrk_mc" in names) == bool(hyb), f"k4_hybrid={hyb}: {sorted(names)}"
        res.append(G)
    assert torch.equal(res[0], res[1])
