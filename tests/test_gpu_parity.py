"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): relative Frobenius ≤ 1e-5 in fp32-accurate modes (FP32, 3×TF32)
and ≤ 2e-3 in BF16 mode; 1×TF32 is in the 2e-3 class; FP64 mode ≤ 1e-12.  The oracle always consumes
exactly the (rounded) tensors the GPU reads, upcast to fp64 (DESIGN.md §4 R11).  Beside every Frobenius
assert, every compared entry is held to the per-entry bound derived from the mode's arithmetic
(tests/entry_bounds.py, reading R22), so a single wrong tile or entry fails.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_2110_01899_b200 as rf  # noqa: E402
import synthetic  # noqa: E402
from entry_bounds import check, gram_bound, phi_bound  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-12, "fp32": 1e-5, "3xtf32": 1e-5, "tf32": 2e-3, "bf16": 2e-3}
DT = {"fp64": torch.float64, "fp32": torch.float32, "3xtf32": torch.float32, "tf32": torch.float32,
      "bf16": torch.bfloat16}
SENTINEL = -7.25


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    assert rf.rf_device_supported(0), "device 0 is not sm_100"
    torch.cuda.set_device(0)
    yield


def dev(a, prec):
    return torch.tensor(np.ascontiguousarray(a), device="cuda").to(DT[prec])


def back(t):
    return t.double().cpu().numpy()


def rel_fro(got, ref):
    return float(np.linalg.norm(got - ref) / np.linalg.norm(ref))


def report(name, got, ref, I, J):
    d = I == J
    err = np.abs(got - ref)
    md = float(err[d].max()) if d.any() else 0.0
    mo = float(err[~d].max()) if (~d).any() else 0.0
    r = rel_fro(got, ref)
    print(f"[parity] {name}: rel-Frobenius {r:.3e}  max-abs diag {md:.3e}  off-diag {mo:.3e}")
    return r


def upper_idx(n):
    return np.triu_indices(n)


# ------------------------------------------------------------------------------------------------ G
def _gram_case(n, p, m, act, prec, out="upper", seed=0, tol=None):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    W = rng.standard_normal((m, p))
    Xd, Wd = dev(X, prec), dev(W, prec)
    G = torch.full((n, n), SENTINEL, dtype=torch.float64 if prec == "fp64" else torch.float32, device="cuda")
    rf.rf_gram(Xd, Wd, act=act, prec=prec, out=out, G=G)
    torch.cuda.synchronize()
    Xo, Wo = back(Xd), back(Wd)
    ref = oracle.gram(Xo, Wo, act)
    Gc = back(G)
    I, J = upper_idx(n)
    r = report(f"G n={n} p={p} m={m} {act} {prec} {out}", Gc[I, J], ref[I, J], I, J)
    assert r <= (TOL[prec] if tol is None else tol)
    check(f"G n={n} p={p} m={m} {act} {prec}", Gc[I, J], ref[I, J], gram_bound(prec, act, Xo, Wo, ref, I, J))
    L = np.tril_indices(n, -1)
    if out == "upper":
        assert np.all(Gc[L] == SENTINEL), "UPPER mode wrote below the diagonal"
    else:
        assert rel_fro(Gc, ref) <= (TOL[prec] if tol is None else tol)
        assert np.array_equal(Gc, Gc.T)


@pytest.mark.parametrize("prec", ["fp64", "fp32", "3xtf32", "tf32", "bf16"])
@pytest.mark.parametrize("act", ["tanh", "erf", "sigmoid_half"])
def test_gram_small_ragged(prec, act):
    # n=200: one partial 128-row tile + one partial 256-col tile; m=300: ragged K for the SYRK;
    # p=72: ragged K for the feature GEMM (72 = 64 + 8 bf16).
    _gram_case(200, 72, 300, act, prec)


@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "tf32", "bf16"])
def test_gram_multi_tile_full(prec):
    _gram_case(1000, 200, 700, "tanh", prec, out="full", seed=1)


@pytest.mark.parametrize("prec", ["fp64", "fp32", "3xtf32", "bf16"])
def test_gram_degenerate_sizes(prec):
    # m = 1 (reading R22): no averaging over features, so G_ij = s_i s_j carries the bf16 rounding of both
    # factors undiluted (unit roundoff 2^-8 each: bf16 keeps 8 significant bits), |ΔG_ij| ≤ (2·2^-8 + 2^-16)|G_ij|
    # + O(e_eval) entry by entry (asserted in _gram_case through gram_bound), hence a relative Frobenius error up to
    # 2·2^-8 + 2^-16 ≈ 7.8e-3, above the 2e-3 that averaging over m ≫ 1 features gives
    r22 = 2 * 2.0 ** -8 + 2.0 ** -16 if prec == "bf16" else None
    _gram_case(1, 8, 1, "erf", prec, out="full", seed=2, tol=r22)
    _gram_case(129, 8, 1, "tanh", prec, seed=3, tol=r22)  # rank one
    _gram_case(256, 8, 512, "tanh", prec, seed=4)           # exact tile multiples


def test_gram_sharded_partials_sum_to_full():
    """Data parallel over m (north star (4)): Σ_r rf_gram(W_r, m_total) == rf_gram(W)."""
    rng = np.random.default_rng(5)
    n, p, m = 300, 64, 768
    X = dev(rng.standard_normal((n, p)) / 8, "bf16")
    W = dev(rng.standard_normal((m, p)), "bf16")
    full = rf.rf_gram(X, W, act="sigmoid_half", prec="bf16", out="upper")
    parts = [rf.rf_gram(X, W[r * 256:(r + 1) * 256].contiguous(), act="sigmoid_half", prec="bf16", out="upper",
                        m_total=m) for r in range(3)]
    torch.cuda.synchronize()
    s = sum(back(g) for g in parts)
    I, J = upper_idx(n)
    assert np.max(np.abs(s[I, J] - back(full)[I, J])) < 1e-6


def test_gram_zero_size_rejected():
    X = torch.zeros((0, 8), dtype=torch.bfloat16, device="cuda")
    W = torch.zeros((4, 8), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(rf.RFError):
        rf.rf_gram(X, W, prec="bf16", G=torch.zeros((1, 4), device="cuda"))


# ------------------------------------------------------------------------------------------------ Φ
def _phi_case(X, act, prec, tau=0.0, out="upper", rows=None, ctx=None):
    n = X.shape[0]
    Xd = dev(X, prec)
    Phi = torch.full((n, n), SENTINEL, dtype=torch.float64 if prec == "fp64" else torch.float32, device="cuda")
    if rows is None:
        rf.rf_phi_closed_form(Xd, act=act, tau=tau, prec=prec, out=out, Phi=Phi, ctx=ctx)
    else:
        for b, e in rows:
            rf.rf_phi_closed_form(Xd, act=act, tau=tau, prec=prec, out=out, row_begin=b, row_end=e, Phi=Phi, ctx=ctx)
    torch.cuda.synchronize()
    Xo = back(Xd)
    t_used = tau if tau > 0 else oracle.tau_hat(Xo)
    ref = oracle.phi_eq1(Xo, act, t_used)
    Pc = back(Phi)
    I, J = upper_idx(n)
    r = report(f"Phi n={n} p={X.shape[1]} {act} {prec} {out}", Pc[I, J], ref[I, J], I, J)
    tol = {"fp64": 1e-12, "fp32": 1e-5, "3xtf32": 1e-5, "tf32": 2e-3, "bf16": 1e-5}[prec]
    assert r <= tol
    check(f"Phi n={n} {act} {prec}", Pc[I, J], ref[I, J], phi_bound(prec, act, Xo, t_used, I, J))
    L = np.tril_indices(n, -1)
    if out == "upper":
        assert np.all(Pc[L] == SENTINEL)
    else:
        assert np.array_equal(Pc, Pc.T)
    return Pc, ref


@pytest.mark.parametrize("prec", ["fp64", "fp32", "3xtf32", "tf32", "bf16"])
@pytest.mark.parametrize("act", ["tanh", "erf", "sigmoid_half"])
def test_phi_small_ragged(prec, act):
    X = synthetic.make_X(4, n=300, p=72)        # unit-scaled rows with norms in [0.5, 1.5]
    _phi_case(X, act, prec)


@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "bf16"])
def test_phi_multi_tile_given_tau_full(prec):
    X = synthetic.make_X(1, n=1100, p=200)
    _phi_case(X, "erf", prec, tau=1.05, out="full")


@pytest.mark.parametrize("prec", ["3xtf32", "bf16"])
def test_phi_general_epilogue_matches_odd_form(prec):
    """The general EQ1 epilogue (A0, A2 terms kept, used for non-odd σ) on an odd σ: same parity, and within
    a few fp32 ulps of the odd-σ form the library selects by default."""
    X = synthetic.make_X(4, n=700, p=96)
    P_odd, _ = _phi_case(X, "tanh", prec)
    ctx = rf.Context(0)
    ctx.set_option("eq1_general", 1)
    P_gen, _ = _phi_case(X, "tanh", prec, ctx=ctx)
    I, J = upper_idx(X.shape[0])
    assert np.max(np.abs(P_gen[I, J] - P_odd[I, J])) <= 1e-6 * np.max(np.abs(P_odd[I, J]))


def test_phi_row_blocks_assemble_to_full():
    X = synthetic.make_X(4, n=1000, p=64)
    ranges = [rf.rf_phi_row_split(1000, 3, r) for r in range(3)]
    _phi_case(X, "tanh", "bf16", rows=ranges)


def test_phi_diagonal_rule_and_zero_norm():
    X = synthetic.make_X(0, n=256, p=64)
    Pc, ref = _phi_case(X, "tanh", "fp32")
    d = np.arange(256)
    assert np.max(np.abs(Pc[d, d] - ref[d, d])) < 1e-6
    Xz = X.copy()
    Xz[5] = 0.0
    with pytest.raises(rf.RFError):
        rf.rf_phi_closed_form(dev(Xz, "bf16"), act="tanh", tau=0.0, prec="bf16")
    # explicit τ (asynchronous call): the zero pivot row is its Gram–Schmidt limit (R23), every entry finite
    Pz, refz = _phi_case(Xz, "sigmoid_half", "bf16", tau=1.0)
    I, J = upper_idx(256)
    assert np.all(np.isfinite(Pz[I, J]))
    assert np.all(np.abs(Pz[5, 5:]) < 1e-12)  # odd σ, ν = 0 on the zero row: Φ = ν·A1·C1 = 0


def test_estimate_tau_lemma1():
    X = synthetic.make_X(2, n=4096, p=3072)
    for prec in ("fp64", "fp32", "bf16"):
        Xd = dev(X, prec)
        t = rf.rf_estimate_tau(Xd)
        assert abs(t - oracle.tau_hat(back(Xd))) < 1e-12 * t


# ------------------------------------------------------------------------------------------------ configs
def _sampled_gram(cfg_idx, prec, count, stride):
    cfg = synthetic.CONFIGS[cfg_idx]
    X = synthetic.make_X(cfg)
    W = synthetic.make_W(cfg)
    Xd, Wd = dev(X, prec), dev(W, prec)
    del X, W
    G = rf.rf_gram(Xd, Wd, act=cfg.act, prec=prec, out="upper")
    torch.cuda.synchronize()
    S = synthetic.sample_indices(cfg.n, count=count, tile_stride=stride)
    St = torch.tensor(S, device="cuda")
    sub = back(G.index_select(0, St).index_select(1, St))
    del G
    Xs = back(Xd.index_select(0, St))
    Wo = back(Wd)
    ref = oracle.gram(Xs, Wo, cfg.act)
    I, J = upper_idx(len(S))
    r = report(f"G configs[{cfg_idx}] {prec} sampled |S|={len(S)}", sub[I, J], ref[I, J], S[I], S[J])
    assert r <= TOL[prec]
    check(f"G configs[{cfg_idx}] {prec}", sub[I, J], ref[I, J], gram_bound(prec, cfg.act, Xs, Wo, ref, I, J))


def _sampled_phi(cfg_idx, prec, count, stride, packed=False):
    cfg = synthetic.CONFIGS[cfg_idx]
    X = synthetic.make_X(cfg)
    Xd = dev(X, prec)
    tau_ref = oracle.tau_hat(back(Xd))
    S = synthetic.sample_indices(cfg.n, count=count, tile_stride=stride)
    St = torch.tensor(S, device="cuda")
    if packed:
        # RF_OUT_PACKED_TRI (the e2e read-back layout): gather the sampled upper-triangle entries on the device by
        # the include/rf.h offsets, tile (I, J) at 65536·(I·T − I(I−1)/2 + J − I), row-major inside
        P = rf.rf_phi_closed_form(Xd, act=cfg.act, tau=0.0, prec=prec, out="packed_tri")
        torch.cuda.synchronize()
        T = -(-cfg.n // 256)
        ii, jj = np.meshgrid(S, S, indexing="ij")
        lo, hi = np.minimum(ii, jj), np.maximum(ii, jj)
        It, Jt = lo // 256, hi // 256
        off = 65536 * (It * T - It * (It - 1) // 2 + Jt - It) + (lo % 256) * 256 + (hi % 256)
        sub = back(P[torch.tensor(off.ravel(), device="cuda")]).reshape(len(S), len(S))
        del P
    else:
        Phi = rf.rf_phi_closed_form(Xd, act=cfg.act, tau=0.0, prec=prec, out="upper")
        torch.cuda.synchronize()
        sub = back(Phi.index_select(0, St).index_select(1, St))
        del Phi
    Xs = back(Xd.index_select(0, St))
    ref = oracle.phi_eq1(Xs, cfg.act, tau_ref)
    I, J = upper_idx(len(S))
    tol = {"fp32": 1e-5, "3xtf32": 1e-5, "tf32": 2e-3, "bf16": 1e-5}[prec]
    r = report(f"Phi configs[{cfg_idx}] {prec} sampled |S|={len(S)}", sub[I, J], ref[I, J], S[I], S[J])
    assert r <= tol
    check(f"Phi configs[{cfg_idx}] {prec}", sub[I, J], ref[I, J], phi_bound(prec, cfg.act, Xs, tau_ref, I, J))


@pytest.mark.parametrize("prec", ["fp64", "fp32", "3xtf32", "tf32", "bf16"])
def test_config0_tiny_full(prec):
    cfg = synthetic.CONFIGS[0]
    X = synthetic.make_X(cfg)
    W = synthetic.make_W(cfg)
    Xd, Wd = dev(X, prec), dev(W, prec)
    G = rf.rf_gram(Xd, Wd, act=cfg.act, prec=prec, out="full")
    torch.cuda.synchronize()
    ref = oracle.gram(back(Xd), back(Wd), cfg.act)
    I, J = upper_idx(cfg.n)
    assert report(f"G configs[0] {prec}", back(G)[I, J], ref[I, J], I, J) <= TOL[prec]
    check(f"G configs[0] {prec}", back(G)[I, J], ref[I, J], gram_bound(prec, cfg.act, back(Xd), back(Wd), ref, I, J))
    _phi_case(X, cfg.act, prec)


@pytest.mark.parametrize("prec", ["fp32", "3xtf32"])
def test_config1_full_size(prec):
    _sampled_gram(1, prec, count=512, stride=256)
    _sampled_phi(1, prec, count=1024, stride=128)


def test_config2_full_size_bf16():
    _sampled_gram(2, "bf16", count=512, stride=512)
    _sampled_phi(2, "bf16", count=512, stride=512)


def test_config3_full_size_bf16():
    # S holds every row ≡ 0, ±1 (mod 256) — each K4 pair tile's first/last rows, the 128-row CTA halves' seams at
    # 256-multiples, and the multicast/pair hybrid split rows (multiples of 512) of K3 and K4 — plus random rows
    _sampled_gram(3, "bf16", count=256, stride=256)
    _sampled_phi(3, "bf16", count=768, stride=128)     # the bench step's Φ on the same X


def test_config4_full_size_phi_packed_tri():
    """configs[4] Φ in the packed upper-triangle layout (16-warp K5, tile-remapped TMA stores), sampled."""
    _sampled_phi(4, "bf16", count=1024, stride=256, packed=True)


@pytest.mark.parametrize("prec", ["bf16", "3xtf32"])
def test_config4_full_size_phi(prec):
    _sampled_phi(4, prec, count=1024, stride=128 if prec == "bf16" else 256)


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
@pytest.mark.parametrize("out", ["upper", "full", "packed_tri"])
def test_phi_wide_epilogue_bit_exact(prec, out):
    """K5's 16-warp epilogue (p ≤ 512: four warps per TMEM lane quarter, chunks dealt round-robin) computes every
    entry with the same arithmetic as the 8-warp kernel: the two agree bit for bit, in every output layout."""
    X = synthetic.make_X(4, n=1100, p=200)
    Xd = dev(X, prec)
    res = []
    ctx = rf.Context(0)
    for wide in (1, 0):
        ctx.set_option("k5_wide", wide)
        P = rf.rf_phi_closed_form(Xd, act="tanh", prec=prec, out=out, ctx=ctx)
        torch.cuda.synchronize()
        res.append(P.cpu().numpy())
    if out == "packed_tri":
        from paper_2110_01899_b200 import layout
        res = [layout.unpack_tri(r, X.shape[0]) for r in res]
        I, J = upper_idx(X.shape[0])
        assert np.array_equal(res[0][I, J], res[1][I, J])
    else:
        assert np.array_equal(res[0], res[1])


@pytest.mark.parametrize("act,prec", [("erf", "bf16"), ("relu", "bf16"), ("erf", "tf32")])
def test_k3_multicast_hybrid_bit_exact(act, prec):
    """K3's multicast + pair hybrid (n ≥ 32 row tiles: 4-CTA clusters sharing each B tile as two multicast 64-row
    halves, pair clusters on the leftover SMs) accumulates in the same order as the pair kernel: G agrees bit for
    bit, and with the oracle.  (TF32 truncates its inputs, so a one-sided σ such as ReLU carries a −2e-3 bias
    there: TF32 is checked with erf.)"""
    n, p, m = 8448 + 77, 128, 1024 + 40          # 34 row tiles, ragged rows and features
    rng = np.random.default_rng(21)
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    W = rng.standard_normal((m, p))
    Xd, Wd = dev(X, prec), dev(W, prec)
    res = []
    ctx = rf.Context(0)
    for mc in (1, 0):
        ctx.set_option("k3_hybrid", mc)
        rf.rf_profile_read()
        rf.rf_profile_enable(True)
        G = rf.rf_gram(Xd, Wd, act=act, prec=prec, out="upper", ctx=ctx)
        torch.cuda.synchronize()
        rf.rf_profile_enable(False)
        names = {nm for nm, _ in rf.rf_profile_read()}
        assert ("K3_gemm_sigma_mc" in names) == bool(mc), f"k3_hybrid={mc}: {sorted(names)}"
        res.append(G)
    assert torch.equal(res[0], res[1])
    S = synthetic.sample_indices(n, count=256, tile_stride=512)
    St = torch.tensor(S, device="cuda")
    sub = back(res[0].index_select(0, St).index_select(1, St))
    Xs = back(Xd.index_select(0, St))
    ref = oracle.gram(Xs, back(Wd), act)
    I, J = upper_idx(len(S))
    assert report(f"G K3-multicast {act} {prec} n={n}", sub[I, J], ref[I, J], S[I], S[J]) <= TOL[prec]
    check(f"G K3-multicast {act} {prec}", sub[I, J], ref[I, J], gram_bound(prec, act, Xs, back(Wd), ref, I, J))


@pytest.mark.parametrize("cl8,dyn,out", [("0", 1, "upper"), ("0", 0, "upper"), ("1", 1, "upper"), ("0", 1, "full"),
                                         ("0", 1, "packed_tri"), ("0", 0, "packed_tri")])
def test_k4_hybrid_bit_exact(cl8, dyn, out):
    """K4's multicast + pair hybrid (n ≥ 64 row tiles) — 4-CTA clusters sharing B, or (k4_cl8) 8-CTA clusters of
    2 × 2 pairs sharing A and B; with the dynamic unit queue (default) or the static split — equals the pair-cluster
    kernel bit for bit (same accumulation order), in the dense, mirrored and packed-triangle layouts."""
    n, p, m = 16384 + 77, 64, 1024
    rng = np.random.default_rng(5)
    Xd = dev(rng.standard_normal((n, p)) / math.sqrt(p), "bf16")
    Wd = dev(rng.standard_normal((m, p)), "bf16")
    ctx = rf.Context(0)
    ctx.set_option("k4_cl8", int(cl8))
    ctx.set_option("k4_dynamic", dyn)      # 1: both kernels pull units from one device counter; 0: static split
    torch.cuda.synchronize()
    rf.rf_profile_read()
    rf.rf_profile_enable(True)
    G1 = rf.rf_gram(Xd, Wd, act="tanh", prec="bf16", out=out, ctx=ctx)
    torch.cuda.synchronize()
    rf.rf_profile_enable(False)
    names = {nm for nm, _ in rf.rf_profile_read()}
    assert "K4_syrk_mc" in names and "K4_syrk_tail" in names, f"the hybrid did not run: {sorted(names)}"
    ctx.set_option("k4_hybrid", 0)
    G0 = rf.rf_gram(Xd, Wd, act="tanh", prec="bf16", out="upper" if out == "packed_tri" else out, ctx=ctx)
    torch.cuda.synchronize()
    if out == "packed_tri":   # the same entries through the packed offsets (include/rf.h), sampled rows
        T = -(-n // 256)
        S = synthetic.sample_indices(n, count=300, tile_stride=1024)
        ii, jj = np.meshgrid(S, S, indexing="ij")
        lo, hi = np.minimum(ii, jj), np.maximum(ii, jj)
        It, Jt = lo // 256, hi // 256
        off = 65536 * (It * T - It * (It - 1) // 2 + Jt - It) + (lo % 256) * 256 + (hi % 256)
        got = G1[torch.tensor(off.ravel(), device="cuda")].reshape(len(S), len(S))
        ref = G0[torch.tensor(lo.ravel(), device="cuda"), torch.tensor(hi.ravel(), device="cuda")].reshape(len(S), len(S))
        assert torch.equal(got, ref)
    else:
        assert torch.equal(G1, G0)


def test_non_current_stream_orders_allocations_and_results():
    """the wrappers allocate outputs and workspace on the stream the kernels are enqueued on, so a
    call on a non-current stream neither races the allocator's zero-fill nor lets the workspace be reused while the
    kernels still run: G from a side stream equals G from the current stream bit for bit, repeatedly, with the
    side stream never synchronized against the current one by the caller."""
    rng = np.random.default_rng(9)
    n, p, m = 2100, 128, 1024
    Xd = dev(rng.standard_normal((n, p)) / math.sqrt(p), "bf16")
    Wd = dev(rng.standard_normal((m, p)), "bf16")
    ref = rf.rf_gram(Xd, Wd, act="tanh", prec="bf16", out="upper")
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    outs = []
    for _ in range(4):
        G = rf.rf_gram(Xd, Wd, act="tanh", prec="bf16", out="upper", stream=side)   # allocated on `side`
        Phi = rf.rf_phi_closed_form(Xd, act="tanh", prec="bf16", stream=side)
        outs.append((G, Phi))
        torch.empty(1 << 26, dtype=torch.uint8, device="cuda")   # allocator churn on the current stream
    side.synchronize()
    Pref = rf.rf_phi_closed_form(Xd, act="tanh", prec="bf16")
    torch.cuda.synchronize()
    for G, Phi in outs:
        assert torch.equal(G, ref)
        assert torch.equal(Phi, Pref)


@pytest.mark.parametrize("ares,dyn", [(1, 1), (1, 0), (2, 1)])
@pytest.mark.parametrize("out,rows", [("upper", None), ("full", None), ("packed_tri", None), ("upper", (512, 1536))])
def test_phi_a_resident_bit_exact(ares, dyn, out, rows):
    """K5 with A-panel residency (RF_OPT_K5_ARES: each CTA keeps its A rows over the whole K = p in shared memory for
    a segment of up to 16 column tiles; column-block-major segment schedule, segments pulled from a device counter
    (RF_OPT_K5_DYNAMIC = 1) or dealt round-robin (0)) computes every entry with the same arithmetic as the K5 without
    residency: bit-identical, in every layout and on a row block."""
    n, p = 2100, 448                     # 7 K-blocks, ragged rows
    X = synthetic.make_X(4, n=n, p=p)
    Xd = dev(X, "bf16")
    ctx = rf.Context(0)
    ctx.set_option("k5_dynamic", dyn)
    res = []
    for a in (ares, 0):
        ctx.set_option("k5_ares", a)
        kw = {} if rows is None else {"row_begin": rows[0], "row_end": rows[1]}
        if out == "packed_tri":
            P = torch.full((rf.rf_packed_tri_elems(n),), float("nan"), device="cuda")
        else:
            P = torch.full((n, n), SENTINEL, device="cuda")
        rf.rf_phi_closed_form(Xd, act="tanh", prec="bf16", out=out, Phi=P, ctx=ctx, **kw)
        torch.cuda.synchronize()
        res.append(P.cpu().numpy())
    if out == "packed_tri":
        from paper_2110_01899_b200 import layout
        res = [layout.unpack_tri(r, n) for r in res]
        I, J = upper_idx(n)
        assert np.array_equal(res[0][I, J], res[1][I, J])
    else:
        assert np.array_equal(res[0], res[1])
