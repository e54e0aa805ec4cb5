"""GPU parity of NEXT-3: the Table-2 activations through the whole path (K3's σ epilogue, rf_moments' Stein-form
moments feeding EQ1) and the six-term EQ2 epilogue (rf_phi_eq2), against the fp64 oracle on the same rounded inputs."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_2110_01899_b200 as rf  # noqa: E402
import synthetic  # noqa: E402
from entry_bounds import check, gram_bound, phi_bound  # noqa: E402

pytestmark = pytest.mark.gpu
TABLE2 = ["relu", "abs", "sign", "step", "cos", "sin", "ident", "quad", "bump"]
DT = {"bf16": torch.bfloat16, "3xtf32": torch.float32, "fp32": torch.float32}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    assert rf.rf_device_supported(0), "device 0 is not sm_100"
    torch.cuda.set_device(0)
    yield


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("act", TABLE2)
@pytest.mark.parametrize("prec", ["bf16", "3xtf32", "fp32"])
def test_gram_table2(act, prec):
    n, p, m = 300, 72, 400
    rng = np.random.default_rng(11)
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    W = rng.standard_normal((m, p))
    Xd, Wd = torch.tensor(X, device="cuda").to(DT[prec]), torch.tensor(W, device="cuda").to(DT[prec])
    G = rf.rf_gram(Xd, Wd, act=act, prec=prec, out="upper")
    torch.cuda.synchronize()
    Xo, Wo = Xd.double().cpu().numpy(), Wd.double().cpu().numpy()
    ref = oracle.gram(Xo, Wo, act)
    I, J = np.triu_indices(n)
    Gc = G.double().cpu().numpy()
    e = _rel(Gc[I, J], ref[I, J])
    tol = 2e-3 if prec == "bf16" else (2e-5 if act in ("sign", "step") else 1e-5)
    print(f"[parity] G {act} {prec}: rel-Frobenius {e:.3e}")
    assert e <= tol
    check(f"G {act} {prec}", Gc[I, J], ref[I, J], gram_bound(prec, act, Xo, Wo, ref, I, J))


@pytest.mark.parametrize("act", TABLE2)
@pytest.mark.parametrize("form", [1, 2])
def test_phi_table2_eq1_eq2(act, form):
    n, p = 520, 96
    X = synthetic.make_X(4, n=n, p=p)
    Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
    Xb = Xd.double().cpu().numpy()
    Phi = rf.rf_phi_closed_form(Xd, act=act, tau=0.0, prec="bf16", out="upper", form=form)
    torch.cuda.synchronize()
    ref = (oracle.phi_eq1 if form == 1 else oracle.phi_eq2)(Xb, act)
    I, J = np.triu_indices(n)
    Pc = Phi.double().cpu().numpy()
    e = _rel(Pc[I, J], ref[I, J])
    print(f"[parity] Φ EQ{form} {act} bf16: rel-Frobenius {e:.3e}")
    assert e <= 1e-5
    check(f"Phi EQ{form} {act}", Pc[I, J], ref[I, J], phi_bound("bf16", act, Xb, oracle.tau_hat(Xb), I, J, form=form))


@pytest.mark.parametrize("act", ["tanh", "erf", "sigmoid_half"])
def test_phi_eq2_north_star_acts_3xtf32(act):
    n, p = 700, 128
    X = synthetic.make_X(1, n=n, p=p)
    Xd = torch.tensor(X, device="cuda").to(torch.float32)
    Phi = rf.rf_phi_closed_form(Xd, act=act, tau=0.0, prec="3xtf32", out="full", form=2)
    torch.cuda.synchronize()
    Xo = Xd.double().cpu().numpy()
    ref = oracle.phi_eq2(Xo, act)
    I, J = np.triu_indices(n)
    Pc = Phi.double().cpu().numpy()
    e = _rel(Pc[I, J], ref[I, J])
    print(f"[parity] Φ EQ2 {act} 3xtf32: rel-Frobenius {e:.3e}")
    assert e <= 1e-5
    check(f"Phi EQ2 {act} 3xtf32", Pc[I, J], ref[I, J], phi_bound("3xtf32", act, Xo, oracle.tau_hat(Xo), I, J, form=2))
    assert np.array_equal(Pc, Pc.T)


def test_trf_thresholds_for_relu_matches_table2_targets():
    """Algorithm 1 for the ReLU kernel (the paper's Fig. 1 setting): thresholds from rf_moments(ReLU)."""
    from oracle import trf
    tau = 1.0
    sm, sp = rf.rf_trf_thresholds_for("relu", tau)
    t = trf.ternary_moments(sm, sp, tau)
    assert abs(t["d1"] - 0.25) < 1e-10 and abs(t["d2"] - 1 / (8 * math.pi)) < 1e-10


def test_phi_eq2_config4_full_size_sampled():
    """configs[4] (n = 131072, p = 512): EQ2 through the 16-warp K5 epilogue, sampled principal submatrix (tile-boundary
    rows included) against the oracle's EQ2 with the τ̂ of all rows."""
    cfg = synthetic.CONFIGS[4]
    X = synthetic.make_X(cfg)
    Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
    Phi = rf.rf_phi_closed_form(Xd, act=cfg.act, tau=0.0, prec="bf16", out="upper", form=2)
    torch.cuda.synchronize()
    S = synthetic.sample_indices(cfg.n, count=768, tile_stride=256)     # every row ≡ 0, ±1 (mod 256)
    St = torch.tensor(S, device="cuda")
    sub = Phi.index_select(0, St).index_select(1, St).double().cpu().numpy()
    del Phi
    Xb = Xd.double().cpu().numpy()
    tau = oracle.tau_hat(Xb)
    ref = oracle.phi_eq2(Xb[S], cfg.act, tau=tau)
    I, J = np.triu_indices(len(S))
    e = _rel(sub[I, J], ref[I, J])
    print(f"[parity] Φ EQ2 configs[4] sampled |S|={len(S)}: rel-Frobenius {e:.3e}")
    assert e <= 1e-5
    check("Phi EQ2 configs[4]", sub[I, J], ref[I, J], phi_bound("bf16", cfg.act, Xb[S], tau, I, J, form=2))


# ------------------------------------------------------------------------------------------ Table 2's parametrised rows
def _param_acts():
    return [rf.rf_act_leaky_relu(1.0, -0.2), rf.rf_act_leaky_relu(0.5, 2.0), rf.rf_act_quadratic(0.4, -1.3, 0.7)]


@pytest.mark.parametrize("k", [0, 1, 2])
@pytest.mark.parametrize("prec", ["bf16", "3xtf32", "fp32"])
def test_gram_param_acts(k, prec):
    """G for Table 2's a₊max(0,t) + a₋max(0,−t) and a₂t² + a₁t + a₀ through K3's runtime σ (tensor
    core) and the SIMT K6, against the oracle's σ written literally; per-entry bounds."""
    act = _param_acts()[k]
    n, p, m = 300, 72, 400
    rng = np.random.default_rng(17 + k)
    Xd = torch.tensor(rng.standard_normal((n, p)) / math.sqrt(p), device="cuda").to(DT[prec])
    Wd = torch.tensor(rng.standard_normal((m, p)), device="cuda").to(DT[prec])
    G = rf.rf_gram(Xd, Wd, act=act, prec=prec, out="upper")
    torch.cuda.synchronize()
    Xo, Wo = Xd.double().cpu().numpy(), Wd.double().cpu().numpy()
    ref = oracle.gram(Xo, Wo, act)
    I, J = np.triu_indices(n)
    Gc = G.double().cpu().numpy()
    e = _rel(Gc[I, J], ref[I, J])
    print(f"[parity] G {act} {prec}: rel-Frobenius {e:.3e}")
    assert e <= (2e-3 if prec == "bf16" else 1e-5)
    check(f"G {act} {prec}", Gc[I, J], ref[I, J], gram_bound(prec, act, Xo, Wo, ref, I, J))


@pytest.mark.parametrize("k", [0, 1, 2])
@pytest.mark.parametrize("form", [1, 2])
def test_phi_param_acts(k, form):
    act = _param_acts()[k]
    n, p = 520, 96
    X = synthetic.make_X(4, n=n, p=p)
    Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
    Xb = Xd.double().cpu().numpy()
    Phi = rf.rf_phi_closed_form(Xd, act=act, tau=0.0, prec="bf16", out="upper", form=form)
    torch.cuda.synchronize()
    ref = (oracle.phi_eq1 if form == 1 else oracle.phi_eq2)(Xb, act)
    I, J = np.triu_indices(n)
    Pc = Phi.double().cpu().numpy()
    e = _rel(Pc[I, J], ref[I, J])
    print(f"[parity] Φ EQ{form} {act} bf16: rel-Frobenius {e:.3e}")
    assert e <= 1e-5
    check(f"Phi EQ{form} {act}", Pc[I, J], ref[I, J], phi_bound("bf16", act, Xb, oracle.tau_hat(Xb), I, J, form=form))
