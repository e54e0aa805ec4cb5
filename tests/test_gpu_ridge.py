"""GPU parity of NEXT-4 (include/rf.h rf_ridge): fp64 blocked Cholesky ridge on the random-features Gram of the
paper's GMM ridge setup, against the fp64 oracle (oracle/ridge.py) on the same fp32 Gram."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import ridge  # noqa: E402
import paper_2110_01899_b200 as rf  # noqa: E402
from paper_2110_01899_b200 import _lib  # noqa: E402
import synthetic  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    torch.cuda.set_device(0)
    yield


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _gram(n_train, n_test, p, m, act="cos", seed=0):
    X, y = synthetic.make_ridge_gmm(n_train, n_test, p, seed=seed)
    rng = np.random.default_rng(seed + 100)
    W = rng.standard_normal((m, p))
    Xd = torch.tensor(X, device="cuda").bfloat16()
    Wd = torch.tensor(W, device="cuda").bfloat16()
    G = rf.rf_gram(Xd, Wd, act=act, prec="bf16", out="upper")
    torch.cuda.synchronize()
    return G, y


@pytest.mark.parametrize("n_train,n_test", [(40, 17), (64, 64), (700, 300), (1024, 512)])
@pytest.mark.parametrize("nrhs", [1, 3])
def test_ridge_matches_oracle(n_train, n_test, nrhs):
    G, y = _gram(n_train, n_test, 96, 512)
    rng = np.random.default_rng(n_train)
    Y = np.concatenate([y, rng.standard_normal((y.shape[0], nrhs - 1))], axis=1) if nrhs > 1 else y
    gammas = [1e-2, 1.0, 1e3]
    a, yh = rf.rf_ridge(G, n_train, gammas, torch.tensor(Y[:n_train], device="cuda"))
    torch.cuda.synchronize()
    ref = ridge.ridge_path(G.double().cpu().numpy(), n_train, Y[:n_train], Y[n_train:], gammas)
    for g, (gam, a_ref, yh_ref, mse_ref) in enumerate(ref):
        ea = _rel(a[g].cpu().numpy(), a_ref)
        ey = _rel(yh[g].cpu().numpy(), yh_ref)
        print(f"[parity] ridge n={n_train}+{n_test} r={nrhs} γ={gam:g}: α {ea:.2e}  Ŷ {ey:.2e}  mse {mse_ref:.4f}")
        assert ea <= 1e-9 and ey <= 1e-9


def test_ridge_large_and_tail_block():
    """128 + 1 panels (n_train = 8256): every kernel of the blocked factorisation, the 64-row tail block included."""
    n_train, n_test = 8256, 256
    G, y = _gram(n_train, n_test, 64, 256, act="sigmoid_half", seed=3)
    a, yh = rf.rf_ridge(G, n_train, [0.5], torch.tensor(y[:n_train], device="cuda"))
    torch.cuda.synchronize()
    ((gam, a_ref, yh_ref, _),) = ridge.ridge_path(G.double().cpu().numpy(), n_train, y[:n_train], y[n_train:], [0.5])
    assert _rel(a[0].cpu().numpy(), a_ref) <= 1e-9
    assert _rel(yh[0].cpu().numpy(), yh_ref) <= 1e-9


def test_ridge_not_positive_definite_is_reported():
    n = 100
    G = -torch.eye(n, device="cuda")
    with pytest.raises(rf.RFError) as e:
        rf.rf_ridge(G, n, [0.5], torch.ones((n, 1), dtype=torch.float64, device="cuda"), n_test=0)
    assert e.value.status == _lib.RF_E_NONFINITE


def test_ridge_mse_trf_matches_relu_on_gmm():
    """The paper's ridge comparison (Fig. 1): TRFs with thresholds matched to the d1, d2 of ReLU
    random features (Algorithm 1) against ReLU features with Gaussian W, on the GMM of P:1177.  Checked loosely (the
    match is asymptotic in m): both beat the trivial predictor, their best test errors are close, and γ → ∞ gives
    the trivial predictor (MSE → E[y²] = 1).  ([cos, sin] RFFs, the paper's other reference, are out of reach of a
    ternary σ at this τ: rf_trf_thresholds rejects d2 = e^{−τ}/4 as infeasible.)"""
    n_train, n_test, p, m = 1024, 512, 512, 4096
    X, y = synthetic.make_ridge_gmm(n_train, n_test, p, seed=1)
    rng = np.random.default_rng(7)
    W = rng.standard_normal((m, p))
    Xd, Wd = torch.tensor(X, device="cuda").bfloat16(), torch.tensor(W, device="cuda").bfloat16()
    G = rf.rf_gram(Xd, Wd, act="relu", prec="bf16", out="upper")
    tau = oracle.tau_hat(Xd.double().cpu().numpy())
    sm, sp = rf.rf_trf_thresholds_for("relu", tau)
    T = torch.tensor(synthetic.make_T(1, 0.9, m=m, p=p), device="cuda").bfloat16()
    Gt = rf.rf_gram_ter(Xd, T, 0.9, sm, sp, out="upper")
    gammas = [1e-2, 1e-1, 1.0, 10.0, 1e6]
    Yt = torch.tensor(y[:n_train], device="cuda")
    _, yh_rf = rf.rf_ridge(G, n_train, gammas, Yt)
    _, yh_ter = rf.rf_ridge(Gt, n_train, gammas, Yt)
    torch.cuda.synchronize()
    e_rf = [ridge.mse(yh_rf[g].cpu().numpy(), y[n_train:]) for g in range(len(gammas))]
    e_ter = [ridge.mse(yh_ter[g].cpu().numpy(), y[n_train:]) for g in range(len(gammas))]
    print(f"[ridge] GMM test MSE γ={gammas}: ReLU RF {np.round(e_rf, 4)}  TRF(ε=0.9) {np.round(e_ter, 4)}")
    assert min(e_rf[:4]) < 0.9 and min(e_ter[:4]) < 0.9              # better than the trivial predictor
    assert abs(min(e_rf[:4]) - min(e_ter[:4])) < 0.05
    assert abs(e_rf[-1] - 1.0) < 0.05 and abs(e_ter[-1] - 1.0) < 0.05
