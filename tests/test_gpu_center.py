"""GPU parity of NEXT-2 (include/rf.h): centred outputs K = P·A·P (RF_OUT_*_CENTERED) of G, G^ter and Φ, and
Theorem 1's K̃ (rf_ktilde), against the fp64 oracle (oracle/center.py) on the same (rounded) inputs."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import center as C  # noqa: E402
from oracle import trf  # noqa: E402
import paper_2110_01899_b200 as rf  # noqa: E402
import synthetic  # noqa: E402
from entry_bounds import center_bound, check, full_pairs, gram_bound, phi_bound  # noqa: E402

pytestmark = pytest.mark.gpu
SENT = -7.25


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    assert rf.rf_device_supported(0), "device 0 is not sm_100"
    torch.cuda.set_device(0)
    yield


def _rel(got, ref):
    return float(np.linalg.norm(got - ref) / np.linalg.norm(ref))


@pytest.mark.parametrize("prec,out,tol", [("bf16", "upper_centered", 2e-3), ("3xtf32", "full_centered", 1e-5),
                                          ("fp32", "upper_centered", 1e-5), ("fp64", "full_centered", 1e-11)])
def test_gram_centered(prec, out, tol):
    n, p, m = 700, 96, 512
    rng = np.random.default_rng(3)
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    W = rng.standard_normal((m, p))
    dt = {"bf16": torch.bfloat16, "3xtf32": torch.float32, "fp32": torch.float32, "fp64": torch.float64}[prec]
    Xd, Wd = torch.tensor(X, device="cuda").to(dt), torch.tensor(W, device="cuda").to(dt)
    G = torch.full((n, n), SENT, dtype=torch.float64 if prec == "fp64" else torch.float32, device="cuda")
    rf.rf_gram(Xd, Wd, act="tanh", prec=prec, out=out, G=G)
    torch.cuda.synchronize()
    Xo, Wo = Xd.double().cpu().numpy(), Wd.double().cpu().numpy()
    A = oracle.gram(Xo, Wo, "tanh")
    ref = C.center(A)
    Gc = G.double().cpu().numpy()
    I, J = np.triu_indices(n)
    e = _rel(Gc[I, J], ref[I, J])
    print(f"[parity] centred G {prec} {out}: rel-Frobenius {e:.3e}")
    assert e <= tol
    FI, FJ = full_pairs(n)
    bA = gram_bound(prec, "tanh", Xo, Wo, A, FI, FJ).reshape(n, n)
    check(f"centred G {prec}", Gc[I, J], ref[I, J],
          center_bound(A, bA, I, J, u=2.0 ** -50 if prec == "fp64" else 2.0 ** -21))
    if out.startswith("upper"):
        assert np.all(Gc[np.tril_indices(n, -1)] == SENT)
    else:
        assert np.abs(Gc.sum(axis=1)).max() < 1e-4 * np.abs(Gc).max() * math.sqrt(n)


def test_phi_and_gram_ter_centered():
    n, p, m, eps = 600, 128, 800, 0.9
    X = synthetic.make_X(4, n=n, p=p)
    Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
    Xb = Xd.double().cpu().numpy()
    Phi = rf.rf_phi_closed_form(Xd, act="tanh", tau=0.0, prec="bf16", out="full_centered")
    torch.cuda.synchronize()
    U = np.nan_to_num(oracle.phi_eq1(Xb, "tanh"), nan=0.0)    # upper triangle (pivot = row), R6
    A = U + np.triu(U, 1).T                                     # FULL mirrors the upper triangle
    ref = C.center(A)
    e = _rel(Phi.double().cpu().numpy(), ref)
    print(f"[parity] centred Φ bf16: rel-Frobenius {e:.3e}")
    assert e < 1e-5
    I, J = np.triu_indices(n)
    bu = np.zeros((n, n))
    bu[I, J] = phi_bound("bf16", "tanh", Xb, oracle.tau_hat(Xb), I, J)
    bA = bu + np.triu(bu, 1).T
    FI, FJ = full_pairs(n)
    check("centred Φ bf16", Phi.double().cpu().numpy().ravel(), ref.ravel(), center_bound(A, bA, FI, FJ))
    with pytest.raises(rf.RFError):
        rf.rf_phi_closed_form(Xd, act="tanh", tau=1.0, prec="bf16", out="upper_centered", row_begin=0, row_end=256)
    T = synthetic.make_T(4, eps, m=m, p=p)
    Td = torch.tensor(T, device="cuda").to(torch.bfloat16)
    sm, sp = rf.rf_trf_thresholds_for("tanh", oracle.tau_hat(Xb))
    Gt = rf.rf_gram_ter(Xd, Td, eps, sm, sp, out="upper_centered")
    torch.cuda.synchronize()
    At = trf.gram_ter(Xb, T, eps, sm, sp)
    reft = C.center(At)
    I, J = np.triu_indices(n)
    e2 = _rel(Gt.double().cpu().numpy()[I, J], reft[I, J])
    print(f"[parity] centred G^ter: rel-Frobenius {e2:.3e}")
    assert e2 < 1e-5
    # G^ter is an exact count / m (test_gpu_trf): only decisions inside the fp32 band of a threshold may differ, each
    # moving an entry by ≤ 2/m; rows' band counts bound the uncentred error
    margin = trf.decision_margin(Xb, T, eps, sm, sp)
    band = (1 - eps) ** -0.5 * (math.ceil(p / 16) + 2) * 2.0 ** -23 * np.sum(np.abs(Xb), axis=1) + \
        2.0 ** -22 * max(abs(sm), abs(sp))                      # test_gpu_trf._band
    fr = np.sum(margin <= band[:, None], axis=1).astype(float)   # decisions that may flip, per row
    bA = (fr[:, None] + fr[None, :]) * 2.0 / m + 2.0 ** -22
    check("centred G^ter", Gt.double().cpu().numpy()[I, J], reft[I, J], center_bound(At, bA, I, J))


def _gmm_stats(n, p, seed):
    rng = np.random.default_rng(seed)
    mu = rng.standard_normal(p)
    mu *= 2 / np.linalg.norm(mu)
    lab = (np.arange(n) >= n // 2).astype(int)
    c2 = np.where(np.arange(p) < p // 2, 0.5, 2.5)
    Z = rng.standard_normal((n, p)) / math.sqrt(p)
    Z[lab == 1] *= np.sqrt(c2)[None, :]
    X = Z + np.where(lab == 0, 1.0, -1.0)[:, None] * mu[None, :] / math.sqrt(p)
    J = np.stack([lab == 0, lab == 1], 1).astype(float)
    trC = np.array([1.0, float(np.mean(c2))])
    tau = float(np.mean(trC[lab]))
    T = np.array([[1.0, trC[1]], [trC[1], float(np.mean(c2 * c2))]])
    phi = np.sum(Z * Z, 1) - trC[lab]
    t = (trC - tau) * math.sqrt(p)
    V, A = C.gmm_V_A(J, phi, t, T, p)
    return X, V, A, tau


@pytest.mark.parametrize("prec,out,n,p", [("bf16", "upper", 1000, 256), ("3xtf32", "full", 777, 300),
                                          ("tf32", "upper", 513, 64)])
def test_ktilde_matches_oracle(prec, out, n, p):
    X, V, A, tau = _gmm_stats(n, p, seed=n)
    mo = oracle.moments("tanh", tau)
    d0, d1, d2 = mo["d0"], mo["d1"], 0.37        # a non-zero d2 exercises the V·A·Vᵀ term
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    Xd = torch.tensor(X, device="cuda").to(dt)
    Vd = torch.tensor(V, device="cuda").to(torch.float32)
    Kt = torch.full((n, n), SENT, dtype=torch.float32, device="cuda")
    rf.rf_ktilde(Xd, Vd, A, d0, d1, d2, prec=prec, out=out, Kt=Kt)
    torch.cuda.synchronize()
    Xo, Vo = Xd.double().cpu().numpy(), Vd.double().cpu().numpy()
    ref = C.ktilde(Xo, Vo, A, d0, d1, d2)
    Kc = Kt.double().cpu().numpy()
    I, J = np.triu_indices(n)
    e = _rel(Kc[I, J], ref[I, J])
    tol = 2e-3 if prec == "tf32" else 1e-5
    print(f"[parity] K̃ {prec} {out} n={n} p={p}: rel-Frobenius {e:.3e}")
    assert e <= tol
    check(f"K̃ {prec}", Kc[I, J], ref[I, J], _ktilde_bound(prec, Xo, Vo, np.asarray(A, float), d0, d1, d2, I, J))
    if out == "upper":
        assert np.all(Kc[np.tril_indices(n, -1)] == SENT)
    else:
        assert np.array_equal(Kc, Kc.T)


def _ktilde_bound(prec, X, V, A, d0, d1, d2, I, J):
    """Per-entry bound of K̃ = d1·g + d2·u_iᵀv_j + d0·δ_ij − r'_i − r'_j (one fp32 epilogue over the XᵀX mainloop):
    g's conversion + accumulation error (entry_bounds.acc_rel), the rank-kv term and the row means in fp32."""
    from entry_bounds import U_OPERAND, acc_rel
    xn = np.sqrt(np.sum(X * X, axis=1))
    U = V @ A.T
    M = d1 * (X @ X.T) + d2 * (U @ V.T) + d0 * np.eye(len(X))
    r = M.mean(axis=1)
    s_ = r.mean()
    dg = (2 * U_OPERAND[prec] + acc_rel(prec, X.shape[1])) * xn[I] * xn[J]
    uv = np.abs(U[I]) @ np.ones(U.shape[1]) * 0 + np.sum(np.abs(U[I] * V[J]), axis=1)
    # r' comes from fp32 x̄ and per-row dot products of length p: same accumulation rule, relative to ‖x_i‖‖x̄‖/n
    xbar = X.sum(axis=0)
    dr = abs(d1) * (2 * U_OPERAND[prec] + acc_rel(prec, X.shape[1]) + 2.0 ** -20) * xn * np.linalg.norm(xbar) / len(X)
    return (abs(d1) * dg + abs(d2) * 2.0 ** -20 * uv + dr[I] + dr[J]
            + 2.0 ** -20 * (np.abs(M[I, J]) + np.abs(r[I]) + np.abs(r[J]) + abs(s_)) + 1e-9)


def test_ktilde_without_v_and_errors():
    n, p = 300, 64
    X = synthetic.make_X(0, n=n, p=p)
    Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
    Kt = rf.rf_ktilde(Xd, None, None, 0.1, 0.6, 0.0, prec="bf16", out="full")
    torch.cuda.synchronize()
    ref = C.ktilde(Xd.double().cpu().numpy(), np.zeros((n, 0)), np.zeros((0, 0)), 0.1, 0.6, 0.0)
    assert _rel(Kt.double().cpu().numpy(), ref) < 1e-5
    with pytest.raises(rf.RFError):
        rf.rf_ktilde(Xd, None, None, 0.1, 0.6, 0.0, prec="bf16", out="upper_centered")
