"""Pins of the NEXT-2 oracle (oracle/center.py): centering by P (Eq. (2)) and Theorem 1's K̃ (EQ6) against what
the paper fixes — the theorem itself: ‖K − K̃‖ → 0 for GMM data, with K computed from EXACT expected kernels
(σ(t) = t²: Isserlis; σ = erf: the arcsine kernel), so no Monte Carlo noise enters.  The quadratic σ has d2 = 1,
d1 = 0, d0 = 2τ² (Table 2) and exercises the V·A·Vᵀ term (t, T, φ) on a heteroscedastic two-class GMM."""
import math

import numpy as np
import pytest

import oracle
from oracle import center as C


def _gmm(n, p, seed, hetero=True):
    """x_i = ±μ/√p + z_i (Eq. (GMM)), ‖μ‖ = 2; class 1: C = I, class 2: C = diag(0.5, 2.5 halves)."""
    rng = np.random.default_rng(seed)
    mu = rng.standard_normal(p)
    mu *= 2 / np.linalg.norm(mu)
    lab = np.repeat([0, 1], n // 2)
    c2 = np.where(np.arange(p) < p // 2, 0.5, 2.5) if hetero else np.ones(p)
    Z = rng.standard_normal((n, p)) / math.sqrt(p)
    Z[lab == 1] *= np.sqrt(c2)[None, :]
    X = Z + np.where(lab == 0, 1.0, -1.0)[:, None] * mu[None, :] / math.sqrt(p)
    J = np.stack([lab == 0, lab == 1], 1).astype(float)
    trC = np.array([1.0, float(np.mean(c2))])                 # tr(C_a)/p
    tau = float(np.mean(trC))                                  # tr(C°)/p with n_1 = n_2
    T = np.array([[1.0, float(np.mean(c2))], [float(np.mean(c2)), float(np.mean(c2 * c2))]])   # tr(C_a C_b)/p
    phi = np.sum(Z * Z, 1) - trC[lab]                          # ‖z_i‖² − E‖z_i‖²
    t = (trC - tau) * math.sqrt(p)                             # tr(C_a°)/√p
    return X, J, phi, t, T, tau


def _rel2(A, B):
    return float(np.linalg.norm(A - B, 2) / np.linalg.norm(A, 2))


def test_centering_projector_identities():
    n = 37
    Pn = C.P(n)
    assert np.allclose(Pn @ Pn, Pn, atol=1e-14) and np.allclose(Pn, Pn.T)
    assert np.allclose(Pn @ np.ones(n), 0, atol=1e-14)
    rng = np.random.default_rng(1)
    A = rng.standard_normal((n, n))
    A = A + A.T
    K = C.center(A)
    assert np.allclose(K.sum(0), 0, atol=1e-12) and np.allclose(K.sum(1), 0, atol=1e-12)
    r = A.mean(1)                                              # row-means form of P·A·P for symmetric A
    assert np.allclose(K, A - r[:, None] - r[None, :] + r.mean(), atol=1e-13)
    assert np.allclose(C.center(np.ones((n, n))), 0, atol=1e-13)


def test_theorem1_quadratic_sigma_converges():
    errs = []
    for n, p in [(512, 256), (2048, 1024)]:
        X, J, phi, t, T, tau = _gmm(n, p, seed=n)
        V, A = C.gmm_V_A(J, phi, t, T, p)
        K = C.center(C.quadratic_kernel(X))
        Kt = C.ktilde(X, V, A, 2 * tau ** 2, 0.0, 1.0)       # σ = t²: d0 = 2τ², d1 = 0, d2 = 1 (Table 2)
        errs.append(_rel2(K, Kt))
        # dropping φ or t, or flipping t, must be visibly worse (pins the V·A·Vᵀ term)
        for tt, ph in [(0 * t, phi), (t, 0 * phi), (-t, phi)]:
            Vw, Aw = C.gmm_V_A(J, ph, tt, T, p)
            assert _rel2(K, C.ktilde(X, Vw, Aw, 2 * tau ** 2, 0.0, 1.0)) > 2 * errs[-1]
        if n == 2048:   # the d0 regulariser (2τ², Table 2) and the d2 weight are pinned too
            assert _rel2(K, C.ktilde(X, V, A, tau ** 2, 0.0, 1.0)) > 1.3 * errs[-1]
            assert _rel2(K, C.ktilde(X, V, A, 2 * tau ** 2, 0.0, 0.5)) > 1.3 * errs[-1]
    assert errs[1] < 0.05 and errs[1] < 0.5 * errs[0], errs


def test_theorem1_T_term_is_the_best_fit():
    """The 2T block of A is a small effect at these sizes; among T, T/2 and the isotropic guess tr(C_a)tr(C_b)/p²,
    the theorem's T fits the exact kernel best (a weak pin on its own; the sharp pin of the 2T block is the class
    contrast in test_theorem1_2T_block_is_pinned_by_the_class_contrast)."""
    n, p = 2048, 1024
    X, J, phi, t, T, tau = _gmm(n, p, seed=5)
    K = C.center(C.quadratic_kernel(X))
    e = {}
    for name, TT in {"T": T, "T/2": 0.5 * T, "outer": np.outer(np.diag(T) ** 0.5, np.diag(T) ** 0.5) * 0 +
                     np.outer([1.0, T[0, 1]], [1.0, T[0, 1]])}.items():
        V, A = C.gmm_V_A(J, phi, t, TT, p)
        e[name] = _rel2(K, C.ktilde(X, V, A, 2 * tau ** 2, 0.0, 1.0))
    assert e["T"] < e["T/2"] and e["T"] < e["outer"], e


@pytest.mark.parametrize("act", ["erf"])
def test_theorem1_erf_converges(act):
    errs = []
    for n, p in [(512, 256), (2048, 1024)]:
        X, J, phi, t, T, tau = _gmm(n, p, seed=n + 1, hetero=False)
        mo = oracle.moments(act, tau)
        V, A = C.gmm_V_A(J, phi, t, T, p)
        K = C.center(C.arcsine_kernel(X))
        Kt = C.ktilde(X, V, A, mo["d0"], mo["d1"], mo["d2"])
        errs.append(_rel2(K, Kt))
    assert errs[1] < 0.03 and errs[1] < 0.75 * errs[0], errs


def _offdiag_block_contrast(D, lab):
    """m_11 − m_12 − m_21 + m_22 of the block means of D over i ≠ j.  Row- or column-additive terms (so also the
    centering by P, and everything ‖x_i‖²‖x_j‖² contributes beyond α_iα_j) cancel in it exactly."""
    D = D.copy()
    np.fill_diagonal(D, 0.0)
    m = np.zeros((2, 2))
    for a in range(2):
        for b in range(2):
            ia, ib = np.where(lab == a)[0], np.where(lab == b)[0]
            cnt = len(ia) * len(ib) - (len(ia) if a == b else 0)
            m[a, b] = D[np.ix_(ia, ib)].sum() / cnt
    return m[0, 0] - m[0, 1] - m[1, 0] + m[1, 1]


def test_theorem1_2T_block_is_pinned_by_the_class_contrast():
    """Sharp pin of the 2T block of A (Theorem 1).  For σ = t² the exact kernel is ‖x‖²‖y‖² + 2(xᵀy)², and
    for i ≠ j in classes a, b: E[2(x_iᵀx_j)²] = 2·tr(C_aC_b)/p² + (terms additive in a and b) — Isserlis.  So the
    double class contrast of (exact kernel − K̃ built with T = 0) must equal that of the (J/√p)(2T)(J/√p)ᵀ block,
    (2/p)(T_11 − 2T_12 + T_22), up to the law-of-large-numbers noise of ≈ n²/4 entries per block (≈ 1 %).  A wrong
    factor (T instead of 2T), a wrong T (tr C_a·tr C_b/p²) or a dropped block misses by 50 %, 80 % or 100 %."""
    n, p = 2048, 1024
    X, J, phi, t, T, tau = _gmm(n, p, seed=7)
    lab = (J[:, 1] > 0).astype(int)
    K = C.center(C.quadratic_kernel(X))
    d0 = 2 * tau ** 2

    def kt(TT):
        V, A = C.gmm_V_A(J, phi, t, TT, p)
        return C.ktilde(X, V, A, d0, 0.0, 1.0)

    K0 = kt(0 * T)
    want = _offdiag_block_contrast(K - K0, lab)                      # what the data say the block must supply
    theory = 2.0 / p * (T[0, 0] - 2 * T[0, 1] + T[1, 1])             # (2/p)(1 − 3 + 3.25) = 2.5/p here
    assert abs(want / theory - 1) < 0.05, (want, theory)
    got = _offdiag_block_contrast(kt(T) - K0, lab)                   # what the oracle's K̃ supplies
    assert abs(got / want - 1) < 0.05, (got, want)
    assert abs(got / theory - 1) < 1e-9                              # and it is exactly the 2T block
    outer = np.outer([1.0, T[0, 1]], [1.0, T[0, 1]])
    for TT in (0.5 * T, outer):
        assert abs(_offdiag_block_contrast(kt(TT) - K0, lab) / want - 1) > 0.4
