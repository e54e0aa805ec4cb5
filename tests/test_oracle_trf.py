"""Pins of the TRF oracle (oracle/trf.py) against what the paper and the mathematics fix (no GPU):
Table 2's sign(t) row, brute-force quadrature of the Stein integrals, the ReLU row as a solver target, the odd-σ
symmetry, exact integer structure of G^ter, the law of W^ter (Eq. (4)), and the Gaussian (CLT) limit of G^ter."""
import math

import numpy as np
import pytest
from scipy import integrate

import oracle
from oracle import trf
import synthetic


def _quad_moments(s_minus, s_plus, tau):
    """E[σ], E[ξσ], E[(ξ²−1)σ], E[σ²] of σ^ter(√τξ) by adaptive quadrature over the three pieces."""
    st = math.sqrt(tau)
    a, b = s_minus / st, s_plus / st
    pdf = lambda x: math.exp(-x * x / 2) / math.sqrt(2 * math.pi)
    def piece(f, lo, hi):
        return integrate.quad(lambda x: f(x) * pdf(x), lo, hi, epsabs=1e-14, epsrel=1e-13, limit=200)[0]
    L, H = -40.0, 40.0
    out = {}
    for name, f in (("E_s", lambda x: 1.0), ("E_xs", lambda x: x), ("E_x2m1s", lambda x: x * x - 1.0)):
        out[name] = -piece(f, L, a) + piece(f, b, H)
    out["E_sq"] = piece(lambda x: 1.0, L, a) + piece(lambda x: 1.0, b, H)
    return out


@pytest.mark.parametrize("s_minus,s_plus,tau", [(0.0, 0.0, 1.0), (-0.7, 0.7, 1.0), (-0.3, 1.1, 0.8),
                                                (0.5, 1.4, 1.0), (-2.0, -0.4, 2.5), (-1.0, 1.0, 0.25)])
def test_ternary_moments_match_quadrature(s_minus, s_plus, tau):
    m = trf.ternary_moments(s_minus, s_plus, tau)
    q = _quad_moments(s_minus, s_plus, tau)
    st = math.sqrt(tau)
    assert abs(m["E_s"] - q["E_s"]) < 1e-12
    assert abs(m["E_sq"] - q["E_sq"]) < 1e-12
    assert abs(m["E_s1"] - q["E_xs"] / st) < 1e-12            # Stein, first weak derivative
    assert abs(m["E_s2"] - q["E_x2m1s"] / tau) < 1e-12         # Stein, second weak derivative


@pytest.mark.parametrize("tau", [0.5, 1.0, 1.0833, 2.0])
def test_sign_row_of_table2(tau):
    """σ^ter with s− = s+ = 0 is sign(t): Table 2 d0 = 1 − 2/π, d1 = 2/(πτ), d2 = 0."""
    m = trf.ternary_moments(0.0, 0.0, tau)
    assert abs(m["d0"] - (1 - 2 / math.pi)) < 1e-14
    assert abs(m["d1"] - 2 / (math.pi * tau)) < 1e-14
    assert m["d2"] == 0.0


def test_eq8_as_printed_disagrees_with_sign_row():
    """Reading R15: Eq. (8) verbatim gives d1 = 4/π² at s± = 0, not Table 2's 2/(πτ) — so the oracle solves
    the thresholds from Eq. (5) directly."""
    d1_printed, _ = trf.eq8_as_printed(0.0, 0.0, 1.0)
    assert abs(d1_printed - 4 / math.pi ** 2) < 1e-15
    assert abs(d1_printed - 2 / math.pi) > 0.2


@pytest.mark.parametrize("act", ["tanh", "erf", "sigmoid_half"])
@pytest.mark.parametrize("tau", [1.0, 1.0133, 1.0833])
def test_thresholds_match_smooth_sigma_and_are_symmetric(act, tau):
    mo = oracle.moments(act, tau)
    sm, sp = trf.solve_thresholds(mo["d1"], mo["d2"], tau)
    t = trf.ternary_moments(sm, sp, tau)
    assert abs(t["d1"] - mo["d1"]) < 1e-12 * max(1.0, mo["d1"])
    assert abs(t["d2"] - mo["d2"]) < 1e-12
    assert abs(sm + sp) < 1e-7, "odd σ (d2 = 0) gives symmetric thresholds"
    # closed form of the symmetric case: 2φ(s+/√τ)/√τ = √d1
    b = sp / math.sqrt(tau)
    assert abs(2 * math.exp(-b * b / 2) / math.sqrt(2 * math.pi) / math.sqrt(tau) - math.sqrt(mo["d1"])) < 1e-10


@pytest.mark.parametrize("tau", [0.5, 1.0])
def test_thresholds_reproduce_relu_row(tau):
    """Table 2 ReLU row: d1 = 1/4, d2 = 1/(8πτ) as the target of Algorithm 1 step 2."""
    d1, d2 = 0.25, 1 / (8 * math.pi * tau)
    sm, sp = trf.solve_thresholds(d1, d2, tau)
    t = trf.ternary_moments(sm, sp, tau)
    assert sm <= sp
    assert abs(t["d1"] - d1) < 1e-12 and abs(t["d2"] - d2) < 1e-12
    sm2, sp2 = trf.solve_thresholds(d1, d2, tau, sign2=-1)       # the mirror solution
    assert abs(sm2 + sp) < 1e-8 and abs(sp2 + sm) < 1e-8


def test_thresholds_infeasible_targets_are_rejected():
    with pytest.raises(ValueError):
        trf.solve_thresholds(2 / math.pi + 0.05, 0.0, 1.0, cap=8.0)     # sign(t) already has the largest d1
    # |E[σ^ter'']| = |aφ(a) + bφ(b)|/τ ≤ 2φ(1)/τ: ReLU's d2 = 1/(8πτ) is out of reach at τ = 2
    assert 2 * math.sqrt(1 / (8 * math.pi * 2.0)) > 2 * math.exp(-0.5) / math.sqrt(2 * math.pi) / 2.0
    with pytest.raises(ValueError):
        trf.solve_thresholds(0.25, 1 / (8 * math.pi * 2.0), 2.0, cap=8.0)


def test_sigma_ter_definition():
    t = np.array([-2.0, -0.5, -0.49, 0.0, 0.5, 0.51, 3.0])
    assert trf.sigma_ter(t, -0.5, 0.5).tolist() == [-1.0, 0.0, 0.0, 0.0, 0.0, 1.0, 1.0]


def test_gram_ter_integer_structure_and_brute_force():
    rng = np.random.default_rng(3)
    n, p, m, eps = 9, 16, 40, 0.5
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    T = synthetic.make_T(0, eps, m=m, p=p)
    sm, sp = -0.3, 0.4
    G = trf.gram_ter(X, T, eps, sm, sp)
    # brute force: loop over features, Eq. (4)/(5) written out
    c = (1 - eps) ** -0.5
    Gb = np.zeros((n, n))
    for k in range(m):
        s = np.zeros(n)
        for i in range(n):
            z = sum(X[i, l] * c * T[k, l] for l in range(p))
            s[i] = -1.0 if z < sm else (1.0 if z > sp else 0.0)
        Gb += np.outer(s, s)
    Gb /= m
    assert np.allclose(G, Gb, atol=1e-15)
    mG = G * m
    assert np.array_equal(mG, np.round(mG))
    S = trf.ternary_features(X, T, eps, sm, sp)
    assert np.array_equal(np.diag(mG), np.sum(S != 0, axis=1).astype(float))
    assert np.array_equal(G, G.T)
    assert np.linalg.eigvalsh(G).min() > -1e-12


@pytest.mark.parametrize("eps", [0.0, 0.5, 0.9])
def test_ternary_weight_law(eps):
    """Eq. (4): P(0) = ε, P(±(1−ε)^{-1/2}) = (1−ε)/2 → E[w] = 0, E[w²] = 1 (Assumption on W)."""
    T = synthetic.make_T(2, eps, m=1024, p=1024)
    w = (1 - eps) ** -0.5 * T
    N = w.size
    nz = np.mean(T != 0)
    assert abs(nz - (1 - eps)) < 4 * math.sqrt(eps * (1 - eps) / N) + 1e-12
    assert abs(np.mean(w)) < 4 / math.sqrt(N)
    assert abs(np.mean(w * w) - 1.0) < 4 * math.sqrt(max(1 / (1 - eps) - 1, 1e-12) / N) + 1e-12


@pytest.mark.parametrize("eps", [0.0, 0.5])
def test_gram_ter_converges_to_gaussian_limit(eps):
    """For large p, wᵀx is Gaussian (CLT) with variance ‖x‖², so G^ter → E[σ^ter(ζ_a)σ^ter(ζ_b)] at the MC rate."""
    rng = np.random.default_rng(11)
    p, m = 1024, 60000
    z = rng.standard_normal((3, p))
    X = np.stack([z[0], 0.6 * z[0] + 0.8 * z[1], z[2] * 1.2]) / math.sqrt(p)
    T = synthetic.make_T(1, eps, m=m, p=p)
    sm, sp = -0.6, 0.8
    S = trf.ternary_features(X, T, eps, sm, sp)
    G = S @ S.T / m
    for i, j in [(0, 1), (0, 2), (1, 1), (0, 0)]:
        k = trf.kappa_ter_gaussian(X[i] @ X[i], X[i] @ X[j], X[j] @ X[j], sm, sp)
        var = np.var(S[i] * S[j])
        assert abs(G[i, j] - k) < 5 * math.sqrt(var / m) + 3e-3, (i, j, G[i, j], k)
