"""Pins for the oracle's EQ1 and its Gram–Schmidt inputs.

The decisive pin: EQ1 is, by its derivation, the expectation of the product of
the two second-order Taylor polynomials
    (f_a + f_a' δ_a + ½ f_a'' δ_a²) (f_b + f_b' δ_b + ½ f_b'' δ_b²),
    f = σ^{(d)}(√τ ξ), δ_a = α√τξ_a, δ_b = β√τξ_b + ν√τξ_a, ξ_a ⊥ ξ_b,
so an independent 2-D Gauss–Hermite integration of that product (SciPy nodes, σ from NumPy)
must reproduce the oracle's 18-term sum to rounding.  A dropped term, a wrong coefficient, a
wrong moment index or the as-printed (garbled) reading fails it.
"""
import math

import numpy as np
import pytest
from scipy import special as sp

import oracle

SIG = {
    "tanh": (np.tanh, lambda x: 1 - np.tanh(x) ** 2, lambda x: -2 * np.tanh(x) * (1 - np.tanh(x) ** 2)),
    "erf": (sp.erf, lambda x: 2 / math.sqrt(math.pi) * np.exp(-x * x),
            lambda x: -4 * x / math.sqrt(math.pi) * np.exp(-x * x)),
    "sigmoid_half": (lambda x: sp.expit(x) - 0.5, lambda x: sp.expit(x) * (1 - sp.expit(x)),
                     lambda x: sp.expit(x) * (1 - sp.expit(x)) * (1 - 2 * sp.expit(x))),
}
# A non-odd activation so every one of the 18 terms is exercised (softplus).
SOFTPLUS = (lambda x: np.logaddexp(0, x), lambda x: sp.expit(x), lambda x: sp.expit(x) * (1 - sp.expit(x)))

PAIRS = [  # (tau, u_a, v_b, u_b)
    (1.0, 1.05, 0.1, 0.97),
    (1.2, 0.9, -0.15, 1.1),
    (0.8, 0.7, 0.3, 0.75),
    (1.0833, 1.0, 1.0, 0.0),
    (1.0, 1.0, 0.0, 1.0),
    (1.5, 1.4, -0.4, 0.6),
]


def taylor_product_2d(fns, tau, u_a, v_b, u_b, N=200):
    f0, f1, f2 = fns
    x, w = sp.roots_hermitenorm(N)
    w = w / w.sum()
    st = math.sqrt(tau)
    al, be, nu = u_a / st - 1, u_b / st - 1, v_b / st
    xa = x[:, None]
    xb = x[None, :]
    da = al * st * xa
    db = be * st * xb + nu * st * xa
    pa = f0(st * xa) + f1(st * xa) * da + 0.5 * f2(st * xa) * da ** 2
    pb = f0(st * xb) + f1(st * xb) * db + 0.5 * f2(st * xb) * db ** 2
    return float(np.sum(w[:, None] * w[None, :] * pa * pb))


@pytest.mark.parametrize("name", ["tanh", "erf", "sigmoid_half", "softplus"])
@pytest.mark.parametrize("pair", PAIRS)
def test_eq1_equals_expectation_of_truncated_taylor_product(name, pair):
    fns = SOFTPLUS if name == "softplus" else SIG[name]
    act = SOFTPLUS if name == "softplus" else name
    tau, u_a, v_b, u_b = pair
    mom = oracle.moments(act, tau, 200)
    got = float(oracle.eq1(mom, u_a, v_b, u_b))
    want = taylor_product_2d(fns, tau, u_a, v_b, u_b)
    assert abs(got - want) < 1e-12 * max(1.0, abs(want)), (got, want)


def test_as_printed_eq1_is_rejected():
    """The printed EQ1 (four garbles) does NOT match the Taylor expectation — proves the pin bites."""
    tau, u_a, v_b, u_b = 1.0, 1.05, 0.1, 0.97
    mom = oracle.moments(SOFTPLUS, tau, 200)
    terms = oracle.eq1_terms(mom, u_a, v_b, u_b)
    M = mom["kd"]
    st = math.sqrt(tau)
    a, b, v = u_a / st - 1, u_b / st - 1, v_b / st
    printed = list(terms)
    printed[4] = M[0, 0] * M[2, 2] / 2 * (u_b - 1) ** 2
    printed[9] = M[0, 2] * M[2, 2] / 2 * v ** 2
    printed[11] = M[0, 1] * (M[2, 1] / tau) * v * a
    printed[13] = M[0, 1] * M[2, 1] / 2 * v * a * b
    want = taylor_product_2d(SOFTPLUS, tau, u_a, v_b, u_b)
    assert abs(sum(terms) - want) < 1e-12
    assert abs(sum(printed) - want) > 1e-5


@pytest.mark.parametrize("act", ["tanh", "erf", "sigmoid_half"])
def test_eq1_error_vs_exact_kernel_is_cubic(act):
    """EQ1 drops O(δ³) ("+O(p^{-3/2})"): shrinking the deviation from the expansion point
    by 2 divides |EQ1 − κ| by ≈ 8, with κ = E[σ(ζ_a)σ(ζ_b)] by 2-D quadrature."""
    tau = 1.0
    errs = []
    for h in (0.2, 0.1, 0.05, 0.025):
        u_a, v_b, u_b = 1 + h, 0.5 * h, 1 - 0.7 * h
        mom = oracle.moments(act, tau)
        errs.append(abs(float(oracle.eq1(mom, u_a, v_b, u_b)) - oracle.phi_exact_pair(act, u_a, v_b, u_b)))
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    for r in ratios[1:]:
        assert 6.5 < r < 9.5, ratios


@pytest.mark.parametrize("pair", PAIRS[:3])
def test_exact_kernel_erf_is_arcsine(pair):
    """For σ = erf, E_w[σ(wᵀx)σ(wᵀy)] = (2/π) arcsin(2xᵀy/√((1+2‖x‖²)(1+2‖y‖²))) (Williams 1997,
    cited at P:450).  Pins the oracle's 2-D quadrature of κ."""
    _, u_a, v_b, u_b = pair
    xx, yy, xy = u_a ** 2, v_b ** 2 + u_b ** 2, u_a * v_b
    want = 2 / math.pi * math.asin(2 * xy / math.sqrt((1 + 2 * xx) * (1 + 2 * yy)))
    assert abs(oracle.phi_exact_pair("erf", u_a, v_b, u_b) - want) < 1e-14


def test_eq1_expansion_point_and_first_order():
    """At u_a = u_b = √τ, v_b = 0: Φ = E[σ]².  ∂Φ/∂g at g = 0 equals E[σ']², the exact
    ∂κ/∂(xᵀy) at orthogonality (Stein) — first-order exactness of the expansion."""
    for act in ("tanh", "erf", "sigmoid_half"):
        tau = 1.1
        mom = oracle.moments(act, tau)
        st = math.sqrt(tau)
        assert abs(float(oracle.eq1(mom, st, 0.0, st)) - mom["kd"][0, 0] ** 2) < 1e-15
        eps = 1e-6
        # g = x_iᵀx_j = u_a v_b  ⇒ v_b = g/u_a; u_b = √(τ − g²/τ)
        f = lambda g: float(oracle.eq1(mom, st, g / st, math.sqrt(tau - g * g / tau)))
        deriv = (f(eps) - f(-eps)) / (2 * eps)
        assert abs(deriv - mom["kd"][0, 1] ** 2) < 1e-8


def test_phi_matrix_structure_and_identities():
    rng = np.random.default_rng(11)
    p, n = 32, 40
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    # odd σ ⇒ Φ_ij = 0 exactly when x_iᵀx_j = 0
    X[1] = X[0][::-1] * np.array([1, -1] * (p // 2))       # construct x_1 ⊥ x_0 below
    X[1] -= X[0] * (X[0] @ X[1]) / (X[0] @ X[0])
    P = oracle.phi_eq1(X, "tanh")
    assert abs(P[0, 1]) < 1e-15
    assert np.all(np.isnan(np.tril(P, -1)[np.tril_indices(n, -1)]))
    # sigmoid − ½ = ½ tanh(·/2)  ⇒  Φ_sig(X; τ) = ¼ Φ_tanh(X/2; τ/4)
    tau = oracle.tau_hat(X)
    a = oracle.phi_eq1(X, "sigmoid_half", tau)
    b = oracle.phi_eq1(X / 2, "tanh", tau / 4)
    iu = np.triu_indices(n)
    assert np.max(np.abs(a[iu] - 0.25 * b[iu])) < 1e-15
    # diagonal rule: Φ_ii = EQ1(u_a = ‖x_i‖, v_b = ‖x_i‖, u_b = 0)
    mom = oracle.moments("tanh", tau)
    r = math.sqrt(X[3] @ X[3])
    assert abs(P[3, 3] - float(oracle.eq1(mom, r, r, 0.0))) < 1e-15


def test_gram_schmidt_reconstructs_bivariate_covariance():
    """(wᵀx_i, wᵀx_j) = (u_a ξ_a, v_b ξ_a + u_b ξ_b): variances ‖x_i‖², ‖x_j‖², covariance x_iᵀx_j."""
    rng = np.random.default_rng(5)
    xi, xj = rng.standard_normal(7), rng.standard_normal(7)
    u_a, v_b, u_b = oracle.gram_schmidt(xi @ xi, xj @ xj, xi @ xj, False)
    assert abs(u_a ** 2 - xi @ xi) < 1e-13
    assert abs(v_b ** 2 + u_b ** 2 - xj @ xj) < 1e-12
    assert abs(u_a * v_b - xi @ xj) < 1e-13


@pytest.mark.parametrize("act", ["tanh", "erf", "sigmoid_half"])
def test_pivot_asymmetry_diagnostic(act):
    """Reading R6: EQ1 with x_i as the Gram–Schmidt pivot is not symmetric.  Both orientations agree with the
    symmetric kernel to second order, so their difference is at least third order in the deviation from the
    expansion point (ratio ≥ 8 per halving asymptotically; sigmoid − ½'s cubic coefficient is tiny, its ratios are
    higher), and it vanishes when the two norms are equal (the swap then leaves u_a, v_b, u_b unchanged)."""
    def pair(h):
        c, d = 0.5 * h, 1.0 - 0.4 * h
        return np.array([[1.0 + 0.7 * h, 0.0], [d * c, d * math.sqrt(1.0 - c * c)]])
    a = [oracle.phi_pivot_asymmetry(pair(h), act, tau=1.0) for h in (0.2, 0.1, 0.05)]
    assert all(x > 0 for x in a)
    r1, r2 = a[0] / a[1], a[1] / a[2]
    assert r1 > 5.0 and r2 > 6.0, (a, r1, r2)
    rng = np.random.default_rng(3)
    Z = rng.standard_normal((6, 16))
    Z /= np.linalg.norm(Z, axis=1, keepdims=True)
    assert oracle.phi_pivot_asymmetry(Z * 1.1, act, tau=1.0) <= 1e-15 < a[2]   # equal norms up to rounding


# ------------------------------------------------------------------------------------------------------------------
# SURVEY.md §8(c)'s 13 survey-computed values (tests/golden/survey_eq1_values.txt): an independent computation of
# the corrected EQ1 and of the exact kernel, which the oracle must reproduce to ≤ 1e-10 (the values are printed to
# 12 decimals).  Includes the diagonal-type rows (u_b = 0) and the exact tanh / sigmoid−½ column.
# ------------------------------------------------------------------------------------------------------------------
import os  # noqa: E402

_SURVEY = os.path.join(os.path.dirname(__file__), "golden", "survey_eq1_values.txt")


def _survey_rows():
    rows = []
    for line in open(_SURVEY):
        if line.startswith("#") or not line.strip():
            continue
        f = [x.strip() for x in line.split("|")]
        rows.append((f[0], *map(float, f[1:])))
    return rows


def test_survey_golden_values_table_complete():
    rows = _survey_rows()
    assert len(rows) == 13
    assert sum(1 for r in rows if r[4] == 0.0) == 3          # one diagonal-type row per σ


@pytest.mark.parametrize("row", _survey_rows(), ids=lambda r: f"{r[0]}-{r[1]}-{r[2]}-{r[3]}-{r[4]}")
def test_oracle_reproduces_survey_golden_values(row):
    act, tau, u_a, v_b, u_b, want_eq1, want_exact = row
    mom = oracle.moments(act, tau, 200)
    got = float(oracle.eq1(mom, u_a, v_b, u_b))
    assert abs(got - want_eq1) <= 1e-10, (got, want_eq1)
    ex = oracle.phi_exact_pair(act, u_a, v_b, u_b, N=120)
    assert abs(ex - want_exact) <= 1e-10, (ex, want_exact)
    if act == "erf":   # the exact column is the arcsine kernel: x = (u_a, 0), y = (v_b, u_b)
        arc = 2 / math.pi * math.asin(2 * u_a * v_b / math.sqrt((1 + 2 * u_a ** 2) * (1 + 2 * (v_b ** 2 + u_b ** 2))))
        assert abs(arc - want_exact) <= 1e-10, (arc, want_exact)


def test_zero_pivot_reading_r23():
    """R23: a zero sample x_i = 0 as the Gram–Schmidt pivot has v_b = 0, u_b = ‖x_j‖ (x_j is orthogonal to it), so
    for odd σ EQ1 gives the exact kernel's value E[σ(0)σ(‖x_j‖ξ)] = 0 (to the quadrature's ⟨0,0⟩ ≈ 1e-17), and Φ is
    finite everywhere."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((6, 16)) / 4
    X[2] = 0.0
    for act in ("tanh", "erf", "sigmoid_half"):
        P = oracle.phi_eq1(X, act, tau=1.0)
        I, J = np.triu_indices(6)
        assert np.all(np.isfinite(P[I, J]))
        assert np.all(np.abs(P[2, 2:]) < 1e-15)
        assert abs(oracle.phi_exact_pair(act, 0.0, 0.0, float(np.linalg.norm(X[4])))) < 1e-15
    u_a, v_b, u_b = oracle.gram_schmidt(np.array([0.0]), np.array([2.25]), np.array([0.0]), np.array([False]))
    assert u_a[0] == 0.0 and v_b[0] == 0.0 and u_b[0] == 1.5
