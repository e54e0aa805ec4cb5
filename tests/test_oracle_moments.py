"""Pins for the oracle's Gauss–Hermite rule, σ derivatives and Gaussian moments.

Nothing here re-types the oracle's own formulas: every check is against something the paper
or the mathematics fixes (paper-printed closed forms, SciPy's independent Hermite rule,
finite differences, Stein's lemma, closed-form erf moments, a trapezoid quadrature).
"""
import math
import os

import numpy as np
import pytest
from scipy import special as sp

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_gaussian_moments.txt")


def _golden_rows():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            act, q, expr, cite = [s.strip() for s in line.split("|")]
            rows.append((act, q, expr, cite))
    return rows


A2, A1, A0 = 0.7, -1.3, 0.4
AP, AM = 1.0, -0.2          # leaky ReLU of slope 0.2 in Table 2's a₊·max(0,t) + a₋·max(0,−t) form
TEST_ACTS = {
    "cos": (np.cos, lambda x: -np.sin(x), lambda x: -np.cos(x)),
    "sin": (np.sin, np.cos, lambda x: -np.sin(x)),
    "ident": (lambda x: x, lambda x: np.ones_like(x), lambda x: np.zeros_like(x)),
    "quad": (lambda x: A2 * x * x + A1 * x + A0, lambda x: 2 * A2 * x + A1, lambda x: 2 * A2 * np.ones_like(x)),
    "bump": (lambda x: np.exp(-x * x / 2), lambda x: -x * np.exp(-x * x / 2),
             lambda x: (x * x - 1) * np.exp(-x * x / 2)),
}


@pytest.mark.parametrize("N", [4, 16, 64, 128, 200])
def test_hermite_rule_matches_scipy(N):
    x, w = oracle.hermite_rule(N)
    xs, ws = sp.roots_hermitenorm(N)
    ws = ws / ws.sum()
    assert np.max(np.abs(x - xs)) < 1e-12 * max(1.0, np.max(np.abs(xs)))
    assert np.max(np.abs(w - ws) / ws) < 1e-9
    assert abs(w.sum() - 1.0) < 1e-13


@pytest.mark.parametrize("N", [10, 40, 128])
def test_hermite_rule_integrates_gaussian_moments_exactly(N):
    # E[ξ^{2k}] = (2k−1)!! — exact for polynomials of degree ≤ 2N−1.
    x, w = oracle.hermite_rule(N)
    for k in range(0, min(N, 12)):
        exact = float(np.prod(np.arange(2 * k - 1, 0, -2))) if k > 0 else 1.0
        assert abs(np.sum(w * x ** (2 * k)) - exact) <= 1e-11 * exact
        assert abs(np.sum(w * x ** (2 * k + 1))) < 1e-9 * max(1.0, exact)


@pytest.mark.parametrize("act", oracle.ACTS)
def test_derivatives_match_finite_differences(act):
    x = np.linspace(-3, 3, 61)
    h = 1e-4
    f = lambda t: oracle.sigma(act, t)
    d1_fd = (-f(x + 2 * h) + 8 * f(x + h) - 8 * f(x - h) + f(x - 2 * h)) / (12 * h)
    d2_fd = (-f(x + 2 * h) + 16 * f(x + h) - 30 * f(x) + 16 * f(x - h) - f(x - 2 * h)) / (12 * h * h)
    assert np.max(np.abs(oracle.dsigma(act, x) - d1_fd)) < 1e-9
    assert np.max(np.abs(oracle.d2sigma(act, x) - d2_fd)) < 1e-6


def test_sigma_definitions_special_values():
    # library definitions: tanh(1), erf(1), sigmoid(1) − 1/2 = (e−1)/(2(e+1))
    assert abs(oracle.sigma("tanh", 1.0) - math.tanh(1.0)) < 1e-16
    assert abs(oracle.sigma("erf", 1.0) - math.erf(1.0)) < 2.3e-16
    assert abs(oracle.sigma("sigmoid_half", 1.0) - (math.e - 1) / (2 * (math.e + 1))) < 1e-15


@pytest.mark.parametrize("tau", [0.3, 1.0, 2.5])
def test_paper_printed_gaussian_moments(tau):
    """Table 2 and the draft tables — values printed in the paper."""
    rows = _golden_rows()
    assert len(rows) >= 25
    env = {"exp": math.exp, "sqrt": math.sqrt, "pi": math.pi, "tau": tau, "a0": A0, "a1": A1, "a2": A2, "ap": AP,
           "am": AM}
    for act, q, expr, cite in rows:
        # analytic derivatives by Gauss–Hermite where the golden row's σ is defined locally; the Table-2
        # activations with kinks/jumps (|t|, ReLU, sign, 1_{t>0}, leaky) go through the oracle's Stein-form moments
        if act == "leaky":
            mom = oracle.moments(f"leaky_relu({AP!r},{AM!r})", tau)
        else:
            mom = oracle.moments(TEST_ACTS[act], tau, N=128) if act in TEST_ACTS else oracle.moments(act, tau)
        kd = mom["kd"]
        got = {"d0": mom["d0"], "d1": mom["d1"], "d2": mom["d2"], "E_s": kd[0, 0], "E_s1": kd[0, 1],
               "E_s2": kd[0, 2], "E_sq": mom["e_sigma_sq"]}[q]
        want = eval(expr, {"__builtins__": {}}, env)
        assert abs(got - want) < 1e-11 * max(1.0, abs(want)), (act, q, cite, got, want)


@pytest.mark.parametrize("tau", [0.5, 1.0, 1.0133, 3.0])
def test_erf_moments_closed_form(tau):
    """E over ξ of erf and its derivatives: with c = 2/√π,
    E[erf'(√τξ)] = c/√(1+2τ), ⟨1,0⟩ = τ⟨0,1⟩, ⟨1,2⟩ = −2cτ(1+2τ)^{-3/2}, ⟨2,1⟩ = cτ(1+2τ)^{-3/2},
    ⟨3,2⟩ = −6cτ²(1+2τ)^{-5/2}, E[erf(√τξ)²] = (2/π) arcsin(2τ/(1+2τ))."""
    c = 2 / math.sqrt(math.pi)
    kd = oracle.moments("erf", tau)["kd"]
    q = 1 + 2 * tau
    assert abs(kd[0, 1] - c / math.sqrt(q)) < 1e-14
    assert abs(kd[1, 0] - tau * c / math.sqrt(q)) < 1e-14
    assert abs(kd[1, 2] - (-2 * c * tau * q ** -1.5)) < 1e-14
    assert abs(kd[2, 1] - c * tau * q ** -1.5) < 1e-14
    assert abs(kd[3, 2] - (-6 * c * tau ** 2 * q ** -2.5)) < 5e-13
    e2 = oracle.moments("erf", tau)["e_sigma_sq"]
    assert abs(e2 - 2 / math.pi * math.asin(2 * tau / (1 + 2 * tau))) < 1e-14


@pytest.mark.parametrize("act", oracle.ACTS)
@pytest.mark.parametrize("tau", [0.7, 1.0, 1.0833])
def test_stein_identities_and_odd_structure(act, tau):
    """Stein's lemma E[√τξ g(√τξ)] = τ E[g'(√τξ)] (draft P:182-189):
    ⟨1,0⟩ = τ⟨0,1⟩, ⟨1,1⟩ = τ⟨0,2⟩, ⟨2,1⟩ = τ(⟨0,1⟩ + ⟨1,2⟩), ⟨2,0⟩ = τ(⟨0,0⟩ + ⟨1,1⟩).
    Odd σ: ⟨k,d⟩ = 0 when k + d is even."""
    kd = oracle.moments(act, tau)["kd"]
    assert abs(kd[1, 0] - tau * kd[0, 1]) < 1e-12
    assert abs(kd[1, 1] - tau * kd[0, 2]) < 1e-12
    assert abs(kd[2, 1] - tau * (kd[0, 1] + kd[1, 2])) < 1e-12
    assert abs(kd[2, 0] - tau * (kd[0, 0] + kd[1, 1])) < 1e-12
    for k in range(5):
        for d in range(3):
            if (k + d) % 2 == 0:
                assert abs(kd[k, d]) < 1e-14


@pytest.mark.parametrize("act", oracle.ACTS)
@pytest.mark.parametrize("tau", [1.0, 1.0133, 1.0833, 4.0])
def test_quadrature_converged_against_trapezoid(act, tau):
    gh = oracle.moments(act, tau)["kd"]
    tr = oracle.moments_trapezoid(act, tau)
    tol = 1e-10 if tau <= 1.1 else 1e-5      # GH degrades for tanh at large τ (poles at ±iπ/(2√τ))
    assert np.max(np.abs(gh - tr)) < tol


@pytest.mark.parametrize("act", oracle.ACTS)
def test_d0_nonnegative_poincare(act):
    for tau in (0.25, 1.0, 4.0):
        assert oracle.moments(act, tau)["d0"] >= -1e-12


def test_sigmoid_half_is_half_tanh_half():
    """σ_sig(x) − ½ = ½ tanh(x/2) ⇒ ⟨k,d⟩_sig(τ) = 2^{k−d−1} ⟨k,d⟩_tanh(τ/4)."""
    for tau in (0.8, 1.0, 2.0):
        a = oracle.moments("sigmoid_half", tau)["kd"]
        b = oracle.moments("tanh", tau / 4)["kd"]
        for k in range(5):
            for d in range(3):
                assert abs(a[k, d] - 2.0 ** (k - d - 1) * b[k, d]) < 1e-14


def test_tau_hat_lemma1():
    X = np.array([[1.0, 0, 0, 0], [0, 1.0, 0, 0]])
    assert oracle.tau_hat(X) == 1.0
    assert oracle.tau_hat(np.zeros((1, 5))) == 0.0
    rng = np.random.default_rng(3)
    Xs = rng.standard_normal((4096, 4096)) / 64.0
    assert abs(oracle.tau_hat(Xs) - 1.0) < 0.05


@pytest.mark.parametrize("tau", [0.3, 1.0, 2.5])
def test_parametrised_quadratic_rows_through_stein(tau):
    """The oracle's parametrised "quadratic(a0,a1,a2)" (Stein-form moments from σ alone) against the same printed
    Table-2 / draft rows the analytic-derivative quad above meets."""
    env = {"exp": math.exp, "sqrt": math.sqrt, "pi": math.pi, "tau": tau, "a0": A0, "a1": A1, "a2": A2}
    mom = oracle.moments(f"quadratic({A0!r},{A1!r},{A2!r})", tau)
    kd = mom["kd"]
    n = 0
    for act, q, expr, cite in _golden_rows():
        if act != "quad":
            continue
        got = {"d0": mom["d0"], "d1": mom["d1"], "d2": mom["d2"], "E_s": kd[0, 0], "E_s1": kd[0, 1],
               "E_s2": kd[0, 2], "E_sq": mom["e_sigma_sq"]}[q]
        want = eval(expr, {"__builtins__": {}}, env)
        assert abs(got - want) < 1e-11 * max(1.0, abs(want)), (q, cite, got, want)
        n += 1
    assert n == 7


def test_parametrised_leaky_reduces_to_relu_and_abs():
    """Table 2's leaky row at (a₊, a₋) = (1, 0) is the ReLU row and at (1, 1) the |t| row."""
    for tau in (0.5, 1.7):
        for name, ref in (("leaky_relu(1.0,0.0)", "relu"), ("leaky_relu(1.0,1.0)", "abs")):
            a, b = oracle.moments(name, tau), oracle.moments(ref, tau)
            assert np.max(np.abs(a["kd"] - b["kd"])) < 1e-13 and abs(a["d0"] - b["d0"]) < 1e-13
