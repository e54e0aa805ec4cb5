"""Pins of the NEXT-3 oracle (oracle/acts.py): Table-2 activations through Stein-form moments, and EQ2.

* Stein-form ⟨k,d⟩ (σ only, weak derivatives) equal Gauss–Hermite with the analytic σ', σ'' wherever σ is smooth.
* Table 2's d0, d1, d2 rows for |t|, ReLU, sign, 1_{t>0} are in tests/golden (test_oracle_moments.py).
* Stein identities and the odd-σ zero pattern hold for every Table-2 activation.
* EQ2 equals EQ1 exactly at the expansion point u_a = u_b = √τ (only α, β terms differ), and on high-dimensional
  data |κ − EQ2| falls like p^{-3/2} (the paper's order) while dropping any one EQ2 term leaves O(p^{-1})."""
import math

import numpy as np
import pytest

import oracle
from oracle import acts
from oracle import center as C

SMOOTH = {
    "cos": (np.cos, lambda x: -np.sin(x), lambda x: -np.cos(x)),
    "sin": (np.sin, np.cos, lambda x: -np.sin(x)),
    "ident": (lambda x: x, lambda x: np.ones_like(x), lambda x: np.zeros_like(x)),
    "quad": (lambda x: x * x, lambda x: 2 * x, lambda x: 2 * np.ones_like(x)),
    "bump": (lambda x: np.exp(-x * x / 2), lambda x: -x * np.exp(-x * x / 2),
             lambda x: (x * x - 1) * np.exp(-x * x / 2)),
}


@pytest.mark.parametrize("act", sorted(SMOOTH))
@pytest.mark.parametrize("tau", [0.5, 1.0, 2.0])
def test_stein_moments_equal_analytic_derivatives(act, tau):
    st = acts.moments_stein(act, tau)
    gh = oracle.moments(SMOOTH[act], tau, N=160)
    assert np.max(np.abs(st["kd"] - gh["kd"])) < 1e-11
    assert abs(st["e_sigma_sq"] - gh["e_sigma_sq"]) < 1e-11


@pytest.mark.parametrize("act", acts.TABLE2)
@pytest.mark.parametrize("tau", [0.7, 1.0833])
def test_stein_identities_and_parity_structure(act, tau):
    kd = oracle.moments(act, tau)["kd"]
    assert abs(kd[1, 0] - tau * kd[0, 1]) < 1e-11
    assert abs(kd[1, 1] - tau * kd[0, 2]) < 1e-11
    assert abs(kd[2, 1] - tau * (kd[0, 1] + kd[1, 2])) < 1e-11
    assert abs(kd[2, 0] - tau * (kd[0, 0] + kd[1, 1])) < 1e-11
    if act in acts.ODD:
        for k in range(5):
            for d in range(3):
                if (k + d) % 2 == 0:
                    assert abs(kd[k, d]) < 1e-13
    else:   # even σ (|t|, cos, t², bump) or neither (ReLU, 1_{t>0}): some even-sum moment is non-zero
        assert max(abs(kd[k, d]) for k in range(5) for d in range(3) if (k + d) % 2 == 0) > 1e-3


def test_relu_weak_second_derivative_is_dirac():
    """ReLU'' = δ: E[σ''(√τξ)] = φ(0)/√τ (Remark 2); ReLU' = 1_{t>0}: E[σ'] = 1/2."""
    for tau in (0.5, 1.0, 3.0):
        kd = oracle.moments("relu", tau)["kd"]
        assert abs(kd[0, 2] - 1 / math.sqrt(2 * math.pi * tau)) < 1e-12
        assert abs(kd[0, 1] - 0.5) < 1e-12


@pytest.mark.parametrize("act", ["tanh", "erf", "relu", "cos", "bump"])
def test_eq2_equals_eq1_at_the_expansion_point(act):
    tau = 1.0833
    mom = oracle.moments(act, tau)
    st = math.sqrt(tau)
    v = np.linspace(-0.4, 0.4, 9)
    assert np.allclose(acts.eq2(mom, st, v, st), oracle.eq1(mom, st, v, st), atol=1e-14, rtol=0)


def test_eq2_matrix_error_vanishes_in_operator_norm():
    """The paper uses EQ2 at matrix level: with n = p growing, ‖P(K − EQ2)P‖ / ‖PKP‖ over the
    off-diagonal entries falls (σ = erf, exact K by the arcsine kernel; rows with ‖x_i‖² fluctuating at O(p^{-1/2})
    so α, β ≠ 0), EQ1 (more terms) is closer still, and dropping EQ2's ν term leaves an O(1) error."""
    rng = np.random.default_rng(0)
    e1s, e2s = [], []
    for p in (128, 512, 2048):
        n = p
        X = rng.standard_normal((n, p)) / math.sqrt(p)
        X *= 1 + 0.3 * rng.standard_normal((n, 1)) / math.sqrt(p)
        tau = oracle.tau_hat(X)
        mom = oracle.moments("erf", tau)
        K = C.arcsine_kernel(X)
        np.fill_diagonal(K, 0.0)
        g = X @ X.T
        nrm2 = np.diag(g)
        I, J = np.triu_indices(n, 1)
        u_a, v_b, u_b = oracle.gram_schmidt(nrm2[I], nrm2[J], g[I, J], I == J)

        def sym(vals):
            M = np.zeros((n, n))
            M[I, J] = vals
            return M + M.T
        Pn = C.P(n)
        nk = np.linalg.norm(Pn @ K @ Pn, 2)
        rel = lambda M: np.linalg.norm(Pn @ (K - M) @ Pn, 2) / nk
        terms = acts.eq2_terms(mom, u_a, v_b, u_b)
        e2s.append(rel(sym(acts.eq2(mom, u_a, v_b, u_b))))
        e1s.append(rel(sym(oracle.eq1(mom, u_a, v_b, u_b))))
        if p == 2048:
            assert rel(sym(acts.eq2(mom, u_a, v_b, u_b) - terms[2])) > 0.5
    assert e2s[2] < 0.02 and e2s[2] < 0.5 * e2s[0], e2s
    assert all(a < b for a, b in zip(e1s, e2s)), (e1s, e2s)


# ------------------------------------------------------------------------------------------------------------------
# EQ2's α / β / ν coefficients, pinned against the exact kernel.  EQ2 is the part of the expansion of
# κ(α, β, ν) = E[σ(√τ(1+α)ξ_a) σ(√τν ξ_a + √τ(1+β)ξ_b)] that the paper keeps:
#   κ(0) + κ_α α + κ_β β + κ_ν ν + κ_αβ αβ + ½κ_νν ν²,
# so every one of its coefficients is a partial derivative of κ at the expansion point.  Those partials are taken
# here by Richardson-extrapolated central differences of κ, with κ from a closed form (σ = cos, t²) or from an
# independent SciPy 2-D Gauss–Hermite rule (softplus, the bump) — no moment routine of the oracle is involved — and
# EQ2's coefficients are read off the oracle's eq2 by the same differences (exact for a quadratic).  A dropped term,
# a wrong sign, a wrong moment or a wrong ½ in any of the six terms fails.
# ------------------------------------------------------------------------------------------------------------------
from scipy import special as _sp  # noqa: E402

_SOFTPLUS = (lambda x: np.logaddexp(0, x), lambda x: _sp.expit(x), lambda x: _sp.expit(x) * (1 - _sp.expit(x)))


def _kappa_closed(name, u_a, v_b, u_b):
    if name == "cos":      # E[cos(u_a ξa) cos(v_b ξa + u_b ξb)] = e^{−(u_a² + v_b² + u_b²)/2} cosh(u_a v_b)
        return math.exp(-0.5 * (u_a * u_a + v_b * v_b + u_b * u_b)) * math.cosh(u_a * v_b)
    if name == "quad":     # E[(u_a ξa)² (v_b ξa + u_b ξb)²] = u_a² (3 v_b² + u_b²)   (Isserlis)
        return u_a * u_a * (3 * v_b * v_b + u_b * u_b)
    raise ValueError(name)


def _kappa_gh(f, u_a, v_b, u_b, N=160):
    x, w = _sp.roots_hermitenorm(N)
    w = w / w.sum()
    return float(np.sum(w[:, None] * w[None, :] * f(u_a * x)[:, None] * f(v_b * x[:, None] + u_b * x[None, :])))


def _partials(fun, h=2e-2):
    """κ and the five partials EQ2 keeps, plus the four second-order ones it drops, at (α, β, ν) = 0, by central
    differences with one Richardson step (error O(h⁴))."""
    def d1(i, hh):
        e = np.zeros(3)
        e[i] = hh
        return (fun(*e) - fun(*(-e))) / (2 * hh)

    def d2(i, j, hh):
        ei, ej = np.zeros(3), np.zeros(3)
        ei[i], ej[j] = hh, hh
        if i == j:
            return (fun(*ei) - 2 * fun(0, 0, 0) + fun(*(-ei))) / (hh * hh)
        return (fun(*(ei + ej)) - fun(*(ei - ej)) - fun(*(ej - ei)) + fun(*(-ei - ej))) / (4 * hh * hh)

    rich = lambda g: (4 * g(h / 2) - g(h)) / 3   # noqa: E731
    out = {"0": fun(0, 0, 0)}
    for k, i in (("a", 0), ("b", 1), ("v", 2)):
        out[k] = rich(lambda hh, i=i: d1(i, hh))
    for k, (i, j) in (("ab", (0, 1)), ("vv", (2, 2)), ("aa", (0, 0)), ("bb", (1, 1)), ("av", (0, 2)),
                      ("bv", (1, 2))):
        out[k] = rich(lambda hh, i=i, j=j: d2(i, j, hh))
    return out


@pytest.mark.parametrize("name", ["cos", "quad", "softplus", "bump"])
@pytest.mark.parametrize("tau", [0.8, 1.2])
def test_eq2_coefficients_are_the_partials_of_the_exact_kernel(name, tau):
    st = math.sqrt(tau)
    if name in ("cos", "quad"):
        kap = lambda a, b, v: _kappa_closed(name, st * (1 + a), st * v, st * (1 + b))   # noqa: E731
    else:
        f = _SOFTPLUS[0] if name == "softplus" else (lambda x: np.exp(-0.5 * x * x))
        kap = lambda a, b, v: _kappa_gh(f, st * (1 + a), st * v, st * (1 + b))        # noqa: E731
    mom = oracle.moments(_SOFTPLUS if name == "softplus" else name, tau)
    e2 = lambda a, b, v: float(acts.eq2(mom, st * (1 + a), st * v, st * (1 + b)))     # noqa: E731
    K = _partials(kap)
    E = _partials(e2)
    scale = max(abs(K["0"]), abs(K["a"]), abs(K["v"]), 1e-3)
    for key in ("0", "a", "b", "v", "ab"):
        assert abs(E[key] - K[key]) <= 1e-7 * scale, (name, key, E[key], K[key])
    # the ν² term carries ½κ_νν: EQ2's second difference in ν equals κ_νν
    assert abs(E["vv"] - K["vv"]) <= 1e-6 * scale, (name, "vv", E["vv"], K["vv"])
    # EQ2 keeps no α², β², αν, βν term (the paper's O(p^{-3/2}) remainder at matrix level, reading R18)
    for key in ("aa", "bb", "av", "bv"):
        assert abs(E[key]) <= 1e-7 * scale, (name, key, E[key])
    # the α and β terms are live for these σ (⟨0,0⟩⟨1,1⟩ ≠ 0), so the pin has teeth
    assert abs(K["a"]) > 1e-2 * scale and abs(K["ab"]) > 1e-2 * scale


def test_eq2_quadratic_hand_evaluated():
    """σ = t²: ⟨0,0⟩ = τ, ⟨1,1⟩ = 2τ, ⟨0,1⟩ = ⟨1,0⟩ = 0, ⟨0,2⟩ = 2, ⟨2,0⟩ = 3τ² (Gaussian moments by hand), so
    EQ2 = τ²(1 + 2α + 2β + 4αβ + 3ν²) — the exact κ = u_a²(3v_b² + u_b²) = τ²(1+α)²(3ν² + (1+β)²) minus its
    α², β², α²β, … terms."""
    for tau, u_a, v_b, u_b in [(1.0, 1.1, 0.2, 0.9), (0.7, 0.6, -0.3, 1.0), (1.3, 1.2, 0.05, 1.25)]:
        st = math.sqrt(tau)
        al, be, nu = u_a / st - 1, u_b / st - 1, v_b / st
        want = tau ** 2 * (1 + 2 * al + 2 * be + 4 * al * be + 3 * nu * nu)
        got = float(acts.eq2(oracle.moments("quad", tau), u_a, v_b, u_b))
        assert abs(got - want) <= 1e-11 * abs(want), (got, want)
