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
