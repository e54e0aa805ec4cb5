"""fp64 CPU ORACLE for Ternary Random Features (TRF, §8(f) NEXT-1): Eq. (3)-(5), Corollary 1, Eq. (8),
Algorithm 1.

TEST INFRASTRUCTURE ONLY (same rule as oracle/rf_oracle.py): only tests/, __graft_entry__.smoke() and
bench.py's CPU legs may import it.  Plain NumPy/SciPy in float64, written to be checked against the paper by
eye.  Citations P:<line> are PAPER.md lines.

  sigma_ter(t, s_minus, s_plus) ...... Eq. (5): σ^ter(t) = −1·δ_{t<s−} + 1·δ_{t>s+} (0 on [s−, s+])
  ternary_moments(s_minus, s_plus, τ)  E[σ^ter], E[σ^ter'], E[σ^ter''], E[σ^ter²] at √τξ and d0, d1, d2
                                       (Theorem 1), derivatives in the weak sense (Remark 2) through
                                       Stein's lemma, integrals written with the normal pdf/cdf
  solve_thresholds(d1, d2, τ) ........ Algorithm 1 step 2: least squares on (ŝ−, ŝ+), search box enlarged from
                                       [−1, 1]² until solved ("gradually enlarging the search range")
  ternary_features(X, T, ε, s−, s+) .. Σ^terᵀ = σ^ter(X·W^terᵀ) with W^ter = (1−ε)^{-1/2}·T  (Eq. (4), Alg. 1 step 4)
  gram_ter(...) ...................... G^ter = (1/m) Σ^terᵀ Σ^ter  (Alg. 1 step 4, Eq. def_Gram)
  decision_margin(...) ............... min |z − s±| per entry (where a rounding of z could flip σ^ter)
  kappa_ter_gaussian(...) ............ E[σ^ter(ζ_a)σ^ter(ζ_b)], (ζ_a, ζ_b) ~ N(0, [[‖x_i‖², g], [g, ‖x_j‖²]]):
                                       the m → ∞ limit of G^ter when wᵀx is Gaussian (CLT in p)

Reading R15: Eq. (8) as printed, d1 = π^{-2}(e^{−s+²/τ} + e^{−s−²/τ})² and
d2 = (2πτ³)^{-1}(s+e^{−s+²/τ} + s−e^{−s−²/τ})², does not follow from Eq. (5): at s− = s+ = 0 (σ^ter = sign) it
gives d1 = 4/π², while Table 2's sign(t) row gives 2/(πτ).  Computed from Eq. (5) with the weak
derivatives of Remark 2 (Stein): E[σ^ter'(√τξ)] = (φ(a) + φ(b))/√τ, E[σ^ter''(√τξ)] = (aφ(a) + bφ(b))/τ with
a = s−/√τ, b = s+/√τ and φ the N(0, 1) density, so
    d1 = (e^{−s−²/(2τ)} + e^{−s+²/(2τ)})² / (2πτ),   d2 = (s−e^{−s−²/(2τ)} + s+e^{−s+²/(2τ)})² / (8πτ³),
which reproduces the sign row.  The thresholds are solved from these.
"""
from __future__ import annotations

import math
from typing import Dict, Optional, Tuple

import numpy as np


def _pdf(x):
    return np.exp(-0.5 * np.asarray(x, dtype=np.float64) ** 2) / math.sqrt(2.0 * math.pi)


def _cdf(x):
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * (1.0 + np.vectorize(math.erf)(x / math.sqrt(2.0)))


# --------------------------------------------------------------------------------------------
# Eq. (5)
# --------------------------------------------------------------------------------------------
def sigma_ter(t, s_minus: float, s_plus: float):
    """σ^ter(t) = −1·δ_{t<s−} + 1·δ_{t>s+}  (Eq. (5)); 0 for s− ≤ t ≤ s+."""
    t = np.asarray(t, dtype=np.float64)
    return np.where(t < s_minus, -1.0, 0.0) + np.where(t > s_plus, 1.0, 0.0)


# --------------------------------------------------------------------------------------------
# Gaussian moments of σ^ter at √τξ (Theorem 1's d0, d1, d2; derivatives via Stein, Remark 2)
# --------------------------------------------------------------------------------------------
def ternary_moments(s_minus: float, s_plus: float, tau: float) -> Dict[str, float]:
    if not s_minus <= s_plus:
        raise ValueError("need s_minus <= s_plus")
    st = math.sqrt(tau)
    a, b = s_minus / st, s_plus / st
    Pa, Pb = float(_cdf(a)), float(_cdf(b))
    pa, pb = float(_pdf(a)), float(_pdf(b))
    E_s = -Pa + (1.0 - Pb)                       # E[σ(√τξ)] = −P(ξ<a) + P(ξ>b)
    E_sq = Pa + (1.0 - Pb)                       # E[σ²] = P(ξ<a) + P(ξ>b)
    E_xs = pa + pb                               # E[ξσ] = −E[ξ1{ξ<a}] + E[ξ1{ξ>b}] = φ(a) + φ(b)
    E_x2m1s = a * pa + b * pb                    # E[(ξ²−1)σ] = −(−aφ(a)) + bφ(b)
    E_s1 = E_xs / st                             # Stein: E[σ'(√τξ)] = E[ξσ(√τξ)]/√τ
    E_s2 = E_x2m1s / tau                         # Stein: E[σ''(√τξ)] = E[(ξ²−1)σ(√τξ)]/τ
    d1 = E_s1 ** 2                               # Theorem 1
    d2 = E_s2 ** 2 / 4.0
    d0 = E_sq - E_s ** 2 - tau * d1
    return {"E_s": E_s, "E_s1": E_s1, "E_s2": E_s2, "E_sq": E_sq, "d0": d0, "d1": d1, "d2": d2}


def eq8_as_printed(s_minus: float, s_plus: float, tau: float) -> Tuple[float, float]:
    """Eq. (8) verbatim — kept only so a test can show it disagrees with Table 2 (R15)."""
    d1 = (math.exp(-s_plus ** 2 / tau) + math.exp(-s_minus ** 2 / tau)) ** 2 / math.pi ** 2
    d2 = (s_plus * math.exp(-s_plus ** 2 / tau) + s_minus * math.exp(-s_minus ** 2 / tau)) ** 2 / (2 * math.pi * tau ** 3)
    return d1, d2


# --------------------------------------------------------------------------------------------
# Algorithm 1 step 2: thresholds by least squares with an enlarging search box
# --------------------------------------------------------------------------------------------
def solve_thresholds(d1: float, d2: float, tau: float, sign2: int = 1, cap: float = 64.0,
                     tol: float = 1e-24) -> Tuple[float, float]:
    """(ŝ−, ŝ+) with ŝ− ≤ ŝ+ whose ternary (d1, d2) equal the targets.  d2 fixes |E[σ'']|; `sign2` picks the sign
    of E[σ''] (the two mirror solutions (s−, s+) and (−s+, −s−) have the same d1, d2)."""
    from scipy.optimize import least_squares

    st = math.sqrt(tau)
    t1 = math.sqrt(d1)
    t2 = sign2 * 2.0 * math.sqrt(max(d2, 0.0))

    def resid(v):
        lo, hi = min(v[0], v[1]), max(v[0], v[1])
        m = ternary_moments(lo, hi, tau)
        return [m["E_s1"] - t1, m["E_s2"] - t2]

    R = 1.0
    best = None
    while R <= cap * st:
        for x0 in ((-0.5 * R, 0.5 * R), (-0.9 * R, 0.1 * R), (-0.1 * R, 0.9 * R), (0.0, 0.0)):
            r = least_squares(resid, x0=np.array(x0, dtype=float), bounds=([-R, -R], [R, R]), xtol=1e-15,
                              ftol=1e-15, gtol=1e-15)
            f = float(np.sum(np.square(r.fun)))
            if best is None or f < best[0]:
                best = (f, min(r.x), max(r.x))
        if best[0] <= tol:
            return best[1], best[2]
        R *= 2.0
    raise ValueError(f"no thresholds reproduce d1={d1}, d2={d2} at tau={tau} (residual {best[0]:.3e})")


# --------------------------------------------------------------------------------------------
# Algorithm 1 step 4: features and Gram
# --------------------------------------------------------------------------------------------
def projections(Xs: np.ndarray, T: np.ndarray, eps: float) -> np.ndarray:
    """z = X·W^terᵀ, W^ter = (1−ε)^{-1/2}·T  (n × m), fp64."""
    return (1.0 - eps) ** -0.5 * (np.asarray(Xs, dtype=np.float64) @ np.asarray(T, dtype=np.float64).T)


def ternary_features(Xs: np.ndarray, T: np.ndarray, eps: float, s_minus: float, s_plus: float) -> np.ndarray:
    """Σ^terᵀ = σ^ter(X W^terᵀ), n × m, values in {−1, 0, +1} (float64)."""
    return sigma_ter(projections(Xs, T, eps), s_minus, s_plus)


def gram_ter(Xs: np.ndarray, T: np.ndarray, eps: float, s_minus: float, s_plus: float,
             m_total: Optional[int] = None) -> np.ndarray:
    """G^ter = (1/m) Σ^terᵀ Σ^ter (n × n)."""
    S = ternary_features(Xs, T, eps, s_minus, s_plus)
    m = S.shape[1] if m_total is None else m_total
    return (S @ S.T) / m


def decision_margin(Xs: np.ndarray, T: np.ndarray, eps: float, s_minus: float, s_plus: float) -> np.ndarray:
    """min(|z − s−|, |z − s+|) per entry: a computed z within this distance of a threshold may decide differently."""
    z = projections(Xs, T, eps)
    return np.minimum(np.abs(z - s_minus), np.abs(z - s_plus))


def kappa_ter_gaussian(u_a2: float, g: float, u_b2: float, s_minus: float, s_plus: float) -> float:
    """E[σ^ter(ζ_a)σ^ter(ζ_b)] for (ζ_a, ζ_b) ~ N(0, [[u_a2, g], [g, u_b2]]) — orthant probabilities of the
    bivariate normal (scipy's CDF): σσ = +1 on {both < s−} ∪ {both > s+}, −1 on the mixed corners."""
    from scipy.stats import multivariate_normal

    cov = np.array([[u_a2, g], [g, u_b2]], dtype=np.float64)
    F = multivariate_normal(mean=[0.0, 0.0], cov=cov, allow_singular=True).cdf
    inf = 1e3 * math.sqrt(max(u_a2, u_b2))
    def box(x0, x1, y0, y1):   # P(x0 < ζa < x1, y0 < ζb < y1)
        return F([x1, y1]) - F([x0, y1]) - F([x1, y0]) + F([x0, y0])
    lo_lo = box(-inf, s_minus, -inf, s_minus)
    hi_hi = box(s_plus, inf, s_plus, inf)
    lo_hi = box(-inf, s_minus, s_plus, inf)
    hi_lo = box(s_plus, inf, -inf, s_minus)
    return float(lo_lo + hi_hi - lo_hi - hi_lo)
