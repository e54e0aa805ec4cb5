"""fp64 CPU ORACLE for the random-features Gram G and the closed-form kernel Φ (EQ1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or call
anything in ``oracle/``.  The product path (``paper_2110_01899_b200``) never
imports it and shares no code, table or constant generator with it.

Everything here is plain NumPy in float64, written to be checked against
PAPER.md by eye.  Citations ``P:<line>`` are PAPER.md lines.

  sigma / dsigma / d2sigma ... the activations of the north star and their
                               analytic derivatives (Assumption 3)
  hermite_rule(N) ............ probabilists' Gauss–Hermite nodes/weights by
                               Newton iteration on the normalised Hermite
                               three-term recurrence (independent of the
                               library's Golub–Welsch eigen-solver)
  moments(act, tau) .......... ⟨k,d⟩ = E[(√τξ)^k σ^(d)(√τξ)], d0, d1, d2
                               ("moments needed", Theorem 1)
  tau_hat(X) ................. Lemma 1 estimator (1/n)Σ‖x_i‖² (Alg. 1)
  gram(X, W, act) ............ G = (1/m) σ(WX)ᵀ σ(WX)  (Eq. def_Gram)
  phi_eq1(X, act, tau) ....... the 18-term EQ1 evaluated from the
                               Gram–Schmidt quantities u_a, v_b, u_b

Readings of garbled / silent passages (DESIGN.md §4 lists all of them):
  R1  EQ1 term 5 prints (u_b−1)²; read ((u_b/√τ)−1)² = β².
  R2  EQ1 term 10 prints E[σ'']E[τξ²σ'']; read E[σ'']E[τξ²σ] (EQ2, prints this).
  R3  EQ1 term 12 prints E[σ']E[ξ²σ']; read E[σ']E[τξ²σ'] (the τ is missing).
  R4  EQ1 term 14 prints ½E[σ']E[τξ²σ']; read E[τξ²σ']E[√τξσ''] (coefficient 1).
  R5  Taylor lines P:1022/P:1029 evaluate σ'' at ξ_a instead of √τξ_a: all
      derivatives are taken at √τξ.
  R6  Pivot: entry (i, j), i ≤ j, uses x_i as the Gram–Schmidt pivot (EQ1 is
      not symmetric).  Diagonal i = j: u_b = 0, v_b = u_a exactly.
  R7  u_b radicand clamped at 0.
  R8  No normalisation of σ (the draft's "E[σ(ξ²)]=1", is not applied).
Every reading is pinned by a test in tests/test_oracle_*.py (2-D Gauss–Hermite
integration of the truncated Taylor product, closed forms, invariants).
"""
from __future__ import annotations

import math
from functools import lru_cache
from typing import Callable, Dict, Optional, Tuple

import numpy as np
from scipy import special as _sp  # erf only (a library definition of σ)

ACTS = ("tanh", "erf", "sigmoid_half")
_TABLE2 = ("relu", "abs", "sign", "step", "cos", "sin", "ident", "quad", "bump")


# --------------------------------------------------------------------------------------------
# Activations (north star: σ ∈ {tanh, erf, sigmoid − 1/2}); written literally.
# --------------------------------------------------------------------------------------------
def _is_table2(act) -> bool:
    if not isinstance(act, str):
        return False
    from .acts import parse_param_act
    return act in _TABLE2 or parse_param_act(act) is not None


def sigma(act: str, x):
    x = np.asarray(x, dtype=np.float64)
    if _is_table2(act):                     # NEXT-3 activations (oracle/acts.py)
        from .acts import sigma2
        return sigma2(act, x)
    if act == "tanh":
        return np.tanh(x)
    if act == "erf":
        return _sp.erf(x)
    if act == "sigmoid_half":
        return 1.0 / (1.0 + np.exp(-x)) - 0.5
    raise ValueError(act)


def dsigma(act: str, x):
    x = np.asarray(x, dtype=np.float64)
    if act == "tanh":
        t = np.tanh(x)
        return 1.0 - t * t
    if act == "erf":
        return 2.0 / math.sqrt(math.pi) * np.exp(-x * x)
    if act == "sigmoid_half":
        s = 1.0 / (1.0 + np.exp(-x))
        return s * (1.0 - s)
    raise ValueError(act)


def d2sigma(act: str, x):
    x = np.asarray(x, dtype=np.float64)
    if act == "tanh":
        t = np.tanh(x)
        return -2.0 * t * (1.0 - t * t)
    if act == "erf":
        return -2.0 * x * (2.0 / math.sqrt(math.pi) * np.exp(-x * x))
    if act == "sigmoid_half":
        s = 1.0 / (1.0 + np.exp(-x))
        return s * (1.0 - s) * (1.0 - 2.0 * s)
    raise ValueError(act)


def derivs(act) -> Tuple[Callable, Callable, Callable]:
    """(σ, σ', σ'') for a named activation, or a user tuple of three callables."""
    if isinstance(act, str):
        return (lambda x: sigma(act, x), lambda x: dsigma(act, x), lambda x: d2sigma(act, x))
    return act


# --------------------------------------------------------------------------------------------
# Gauss–Hermite rule for the N(0,1) density, by Newton on the normalised recurrence.
#   ψ_0 = 1, ψ_1 = x, ψ_{k+1} = (x ψ_k − √k ψ_{k−1}) / √(k+1)     (ψ_k = He_k/√k!)
#   nodes = roots of ψ_N;  weights w_i = 1 / (N ψ_{N−1}(x_i)²)       (Σ w_i = 1)
# --------------------------------------------------------------------------------------------
def _psi(N: int, x: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    pm1 = np.zeros_like(x)
    p = np.ones_like(x)
    for k in range(N):
        pm1, p = p, (x * p - math.sqrt(k) * pm1) / math.sqrt(k + 1)
    return p, pm1            # ψ_N(x), ψ_{N−1}(x)


@lru_cache(maxsize=None)
def hermite_rule(N: int) -> Tuple[np.ndarray, np.ndarray]:
    if N < 1:
        raise ValueError("N >= 1")
    # Bracket the N real roots by sign changes of ψ_N on a fine grid (all roots lie in
    # |x| < √(4N+2)), then polish each bracket by safeguarded Newton steps.
    L = math.sqrt(4.0 * N + 2.0) + 1.0
    grid = np.linspace(-L, L, 400 * N + 1)
    f, _ = _psi(N, grid)
    idx = np.nonzero(np.sign(f[:-1]) * np.sign(f[1:]) < 0)[0]
    if len(idx) != N:
        raise RuntimeError(f"hermite_rule: bracketed {len(idx)} roots, expected {N}")
    lo, hi = grid[idx].copy(), grid[idx + 1].copy()
    x = 0.5 * (lo + hi)
    for _ in range(100):
        pN, pNm1 = _psi(N, x)
        # ψ_N' = √N ψ_{N−1}
        step = pN / (math.sqrt(N) * pNm1)
        xn = x - step
        bad = (xn <= lo) | (xn >= hi)
        xn = np.where(bad, 0.5 * (lo + hi), xn)
        fl, _ = _psi(N, lo)
        fx, _ = _psi(N, xn)
        same = np.sign(fx) == np.sign(fl)
        lo = np.where(same, xn, lo)
        hi = np.where(same, hi, xn)
        done = np.max(np.abs(xn - x)) < 1e-15 * L
        x = xn
        if done:
            break
    x = 0.5 * (x - x[::-1])           # enforce exact symmetry of the rule
    with np.errstate(over="ignore"):
        _, pNm1 = _psi(N, x)
        w = 1.0 / (N * pNm1 * pNm1)          # far-tail weights underflow to 0 for large N
    w = 0.5 * (w + w[::-1])
    return x, w


def gauss_expect(f: Callable, N: int = 128) -> float:
    """E[f(ξ)], ξ ~ N(0,1), by the N-point rule."""
    x, w = hermite_rule(N)
    return float(np.sum(w * f(x)))


# --------------------------------------------------------------------------------------------
# Moments ⟨k,d⟩ = E[(√τ ξ)^k σ^(d)(√τ ξ)]  (EQ1 coefficients) and Theorem 1's d0, d1, d2.
# --------------------------------------------------------------------------------------------
def moments(act, tau: float, N: int = 200) -> Dict[str, object]:
    if not (tau > 0.0):
        raise ValueError("tau must be > 0")
    if _is_table2(act):                           # weak derivatives through Stein (oracle/acts.py)
        from .acts import moments_stein
        return moments_stein(act, tau)
    s0, s1, s2 = derivs(act)
    x, w = hermite_rule(N)
    t = math.sqrt(tau) * x
    f = (s0(t), s1(t), s2(t))
    kd = np.zeros((5, 3))
    for k in range(5):
        for d in range(3):
            kd[k, d] = np.sum(w * t ** k * f[d])
    e_sig2 = float(np.sum(w * f[0] * f[0]))
    # Theorem 1
    d0 = e_sig2 - kd[0, 0] ** 2 - tau * kd[0, 1] ** 2
    d1 = kd[0, 1] ** 2
    d2 = 0.25 * kd[0, 2] ** 2
    return {"tau": float(tau), "kd": kd, "e_sigma_sq": e_sig2, "d0": d0, "d1": d1, "d2": d2, "nodes": N}


def moments_trapezoid(act, tau: float, h: float = 0.05, L: float = 40.0) -> np.ndarray:
    """Cross-check of ⟨k,d⟩ by the composite trapezoid rule on [−L, L] (geometric convergence
    for integrands analytic in a strip); used only to bound the Gauss–Hermite error."""
    s0, s1, s2 = derivs(act)
    x = np.arange(-L, L + 0.5 * h, h)
    dens = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    t = math.sqrt(tau) * x
    f = (s0(t), s1(t), s2(t))
    kd = np.zeros((5, 3))
    for k in range(5):
        for d in range(3):
            kd[k, d] = h * np.sum(dens * t ** k * f[d])
    return kd


# --------------------------------------------------------------------------------------------
# Lemma 1: τ̂ = (1/n) Σ_i ‖x_i‖²
# --------------------------------------------------------------------------------------------
def tau_hat(Xs: np.ndarray) -> float:
    """Xs is sample-major (n × p): row i = x_i."""
    Xs = np.asarray(Xs, dtype=np.float64)
    return float(np.mean(np.sum(Xs * Xs, axis=1)))


# --------------------------------------------------------------------------------------------
# G = (1/m) σ(WX)ᵀ σ(WX)   (Eq. def_Gram; draft P:7-11)
# --------------------------------------------------------------------------------------------
def sigma_features(Xs: np.ndarray, W: np.ndarray, act: str) -> np.ndarray:
    """Σ = σ(WX) ∈ R^{m×n}.  Xs sample-major n×p, W m×p."""
    X = np.asarray(Xs, dtype=np.float64).T          # paper layout p×n
    Z = np.asarray(W, dtype=np.float64) @ X         # Z = WX (library matmul as one step)
    return sigma(act, Z)


def gram(Xs: np.ndarray, W: np.ndarray, act: str, m_total: Optional[int] = None) -> np.ndarray:
    """Full symmetric n×n G.  `m_total` defaults to the number of rows of W (the 1/m of P:472)."""
    S = sigma_features(Xs, W, act)
    m = S.shape[0] if m_total is None else m_total
    return (S.T @ S) / m


def gram_entries(Xs: np.ndarray, W: np.ndarray, act: str, I: np.ndarray, J: np.ndarray) -> np.ndarray:
    """G_ij for explicit index pairs (I[t], J[t]) — the sampled oracle at full sizes.
    G_ij = (1/m) Σ_k σ(w_kᵀx_i) σ(w_kᵀx_j)."""
    I = np.asarray(I); J = np.asarray(J)
    rows = np.unique(np.concatenate([I, J]))
    S = sigma_features(np.asarray(Xs)[rows], W, act)            # m × |rows|
    pos = {int(r): q for q, r in enumerate(rows)}
    a = S[:, [pos[int(i)] for i in I]]
    b = S[:, [pos[int(j)] for j in J]]
    return np.sum(a * b, axis=0) / S.shape[0]


# --------------------------------------------------------------------------------------------
# Φ by EQ1, step by step in the paper's order and notation.
# --------------------------------------------------------------------------------------------
def gram_schmidt(xi_norm2, xj_norm2, g, diag):
    """u_a = ‖x_i‖, v_b = x_iᵀx_j/‖x_i‖, u_b = √(‖x_j‖² − (x_iᵀx_j)²/‖x_i‖²).
    Readings R6 (diagonal), R7 (clamp) and R23 (a zero pivot x_i = 0: x_j has no component along it, v_b = 0 and
    u_b = ‖x_j‖)."""
    xi_norm2 = np.asarray(xi_norm2, dtype=np.float64)
    zero = xi_norm2 == 0.0
    safe = np.where(zero, 1.0, xi_norm2)
    u_a = np.sqrt(xi_norm2)
    v_b = np.where(zero, 0.0, g / np.sqrt(safe))
    u_b = np.where(zero, np.sqrt(xj_norm2), np.sqrt(np.maximum(0.0, xj_norm2 - g * g / safe)))
    v_b = np.where(diag, u_a, v_b)
    u_b = np.where(diag, 0.0, u_b)
    return u_a, v_b, u_b


def eq1_terms(mom: Dict[str, object], u_a, v_b, u_b) -> list:
    """The 18 terms of EQ1 in the printed order, with readings R1-R4.
    M[k][d] = ⟨k,d⟩ = E[(√τξ)^k σ^(d)(√τξ)]."""
    tau = mom["tau"]
    M = mom["kd"]
    st = math.sqrt(tau)
    a = u_a / st - 1.0            # (u_a/√τ − 1)
    b = u_b / st - 1.0            # (u_b/√τ − 1)
    v = v_b / st                  # v_b/√τ
    E_s, E_xs1, E_s1 = M[0, 0], M[1, 1], M[0, 1]        # E[σ], E[√τξσ'], E[σ']
    E_xs, E_x2s2, E_xs2 = M[1, 0], M[2, 2], M[1, 2]     # E[√τξσ], E[τξ²σ''], E[√τξσ'']
    E_s2, E_x2s, E_x2s1 = M[0, 2], M[2, 0], M[2, 1]     # E[σ''], E[τξ²σ], E[τξ²σ']
    E_x3s1, E_x3s2, E_x4s2 = M[3, 1], M[3, 2], M[4, 2]  # E[τ√τξ³σ'], E[τ√τξ³σ''], E[τ²ξ⁴σ'']
    return [
        E_s ** 2,                                        # 1
        E_s * E_xs1 * b,                                 # 2
        E_s1 * E_xs * v,                                 # 3
        E_xs1 ** 2 * a * b,                              # 4
        E_s * E_x2s2 / 2.0 * b ** 2,                     # 5  (R1)
        E_xs1 * E_x2s2 / 2.0 * a * b ** 2,               # 6
        E_xs1 * E_x2s2 / 2.0 * a ** 2 * b,               # 7
        E_x2s2 ** 2 / 4.0 * a ** 2 * b ** 2,             # 8
        E_xs * E_xs2 * v * b,                            # 9
        E_s2 * E_x2s / 2.0 * v ** 2,                     # 10 (R2)
        E_s * E_xs1 * a,                                 # 11
        E_s1 * E_x2s1 * v * a,                           # 12 (R3)
        E_s2 * E_x3s1 / 2.0 * v ** 2 * a,                # 13
        E_x2s1 * E_xs2 * v * a * b,                      # 14 (R4)
        E_s * E_x2s2 / 2.0 * a ** 2,                     # 15
        E_s1 * E_x3s2 / 2.0 * v * a ** 2,                # 16
        E_s2 * E_x4s2 / 4.0 * v ** 2 * a ** 2,           # 17
        E_xs2 * E_x3s2 / 2.0 * v * b * a ** 2,           # 18
    ]


def eq1(mom: Dict[str, object], u_a, v_b, u_b):
    terms = eq1_terms(mom, np.asarray(u_a, float), np.asarray(v_b, float), np.asarray(u_b, float))
    out = terms[0] * np.ones(np.broadcast(np.asarray(u_a), np.asarray(v_b), np.asarray(u_b)).shape)
    for t in terms[1:]:
        out = out + t
    return out


def phi_eq1(Xs: np.ndarray, act: str, tau: Optional[float] = None, mom=None, N: int = 200,
            rows: Optional[np.ndarray] = None) -> np.ndarray:
    """Φ on the upper triangle (j ≥ i) of the |rows|×|rows| principal submatrix (all rows by
    default); lower triangle left as NaN.  Steps: τ (Lemma 1 unless given) → moments →
    g = x_iᵀx_j → (u_a, v_b, u_b) → EQ1."""
    Xs = np.asarray(Xs, dtype=np.float64)
    if tau is None:
        tau = tau_hat(Xs)
    if mom is None:
        mom = moments(act, tau, N)
    Xr = Xs if rows is None else Xs[rows]
    g = Xr @ Xr.T                                     # XᵀX restricted to rows (library matmul)
    nrm2 = np.sum(Xr * Xr, axis=1)
    k = len(Xr)
    I, J = np.triu_indices(k)
    u_a, v_b, u_b = gram_schmidt(nrm2[I], nrm2[J], g[I, J], I == J)
    out = np.full((k, k), np.nan)
    out[I, J] = eq1(mom, u_a, v_b, u_b)
    return out


def phi_pivot_asymmetry(Xs: np.ndarray, act: str, tau: Optional[float] = None, mom=None, N: int = 200) -> float:
    """Diagnostic of reading R6: max_{i<j} |Φ(x_i, x_j) − Φ(x_j, x_i)|, each side by EQ1 with its first argument
    as the Gram–Schmidt pivot.  EQ1 is not symmetric; the swap changes u_a, v_b, u_b only when
    ‖x_i‖ ≠ ‖x_j‖, so the asymmetry vanishes for equal norms."""
    Xs = np.asarray(Xs, dtype=np.float64)
    if tau is None:
        tau = tau_hat(Xs)
    if mom is None:
        mom = moments(act, tau, N)
    g = Xs @ Xs.T
    nrm2 = np.sum(Xs * Xs, axis=1)
    I, J = np.triu_indices(len(Xs), 1)
    if len(I) == 0:
        return 0.0
    fwd = eq1(mom, *gram_schmidt(nrm2[I], nrm2[J], g[I, J], I == J))
    bwd = eq1(mom, *gram_schmidt(nrm2[J], nrm2[I], g[I, J], I == J))
    return float(np.max(np.abs(fwd - bwd)))


def phi_exact_pair(act, u_a: float, v_b: float, u_b: float, N: int = 120) -> float:
    """κ(x_i,x_j) = E[σ(u_a ξ_a) σ(v_b ξ_a + u_b ξ_b)] by the N×N tensor Gauss–Hermite rule
    (the quantity EQ1 approximates, Eq. (1) P:360-364 after Gram–Schmidt)."""
    s0 = derivs(act)[0]
    x, w = hermite_rule(N)
    fa = s0(u_a * x)                                   # over ξ_a
    fb = s0(v_b * x[:, None] + u_b * x[None, :])       # [ξ_a, ξ_b]
    return float(np.sum(w[:, None] * w[None, :] * fa[:, None] * fb))


def phi_eq2(Xs: np.ndarray, act: str, tau: Optional[float] = None, mom=None, N: int = 200,
            rows: Optional[np.ndarray] = None) -> np.ndarray:
    """As phi_eq1 with the six-term EQ2 instead of EQ1 (NEXT-3)."""
    from .acts import eq2
    Xs = np.asarray(Xs, dtype=np.float64)
    if tau is None:
        tau = tau_hat(Xs)
    if mom is None:
        mom = moments(act, tau, N)
    Xr = Xs if rows is None else Xs[rows]
    g = Xr @ Xr.T
    nrm2 = np.sum(Xr * Xr, axis=1)
    k = len(Xr)
    I, J = np.triu_indices(k)
    u_a, v_b, u_b = gram_schmidt(nrm2[I], nrm2[J], g[I, J], I == J)
    out = np.full((k, k), np.nan)
    out[I, J] = eq2(mom, u_a, v_b, u_b)
    return out
