"""fp64 CPU ORACLE for NEXT-3: the Table-2 activations, their Gaussian moments through Stein's lemma
(derivatives in the weak sense, Remark 2), and EQ2.

TEST INFRASTRUCTURE ONLY (same rule as oracle/rf_oracle.py).

  TABLE2 ............................. relu, abs, sign, step (1_{t>0}), cos, sin, ident (t), quad (t²), bump (e^{−t²/2})
  parametrised rows .... "leaky_relu(a₊,a₋)" = a₊·max(0,t) + a₋·max(0,−t),
                                       "quadratic(a₀,a₁,a₂)" = a₂t² + a₁t + a₀ (the library's activation names)
  sigma2(act, t) ..................... the activation, written literally
  moments_stein(act, τ) .............. ⟨k,d⟩ = E[(√τξ)^k σ^{(d)}(√τξ)], k ≤ 4, d ≤ 2, from M_j = E[ξ^j σ(√τξ)] only:
                                         ⟨k,0⟩ = τ^{k/2} M_k
                                         ⟨k,1⟩ = τ^{(k−1)/2} (M_{k+1} − k M_{k−1})              (Stein once)
                                         ⟨k,2⟩ = τ^{k/2−1} (M_{k+2} − (2k+1) M_k + k(k−1) M_{k−2}) (Stein twice)
                                       with M_j by adaptive quadrature split at the kink / jump t = 0
  eq2(mom, u_a, v_b, u_b) ............ the six terms of EQ2 in the printed order (term 5 read as
                                       E[σ'']E[τξ²σ]/2 · (v_b/√τ)², as printed there)
"""
from __future__ import annotations

import math
from typing import Dict

import numpy as np
from scipy import integrate

TABLE2 = ("relu", "abs", "sign", "step", "cos", "sin", "ident", "quad", "bump")
ODD = ("sign", "sin", "ident")          # σ(−t) = −σ(t): ⟨k,d⟩ = 0 for k + d even


def parse_param_act(act: str):
    """("leaky_relu", (a₊, a₋)) or ("quadratic", (a₀, a₁, a₂)) for a parametrised Table-2 name, else None."""
    for kind, k in (("leaky_relu", 2), ("quadratic", 3)):
        if act.startswith(kind + "(") and act.endswith(")"):
            vals = tuple(float(v) for v in act[len(kind) + 1:-1].split(","))
            if len(vals) == k:
                return kind, vals
    return None


def sigma2(act: str, t):
    t = np.asarray(t, dtype=np.float64)
    pa = parse_param_act(act)
    if pa is not None and pa[0] == "leaky_relu":        # Table 2
        ap, am = pa[1]
        return ap * np.maximum(t, 0.0) + am * np.maximum(-t, 0.0)
    if pa is not None:                                  # Table 2
        a0, a1, a2 = pa[1]
        return a2 * t * t + a1 * t + a0
    if act == "relu":
        return np.maximum(t, 0.0)
    if act == "abs":
        return np.abs(t)
    if act == "sign":
        return np.sign(t)
    if act == "step":
        return (t > 0).astype(np.float64)
    if act == "cos":
        return np.cos(t)
    if act == "sin":
        return np.sin(t)
    if act == "ident":
        return t.copy()
    if act == "quad":
        return t * t
    if act == "bump":
        return np.exp(-0.5 * t * t)
    raise ValueError(act)


def _M(act: str, tau: float, j: int, square: bool = False) -> float:
    """E[ξ^j σ(√τξ)] (or E[ξ^j σ(√τξ)²]) by adaptive quadrature on (−∞, 0] and [0, ∞)."""
    st = math.sqrt(tau)
    pdf = lambda x: math.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    def f(x):
        s = float(sigma2(act, st * x))
        return (x ** j) * (s * s if square else s) * pdf(x)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", integrate.IntegrationWarning)   # tolerances at machine precision
        a = integrate.quad(f, -40.0, 0.0, epsabs=1e-15, epsrel=1e-14, limit=400)[0]
        b = integrate.quad(f, 0.0, 40.0, epsabs=1e-15, epsrel=1e-14, limit=400)[0]
    return a + b


def moments_stein(act: str, tau: float) -> Dict[str, object]:
    if not (tau > 0):
        raise ValueError("tau must be > 0")
    M = [_M(act, tau, j) for j in range(7)]
    Mm = lambda j: M[j] if j >= 0 else 0.0
    kd = np.zeros((5, 3))
    for k in range(5):
        kd[k, 0] = tau ** (k / 2) * M[k]
        kd[k, 1] = tau ** ((k - 1) / 2) * (M[k + 1] - k * Mm(k - 1))
        kd[k, 2] = tau ** (k / 2 - 1) * (M[k + 2] - (2 * k + 1) * M[k] + k * (k - 1) * Mm(k - 2))
    e_sig2 = _M(act, tau, 0, square=True)
    d0 = e_sig2 - kd[0, 0] ** 2 - tau * kd[0, 1] ** 2       # Theorem 1
    d1 = kd[0, 1] ** 2
    d2 = 0.25 * kd[0, 2] ** 2
    return {"tau": float(tau), "kd": kd, "e_sigma_sq": e_sig2, "d0": d0, "d1": d1, "d2": d2, "nodes": 0}


def eq2_terms(mom: Dict[str, object], u_a, v_b, u_b) -> list:
    """EQ2, printed order.  ⟨k,d⟩ = mom["kd"][k][d]."""
    tau = mom["tau"]
    K = mom["kd"]
    st = math.sqrt(tau)
    a = np.asarray(u_a, float) / st - 1.0
    b = np.asarray(u_b, float) / st - 1.0
    v = np.asarray(v_b, float) / st
    E_s, E_xs1, E_s1, E_xs, E_s2, E_x2s = K[0, 0], K[1, 1], K[0, 1], K[1, 0], K[0, 2], K[2, 0]
    return [
        E_s ** 2,                          # (E[σ])²
        E_s * E_xs1 * b,                   # E[σ]E[√τξσ'] (u_b/√τ − 1)
        E_s1 * E_xs * v,                   # E[σ']E[√τξσ] v_b/√τ
        E_xs1 ** 2 * a * b,                # E[√τξσ']² (u_a/√τ − 1)(u_b/√τ − 1)
        E_s2 * E_x2s / 2.0 * v ** 2,       # E[σ'']E[τξ²σ]/2 (v_b/√τ)²
        E_s * E_xs1 * a,                   # E[σ]E[√τξσ'] (u_a/√τ − 1)
    ]


def eq2(mom: Dict[str, object], u_a, v_b, u_b):
    t = eq2_terms(mom, u_a, v_b, u_b)
    out = t[0] * np.ones(np.broadcast(np.asarray(u_a), np.asarray(v_b), np.asarray(u_b)).shape)
    for x in t[1:]:
        out = out + x
    return out
