"""fp64 CPU ORACLE for NEXT-2: centering K = P·G·P (Eq. (2)) and Theorem 1's asymptotic equivalent
K̃ (EQ6).

TEST INFRASTRUCTURE ONLY (same rule as oracle/rf_oracle.py).  Plain NumPy in float64, written literally.

  P(n) ..................... P = I_n − (1/n)1_n1_nᵀ
  center(A) ................ P·A·P  (two dense matrix products, as written)
  ktilde(X, V, A, d0, d1, d2)  K̃ = P(d1·XᵀX + d2·V·A·Vᵀ + d0·I_n)P   (EQ6 with Z + M Jᵀ/√p = X, Eq. (GMM))
  gmm_V_A(J, phi, t, T, p) . V = [J/√p, φ],  A = [[t tᵀ + 2T, t], [tᵀ, 1]]  (Theorem 1)
  quadratic_kernel(X) ...... κ(x, y) = ‖x‖²‖y‖² + 2(xᵀy)² for σ(t) = t², Gaussian w (exact; pins d2·VAVᵀ)
  arcsine_kernel(X) ........ κ for σ = erf, Gaussian w (Williams 1997): (2/π)·asin(2xᵀy/√((1+2‖x‖²)(1+2‖y‖²)))

Layout: X is sample-major (n × p) like the rest of the oracle, so the paper's XᵀX (p × n data) is X·Xᵀ here.
"""
from __future__ import annotations

import math

import numpy as np


def P(n: int) -> np.ndarray:
    return np.eye(n) - np.ones((n, n)) / n


def center(A: np.ndarray) -> np.ndarray:
    """P·A·P (Eq. (2)): left- and right-multiplication by the centering projector."""
    Pn = P(A.shape[0])
    return Pn @ np.asarray(A, dtype=np.float64) @ Pn


def gmm_V_A(J: np.ndarray, phi: np.ndarray, t: np.ndarray, T: np.ndarray, p: int):
    """V = [J/√p, φ] (n × (K+1)),  A = [[t tᵀ + 2T, t], [tᵀ, 1]] ((K+1) × (K+1))  (Theorem 1)."""
    J = np.asarray(J, dtype=np.float64)
    K = J.shape[1]
    V = np.concatenate([J / math.sqrt(p), np.asarray(phi, dtype=np.float64)[:, None]], axis=1)
    A = np.zeros((K + 1, K + 1))
    A[:K, :K] = np.outer(t, t) + 2.0 * np.asarray(T, dtype=np.float64)
    A[:K, K] = t
    A[K, :K] = t
    A[K, K] = 1.0
    return V, A


def ktilde(Xs: np.ndarray, V: np.ndarray, A: np.ndarray, d0: float, d1: float, d2: float) -> np.ndarray:
    """K̃ = P(d1·XᵀX + d2·V A Vᵀ + d0·I)P  (EQ6); Xs sample-major so XᵀX is Xs·Xsᵀ."""
    Xs = np.asarray(Xs, dtype=np.float64)
    n = Xs.shape[0]
    inner = d1 * (Xs @ Xs.T) + d2 * (V @ A @ V.T) + d0 * np.eye(n)
    return center(inner)


def quadratic_kernel(Xs: np.ndarray) -> np.ndarray:
    """E_w[(wᵀx)²(wᵀy)²] for w ~ N(0, I): ‖x‖²‖y‖² + 2(xᵀy)² (Isserlis)."""
    g = np.asarray(Xs, dtype=np.float64) @ np.asarray(Xs, dtype=np.float64).T
    d = np.diag(g)
    return np.outer(d, d) + 2.0 * g * g


def arcsine_kernel(Xs: np.ndarray) -> np.ndarray:
    g = np.asarray(Xs, dtype=np.float64) @ np.asarray(Xs, dtype=np.float64).T
    d = np.diag(g)
    return (2.0 / math.pi) * np.arcsin(2.0 * g / np.sqrt(np.outer(1.0 + 2.0 * d, 1.0 + 2.0 * d)))
