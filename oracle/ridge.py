"""fp64 CPU ORACLE for NEXT-4: random-features kernel ridge regression on G, the paper's downstream
use of the Gram matrix (Section 5; App. A; its figures P:798, P:1177-1325 plot the test MSE
against the ridge parameter γ).

TEST INFRASTRUCTURE ONLY (same rule as oracle/rf_oracle.py): imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs; never by the product path.  Plain NumPy / SciPy in float64.

The paper does not print the estimator (it cites kernel ridge regression); the reading (R20) is the
textbook one on the random-features Gram of the training samples and the cross Gram to the test samples:
  fit ........... α = (G_train + γ I)^{-1} Y           (one library Cholesky solve, SciPy cho_factor / cho_solve)
  predict ....... Ŷ_test = G_cross α,  G_cross[t][i] = (1/m) σ(W x_test,t)ᵀ σ(W x_train,i)
  mse ........... (1/(n_test·r)) ‖Ŷ_test − Y_test‖²_F
Both Grams come from ONE Gram over the stacked samples [X_train; X_test] (its leading n_train × n_train block and the
block of rows < n_train, columns ≥ n_train), which is how the library is called too.
"""
from __future__ import annotations

import numpy as np
from scipy import linalg


def split_gram(G_all: np.ndarray, n_train: int):
    """(G_train, G_cross) from the symmetric Gram of [X_train; X_test]; only entries j ≥ i of G_all are read."""
    G = np.asarray(G_all, dtype=np.float64)
    U = np.triu(G)
    S = U + np.triu(U, 1).T                     # symmetric from the upper triangle
    return S[:n_train, :n_train], S[n_train:, :n_train]


def ridge_fit(G_train: np.ndarray, Y: np.ndarray, gamma: float) -> np.ndarray:
    """α = (G_train + γ I)^{-1} Y by a Cholesky factorisation (γ > 0 and G PSD make the matrix SPD)."""
    A = np.asarray(G_train, dtype=np.float64) + gamma * np.eye(G_train.shape[0])
    return linalg.cho_solve(linalg.cho_factor(A, lower=True), np.asarray(Y, dtype=np.float64))


def ridge_predict(G_cross: np.ndarray, alpha: np.ndarray) -> np.ndarray:
    return np.asarray(G_cross, dtype=np.float64) @ alpha


def mse(Y_hat: np.ndarray, Y: np.ndarray) -> float:
    d = np.asarray(Y_hat, dtype=np.float64) - np.asarray(Y, dtype=np.float64)
    return float(np.mean(d * d))


def ridge_path(G_all: np.ndarray, n_train: int, Y_train: np.ndarray, Y_test: np.ndarray, gammas):
    """[(γ, α, Ŷ_test, test MSE)] for each γ (the curves of P:798 / P:1177)."""
    Gt, Gc = split_gram(G_all, n_train)
    out = []
    for g in gammas:
        a = ridge_fit(Gt, Y_train, g)
        yh = ridge_predict(Gc, a)
        out.append((g, a, yh, mse(yh, Y_test)))
    return out
