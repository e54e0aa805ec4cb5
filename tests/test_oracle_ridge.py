"""Pins for the NEXT-4 ridge oracle (oracle/ridge.py) against closed forms: the identity Gram, a rank-one Gram
(Sherman–Morrison), the large-γ expansion, and the stacked-Gram split."""
import numpy as np
import pytest

from oracle import ridge
import synthetic


def test_identity_gram():
    rng = np.random.default_rng(0)
    Y = rng.standard_normal((50, 3))
    for g in (1e-3, 0.5, 20.0):
        assert np.allclose(ridge.ridge_fit(np.eye(50), Y, g), Y / (1.0 + g), rtol=1e-14, atol=0)


def test_rank_one_sherman_morrison():
    """(vvᵀ + γI)^{-1} y = (y − v·vᵀy/(γ + vᵀv))/γ."""
    rng = np.random.default_rng(1)
    v = rng.standard_normal(40)
    y = rng.standard_normal(40)
    for g in (0.1, 3.0):
        exp = (y - v * (v @ y) / (g + v @ v)) / g
        assert np.allclose(ridge.ridge_fit(np.outer(v, v), y[:, None], g)[:, 0], exp, rtol=1e-11, atol=1e-13)


def test_large_gamma_expansion():
    """α = y/γ − G y/γ² + O(γ^{-3}): the remainder falls 8× per doubling of γ."""
    rng = np.random.default_rng(2)
    F = rng.standard_normal((30, 60))
    G = F @ F.T / 60
    y = rng.standard_normal((30, 1))
    rem = []
    for g in (1e3, 2e3, 4e3):
        a = ridge.ridge_fit(G, y, g)
        rem.append(np.linalg.norm(a - (y / g - G @ y / g ** 2)))
    assert 7.0 < rem[0] / rem[1] < 9.0 and 7.0 < rem[1] / rem[2] < 9.0


def test_split_gram_reads_upper_triangle_only():
    rng = np.random.default_rng(3)
    F = rng.standard_normal((12, 5))
    S = F @ F.T
    G_upper = np.triu(S) + np.tril(np.full_like(S, 7.0), -1)  # garbage below the diagonal (UPPER layout)
    Gt, Gc = ridge.split_gram(G_upper, 8)
    assert np.array_equal(Gt, S[:8, :8]) and np.array_equal(Gc, S[8:, :8])


def test_ridge_path_and_gmm_inputs():
    X, y = synthetic.make_ridge_gmm(64, 32, 16)
    assert X.shape == (96, 16) and y.shape == (96, 1) and set(np.unique(y)) == {-1.0, 1.0}
    assert abs(int((y > 0).sum()) - 48) <= 1
    G = X @ X.T                                              # any PSD Gram exercises the path
    out = ridge.ridge_path(G, 64, y[:64], y[64:], [1e-2, 1.0, 1e4])
    assert len(out) == 3
    # γ → ∞: predictions → 0, so the MSE → mean(y²) = 1
    assert abs(out[-1][3] - 1.0) < 1e-2
