"""Pins for the oracle's G = (1/m) σ(WX)ᵀσ(WX) (Eq. def_Gram).

G is a sample mean over features of σ(w_kᵀx_i)σ(w_kᵀx_j) ("sample mean of the expected
kernel"), so for σ = erf it converges to the arcsine kernel at the Monte-Carlo rate with an
exactly predictable mean-squared error — that ties the oracle to an independent closed form.
"""
import math

import numpy as np
import pytest
from scipy import special as sp

import oracle
import synthetic


def arcsine_kernel(X):
    g = X @ X.T
    d = 1 + 2 * np.diag(g)
    return 2 / math.pi * np.arcsin(2 * g / np.sqrt(np.outer(d, d)))


def predicted_mse_erf(X, N=48):
    """E‖G − K‖_F² = (1/m) Σ_ij Var_w[σ(wᵀx_i)σ(wᵀx_j)], by 2-D Gauss–Hermite over (ξ_a, ξ_b)."""
    x, w = sp.roots_hermitenorm(N)
    w = w / w.sum()
    g = X @ X.T
    n = len(X)
    tot = 0.0
    for i in range(n):
        ua = math.sqrt(g[i, i])
        fa = sp.erf(ua * x)                                     # [qa]
        for j in range(n):
            vb = g[i, j] / ua
            ub = math.sqrt(max(0.0, g[j, j] - vb * vb))
            fb = sp.erf(vb * x[:, None] + ub * x[None, :])      # [qa, qb]
            prod = fa[:, None] * fb
            e1 = np.sum(w[:, None] * w[None, :] * prod)
            e2 = np.sum(w[:, None] * w[None, :] * prod * prod)
            tot += e2 - e1 * e1
    return tot


def test_gram_symmetric_psd_and_shape():
    X = synthetic.make_X(0)
    W = synthetic.make_W(0)
    G = oracle.gram(X, W, "tanh")
    assert G.shape == (256, 256)
    assert np.max(np.abs(G - G.T)) == 0.0
    ev = np.linalg.eigvalsh(G)
    assert ev.min() >= -1e-10 * np.abs(ev).max()


def test_gram_m1_rank_one_and_duplicate_rows_invariance():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((20, 8)) / math.sqrt(8)
    W = rng.standard_normal((1, 8))
    G = oracle.gram(X, W, "erf")
    s = sp.erf(X @ W[0])
    assert np.max(np.abs(G - np.outer(s, s))) < 1e-15
    W2 = rng.standard_normal((5, 8))
    assert np.max(np.abs(oracle.gram(X, W2, "tanh") - oracle.gram(X, np.vstack([W2, W2]), "tanh"))) < 1e-15


def test_gram_sigmoid_tanh_identity():
    """sigmoid(x) − ½ = ½ tanh(x/2)  ⇒  G_sig(W, X) = ¼ G_tanh(W, X/2)."""
    rng = np.random.default_rng(2)
    X = rng.standard_normal((30, 16)) / 4
    W = rng.standard_normal((64, 16))
    a = oracle.gram(X, W, "sigmoid_half")
    b = oracle.gram(X / 2, W, "tanh")
    assert np.max(np.abs(a - 0.25 * b)) < 1e-15


def test_gram_entries_matches_full():
    X = synthetic.make_X(0)
    W = synthetic.make_W(0)
    G = oracle.gram(X, W, "tanh")
    I = np.array([0, 5, 17, 255, 128])
    J = np.array([0, 200, 17, 3, 129])
    assert np.max(np.abs(oracle.gram_entries(X, W, "tanh", I, J) - G[I, J])) < 1e-15


def test_gram_erf_converges_to_arcsine_at_mc_rate():
    """‖G − K_arcsine‖_F² / predicted ∈ [0.75, 1.33] averaged over seeds, and the log-log slope
    of the error vs m is −½ (Monte-Carlo rate of the sample mean P:472)."""
    rng = np.random.default_rng(123)
    n, p = 48, 32
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    K = arcsine_kernel(X)
    base = predicted_mse_erf(X)
    ms = [256, 1024, 4096, 16384]
    rms = []
    for m in ms:
        ratios = []
        for seed in range(6):
            W = np.random.default_rng(1000 * m + seed).standard_normal((m, p))
            G = oracle.gram(X, W, "erf")
            ratios.append(np.sum((G - K) ** 2) / (base / m))
        r = float(np.mean(ratios))
        assert 0.75 < r < 1.33, (m, r)
        rms.append(math.sqrt(r * base / m))
    slope = np.polyfit(np.log(ms), np.log(rms), 1)[0]
    assert abs(slope + 0.5) < 0.1


def test_synthetic_configs_have_the_stated_laws():
    """The inputs generator (shared by both sides) draws what BASELINE.json configs state."""
    c1 = synthetic.CONFIGS[1]
    X = synthetic.make_X(c1, rows=np.arange(0, 4096, 7))
    nrm = np.sqrt(np.sum(X * X, axis=1))
    assert nrm.min() >= 0.8 - 1e-12 and nrm.max() <= 1.2 + 1e-12
    X0 = synthetic.make_X(0)
    assert abs(oracle.tau_hat(X0) - 1.0) < 0.05
    # row subsets regenerate identical rows
    rows = np.array([5, 4097, 2, 9000])
    c2 = synthetic.CONFIGS[2]
    a = synthetic.make_X(c2, rows=rows, n=10000, p=64)
    b = synthetic.make_X(c2, n=10000, p=64)[rows]
    assert np.array_equal(a, b)
    lab = synthetic.class_labels(c2, 10000)
    assert lab.sum() == 5000
    mu = synthetic.mean_vector(c2, 64)
    assert abs(np.linalg.norm(mu) - 2 / 8) < 1e-14
