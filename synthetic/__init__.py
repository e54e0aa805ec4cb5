"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no σ, no Gram, no EQ1, no
moments): it only draws the data X and the projection W of the workloads in
BASELINE.json ``configs`` so that both implementations consume identical
numbers.  It imports neither ``oracle`` nor ``paper_2110_01899_b200``.

Layouts:
  X is returned sample-major, shape (n, p): row i is the paper's column x_i
    (PAPER.md:5 / P:470, X = [x_1, ..., x_n] ∈ R^{p×n}).
  W is returned row-major, shape (m, p): row k is w_k (W ∈ R^{m×p}).

Generator: NumPy PCG64 in float64; every block of ``BLOCK`` rows has its own
substream SeedSequence([seed, block]) so any subset of rows can be regenerated
without drawing the whole matrix (used by the sampled oracle at full size).
Seeds: seed = 211001899 + 100*cfg + t, t = 0 for X, 1 for W, 2 for norm
factors, 3 for class labels / mean direction.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

BLOCK = 4096
SEED_BASE = 211001899


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json config (index ``idx`` is 0-based into ``configs``)."""
    idx: int
    name: str
    p: int
    n: int
    m: int            # 0 for the Φ-only config
    act: str          # "tanh" | "erf" | "sigmoid_half"
    x_law: str        # "iid" | "unit_scaled" | "gmm2"
    scale_lo: float = 1.0
    scale_hi: float = 1.0
    modes: Sequence[str] = ()
    gram: bool = True
    phi: bool = True


CONFIGS = [
    Config(0, "tiny", 64, 256, 512, "tanh", "iid", modes=("fp64", "fp32", "3xtf32", "tf32", "bf16")),
    Config(1, "p784_n4096_m8192_erf", 784, 4096, 8192, "erf", "unit_scaled", 0.8, 1.2,
           modes=("fp32", "3xtf32")),
    Config(2, "p3072_n16384_m32768_gmm_tanh", 3072, 16384, 32768, "tanh", "gmm2", modes=("bf16",)),
    Config(3, "p1024_n65536_m65536_sigmoid", 1024, 65536, 65536, "sigmoid_half", "iid",
           modes=("bf16",), phi=False),
    Config(4, "phi_p512_n131072_tanh", 512, 131072, 0, "tanh", "unit_scaled", 0.5, 1.5,
           modes=("bf16", "tf32", "3xtf32"), gram=False),
]


def seed_of(cfg: int, t: int) -> int:
    return SEED_BASE + 100 * (cfg + 1) + t


def _block_rng(seed: int, block: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, block])))


def _normal_rows(seed: int, rows: np.ndarray, ncols: int, total_rows: int) -> np.ndarray:
    """Rows `rows` of a (total_rows × ncols) iid N(0,1) matrix drawn blockwise."""
    out = np.empty((len(rows), ncols), dtype=np.float64)
    rows = np.asarray(rows, dtype=np.int64)
    order = np.argsort(rows, kind="stable")
    srt = rows[order]
    blocks = srt // BLOCK
    for b in np.unique(blocks):
        b = int(b)
        nb = min(BLOCK, total_rows - b * BLOCK)
        full = _block_rng(seed, b).standard_normal((nb, ncols))
        sel = blocks == b
        out[order[sel]] = full[srt[sel] - b * BLOCK]
    return out


def _uniform_rows(seed: int, rows: np.ndarray, total_rows: int, lo: float, hi: float) -> np.ndarray:
    rows = np.asarray(rows, dtype=np.int64)
    out = np.empty(len(rows), dtype=np.float64)
    blocks = rows // BLOCK
    for b in np.unique(blocks):
        b = int(b)
        nb = min(BLOCK, total_rows - b * BLOCK)
        full = _block_rng(seed, b).uniform(lo, hi, size=nb)
        sel = blocks == b
        out[sel] = full[rows[sel] - b * BLOCK]
    return out


def make_X(cfg: Config | int, rows: Optional[np.ndarray] = None, *, n: Optional[int] = None,
           p: Optional[int] = None) -> np.ndarray:
    """Data matrix, sample-major (len(rows) × p), float64.

    iid:         x_i ~ N(0, I/p)                                   (configs[0], [3])
    unit_scaled: z_i ~ N(0, I/p), x_i = c_i z_i/‖z_i‖, c_i ~ U[lo,hi]  (configs[1], [4])
    gmm2:        x_i = ±μ + z_i, ‖μ‖ = 2/√p, z_i ~ N(0, I/p), balanced labels (configs[2];
                 Eq. (GMM) at P:479-482 with μ_a/√p, ‖μ_a‖ = 2)
    ``n``/``p`` override the config's sizes (for reduced-size parity cases).
    """
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    n = cfg.n if n is None else n
    p = cfg.p if p is None else p
    if rows is None:
        rows = np.arange(n, dtype=np.int64)
    rows = np.asarray(rows, dtype=np.int64)
    z = _normal_rows(seed_of(cfg.idx, 0), rows, p, n) / math.sqrt(p)
    if cfg.x_law == "iid":
        return z
    if cfg.x_law == "unit_scaled":
        c = _uniform_rows(seed_of(cfg.idx, 2), rows, n, cfg.scale_lo, cfg.scale_hi)
        nrm = np.sqrt(np.sum(z * z, axis=1))
        return z * (c / nrm)[:, None]
    if cfg.x_law == "gmm2":
        labels = class_labels(cfg, n)[rows]
        mu = mean_vector(cfg, p)
        sign = np.where(labels == 0, 1.0, -1.0)
        return z + sign[:, None] * mu[None, :]
    raise ValueError(cfg.x_law)


def class_labels(cfg: Config | int, n: Optional[int] = None) -> np.ndarray:
    """Balanced labels for gmm2: a seeded permutation of n/2 zeros and n/2 ones."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    n = cfg.n if n is None else n
    rng = np.random.Generator(np.random.PCG64(seed_of(cfg.idx, 3)))
    lab = np.zeros(n, dtype=np.int64)
    lab[n // 2:] = 1
    return rng.permutation(lab)


def mean_vector(cfg: Config | int, p: Optional[int] = None) -> np.ndarray:
    """μ = (2/√p)·u with u a seeded unit vector (‖μ‖ = 2/√p)."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    p = cfg.p if p is None else p
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed_of(cfg.idx, 3), 1])))
    u = rng.standard_normal(p)
    u /= np.sqrt(np.sum(u * u))
    return (2.0 / math.sqrt(p)) * u


def make_W(cfg: Config | int, rows: Optional[np.ndarray] = None, *, m: Optional[int] = None,
           p: Optional[int] = None) -> np.ndarray:
    """Projection matrix, row-major (len(rows) × p), iid N(0,1) (Assumption 2 with Gaussian law)."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    m = cfg.m if m is None else m
    p = cfg.p if p is None else p
    if rows is None:
        rows = np.arange(m, dtype=np.int64)
    return _normal_rows(seed_of(cfg.idx, 1), np.asarray(rows, dtype=np.int64), p, m)


def sample_indices(n: int, count: int = 1024, seed: int = 7, tile_stride: int = 128) -> np.ndarray:
    """Sampled index set S for full-size parity (SURVEY.md §8c "Oracle at scale"):
    `count` random indices ∪ first/last 256 ∪ every multiple of `tile_stride` ± 1, sorted, unique."""
    rng = np.random.Generator(np.random.PCG64(seed))
    s = set(rng.choice(n, size=min(count, n), replace=False).tolist())
    s.update(range(min(256, n)))
    s.update(range(max(0, n - 256), n))
    for t in range(0, n + 1, tile_stride):
        for d in (-1, 0, 1):
            if 0 <= t + d < n:
                s.add(t + d)
    return np.array(sorted(s), dtype=np.int64)


def make_T(cfg: Config | int, eps: float, rows: Optional[np.ndarray] = None, *, m: Optional[int] = None,
           p: Optional[int] = None) -> np.ndarray:
    """Sign/sparsity pattern T ∈ {−1, 0, +1}^{len(rows)×p} of the ternary projection (Eq. (4)):
    entry 0 with probability ε, −1 or +1 each with probability (1−ε)/2.  W^ter = (1−ε)^{-1/2}·T; the scale
    belongs to the method and is applied by each implementation, not here.  Returned as float64 (exact).
    Seed t = 4 of the config; blockwise substreams as make_W."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    if not (0.0 <= eps < 1.0):
        raise ValueError("eps must be in [0, 1)")
    m = cfg.m if m is None else m
    p = cfg.p if p is None else p
    if rows is None:
        rows = np.arange(m, dtype=np.int64)
    rows = np.asarray(rows, dtype=np.int64)
    out = np.empty((len(rows), p), dtype=np.float64)
    blocks = rows // BLOCK
    seed = seed_of(cfg.idx, 4)
    for b in np.unique(blocks):
        b = int(b)
        nb = min(BLOCK, m - b * BLOCK)
        u = _block_rng(seed, b).random((nb, p))
        full = np.where(u < eps, 0.0, np.where(u < eps + (1.0 - eps) / 2.0, -1.0, 1.0))
        sel = blocks == b
        out[sel] = full[rows[sel] - b * BLOCK]
    return out


def make_ridge_gmm(n_train: int, n_test: int, p: int, seed: int = 0):
    """Two-class GMM of the paper's ridge experiments (Eq. (GMM)): x = μ_a/√p + z,
    z ~ N(0, C_a/p), μ_a = 4·e_a (a = 1, 2), C_a = (1 + 4(a − 1)/√p)·I_p; balanced classes in random order; the
    regression target is the class sign y = −1 (a = 1) / +1 (a = 2).  Returns X (n_train + n_test, p) with the
    training samples first, and y (n_train + n_test, 1).  Stands in for the paper's MNIST / Cov-Type / Census data.
    Data only: no arithmetic of the method."""
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 7001 + seed))
    n = n_train + n_test
    lab = np.concatenate([np.zeros(n // 2, dtype=np.int64), np.ones(n - n // 2, dtype=np.int64)])
    rng.shuffle(lab)
    X = rng.standard_normal((n, p))
    scale = np.where(lab == 0, 1.0, math.sqrt(1.0 + 4.0 / math.sqrt(p)))
    X *= scale[:, None] / math.sqrt(p)
    X[np.arange(n), lab] += 4.0 / math.sqrt(p)
    y = np.ascontiguousarray(np.where(lab == 0, -1.0, 1.0)[:, None])
    return X, y

