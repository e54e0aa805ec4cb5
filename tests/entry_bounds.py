"""Per-entry error bounds for the GPU parity tests (reading R22), beside the north star's
relative-Frobenius tolerances.  A Frobenius norm over a large matrix barely moves when one tile is wrong; these
bounds are asserted entry by entry, so one wrong tile (or one wrong entry) fails.

The bounds are derived from the arithmetic each precision mode performs, not fitted:

Gram G = (1/m) Σ_k s_ki s_kj with s_ki the stored feature σ(z_ki) (z_ki = w_kᵀx_i):
  * stored-feature perturbation s = σ(ẑ)(1 + δ), |δ| ≤ u_s (bf16 round-to-nearest: 8 significant bits, unit roundoff 2^-8; tf32 truncation of the
    fp32 feature by the tensor pipe 2^-10; 3×TF32 hi/lo split ≈ 2^-20; fp32 / fp64 0);
  * ẑ − z from the operand conversion (tf32 truncation 2^-10 per operand, 3×TF32 ≈ 2^-20) and the accumulation over
    p (tensor pipe: ≤ 2^-23 per accumulated MMA, truncating, DESIGN.md §6 finding 4; SIMT FFMA: 2^-24 per FMA),
    bounded by c·‖w_k‖‖x_i‖; it moves σ by at most L_σ·|ẑ − z| (L_σ = max|σ'|), plus σ's own evaluation error;
  * the accumulation over the m features, the same per-step rule (3×TF32: K-chunks of 128 features summed in fp32
    round-to-nearest), and the final 1/m scaling (one fp32 rounding).
  Cauchy–Schwarz turns Σ_k |σ_ki σ_kj| into m·√(G_ii G_jj) and Σ_k |σ_kj| into m·√G_jj, so with
  e_i = L_σ·Δz_i + e_eval:
      |ΔG_ij| ≤ (2u_s + u_s² + acc_m)·√(G_ii G_jj) + e_i √G_jj + e_j √G_ii + e_i e_j.
  At m = 1 (no averaging) this is the R22 reading: |ΔG_ij| ≤ (2·2^-8 + 2^-16 + ε)|G_ij| + O(e).

Φ by EQ1 from g = x_iᵀx_j:
  * Δg from the operand conversion and accumulation over p as above, ≤ c_g·‖x_i‖‖x_j‖;
  * its effect, |EQ1(g + Δg) − EQ1(g − Δg)|/2, evaluated with the oracle's own EQ1 (diagonal entries do not depend
    on g, reading R6);
  * the fp32 evaluation of the regrouped polynomial (≈ 10 roundings, a sqrt.approx at 2^-22, coefficients rounded to
    fp32): 2^-18 × the sum of the absolute values of EQ1's 18 terms (2^-47 in FP64 mode), plus 2e-12 of it for the
    two independent quadrature rules (library Golub–Welsch vs oracle Newton; they agree to ≤ 5e-13 per moment).
"""
from __future__ import annotations

import math

import numpy as np

import oracle

# max |σ'| of the smooth north-star activations (and the Lipschitz constants of the continuous Table-2 ones)
LIP = {"tanh": 1.0, "erf": 2.0 / math.sqrt(math.pi), "sigmoid_half": 0.25, "relu": 1.0, "abs": 1.0, "cos": 1.0,
       "sin": 1.0, "ident": 1.0, "bump": math.exp(-0.5)}
U_STORE = {"bf16": 2.0 ** -8, "tf32": 2.0 ** -10, "3xtf32": 2.0 ** -20, "fp32": 0.0, "fp64": 0.0}
U_OPERAND = {"bf16": 0.0, "tf32": 2.0 ** -10, "3xtf32": 2.0 ** -20, "fp32": 0.0, "fp64": 0.0}
E_EVAL = {"bf16": 5e-7, "tf32": 5e-7, "3xtf32": 5e-7, "fp32": 5e-7, "fp64": 1e-15}


def acc_rel(prec: str, K: int) -> float:
    """Worst-case relative error (to Σ|products|) of accumulating K products in the mode's accumulator."""
    if prec == "bf16":
        return (K / 16.0 + 1.0) * 2.0 ** -23          # one truncating add per kind::f16 MMA (K = 16)
    if prec == "tf32":
        return (K / 8.0 + 1.0) * 2.0 ** -23           # kind::tf32, K = 8
    if prec == "3xtf32":                               # 3 MMAs per K-step, chunks of 128 summed in fp32 (RN)
        return (3.0 * min(K, 128) / 8.0 + 1.0) * 2.0 ** -23 + (K / 128.0 + 1.0) * 2.0 ** -24
    if prec == "fp32":
        return (K + 1.0) * 2.0 ** -24
    return (K + 1.0) * 2.0 ** -53


def gram_bound(prec: str, act: str, Xs: np.ndarray, W: np.ndarray, Gref: np.ndarray, I, J) -> np.ndarray:
    """Per-entry bound on |G_gpu − G_oracle| at pairs (I, J) of the principal submatrix whose rows are Xs.
    Xs: |S| × p (fp64 copy of what the GPU read), W: the m × p rows that were summed, Gref: |S| × |S| oracle G."""
    m, p = W.shape
    d = np.sqrt(np.maximum(np.diag(Gref), 0.0))
    u = U_STORE[prec]
    rel = 2 * u + u * u + acc_rel(prec, m) + 2.0 ** -23
    wmax = float(np.sqrt(np.max(np.sum(np.asarray(W, float) ** 2, axis=1))))
    xn = np.sqrt(np.sum(np.asarray(Xs, float) ** 2, axis=1))
    dz = (2 * U_OPERAND[prec] + acc_rel(prec, p)) * xn * wmax
    extra = 0.0
    from oracle.acts import parse_param_act
    pa = parse_param_act(act) if isinstance(act, str) else None
    quad = (0.0, 0.0, 1.0) if act == "quad" else (pa[1] if pa and pa[0] == "quadratic" else None)
    if quad is not None or act in ("sign", "step"):
        Z = np.asarray(Xs, float) @ np.asarray(W, float).T            # |S| × m, fp64
    if quad is not None:     # σ' = 2a₂t + a₁ is not bounded: the local Lipschitz constant on each row's range of z
        a0, a1, a2 = quad
        zmax = np.max(np.abs(Z), axis=1) + dz
        L = 2.0 * abs(a2) * zmax + abs(a1)
        e = L * dz + E_EVAL[prec] * (1.0 + abs(a2) * zmax * zmax + abs(a1) * zmax + abs(a0))
    elif pa is not None:     # leaky ReLU: Lipschitz max(|a₊|, |a₋|)
        e = max(abs(pa[1][0]), abs(pa[1][1])) * dz + E_EVAL[prec] * max(1.0, abs(pa[1][0]), abs(pa[1][1]))
    else:
        e = LIP.get(act, 1.0) * dz + E_EVAL[prec]
    bound = rel * d[I] * d[J] + e[I] * d[J] + e[J] * d[I] + e[I] * e[J]
    if act in ("sign", "step"):
        # a jump of σ: a feature whose exact z lies within Δz of 0 may be decided either way; each such feature moves
        # G_ij by at most jump·max|σ| / m
        jump = 2.0 if act == "sign" else 1.0
        flips = np.sum(np.abs(Z) <= dz[:, None], axis=1).astype(float)
        extra = jump * (flips[I] + flips[J]) / m
    return bound + extra


def phi_bound(prec: str, act: str, Xs: np.ndarray, tau: float, I, J, mom=None, form: int = 1) -> np.ndarray:
    """Per-entry bound on |Φ_gpu − Φ_oracle| at pairs (I, J), i ≤ j, of the principal submatrix whose rows are Xs.
    form = 2: the six-term EQ2 (oracle/acts.py) instead of EQ1."""
    Xs = np.asarray(Xs, float)
    p = Xs.shape[1]
    if mom is None:
        mom = oracle.moments(act, tau)
    if form == 2:
        from oracle import acts
        f_val, f_terms = acts.eq2, acts.eq2_terms
    else:
        f_val, f_terms = oracle.eq1, oracle.eq1_terms
    nrm2 = np.sum(Xs * Xs, axis=1)
    xn = np.sqrt(nrm2)
    g = np.einsum("ij,ij->i", Xs[I], Xs[J])
    dg = (2 * U_OPERAND[prec] + acc_rel(prec, p)) * xn[I] * xn[J]
    diag = np.asarray(I) == np.asarray(J)
    hi = f_val(mom, *oracle.gram_schmidt(nrm2[I], nrm2[J], g + dg, diag))
    lo = f_val(mom, *oracle.gram_schmidt(nrm2[I], nrm2[J], g - dg, diag))
    sens = 0.5 * np.abs(hi - lo)
    # a sample pair with Gram–Schmidt residual u_b ≈ 0 off the diagonal (near-parallel rows) makes ∂Φ/∂g large;
    # the secant over ±Δg above captures it
    T = sum(np.abs(t) for t in f_terms(mom, *oracle.gram_schmidt(nrm2[I], nrm2[J], g, diag)))
    # + the library's Golub–Welsch moments vs the oracle's Newton Gauss–Hermite rule: they agree to ≤ 5e-13 relative
    # (tests/test_abi.py), each EQ1 term is a product of two moments
    arith = ((2.0 ** -47 if prec == "fp64" else 2.0 ** -18) + 2e-12) * T
    return sens + arith + 1e-30


def check(name: str, got: np.ndarray, ref: np.ndarray, bound: np.ndarray) -> float:
    """Assert |got − ref| ≤ bound entry by entry; return (and print) the worst ratio."""
    err = np.abs(np.asarray(got, float) - np.asarray(ref, float))
    ratio = err / bound
    worst = float(np.max(ratio)) if ratio.size else 0.0
    k = int(np.argmax(ratio)) if ratio.size else 0
    print(f"[entry] {name}: max |err|/bound {worst:.3f} (max-abs {float(err.max()) if err.size else 0:.3e})")
    assert worst <= 1.0, f"{name}: entry {k} err {float(err.flat[k]):.3e} > bound {float(bound.flat[k]):.3e}"
    return worst


def psd_bound(ref: np.ndarray, I, J, rel: float) -> np.ndarray:
    """rel·√(|A_ii A_jj|): the Cauchy–Schwarz scale of entry (i, j) of a PSD-like matrix (centred G, K̃, G^ter), for
    outputs whose arithmetic is the Gram's plus an O(1)-ulp post-pass; rel is the mode's Gram coefficient."""
    d = np.sqrt(np.abs(np.diag(ref)))
    return rel * d[I] * d[J] + 1e-12


def center_bound(A: np.ndarray, bA: np.ndarray, I, J, u: float = 2.0 ** -21) -> np.ndarray:
    """Per-entry bound for K = P·A·P (NEXT-2 centring post-pass) given the uncentred reference A (n × n, symmetric)
    and a per-entry bound bA (n × n) of the uncentred result: K_ij − K̂_ij = ΔA_ij − Δr_i − Δr_j + Δs with
    |Δr_i| ≤ max_j bA_ij and |Δs| ≤ max bA, plus the post-pass's own fp32/fp64 roundings (u per operand)."""
    r = A.mean(axis=1)
    s = r.mean()
    rb = bA.max(axis=1)
    return bA[I, J] + rb[I] + rb[J] + bA.max() + u * (np.abs(A[I, J]) + np.abs(r[I]) + np.abs(r[J]) + abs(s))


def full_pairs(n: int):
    I, J = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    return I.ravel(), J.ravel()
