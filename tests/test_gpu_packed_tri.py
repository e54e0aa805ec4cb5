"""GPU parity of RF_OUT_PACKED_TRI (include/rf.h): G (K4 SYRK epilogue), Φ (K5 EQ1 epilogue) and G^ter written as
the packed upper triangle.  The packed tiles decode (layout.unpack_tri) to exactly the UPPER output of the same
call — same kernels, same arithmetic, only the store address differs — and that output is checked against the fp64
oracle here as well; sizes cover one partial tile, several tiles with a ragged tail, and the 3×TF32 K-chunked
accumulation that re-reads the packed partial."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_2110_01899_b200 as rf  # noqa: E402
import synthetic  # noqa: E402
from paper_2110_01899_b200 import layout  # noqa: E402
from entry_bounds import check, gram_bound, phi_bound  # noqa: E402

pytestmark = pytest.mark.gpu
DT = {"bf16": torch.bfloat16, "tf32": torch.float32, "3xtf32": torch.float32}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    torch.cuda.set_device(0)
    yield


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,p,m", [(200, 64, 300), (1300, 128, 1024), (777, 96, 1500)])
@pytest.mark.parametrize("prec", ["bf16", "tf32", "3xtf32"])
def test_gram_packed_tri_equals_upper(n, p, m, prec):
    rng = np.random.default_rng(n + m)
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    W = rng.standard_normal((m, p))
    Xd, Wd = torch.tensor(X, device="cuda").to(DT[prec]), torch.tensor(W, device="cuda").to(DT[prec])
    P = torch.full((rf.rf_packed_tri_elems(n),), float("nan"), device="cuda")
    rf.rf_gram(Xd, Wd, act="tanh", prec=prec, out="packed_tri", G=P)
    G = rf.rf_gram(Xd, Wd, act="tanh", prec=prec, out="upper")
    torch.cuda.synchronize()
    D = layout.unpack_tri(P.cpu().numpy(), n, out=np.zeros((n, n), np.float32))
    I, J = np.triu_indices(n)
    Gc = G.cpu().numpy()
    assert np.array_equal(D[I, J], Gc[I, J])
    Xo, Wo = Xd.double().cpu().numpy(), Wd.double().cpu().numpy()
    ref = oracle.gram(Xo, Wo, "tanh")
    e = _rel(D[I, J].astype(np.float64), ref[I, J])
    print(f"[parity] packed G {prec} n={n}: rel-Frobenius {e:.3e}")
    assert e <= (2e-3 if prec in ("bf16", "tf32") else 1e-5)
    check(f"packed G {prec} n={n}", D[I, J], ref[I, J], gram_bound(prec, "tanh", Xo, Wo, ref, I, J))


@pytest.mark.parametrize("act", ["sigmoid_half", "relu"])
@pytest.mark.parametrize("n", [300, 1100])
def test_phi_packed_tri_equals_upper(act, n):
    X = synthetic.make_X(3, n=n, p=128)
    Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
    P = torch.full((rf.rf_packed_tri_elems(n),), float("nan"), device="cuda")
    rf.rf_phi_closed_form(Xd, act=act, prec="bf16", out="packed_tri", Phi=P)
    Phi = rf.rf_phi_closed_form(Xd, act=act, prec="bf16", out="upper")
    torch.cuda.synchronize()
    D = layout.unpack_tri(P.cpu().numpy(), n, out=np.zeros((n, n), np.float32))
    I, J = np.triu_indices(n)
    assert np.array_equal(D[I, J], Phi.cpu().numpy()[I, J])
    Xo = Xd.double().cpu().numpy()
    ref = oracle.phi_eq1(Xo, act)
    e = _rel(D[I, J].astype(np.float64), ref[I, J])
    print(f"[parity] packed Φ {act} n={n}: rel-Frobenius {e:.3e}")
    assert e <= 1e-5
    check(f"packed Φ {act} n={n}", D[I, J], ref[I, J], phi_bound("bf16", act, Xo, oracle.tau_hat(Xo), I, J))


def test_phi_packed_tri_row_ranges_compose():
    """Two row-range calls into one packed buffer fill the same triangle as one call (the multi-GPU row split)."""
    n = 1000
    X = synthetic.make_X(2, n=n, p=64)
    Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
    P1 = torch.zeros(rf.rf_packed_tri_elems(n), device="cuda")
    P2 = torch.zeros_like(P1)
    rf.rf_phi_closed_form(Xd, act="tanh", prec="bf16", out="packed_tri", Phi=P1)
    rf.rf_phi_closed_form(Xd, act="tanh", prec="bf16", out="packed_tri", Phi=P2, row_begin=0, row_end=512)
    rf.rf_phi_closed_form(Xd, act="tanh", prec="bf16", out="packed_tri", Phi=P2, row_begin=512, row_end=n)
    torch.cuda.synchronize()
    D1 = layout.unpack_tri(P1.cpu().numpy(), n)
    D2 = layout.unpack_tri(P2.cpu().numpy(), n)
    assert np.array_equal(D1, D2)


def test_gram_ter_packed_tri_equals_upper():
    n, p, m = 900, 128, 2048
    rng = np.random.default_rng(7)
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    T = rng.standard_normal((m, p))
    Xd, Td = torch.tensor(X, device="cuda").bfloat16(), torch.tensor(T, device="cuda").bfloat16()
    sm, sp = rf.rf_trf_thresholds_for("tanh", 1.0)
    P = torch.full((rf.rf_packed_tri_elems(n),), float("nan"), device="cuda")
    rf.rf_gram_ter(Xd, Td, 0.9, sm, sp, out="packed_tri", G=P)
    G = rf.rf_gram_ter(Xd, Td, 0.9, sm, sp, out="upper")
    torch.cuda.synchronize()
    D = layout.unpack_tri(P.cpu().numpy(), n, out=np.zeros((n, n), np.float32))
    I, J = np.triu_indices(n)
    assert np.array_equal(D[I, J], G.cpu().numpy()[I, J])
