"""GPU parity of step G1 (include/rf.h rf_round_bf16): fp32 → bf16 round to nearest, ties to even, bit-exact against
the CPU oracle (oracle/rounding.py) — on the 16-B vector path and the scalar path (ragged column count, padded
strides), on values built to hit ties, carries into the exponent, overflow, subnormals, ±inf and NaN, and at the
size of configs[3]'s X; then the BF16 G computed from rf_round_bf16's output equals the G of bf16 inputs rounded by
the oracle, bit for bit (same bf16 operands ⇒ same kernel arithmetic)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2110_01899_b200 as rf  # noqa: E402
from oracle.rounding import round_bf16_bits  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    torch.cuda.set_device(0)
    yield


def _bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def _edge_values(rng, k):
    keep = rng.integers(0, 0x7F80, k, dtype=np.uint32) | (rng.integers(0, 2, k, dtype=np.uint32) << 15)
    rest = rng.choice(np.array([0x0000, 0x7FFF, 0x8000, 0x8001, 0xFFFF], dtype=np.uint32), k)
    return ((keep << 16) | rest).view(np.float32)


@pytest.mark.parametrize("rows,cols,lds,ldd", [(1, 1, 1, 1), (37, 1000, 1000, 1000), (37, 1000, 1004, 1008),
                                               (65, 1023, 1023, 1024), (5, 7, 9, 11), (300, 4096, 4100, 4096)])
def test_round_bf16_bit_exact(rows, cols, lds, ldd):
    rng = np.random.default_rng(rows * 7 + cols)
    x = np.empty((rows, lds), dtype=np.float32)
    x[:] = rng.standard_normal((rows, lds)).astype(np.float32) * np.float32(3.0)
    x.reshape(-1)[: x.size // 2] = _edge_values(rng, x.size // 2)
    x[0, : min(cols, 6)] = np.array([np.inf, -np.inf, np.nan, 3.4e38, 1e-45, -0.0], dtype=np.float32)[: min(cols, 6)]
    src = torch.from_numpy(x).cuda()[:, :cols]
    out_full = torch.full((rows, ldd), -7.0, dtype=torch.bfloat16, device="cuda")
    out = out_full[:, :cols]
    rf.rf_round_bf16(src, out=out)
    torch.cuda.synchronize()
    got = _bits(out_full)
    ref = round_bf16_bits(x[:, :cols])
    nan = np.isnan(x[:, :cols])
    g = got[:, :cols]
    assert np.array_equal(g[~nan], ref[~nan])
    assert np.all(((g[nan] & 0x7F80) == 0x7F80) & ((g[nan] & 0x7F) != 0))      # NaN stays NaN
    if ldd > cols:                                                               # padding untouched
        assert np.all(got[:, cols:] == _bits(torch.full((1,), -7.0, dtype=torch.bfloat16))[0])


def test_round_bf16_configs3_size():
    import synthetic
    cfg = synthetic.CONFIGS[3]
    x = synthetic.make_X(cfg).astype(np.float32)
    out = rf.rf_round_bf16(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    assert rf.rf_last_launch_count() == 1
    idx = np.random.default_rng(3).integers(0, x.size, 200000)
    assert np.array_equal(_bits(out).reshape(-1)[idx], round_bf16_bits(x.reshape(-1)[idx]))


def test_round_bf16_empty_and_invalid():
    e = torch.empty((0, 16), dtype=torch.float32, device="cuda")
    assert rf.rf_round_bf16(e).shape == (0, 16)
    x = torch.zeros((4, 8), dtype=torch.float32, device="cuda")
    with pytest.raises(rf.RFError):
        rf.rf_round_bf16(x, out=torch.empty((4, 9), dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(rf.RFError):
        rf.rf_round_bf16(x.double())


def test_gram_from_rounded_inputs():
    import synthetic
    cfg = synthetic.CONFIGS[1]
    X = synthetic.make_X(cfg).astype(np.float32)
    W = synthetic.make_W(cfg).astype(np.float32)
    Xb = rf.rf_round_bf16(torch.from_numpy(X).cuda())
    Wb = rf.rf_round_bf16(torch.from_numpy(W).cuda())
    Xr = torch.from_numpy(round_bf16_bits(X).view(np.int16)).view(torch.bfloat16).cuda()
    Wr = torch.from_numpy(round_bf16_bits(W).view(np.int16)).view(torch.bfloat16).cuda()
    G1 = rf.rf_gram(Xb, Wb, act=cfg.act, prec="bf16")
    G2 = rf.rf_gram(Xr, Wr, act=cfg.act, prec="bf16")
    torch.cuda.synchronize()
    assert torch.equal(torch.triu(G1), torch.triu(G2))
