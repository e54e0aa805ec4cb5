"""The tcgen05 CTA-pair mainloop in isolation (rf_debug_gemm_nt test hook): exact-in-fp32 integer inputs
must give bit-exact products at every tile / ragged-edge position, for BF16, TF32 and 3×TF32 operand
paths, with and without K-chunked accumulation."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2110_01899_b200 as rf  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available() and rf.rf_device_supported(0)
    yield


@pytest.mark.parametrize("prec", ["bf16", "tf32", "3xtf32"])
@pytest.mark.parametrize("shape", [(256, 256, 64), (300, 520, 200), (1, 1, 8), (513, 257, 1000)])
@pytest.mark.parametrize("kchunk", [0, 1, 3])
def test_integer_gemm_bit_exact(prec, shape, kchunk):
    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.integers(-4, 5, size=(M, K)).astype(np.float64)
    B = rng.integers(-4, 5, size=(N, K)).astype(np.float64)
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    Ad = torch.tensor(A, device="cuda").to(dt)
    Bd = torch.tensor(B, device="cuda").to(dt)
    C = rf.rf_debug_gemm_nt(Ad, Bd, prec=prec, kchunk=kchunk)
    torch.cuda.synchronize()
    ref = A @ B.T                     # |entries| ≤ 16·K < 2^24: exact in fp32 whatever the order
    assert np.array_equal(C.double().cpu().numpy(), ref)


def test_3xtf32_split_recovers_fp32_operands():
    """3×TF32 on operands that are not tf32-representable: per-product error ≈ 2^-22 relative."""
    rng = np.random.default_rng(9)
    M, N, K = 256, 256, 32
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    C = rf.rf_debug_gemm_nt(torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda"), prec="3xtf32")
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    err = np.abs(C.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err < 2e-6
