"""Pins of the G1 oracle (oracle/rounding.py): bf16 round to nearest, ties to even, on the binary32 bit pattern.

Pinned by (1) values whose rounding is fixed by the definition (exact bf16 values, halfway ties both ways, just-off
ties, the carry into the exponent, overflow to inf, subnormals), (2) brute force over every bf16 neighbourhood of a
sample of binary32 values (the result is the nearest of the two bf16 neighbours, the even one on a tie), and
(3) a library routine that implements the same IEEE rounding (torch's float32 → bfloat16 cast on the CPU)."""
import numpy as np
import pytest

from oracle.rounding import bf16_bits_to_f64, round_bf16, round_bf16_bits


def f32(bits):
    return np.array(bits, dtype=np.uint32).view(np.float32)


def test_exact_values_unchanged():
    for v in [0.0, -0.0, 1.0, -2.5, 0.15625, 2.0 ** 127, -3.0 * 2.0 ** 100, 2.0 ** -126, 2.0 ** -133]:
        assert round_bf16(v)[()] == v


def test_ties_go_to_even():
    # 1 + 2^-8 lies halfway between 1 (even fraction) and 1 + 2^-7 (odd): rounds to 1
    assert round_bf16(f32(0x3F808000))[()] == 1.0
    # 1 + 3·2^-8 lies halfway between 1 + 2^-7 (odd) and 1 + 2^-6 (even): rounds up
    assert round_bf16(f32(0x3F818000))[()] == 1.0 + 2.0 ** -6
    # just above / below a tie
    assert round_bf16(f32(0x3F808001))[()] == 1.0 + 2.0 ** -7
    assert round_bf16(f32(0x3F807FFF))[()] == 1.0
    # negative tie: sign-magnitude, same rule
    assert round_bf16(f32(0xBF818000))[()] == -(1.0 + 2.0 ** -6)


def test_carry_into_exponent_and_overflow():
    # the largest bf16 fraction below 2 plus more than half an ulp rounds to 2
    assert round_bf16(f32(0x3FFFC000))[()] == 2.0
    # above the largest finite bf16 (0x7F7F) by at least half an ulp: +inf
    assert round_bf16(f32(0x7F7FFFFF))[()] == np.inf
    assert round_bf16(f32(0xFF7FFFFF))[()] == -np.inf
    assert round_bf16(np.float32(np.inf))[()] == np.inf


def test_nan_stays_nan():
    b = round_bf16_bits(np.array([np.nan, -np.nan], dtype=np.float32))
    assert np.all(np.isnan(bf16_bits_to_f64(b)))


def test_nearest_neighbour_brute_force():
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 0x7F7F0000, size=20000, dtype=np.uint32)   # positive finite binary32 below bf16 max
    x = bits.view(np.float32).astype(np.float64)
    lo = bf16_bits_to_f64((bits >> 16).astype(np.uint16))
    hi = bf16_bits_to_f64(((bits >> 16) + 1).astype(np.uint16))
    r = round_bf16(bits.view(np.float32))
    dlo, dhi = x - lo, hi - x
    assert np.all((r == lo) | (r == hi))
    assert np.all(r[dlo < dhi] == lo[dlo < dhi])
    assert np.all(r[dhi < dlo] == hi[dhi < dlo])
    tie = dlo == dhi
    even_lo = ((bits >> 16) & 1) == 0
    assert np.all(r[tie & even_lo] == lo[tie & even_lo]) and np.all(r[tie & ~even_lo] == hi[tie & ~even_lo])


def test_matches_library_cast():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    a = (rng.standard_normal(50000) * 10.0 ** rng.integers(-30, 30, 50000)).astype(np.float32)
    b = f32(rng.integers(0, 2 ** 32, 50000, dtype=np.uint64).astype(np.uint32))
    b = b[np.isfinite(b)]                       # random bit patterns: drop NaN / inf before any float cast
    x = np.concatenate([a, b]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(round_bf16_bits(x), ref)
