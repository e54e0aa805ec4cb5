"""CPU ORACLE for step G1: the BF16 mode's fp32 → bf16 input rounding.

TEST INFRASTRUCTURE ONLY (same rule as oracle/rf_oracle.py): imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs; never by the product path.

The paper is silent on precision (X, W are real matrices); BF16 is the north star's mode, and bf16 is binary32 with the low 16 fraction bits
dropped (1 sign, 8 exponent, 7 fraction bits), and the rounding is IEEE 754's default, round to nearest, ties to even.
Written out on the bit pattern u of the binary32 value:
  keep = u >> 16;  rest = u & 0xFFFF
  round up iff rest > 0x8000, or rest == 0x8000 and keep is odd (the tie goes to the even neighbour)
A carry out of the fraction bumps the exponent, which is exactly the next representable value (and turns the largest
finite values into ±inf, as IEEE overflow under round-to-nearest requires).  NaN inputs stay NaN (quiet bit set).
"""
from __future__ import annotations

import numpy as np


def round_bf16_bits(x) -> np.ndarray:
    """The bf16 bit patterns (uint16) of round-to-nearest-even(x), x cast to binary32 first."""
    u = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).view(np.uint32).astype(np.uint64)
    keep = u >> 16
    rest = u & 0xFFFF
    up = (rest > 0x8000) | ((rest == 0x8000) & ((keep & 1) == 1))
    out = keep + up.astype(np.uint64)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    out = np.where(nan, keep | 0x0040, out)          # quiet NaN, sign kept
    return out.astype(np.uint16)


def bf16_bits_to_f64(b) -> np.ndarray:
    """Value of bf16 bit patterns, exactly, as float64 (bf16 → binary32 is exact: append 16 zero bits)."""
    b = np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def round_bf16(x) -> np.ndarray:
    """round-to-nearest-even(x) to bf16, returned as float64 values."""
    return bf16_bits_to_f64(round_bf16_bits(x))
