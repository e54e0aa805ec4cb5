"""Host-side decoding of the RF_OUT_PACKED_TRI layout (include/rf.h): tile (I, J ≥ I) of the T × T grid of
256 × 256 tiles, T = ceil(n/256), at float offset 65536·(I·T − I(I−1)/2 + J − I), row-major inside.

Used by tests and by callers that copied a packed G or Φ to the host; it is data movement only (no arithmetic of
the method) and never runs on the product path."""
from __future__ import annotations

import numpy as np

TILE = 256


def tri_tile_index(I: int, J: int, T: int) -> int:
    return I * T - I * (I - 1) // 2 + (J - I)


def packed_tri_elems(n: int) -> int:
    T = (n + TILE - 1) // TILE
    return T * (T + 1) // 2 * TILE * TILE


def unpack_tri(P, n: int, out=None, mirror: bool = False):
    """Packed triangle (1-D array-like, host) → n × n array with the upper triangle filled (lower untouched unless
    mirror, then mirrored)."""
    P = np.asarray(P)
    T = (n + TILE - 1) // TILE
    if out is None:
        out = np.zeros((n, n), dtype=P.dtype)
    tiles = P[:T * (T + 1) // 2 * TILE * TILE].reshape(-1, TILE, TILE)
    for I in range(T):
        r0, r1 = I * TILE, min(n, I * TILE + TILE)
        for J in range(I, T):
            c0, c1 = J * TILE, min(n, J * TILE + TILE)
            blk = tiles[tri_tile_index(I, J, T), :r1 - r0, :c1 - c0]
            if I == J:
                iu = np.triu_indices(r1 - r0)
                out[r0 + iu[0], c0 + iu[1]] = blk[iu]
            else:
                out[r0:r1, c0:c1] = blk
    if mirror:
        il = np.tril_indices(n, -1)
        out[il] = out.T[il]
    return out
