"""G5 — the one exchange step of the path: sum the ranks' partial G.

G is data parallel over the features m (Eq. def_Gram: G is a sum over the m features): rank r
holds W rows [m0, m1) and computes, with rf_gram, the partial upper triangle
G_r = (1/m_total) Σ_{k ∈ [m0, m1)} σ(Xᵀw_k)σ(w_kᵀX).  G = Σ_r G_r is formed by a reduce-scatter over NCCL
(NVLink / NVSwitch on the 8×B200 box) of the UPPER TRAPEZOIDS only: ownership is by row blocks of equal
triangle area (rf_phi_row_split, 256-row boundaries), and block b is the dense sub-matrix
G[r_b:r_{b+1}, r_b:n] — the part of the upper triangle in those rows — so the bytes on the wire are ≈ half
of a dense n×n reduce-scatter.  Rank r ends with block r of G, summed.

torch.distributed is plumbing here (process group + NCCL); the compute stays in librf_b200.so.
"""
from __future__ import annotations

from typing import List, Tuple

from . import rf_phi_row_split


def feature_shard(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [m0, m1) of W owned by `rank` (contiguous, sizes differ by at most one)."""
    base, rem = divmod(m, world)
    m0 = rank * base + min(rank, rem)
    return m0, m0 + base + (1 if rank < rem else 0)


def row_blocks(n: int, world: int) -> List[Tuple[int, int]]:
    """Row block per rank, balanced by upper-triangle area (same split as Φ's row sharding)."""
    return [rf_phi_row_split(n, world, r) for r in range(world)]


def block_numel(n: int, blk: Tuple[int, int]) -> int:
    r0, r1 = blk
    return (r1 - r0) * (n - r0)


def pack_upper_blocks(G, blocks, out):
    """Copy block b = G[r_b:r_{b+1}, r_b:n] of the (partial) upper triangle into out[b, :numel_b]."""
    n = G.shape[0]
    for b, (r0, r1) in enumerate(blocks):
        k = block_numel(n, (r0, r1))
        if k:
            out[b, :k].view(r1 - r0, n - r0).copy_(G[r0:r1, r0:n])
    return out


def gram_reduce_scatter(G, group=None, send=None, recv=None):
    """Sum the ranks' partial upper triangles; returns (recv_block, (r0, r1)) where recv_block is the summed
    G[r0:r1, r0:n] of this rank's row block.  `send`/`recv` may be preallocated
    (shape (world, max_numel) and (max_numel,))."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = G.shape[0]
    blocks = row_blocks(n, world)
    width = max(block_numel(n, b) for b in blocks)
    if send is None:
        send = torch.zeros((world, width), dtype=G.dtype, device=G.device)
    if recv is None:
        recv = torch.empty((width,), dtype=G.dtype, device=G.device)
    pack_upper_blocks(G, blocks, send)
    dist.reduce_scatter_tensor(recv, send.view(-1), op=dist.ReduceOp.SUM, group=group)
    r0, r1 = blocks[rank]
    return recv[: block_numel(n, (r0, r1))].view(r1 - r0, n - r0), (r0, r1)
