"""G5 — the one exchange step of the path: sum the ranks' partial G.

G is data parallel over the features m (Eq. def_Gram: G is a sum over the m features).  Rank r holds W
rows [m0, m1) (`feature_shard`) and computes the partial G_r = (1/m_total) Σ_{k ∈ [m0, m1)} σ(Xᵀw_k)σ(w_kᵀX);
G = Σ_r G_r.  The whole exchange runs inside the library's collective rf_gram (include/rf.h "G5"): K4's epilogue
writes each upper-triangle tile of the partial into its owner's exchange slot and rank r ends with its owned tiles
summed (rf_tile_map says which).  This module only sets the context up — it exchanges the 64-byte CUDA IPC handles
of the staging buffers (peer-memory exchange, the product path) or broadcasts the NCCL unique id (NCCL baseline)
over the caller's process group — and decodes owned tiles on the host for tests.  No host synchronization or
barrier happens per call.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

from . import RF_PACK_TILE, Context, rf_gram, rf_nccl_get_unique_id, rf_tile_map, rf_workspace_size

TILE_ELEMS = RF_PACK_TILE * RF_PACK_TILE


def feature_shard(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [m0, m1) of W owned by `rank` (contiguous, sizes differ by at most one)."""
    base, rem = divmod(m, world)
    m0 = rank * base + min(rank, rem)
    return m0, m0 + base + (1 if rank < rem else 0)


def owned_tiles(n: int, world: int, rank: int) -> np.ndarray:
    """(row tile, col tile) of each receive slot of `rank`; (−1, −1) marks padding slots (include/rf.h rf_tile_map)."""
    return rf_tile_map(n, world, rank)


def scatter_owned(recv, tiles: np.ndarray, n: int, out, upper_only: bool = True):
    """Copy the received tiles of one rank into a dense n×n buffer `out` (torch or numpy, same device as recv);
    entries (i, j) with j ≥ i only when upper_only.  Returns a boolean mask (numpy) of the entries written."""
    written = np.zeros((n, n), dtype=bool)
    T = RF_PACK_TILE
    for k, (I, J) in enumerate(tiles):
        if I < 0:
            continue
        i0, j0 = int(I) * T, int(J) * T
        i1, j1 = min(i0 + T, n), min(j0 + T, n)
        blk = recv[k * TILE_ELEMS:(k + 1) * TILE_ELEMS].reshape(T, T)[: i1 - i0, : j1 - j0]
        m = np.ones((i1 - i0, j1 - j0), dtype=bool)
        if upper_only:
            m = np.arange(j0, j1)[None, :] >= np.arange(i0, i1)[:, None]
        if m.all():
            out[i0:i1, j0:j1] = blk
        else:
            idx = np.nonzero(m)
            out[i0:i1, j0:j1][idx] = blk[idx]
        written[i0:i1, j0:j1] |= m
    return written


def exchange_peer_handles(handle: bytes, group=None) -> list:
    """All ranks' 64-byte IPC handles, in rank order (process-group plumbing only)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return out


def broadcast_nccl_id(group=None) -> bytes:
    """Rank 0's ncclUniqueId (from the library's NCCL), broadcast over the process group."""
    import torch.distributed as dist
    obj = [rf_nccl_get_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class GramCollective:
    """Multi-GPU G through the library's collective rf_gram (one process per GPU).

        gc = GramCollective(n, p, m_local, m_total, act, prec, group, mode="peers")   # or mode="nccl"
        recv = gc(X, W_local)      # this rank's summed tiles, layout per gc.owned_tiles()
    The process group is used at construction only (handle exchange / NCCL id broadcast)."""

    def __init__(self, n: int, p: int, m_local: int, m_total: int, act: str, prec: str, group=None,
                 mode: str = "peers", device=None, ctx: Context = None):
        import torch
        import torch.distributed as dist
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n, self.p, self.m_local, self.m_total, self.act, self.prec = n, p, m_local, m_total, act, prec
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ctx = ctx if ctx is not None else Context(dev.index if dev.index is not None else 0)
        self.mode = mode
        if mode == "peers":
            self.ctx.attach_peers(self.rank, self.world, n)
            self.ctx.open_peers(exchange_peer_handles(self.ctx.peer_handle(), group))
        elif mode == "nccl":
            self.ctx.init_nccl(broadcast_nccl_id(group), self.rank, self.world)
        else:
            raise ValueError(mode)
        self.tiles = owned_tiles(n, self.world, self.rank)
        self.recv = torch.empty(len(self.tiles) * TILE_ELEMS, dtype=torch.float32, device=dev)
        self.ws = torch.empty(rf_workspace_size("gram", p, n, m_local, prec, "packed_tiles", ctx=self.ctx),
                              dtype=torch.uint8, device=dev)

    def __call__(self, X, W, stream=None):
        return rf_gram(X, W, act=self.act, prec=self.prec, out="packed_tiles", m_total=self.m_total, G=self.recv,
                       ws=self.ws, stream=stream, ctx=self.ctx)

    def owned_tiles(self) -> np.ndarray:
        return self.tiles

    def close(self):
        self.ctx.destroy()
