"""G5 — the one exchange step of the path: sum the ranks' partial G.

G is data parallel over the features m (Eq. def_Gram: G is a sum over the m features).  Rank r
holds W rows [m0, m1) (`feature_shard`) and computes the partial G_r = (1/m_total) Σ_{k ∈ [m0, m1)}
σ(Xᵀw_k)σ(w_kᵀX); G = Σ_r G_r.

The partial never exists as a dense n×n matrix: K4 (rf_gram_packed) writes every 256×256 tile of the upper
triangle straight into a chunk-major, owner-major SEND buffer (include/rf.h, rf_pack_plan_t) and counts
finished tiles per chunk.  A communication stream waits for chunk c (rf_stream_wait_chunk, a driver
stream-memory wait) and runs the reduce-scatter of chunk c while K4 computes chunk c+1, so only the last
chunk's collective is exposed.  Rank r ends with the summed tiles it owns (rf_pack_tile_map says which).
Bytes on the wire ≈ the triangle (half of a dense n×n reduce-scatter).

torch.distributed (NCCL over NVLink/NVSwitch on the 8×B200 box; gloo in the CPU tests) is plumbing here:
it moves and sums bytes the library's kernels produced.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

from . import RF_PACK_TILE, rf_gram_packed, rf_gram_workspace_size, rf_pack_plan, rf_pack_tile_map, \
    rf_stream_wait_chunk

TILE_ELEMS = RF_PACK_TILE * RF_PACK_TILE


def feature_shard(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [m0, m1) of W owned by `rank` (contiguous, sizes differ by at most one)."""
    base, rem = divmod(m, world)
    m0 = rank * base + min(rank, rem)
    return m0, m0 + base + (1 if rank < rem else 0)


def chunk_views(plan, send, recv):
    """[(send slice, recv slice)] per chunk: send chunk c = [owner 0 | … | owner R−1] blocks of
    chunk_slots[c] tiles, recv chunk c = this rank's block."""
    out = []
    for c in range(plan.nchunks):
        s0, s1 = plan.chunk_send_off[c], plan.chunk_send_off[c + 1]
        r0, r1 = plan.chunk_recv_off[c], plan.chunk_recv_off[c + 1]
        out.append((send[s0:s1], recv[r0:r1]))
    return out


def owned_tiles(plan, rank: int) -> np.ndarray:
    """(row tile, col tile) of each receive slot of `rank`; (−1, −1) marks padding slots."""
    return rf_pack_tile_map(plan, rank)


def scatter_owned(recv, tiles: np.ndarray, n: int, out, upper_only: bool = True):
    """Copy the received tiles of one rank into a dense n×n buffer `out` (torch or numpy, same device as
    recv); entries (i, j) with j ≥ i only when upper_only.  Returns a boolean mask (numpy) of the entries
    written."""
    written = np.zeros((n, n), dtype=bool)
    T = RF_PACK_TILE
    for k, (I, J) in enumerate(tiles):
        if I < 0:
            continue
        i0, j0 = int(I) * T, int(J) * T
        i1, j1 = min(i0 + T, n), min(j0 + T, n)
        if i0 >= n or j0 >= n:
            continue
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


class GramReduceScatter:
    """Multi-GPU G: rf_gram_packed on the caller's stream, chunked reduce-scatter overlapped on a
    communication stream (one process per GPU, process group over NCCL).

        rs = GramReduceScatter(n, p, m_local, m_total, act, prec, group)
        recv = rs(X, W_local)          # this rank's summed tiles, layout per owned_tiles(rs.plan, rank)
    """

    def __init__(self, n: int, p: int, m_local: int, m_total: int, act: str, prec: str, group=None,
                 nchunks: int = 16, max_sms: int = 0, device=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n, self.p, self.m_local, self.m_total, self.act, self.prec = n, p, m_local, m_total, act, prec
        self.plan = rf_pack_plan(n, self.world, nchunks, prec)
        self.max_sms = max_sms
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.send = torch.empty(self.plan.send_elems, dtype=torch.float32, device=dev)
        self.recv = torch.empty(self.plan.recv_elems, dtype=torch.float32, device=dev)
        self.sync = torch.zeros(self.plan.nchunks, dtype=torch.int32, device=dev)
        self.ws = torch.empty(rf_gram_workspace_size(p, n, m_local, prec), dtype=torch.uint8, device=dev)
        self.comm = torch.cuda.Stream(device=dev)
        self.epoch = 0
        self.views = chunk_views(self.plan, self.send, self.recv)

    def __call__(self, X, W):
        import torch
        import torch.distributed as dist
        cur = torch.cuda.current_stream()
        cur.wait_stream(self.comm)             # the previous call's collectives still read `send`
        self.epoch += 1
        rf_gram_packed(X, W, self.plan, self.send, self.sync, self.epoch, act=self.act, prec=self.prec,
                       m_total=self.m_total, max_sms=self.max_sms, ws=self.ws, stream=cur)
        with torch.cuda.stream(self.comm):
            for c, (snd, rcv) in enumerate(self.views):
                rf_stream_wait_chunk(self.plan, self.sync, c, self.epoch, stream=self.comm)
                dist.reduce_scatter_tensor(rcv, snd, op=dist.ReduceOp.SUM, group=self.group)
        cur.wait_stream(self.comm)
        return self.recv

    def owned_tiles(self) -> np.ndarray:
        return owned_tiles(self.plan, self.rank)


class GramFusedP2P:
    """Fused G5 (the product path for R > 1): K4's epilogue stores each tile of this rank's partial G straight into
    the owner's staging buffer over NVLink (peer memory mapped with CUDA IPC), so the exchange overlaps the SYRK
    tile by tile and no collective kernel runs; then each owner sums its R staging slices in rank order.

        fz = GramFusedP2P(n, p, m_local, m_total, act, prec, group)
        recv = fz(X, W_local)          # same layout as GramReduceScatter (owned_tiles)
    The process group only exchanges the 64-byte IPC handles and provides the barrier between the two phases.
    """

    def __init__(self, n: int, p: int, m_local: int, m_total: int, act: str, prec: str, group=None,
                 nchunks: int = 16, max_sms: int = 0, device=None):
        import torch
        import torch.distributed as dist
        from . import rf_ipc_handle, rf_ipc_open
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n, self.p, self.m_local, self.m_total, self.act, self.prec = n, p, m_local, m_total, act, prec
        self.plan = rf_pack_plan(n, self.world, nchunks, prec)
        self.max_sms = max_sms
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.staging = torch.empty(self.world * self.plan.recv_elems, dtype=torch.float32, device=dev)
        self.recv = torch.empty(self.plan.recv_elems, dtype=torch.float32, device=dev)
        self.ws = torch.empty(rf_gram_workspace_size(p, n, m_local, prec), dtype=torch.uint8, device=dev)
        handles = [None] * self.world
        dist.all_gather_object(handles, rf_ipc_handle(self.staging), group=group)
        self.opened = []
        self.ptrs = []
        for r, h in enumerate(handles):
            if r == self.rank:
                self.ptrs.append(self.staging.data_ptr())
            else:
                a = rf_ipc_open(h)
                self.opened.append(a)
                self.ptrs.append(a)

    def __call__(self, X, W):
        import torch
        import torch.distributed as dist
        from . import rf_gram_packed_p2p, rf_pack_reduce
        torch.cuda.current_stream().synchronize()   # my previous rf_pack_reduce has finished reading staging
        dist.barrier(group=self.group)          # every owner has finished reading its staging buffer
        rf_gram_packed_p2p(X, W, self.plan, self.rank, self.ptrs, act=self.act, prec=self.prec,
                           m_total=self.m_total, max_sms=self.max_sms, ws=self.ws)
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)          # every rank's stores into my staging buffer have landed
        rf_pack_reduce(self.plan, self.staging, self.recv)
        return self.recv

    def owned_tiles(self) -> np.ndarray:
        return owned_tiles(self.plan, self.rank)

    def close(self):
        from . import rf_ipc_close
        for a in self.opened:
            rf_ipc_close(a)
        self.opened = []
