"""CPU tests of the multi-GPU host logic (include/rf.h "G5"): the canonical tile ownership rf_tile_map (host-only C ABI
call, no GPU needed), feature sharding of W, and a world-size-2 gloo run of the exchange layout: each rank's partial
G over its W rows (the oracle stands in for rf_gram on that rank's shard) is cut into the owners' slots by
rf_tile_map and summed with a reduce-scatter — the data movement the library's collective rf_gram does on the GPU
(peer-memory stores into the owners' staging buffers, or NCCL), here over gloo."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2110_01899_b200 as rf
from paper_2110_01899_b200 import collective

T_ = collective.RF_PACK_TILE


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [1, 255, 256, 600, 1024, 4097, 65536])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_tile_map_covers_upper_triangle_exactly_once(n, world):
    T = -(-n // T_)
    seen = np.zeros((T, T), dtype=int)
    slots = None
    for r in range(world):
        ij = rf.rf_tile_map(n, world, r)
        slots = len(ij) if slots is None else slots
        assert len(ij) == slots, "every rank receives the same number of slots"
        for I, J in ij:
            if I < 0:
                assert J < 0
                continue
            assert 0 <= I <= J < T
            seen[I, J] += 1
    iu = np.triu_indices(T)
    assert np.all(seen[iu] == 1)
    assert seen.sum() == T * (T + 1) // 2
    # padding: at most one slot per chunk and rank (≤ 16 chunks)
    assert slots * world - T * (T + 1) // 2 <= 16 * world


def test_tile_map_chunks_are_row_ordered_and_balanced():
    """Slots follow chunk order (chunks = runs of 8-row-tile groups, the order K4 finishes them), and inside a chunk
    the owned tiles go row-major; owners' real tiles differ by at most one per chunk."""
    n, world = 65536, 8
    maps = [rf.rf_tile_map(n, world, r) for r in range(world)]
    for ij in maps:
        real = ij[ij[:, 0] >= 0]
        key = real[:, 0] * 10 ** 6 + real[:, 1]
        assert np.all(np.diff(key) > 0), "slots are in (row, column) order"
    counts = [int(np.sum(ij[:, 0] >= 0)) for ij in maps]
    assert max(counts) - min(counts) <= 16


def test_tile_map_rejects_bad_arguments():
    for args in [(0, 1, 0), (100, 0, 0), (100, 2, 2), (100, 2, -1)]:
        with pytest.raises(rf.RFError):
            rf.rf_tile_map(*args)


def _worker(rank, world, port, n, p, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, p)) / np.sqrt(p)
        W = rng.standard_normal((m, p))
        m0, m1 = collective.feature_shard(m, world, rank)
        Gp = oracle.gram(X, W[m0:m1], "tanh", m_total=m)          # this rank's partial, scaled by 1/m_total
        T = -(-n // T_)
        Gpad = np.zeros((T * T_, T * T_))
        Gpad[:n, :n] = Gp
        maps = [rf.rf_tile_map(n, world, o) for o in range(world)]
        # the staging layout's content: for every owner o, o's slots cut from this rank's partial (whole tiles)
        send = np.zeros((world, len(maps[0]), T_ * T_), dtype=np.float32)
        for o in range(world):
            for k, (I, J) in enumerate(maps[o]):
                if I >= 0:
                    send[o, k] = Gpad[I * T_:(I + 1) * T_, J * T_:(J + 1) * T_].reshape(-1)
        recv = torch.empty(len(maps[0]) * T_ * T_, dtype=torch.float32)
        dist.reduce_scatter_tensor(recv, torch.from_numpy(send.reshape(-1)), op=dist.ReduceOp.SUM)
        got = np.full((n, n), np.nan)
        written = collective.scatter_owned(recv.numpy(), maps[rank], n, got)
        Gfull = oracle.gram(X, W, "tanh")
        err = float(np.max(np.abs(got[written] - Gfull[written]))) if written.any() else 0.0
        hs = collective.exchange_peer_handles(bytes([rank]) * 64)            # the IPC-handle exchange helper
        q.put((rank, written, err, hs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [600, 1024, 1300])
def test_g5_exchange_layout_gloo_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world, p, m = 2, 32, 301
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, m, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort(key=lambda r: r[0])
    cover = res[0][1].astype(int) + res[1][1].astype(int)
    iu = np.triu_indices(n)
    assert np.all(cover[iu] == 1), "owned tiles must cover the upper triangle exactly once"
    for _, written, err, hs in res:
        assert written.sum() > 0
        assert err < 1e-6, err       # fp32 slots: sums of two fp32-rounded partials
        assert hs == [bytes([0]) * 64, bytes([1]) * 64]


def test_feature_shard_partition():
    for m in (1, 7, 65536, 65537):
        for world in (1, 2, 3, 8):
            sh = [collective.feature_shard(m, world, r) for r in range(world)]
            assert sh[0][0] == 0 and sh[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            sizes = [b - a for a, b in sh]
            assert max(sizes) - min(sizes) <= 1
