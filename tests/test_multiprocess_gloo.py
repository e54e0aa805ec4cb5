"""World-size-2 CPU (gloo) tests of the multi-GPU host logic: feature sharding of W and the chunked
reduce-scatter of the packed triangle tiles of the partial G (include/rf.h G5: the library's plan and tile
map, the chunk views of collective.py).  The partial G of each rank
is produced by the oracle (the CPU stand-in for rf_gram on that rank's W shard) so the collective logic
runs exactly as in bench.py, over gloo instead of NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2110_01899_b200 import collective


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def pack_host(G, plan):
    """Test stand-in for K4's packed epilogue: place every slot's 256×256 tile of the (full, symmetric) partial
    G into the chunk-major / owner-major send layout of include/rf.h (zero padding past n)."""
    n = G.shape[0]
    T = collective.RF_PACK_TILE
    send = np.zeros(plan.send_elems, dtype=np.float32)
    Gp = np.zeros((((n + 511) // 512) * 512,) * 2)
    Gp[:n, :n] = G
    maps = [collective.owned_tiles(plan, o) for o in range(plan.world)]
    for c in range(plan.nchunks):
        S = plan.chunk_slots[c]
        k0 = plan.chunk_recv_off[c] // collective.TILE_ELEMS
        for o in range(plan.world):
            for s in range(S):
                I, J = maps[o][k0 + s]
                if I < 0:
                    continue
                off = plan.chunk_send_off[c] + (o * S + s) * collective.TILE_ELEMS
                send[off:off + collective.TILE_ELEMS] = Gp[I * T:(I + 1) * T, J * T:(J + 1) * T].reshape(-1)
    return send


def _worker(rank, world, port, n, p, m, prec, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, p)) / np.sqrt(p)
        W = rng.standard_normal((m, p))
        m0, m1 = collective.feature_shard(m, world, rank)
        # partial G of this rank, scaled by 1/m_total (what rf_gram_packed computes on its W rows)
        Gp = oracle.gram(X, W[m0:m1], "tanh", m_total=m)
        plan = collective.rf_pack_plan(n, world, 5, prec)
        send = torch.from_numpy(pack_host(Gp, plan))
        recv = torch.empty(plan.recv_elems, dtype=torch.float32)
        for snd, rcv in collective.chunk_views(plan, send, recv):      # the chunked collective of G5
            dist.reduce_scatter_tensor(rcv, snd, op=dist.ReduceOp.SUM)
        got = np.full((n, n), np.nan)
        written = collective.scatter_owned(recv.numpy(), collective.owned_tiles(plan, rank), n, got)
        Gfull = oracle.gram(X, W, "tanh")
        err = float(np.max(np.abs(got[written] - Gfull[written]))) if written.any() else 0.0
        q.put((rank, written, err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,prec", [(600, "bf16"), (1024, "bf16"), (700, "3xtf32")])
def test_gram_packed_reduce_scatter_gloo_world2(n, prec):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world, p, m = 2, 32, 301
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, m, prec, q)) for r in range(world)]
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
    for _, written, err in res:
        assert written.sum() > 0
        assert err < 1e-6, err       # fp32 send buffer: sums of two fp32-rounded partials


def test_feature_shard_partition():
    for m in (1, 7, 65536, 65537):
        for world in (1, 2, 3, 8):
            sh = [collective.feature_shard(m, world, r) for r in range(world)]
            assert sh[0][0] == 0 and sh[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            sizes = [b - a for a, b in sh]
            assert max(sizes) - min(sizes) <= 1
