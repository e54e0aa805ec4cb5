"""World-size-2 CPU (gloo) tests of the multi-GPU host logic: feature sharding of W, the packed
upper-trapezoid reduce-scatter of the partial G, and Φ's row-block ownership.  The partial G of each rank
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
from paper_2110_01899_b200 import collective, rf_phi_row_split


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, p, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, p)) / np.sqrt(p)
        W = rng.standard_normal((m, p))
        m0, m1 = collective.feature_shard(m, world, rank)
        # partial upper triangle of this rank, scaled by 1/m_total (what rf_gram(m_total=m) returns)
        Gp = oracle.gram(X, W[m0:m1], "tanh", m_total=m)
        Gp[np.tril_indices(n, -1)] = np.nan              # garbage below the diagonal must not matter
        blk, (r0, r1) = collective.gram_reduce_scatter(torch.tensor(Gp))
        Gfull = oracle.gram(X, W, "tanh")
        got = blk.numpy()
        ref = Gfull[r0:r1, r0:n]
        iu = np.triu_indices(r1 - r0)                    # entries j >= i inside the block
        mask = np.zeros_like(got, dtype=bool)
        for i in range(r1 - r0):
            mask[i, i:] = True
        err = float(np.max(np.abs(got[mask] - ref[mask]))) if mask.any() else 0.0
        q.put((rank, r0, r1, err, len(iu[0]) >= 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [600, 1024])
def test_gram_reduce_scatter_gloo_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world, p, m = 2, 32, 301
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, m, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    assert res[0][1] == 0 and res[-1][2] == n and res[0][2] == res[1][1]
    for _, r0, r1, err, _ in res:
        assert err < 1e-12, (r0, r1, err)


def test_feature_shard_partition():
    for m in (1, 7, 65536, 65537):
        for world in (1, 2, 3, 8):
            sh = [collective.feature_shard(m, world, r) for r in range(world)]
            assert sh[0][0] == 0 and sh[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            sizes = [b - a for a, b in sh]
            assert max(sizes) - min(sizes) <= 1


def test_trapezoid_blocks_cover_upper_triangle_once():
    n, world = 1000, 3
    blocks = collective.row_blocks(n, world)
    cover = np.zeros((n, n), dtype=int)
    for r0, r1 in blocks:
        for i in range(r0, r1):
            cover[i, i:] += 1
    assert np.all(cover[np.triu_indices(n)] == 1)
    assert blocks == [rf_phi_row_split(n, world, r) for r in range(world)]
