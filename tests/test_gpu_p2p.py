"""GPU tests of the fused G5 (include/rf.h rf_gram_packed_p2p / rf_pack_reduce, collective.GramFusedP2P): K4's
epilogue stores each packed tile of the partial G straight into its owner's staging buffer through a CUDA-IPC
mapping, then each owner sums its R slices.

* world 1 (in-process gloo group): the fused path equals the dense K4 bit for bit.
* world 2 as two processes on the one GPU of this box: each maps the other's staging buffer by CUDA IPC and its K4
  stores half of its tiles into it.  No kernel waits on another (the two phases are separated by host barriers), so
  this is a faithful two-rank run of the data path; the summed owned tiles are checked against the fp64 oracle.
"""
import math
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(n, p, m):
    rng = np.random.default_rng(5)
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    W = rng.standard_normal((m, p))
    return X, W


def test_fused_world1_equals_dense_gram():
    import torch.distributed as dist
    import paper_2110_01899_b200 as rf
    from paper_2110_01899_b200 import collective
    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        n, p, m = 1300, 128, 1024
        X, W = _inputs(n, p, m)
        Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
        Wd = torch.tensor(W, device="cuda").to(torch.bfloat16)
        fz = collective.GramFusedP2P(n, p, m, m, "tanh", "bf16", nchunks=5)
        for _ in range(2):
            recv = fz(Xd, Wd)
        torch.cuda.synchronize()
        G = rf.rf_gram(Xd, Wd, act="tanh", prec="bf16", out="upper")
        torch.cuda.synchronize()
        got = np.full((n, n), np.nan, dtype=np.float32)
        w = collective.scatter_owned(recv.cpu().numpy(), fz.owned_tiles(), n, got)
        I, J = np.triu_indices(n)
        assert w[I, J].all()
        assert np.array_equal(got[I, J], G.cpu().numpy()[I, J])
        fz.close()
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, n, p, m, q):
    import torch.distributed as dist
    import oracle
    from paper_2110_01899_b200 import collective
    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, W = _inputs(n, p, m)
        m0, m1 = collective.feature_shard(m, world, rank)
        Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
        Wd = torch.tensor(W[m0:m1], device="cuda").to(torch.bfloat16)
        fz = collective.GramFusedP2P(n, p, m1 - m0, m, "sigmoid_half", "bf16", nchunks=4)
        for _ in range(2):                                   # the second call reuses the mapped buffers
            recv = fz(Xd, Wd)
        torch.cuda.synchronize()
        got = np.full((n, n), np.nan)
        written = collective.scatter_owned(recv.cpu().numpy().astype(np.float64), fz.owned_tiles(), n, got)
        Xb = Xd.double().cpu().numpy()
        Wb = torch.tensor(W, device="cuda").to(torch.bfloat16).double().cpu().numpy()
        ref = oracle.gram(Xb, Wb, "sigmoid_half")
        e = float(np.linalg.norm(got[written] - ref[written]) / np.linalg.norm(ref[written]))
        dist.barrier()
        fz.close()
        q.put((rank, written, e))
    finally:
        dist.destroy_process_group()


def test_fused_two_processes_on_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n, p, m, world = 1100, 96, 768, 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, m, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    cover = res[0][1].astype(int) + res[1][1].astype(int)
    I, J = np.triu_indices(n)
    assert np.all(cover[I, J] == 1)
    for rank, _, e in res:
        print(f"[parity] fused G5 rank {rank}/2: rel-Frobenius {e:.3e}")
        assert e < 2e-3
