"""GPU tests of G5 (include/rf.h): K4 writing packed triangle tiles for the multi-GPU reduce-scatter.

* Emulated ranks on ONE GPU: rank r's rf_gram_packed runs on its W shard into its own send buffer (no kernel
  waits on another); the reduce-scatter's sum is taken with torch; each owner's slots are decoded with
  rf_pack_tile_map and compared with the fp64 oracle G of the full W (north-star tolerances).
* The real path at world size 1: GramReduceScatter over an NCCL process group of one rank (the collective
  is a copy), whose result must equal the dense rf_gram bit for bit, and the chunk counters K4 publishes.
"""
import math
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_2110_01899_b200 as rf  # noqa: E402
from paper_2110_01899_b200 import collective  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {"3xtf32": 1e-5, "tf32": 2e-3, "bf16": 2e-3}
DT = {"3xtf32": torch.float32, "tf32": torch.float32, "bf16": torch.bfloat16}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    assert rf.rf_device_supported(0), "device 0 is not sm_100"
    torch.cuda.set_device(0)
    yield


@pytest.mark.parametrize("n,p,m,world,prec,nchunks", [
    (600, 64, 384, 2, "bf16", 4),        # ragged n (not a multiple of 256 / 512)
    (1024, 96, 512, 3, "bf16", 16),      # tile multiple, world not a power of two
    (777, 784, 1000, 4, "3xtf32", 3),    # fp32-accurate mode (256-wide K4 tiles, K-chunked accumulation)
    (1300, 128, 640, 2, "tf32", 64),     # more chunks requested than raster groups
])
def test_packed_emulated_ranks_match_oracle(n, p, m, world, prec, nchunks):
    rng = np.random.default_rng(n + world)
    X = rng.standard_normal((n, p)) / math.sqrt(p)
    W = rng.standard_normal((m, p))
    Xd = torch.tensor(X, device="cuda").to(DT[prec])
    Wd = torch.tensor(W, device="cuda").to(DT[prec])
    plan = rf.rf_pack_plan(n, world, nchunks, prec)
    total = torch.zeros(plan.send_elems, dtype=torch.float32, device="cuda")
    for r in range(world):
        m0, m1 = collective.feature_shard(m, world, r)
        send = torch.full((plan.send_elems,), float("nan"), dtype=torch.float32, device="cuda")
        sync = torch.zeros(plan.nchunks, dtype=torch.int32, device="cuda")
        rf.rf_gram_packed(Xd, Wd[m0:m1].contiguous(), plan, send, sync, 1, act="tanh", prec=prec, m_total=m)
        torch.cuda.synchronize()
        snd = send.view(-1, collective.TILE_ELEMS).cpu()
        for c in range(plan.nchunks):
            nt = (plan.chunk_tile0[c + 1] - plan.chunk_tile0[c]) * plan.tiles_per_pair
            base = plan.chunk_send_off[c] // collective.TILE_ELEMS
            for o in range(world):
                for sl in range(plan.chunk_slots[c]):
                    used = sl * world + o < nt
                    k = base + o * plan.chunk_slots[c] + sl
                    assert bool(torch.isnan(snd[k]).any()) != used, (c, o, sl, used)
        per_chunk = [16 * (plan.chunk_tile0[c + 1] - plan.chunk_tile0[c]) for c in range(plan.nchunks)]
        assert sync.cpu().tolist() == per_chunk
        total += torch.nan_to_num(send, nan=0.0)
    ref = oracle.gram(Xd.double().cpu().numpy(), Wd.double().cpu().numpy(), "tanh")
    got = np.full((n, n), np.nan)
    cover = np.zeros((n, n), dtype=int)
    tot = total.cpu().numpy()
    for r in range(world):
        recv = np.concatenate([tot[plan.chunk_send_off[c] + r * plan.chunk_slots[c] * collective.TILE_ELEMS:
                                   plan.chunk_send_off[c] + (r + 1) * plan.chunk_slots[c] * collective.TILE_ELEMS]
                               for c in range(plan.nchunks)])
        cover += collective.scatter_owned(recv, rf.rf_pack_tile_map(plan, r), n, got)
    I, J = np.triu_indices(n)
    assert np.all(cover[I, J] == 1)
    e = float(np.linalg.norm(got[I, J] - ref[I, J]) / np.linalg.norm(ref[I, J]))
    print(f"[parity] packed G n={n} world={world} {prec}: rel-Frobenius {e:.3e}")
    assert e <= TOL[prec]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_reduce_scatter_world1_nccl_equals_dense_gram():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, p, m = 1500, 128, 1024
        rng = np.random.default_rng(7)
        Xd = torch.tensor(rng.standard_normal((n, p)) / math.sqrt(p), device="cuda").to(torch.bfloat16)
        Wd = torch.tensor(rng.standard_normal((m, p)), device="cuda").to(torch.bfloat16)
        rs = collective.GramReduceScatter(n, p, m, m, "sigmoid_half", "bf16", nchunks=4, max_sms=120)
        for _ in range(3):                          # epochs 1..3 reuse the counters and buffers
            recv = rs(Xd, Wd)
        torch.cuda.synchronize()
        per = [16 * (rs.plan.chunk_tile0[c + 1] - rs.plan.chunk_tile0[c]) for c in range(rs.plan.nchunks)]
        assert rs.sync.cpu().tolist() == [3 * x for x in per]
        G = rf.rf_gram(Xd, Wd, act="sigmoid_half", prec="bf16", out="upper")
        torch.cuda.synchronize()
        got = np.full((n, n), np.nan, dtype=np.float32)
        w = collective.scatter_owned(recv.cpu().numpy(), rs.owned_tiles(), n, got)
        I, J = np.triu_indices(n)
        assert w[I, J].all()
        assert np.array_equal(got[I, J], G.cpu().numpy()[I, J]), "packed path must equal the dense K4 bit for bit"
    finally:
        dist.destroy_process_group()
