"""GPU tests of the peer-memory G5 across PROCESSES (include/rf.h "G5", collective.GramCollective): two processes share
the one GPU of the box, each attaches its context as rank r of 2, and the 64-byte CUDA IPC handles of the staging
buffers are exchanged over a gloo process group (construction only).  Each call is the collective rf_gram: K4 of
rank s stores its tiles into rank o's staging buffer through the IPC mapping, and the device epoch flags (written
across the processes) order the sums — no host barrier or synchronize inside the calls.  No kernel waits on another:
the cross-process waits are stream-memory waits.  Before the context is created each process allocates and frees a
large tensor, so the caching allocator's blocks do not coincide with the staging buffer (the library owns it:
one cudaMalloc, the handle names exactly it).  Also: bench.py's N>1 branch, run as 2 processes on the one GPU.
"""
import json
import math
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


def _worker(rank, world, port, n, p, m, calls, q):
    import torch.distributed as dist
    import oracle
    from paper_2110_01899_b200 import collective
    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        junk = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")     # occupy, then free, a large block
        del junk
        X, W = _inputs(n, p, m)
        m0, m1 = collective.feature_shard(m, world, rank)
        Xd = torch.tensor(X, device="cuda").to(torch.bfloat16)
        Wd = torch.tensor(W[m0:m1], device="cuda").to(torch.bfloat16)
        gc = collective.GramCollective(n, p, m1 - m0, m, "sigmoid_half", "bf16", mode="peers")
        res = []
        for _ in range(calls):                      # epochs 1..calls, no host synchronization in between
            res.append(gc(Xd, Wd).clone())
        torch.cuda.synchronize()
        same = all(torch.equal(r, res[0]) for r in res)
        got = np.full((n, n), np.nan)
        written = collective.scatter_owned(res[-1].cpu().numpy().astype(np.float64), gc.owned_tiles(), n, got)
        Xb = Xd.double().cpu().numpy()
        Wb = torch.tensor(W, device="cuda").to(torch.bfloat16).double().cpu().numpy()
        ref = oracle.gram(Xb, Wb, "sigmoid_half")
        e = float(np.linalg.norm(got[written] - ref[written]) / np.linalg.norm(ref[written]))
        dist.barrier()                               # the peer's kernels are done before the mappings go
        gc.close()
        q.put((rank, written, e, same))
    finally:
        dist.destroy_process_group()


def test_peers_two_processes_on_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n, p, m, world = 1100, 96, 768, 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, m, 3, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    cover = res[0][1].astype(int) + res[1][1].astype(int)
    I, J = np.triu_indices(n)
    assert np.all(cover[I, J] == 1)
    for rank, _, e, same in res:
        print(f"[parity] G5 peers rank {rank}/2 (two processes): rel-Frobenius {e:.3e}, 3 calls identical {same}")
        assert same
        assert e < 2e-3


def test_bench_two_ranks_on_one_gpu():
    """bench.py's N > 1 branch (feature-sharded G with the peer-memory G5, row-block Φ) as 2 processes sharing GPU 0
    over gloo (--same-gpu: the device map for this one-GPU box), so a driver scaling run is not that code's first.
    configs[1] in TF32 (n = 4096): below the multicast hybrids' thresholds, because two processes on one GPU are
    time-sliced and the 4-CTA multicast kernels can hang under that preemption (DESIGN.md §9,
    scripts/timeslice_probe.py; pair kernels never did).  The hybrids' packed G5 is covered by the emulated ranks of
    test_gpu_packed.py (one process, no time-slicing)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--config", "1", "--prec", "tf32", "--same-gpu",
           "--phi4-n", "8192", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, "rank 0 prints exactly one JSON line"
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "G5_pack_reduce" in d["kernels"]
    assert d["trf"]["ms_per_step"] > 0                 # the NEXT-1 leg's N > 1 branch
    # the configs[4]-shaped Φ leg in its N > 1 form (row blocks, max over ranks), at a reduced n
    assert d["phi_configs4"]["K5_ms"] > 0 and d["phi_configs4"]["entries_per_s"] > 0
