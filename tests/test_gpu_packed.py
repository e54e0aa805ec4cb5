"""GPU tests of the multi-GPU G (include/rf.h "G5"): the collective rf_gram(ctx, …, RF_OUT_PACKED_TILES).

* Emulated ranks on ONE GPU: R contexts in this process, each attached as rank r of R with its own staging buffer,
  connected by raw device pointers (rf_ctx_connect_peers).  The exchange is the real one: K4's epilogue stores every
  tile into its owner's staging buffer, one-thread kernels write the device epoch flags with system-scope release,
  stream-memory waits order the owner-side sums and the next call's stores.  On one GPU in one process the ranks'
  streams may share a hardware queue, so a wait could head a queue its producer sits behind: the emulation enqueues
  each call in its two halves (RF_OPT_G5_PHASES test hook: phase 1 of every rank, then phase 2 of every rank) on one
  stream, where every wait's producer is already ahead of it; or (piped) each call has one rank t run the whole
  pipelined call — per-chunk arrival flags and per-chunk owner-side sums on its context's comm / reduce streams beside
  its K4 — after the others' first halves.  No kernel ever waits on another.  Three calls in a row (epochs 1..3) are
  bit-identical, and the summed owned tiles match the fp64 oracle G of the full W.
* world 1, peers and NCCL (the library's own communicator from rf_nccl_get_unique_id): the packed tiles equal the
  dense K4 bit for bit, in BF16, TF32 and (NCCL) 3×TF32, and the NCCL chunk counters K4 publishes reach their
  per-epoch targets.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_2110_01899_b200 as rf  # noqa: E402
from paper_2110_01899_b200 import collective  # noqa: E402
from entry_bounds import check, gram_bound  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {"3xtf32": 1e-5, "tf32": 2e-3, "bf16": 2e-3}
DT = {"3xtf32": torch.float32, "tf32": torch.float32, "bf16": torch.bfloat16}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    assert rf.rf_device_supported(0), "device 0 is not sm_100"
    torch.cuda.set_device(0)
    yield


def _emulated(n, p, m, world, prec, act, calls=3, seed=0, piped=False):
    rng = np.random.default_rng(seed + n + world)
    Xd = torch.tensor(rng.standard_normal((n, p)) / math.sqrt(p), device="cuda").to(DT[prec])
    Wd = torch.tensor(rng.standard_normal((m, p)), device="cuda").to(DT[prec])
    ctxs = [rf.Context(0) for _ in range(world)]
    for r, c in enumerate(ctxs):
        c.attach_peers(r, world, n)
    bases = [c.peer_base() for c in ctxs]
    for c in ctxs:
        c.connect_peers(bases)
    shards = [Wd[slice(*collective.feature_shard(m, world, r))].contiguous() for r in range(world)]
    recvs = [torch.full((len(rf.rf_tile_map(n, world, r)) * collective.TILE_ELEMS,), float("nan"), device="cuda")
             for r in range(world)]
    torch.cuda.synchronize()
    outs = []

    def go(r, phase):
        ctxs[r].set_option("g5_phases", phase)
        rf.rf_gram(Xd, shards[r], act=act, prec=prec, out="packed_tiles", m_total=m, G=recvs[r], ctx=ctxs[r])

    for call in range(calls):
        if not piped:
            for phase in (1, 2):     # no host synchronization between the halves or between calls
                for r in range(world):
                    go(r, phase)
        else:
            # rank t arrives last and runs the whole pipelined call (phases 3: its per-chunk arrival flags and
            # owner-side sums on the context's comm / reduce streams beside its K4); the others run their halves
            # around it, each half after the previous has finished (one GPU: no wait may head its producer's queue)
            t = call % world
            for r in range(world):
                if r != t:
                    go(r, 1)
                    torch.cuda.synchronize()
            go(t, 3)
            torch.cuda.synchronize()
            for r in range(world):
                if r != t:
                    go(r, 2)
        torch.cuda.synchronize()
        outs.append([x.cpu().numpy().copy() for x in recvs])
    for c in ctxs:
        c.destroy()
    return Xd, Wd, outs


@pytest.mark.parametrize("n,p,m,world,prec,act,piped", [
    (600, 64, 384, 2, "bf16", "tanh", False),         # ragged n (not a multiple of 256 / 512)
    (1024, 96, 512, 3, "bf16", "erf", False),         # tile multiple, world not a power of two
    (2100, 128, 640, 4, "tf32", "sigmoid_half", False),
    (17000, 64, 256, 2, "bf16", "sigmoid_half", False),   # ≥ 64 row tiles: K4's multicast + pair hybrid, packed tiles
    (1024, 96, 512, 3, "bf16", "erf", True),          # the pipelined call (per-chunk flags and sums), each rank last
    (17000, 64, 256, 3, "bf16", "sigmoid_half", True),    # … with the hybrid K4 and all 16 chunks
])
def test_peer_exchange_emulated_ranks(n, p, m, world, prec, act, piped):
    Xd, Wd, outs = _emulated(n, p, m, world, prec, act, piped=piped)
    for k in range(1, len(outs)):
        for r in range(world):
            assert np.array_equal(outs[k][r], outs[0][r]), f"call {k + 1} differs from call 1 on rank {r}"
    Xo, Wo = Xd.double().cpu().numpy(), Wd.double().cpu().numpy()
    S = np.arange(n) if n <= 2100 else collective_sample(n)
    ref = oracle.gram(Xo[S], Wo, act)
    pos = -np.ones(n, dtype=np.int64)
    pos[S] = np.arange(len(S))
    got = np.full((len(S), len(S)), np.nan)
    cover = np.zeros((len(S), len(S)), dtype=int)
    T = collective.RF_PACK_TILE
    for r in range(world):
        for k, (I, J) in enumerate(rf.rf_tile_map(n, world, r)):
            if I < 0:
                continue
            tile = outs[0][r][k * collective.TILE_ELEMS:(k + 1) * collective.TILE_ELEMS].reshape(T, T)
            rows = S[(S >= I * T) & (S < (I + 1) * T)]
            cols = S[(S >= J * T) & (S < (J + 1) * T)]
            for i in rows:
                js = cols[cols >= i]
                got[pos[i], pos[js]] = tile[i - I * T, js - J * T]
                cover[pos[i], pos[js]] += 1
    iu = np.triu_indices(len(S))
    assert np.all(cover[iu] == 1)
    e = float(np.linalg.norm(got[iu] - ref[iu]) / np.linalg.norm(ref[iu]))
    print(f"[parity] G5 peers emulated n={n} world={world} {prec}: rel-Frobenius {e:.3e}")
    assert e <= TOL[prec]
    check(f"G5 peers n={n} world={world} {prec}", got[iu], ref[iu], gram_bound(prec, act, Xo[S], Wo, ref, *iu))


def collective_sample(n):
    import synthetic
    return synthetic.sample_indices(n, count=200, tile_stride=512)


def _dense_vs_packed(ctx, n, p, m, prec, act, calls=2):
    rng = np.random.default_rng(7)
    Xd = torch.tensor(rng.standard_normal((n, p)) / math.sqrt(p), device="cuda").to(DT[prec])
    Wd = torch.tensor(rng.standard_normal((m, p)), device="cuda").to(DT[prec])
    for _ in range(calls):
        recv = rf.rf_gram(Xd, Wd, act=act, prec=prec, out="packed_tiles", ctx=ctx)
    G = rf.rf_gram(Xd, Wd, act=act, prec=prec, out="upper", ctx=ctx)
    torch.cuda.synchronize()
    got = np.full((n, n), np.nan, dtype=np.float32)
    w = collective.scatter_owned(recv.cpu().numpy(), rf.rf_tile_map(n, 1, 0), n, got)
    I, J = np.triu_indices(n)
    assert w[I, J].all()
    assert np.array_equal(got[I, J], G.cpu().numpy()[I, J]), "packed tiles must equal the dense K4 bit for bit"


@pytest.mark.parametrize("prec,pipe", [("bf16", 1), ("tf32", 1), ("bf16", 0)])
def test_peers_world1_equals_dense(prec, pipe):
    """World-1 peers: the packed tiles equal the dense K4 bit for bit, with the per-chunk sums beside K4 (pipe 1, the
    default) or after it on the caller's stream (RF_OPT_G5_PIPE = 0)."""
    ctx = rf.Context(0)
    ctx.set_option("g5_pipe", pipe)
    ctx.attach_peers(0, 1, 1500)
    assert ctx.collective() == (0, 1, 2)
    _dense_vs_packed(ctx, 1500, 128, 1024, prec, "tanh", calls=3)
    ctx.destroy()


@pytest.mark.parametrize("prec", ["bf16", "tf32", "3xtf32"])
def test_nccl_world1_equals_dense(prec):
    ctx = rf.Context(0)
    ctx.init_nccl(rf.rf_nccl_get_unique_id(), 0, 1)
    assert ctx.collective() == (0, 1, 1)
    _dense_vs_packed(ctx, 1300, 96, 768, prec, "sigmoid_half", calls=3)
    ctx.destroy()


@pytest.mark.parametrize("mode", ["peers", "nccl"])
def test_world1_n_changes_between_calls(mode):
    """The per-chunk counter targets are running sums over the calls (not epoch × this call's tiles), so n may change
    between collective calls on one context."""
    ctx = rf.Context(0)
    if mode == "peers":
        ctx.attach_peers(0, 1, 1500)
    else:
        ctx.init_nccl(rf.rf_nccl_get_unique_id(), 0, 1)
    for n in (1500, 700, 1300):
        _dense_vs_packed(ctx, n, 96, 512, "bf16", "tanh", calls=2)
    ctx.destroy()


def test_peers_world1_on_side_stream():
    """The pipelined call on a non-current stream: its comm / reduce streams order after the caller's stream, and the
    caller's stream after them (recv complete on `stream`)."""
    n, p, m = 1400, 64, 512
    rng = np.random.default_rng(11)
    Xd = torch.tensor(rng.standard_normal((n, p)) / math.sqrt(p), device="cuda").to(torch.bfloat16)
    Wd = torch.tensor(rng.standard_normal((m, p)), device="cuda").to(torch.bfloat16)
    ctx = rf.Context(0)
    ctx.attach_peers(0, 1, n)
    side = torch.cuda.Stream()
    recv = torch.full((len(rf.rf_tile_map(n, 1, 0)) * collective.TILE_ELEMS,), float("nan"), device="cuda")
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            rf.rf_gram(Xd, Wd, act="erf", out="packed_tiles", G=recv, stream=side, ctx=ctx)
        got_s = recv.clone()
    torch.cuda.current_stream().wait_stream(side)
    G = rf.rf_gram(Xd, Wd, act="erf", out="upper", ctx=ctx)
    torch.cuda.synchronize()
    got = np.full((n, n), np.nan, dtype=np.float32)
    w = collective.scatter_owned(got_s.cpu().numpy(), rf.rf_tile_map(n, 1, 0), n, got)
    I, J = np.triu_indices(n)
    assert w[I, J].all()
    assert np.array_equal(got[I, J], G.cpu().numpy()[I, J])
    ctx.destroy()


def test_collective_errors():
    ctx = rf.Context(0)
    X = torch.zeros((300, 64), dtype=torch.bfloat16, device="cuda")
    W = torch.zeros((128, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(rf.RFError):      # no collective attached
        rf.rf_gram(X, W, out="packed_tiles", ctx=ctx, G=torch.zeros(65536 * 4, device="cuda"))
    ctx.attach_peers(0, 2, 300)
    with pytest.raises(rf.RFError):      # attached but the peer is not connected
        rf.rf_gram(X, W, out="packed_tiles", ctx=ctx)
    with pytest.raises(rf.RFError):      # already attached
        ctx.attach_peers(0, 2, 300)
    ctx.connect_peers([ctx.peer_base(), ctx.peer_base()])
    with pytest.raises(rf.RFError):      # n above the n_max of the attach
        rf.rf_gram(torch.zeros((5000, 64), dtype=torch.bfloat16, device="cuda"), W, out="packed_tiles", ctx=ctx)
    with pytest.raises(rf.RFError):      # 3×TF32 reads tiles back: not over peers
        rf.rf_gram(X.float(), W.float(), prec="3xtf32", out="packed_tiles", ctx=ctx)
    ctx.destroy()
    with pytest.raises(rf.RFError):
        rf.Context(0).set_option("k5_wide", 7)


def test_peers_pipelined_timeline():
    """The pipelined call's launch timeline (rf_profile_timeline): one arrival-flag kernel and one owner-side sum per
    G5 chunk (C = min(16, ⌈T/8⌉) chunks of 8-row-tile groups), each chunk's sum starting after its flag, and the
    whole call's result equal to the dense K4."""
    n, p, m = 16400, 64, 256                   # 65 row tiles: the K4 multicast + pair hybrid, 9 chunks
    T = (n + 255) // 256
    C = min(16, (T + 7) // 8)
    rng = np.random.default_rng(3)
    Xd = torch.tensor(rng.standard_normal((n, p)) / math.sqrt(p), device="cuda").to(torch.bfloat16)
    Wd = torch.tensor(rng.standard_normal((m, p)), device="cuda").to(torch.bfloat16)
    ctx = rf.Context(0)
    ctx.attach_peers(0, 1, n)
    recv = rf.rf_gram(Xd, Wd, act="tanh", out="packed_tiles", ctx=ctx)
    torch.cuda.synchronize()
    rf.rf_profile_read()
    rf.rf_profile_enable(True)
    rf.rf_gram(Xd, Wd, act="tanh", out="packed_tiles", G=recv, ctx=ctx)
    torch.cuda.synchronize()
    rf.rf_profile_enable(False)
    tl = rf.rf_profile_timeline()
    sig = [t0 for nm, t0, _ in tl if nm == "G5_signal_arrived"]
    red = [t0 for nm, t0, _ in tl if nm == "G5_pack_reduce"]
    k4 = [t0 for nm, t0, _ in tl if nm.startswith("K4_syrk_packed")]
    assert len(sig) == C and len(red) == C and k4
    assert all(np.isfinite(v) and v >= 0 for _, v, _ in tl)
    for s_, r_ in zip(sorted(sig), sorted(red)):
        assert r_ >= s_ - 1e-3, "a chunk's sum started before its arrival flag"
    G = rf.rf_gram(Xd, Wd, act="tanh", out="upper", ctx=ctx)
    torch.cuda.synchronize()
    tiles = rf.rf_tile_map(n, 1, 0)
    TE = collective.TILE_ELEMS
    for k in list(range(0, len(tiles), max(1, len(tiles) // 40))) + [len(tiles) - 1]:   # sampled whole tiles
        I, J = (int(v) for v in tiles[k])
        if I < 0:
            continue
        i0, j0 = I * 256, J * 256
        i1, j1 = min(i0 + 256, n), min(j0 + 256, n)
        blk = recv[k * TE:(k + 1) * TE].view(256, 256)[: i1 - i0, : j1 - j0]
        ref = G[i0:i1, j0:j1]
        mask = torch.arange(j0, j1, device="cuda")[None, :] >= torch.arange(i0, i1, device="cuda")[:, None]
        assert torch.equal(blk[mask], ref[mask]), f"tile ({I}, {J}) differs from the dense K4"
    ctx.destroy()
