#!/usr/bin/env python
"""Benchmark of the hot path: one step = the whole path of SURVEY.md §8(a) over one batch:
  G  : G1 (BF16: fp32 X, W rounded to bf16 on the device, rf_round_bf16) / K2 (3×TF32 split) → K3 Σᵀ = σ(X Wᵀ) → K4 upper-triangular SYRK G = ΣᵀΣ/m → (N>1) reduce-scatter of G
  Φ  : K1 row norms + Lemma-1 τ̂ (one 8-byte D2H) → Gauss–Hermite moments (host) → per-row
       coefficients → K5 fused XᵀX + EQ1 epilogue over the rank's upper-triangle rows.

Default workload: BASELINE.json configs[3] (p=1024, n=65536, m=65536, σ = sigmoid − ½, BF16) — the
config the metric's "1/2/4/8 B200" scaling is quoted on — with Φ evaluated on the same X.

  python bench.py [--gpus N --steps K --warmup W] [--config i --prec bf16|3xtf32|tf32|fp32]
  python bench.py --impl reference ...   (the fp64 CPU oracle as the reference arm)

Prints ONE JSON line on rank 0.  Timing: W untimed warm-ups, then K steps bracketed by barrier +
synchronize, CUDA events on the launching stream, max over ranks.  Inputs + workspaces are far larger
than the 126 MB L2 (no flush needed).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gram TFLOP/s and kernel entries/s at 1/2/4/8 B200; % of tensor-core peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--prec", default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-phi", action="store_true")
    ap.add_argument("--no-trf", action="store_true", help="skip the NEXT-1 ternary G^ter measurement")
    ap.add_argument("--no-phi4", action="store_true", help="skip the configs[4] Φ-only measurement")
    ap.add_argument("--phi4-n", type=int, default=0,
                    help="testing only: run the configs[4] Φ leg with this n (also on --same-gpu, where the full n "
                         "would not fit N dense Φ buffers on one GPU)")
    ap.add_argument("--g5", default="peers", choices=["peers", "nccl"],
                    help="N>1: G5 as the peer-memory exchange in K4's epilogue (default) or chunked NCCL reduce-scatter")
    ap.add_argument("--same-gpu", action="store_true",
                    help="testing only: every rank on cuda:0 with a gloo process group (peer G5 over CUDA IPC), so the "
                         "N>1 branch runs on a one-GPU box")
    return ap.parse_args()


def source_hash() -> str:
    """sha256 (12 hex digits) of the library's sources (csrc/* and include/rf.h): the key of the ncu DRAM-traffic
    records in profiles/ncu_traffic.json, so a kernel change can never be reported with stale bytes."""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2110_01899_b200", "csrc")
    for f in sorted(os.listdir(csrc)) + ["../../include/rf.h"]:
        path = os.path.normpath(os.path.join(csrc, f))
        if os.path.isfile(path):
            h.update(os.path.basename(path).encode())
            h.update(open(path, "rb").read())
    return h.hexdigest()[:12]


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: float(m[k]) for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    return p


def tf32_peak_tflops(device):
    """Dense TF32 tensor peak measured in this run (MEASURED_PEAKS has no TF32 entry): cuBLAS
    torch.matmul at 8192³ with TF32 allowed, best of 5 after warm-up.  Only a roofline denominator."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(8192, 8192, device=device)
        b = torch.randn(8192, 8192, device=device)
        for _ in range(3):
            a @ b
        best = float("inf")
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2.0 * 8192 ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def fp8_peak_tflops(device):
    """Dense FP8 (e4m3) tensor peak measured in this run for the TRF leg's fp8 SYRK roofline: cuBLASLt through
    torch._scaled_mm at 8192³ (row-major A, column-major B, unit scales), best of 5 after warm-up; None if the
    call is unavailable.  Only a roofline denominator."""
    import torch
    try:
        a = torch.randn(8192, 8192, device=device).to(torch.float8_e4m3fn)
        b = torch.randn(8192, 8192, device=device).to(torch.float8_e4m3fn).t()
        one = torch.ones((), device=device)
        for _ in range(3):
            torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
        best = float("inf")
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2.0 * 8192 ** 3 / (best * 1e-3) / 1e12
    except Exception:
        return None


def cores_used():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return os.cpu_count() or 1


# ------------------------------------------------------------------------------------------ oracle arm
def oracle_sample(cfg, size, seed=0):
    """Time the fp64 oracle on a principal sample S (|S| = size) of the workload: G_SS (needs σ(W x_i) for
    all m features, i ∈ S) and Φ_SS.  Returns (seconds, algorithmic flops of the sample)."""
    import numpy as np
    import oracle
    import synthetic
    rng = np.random.default_rng(seed)
    S = np.sort(rng.choice(cfg.n, size=size, replace=False))
    Xs = synthetic.make_X(cfg, rows=S)
    W = synthetic.make_W(cfg) if cfg.m else None
    t0 = time.perf_counter()
    flops = 0.0
    if cfg.m:
        oracle.gram(Xs, W, cfg.act)
        flops += 2.0 * cfg.m * size * cfg.p + cfg.m * size * (size + 1.0)
    oracle.phi_eq1(Xs, cfg.act, oracle.tau_hat(Xs))
    flops += cfg.p * size * (size + 1.0)
    return time.perf_counter() - t0, flops


# |S| of the oracle's principal sample per config (rows i ∈ S: G_SS over all m features + Φ_SS), shared by the
# reference arm and the cpu_baseline so the two time the same work; about 5-10 s of fp64 work on 16 host cores
ORACLE_SAMPLE = {0: 256, 1: 1024, 2: 2048, 3: 4096, 4: 4096}
ORACLE_SAMPLE_1T = {0: 256, 1: 512, 2: 1024, 3: 1024, 4: 1024}     # the single-thread leg (same work per entry)


def blas_threads(k):
    """Context manager limiting the BLAS pool (NumPy's matmul) to k threads (None: no limit)."""
    import contextlib
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=k, user_api="blas") if k else contextlib.nullcontext()
    except Exception:
        return contextlib.nullcontext()


def workload_flops(cfg, do_gram=True, do_phi=True):
    return ((2.0 * cfg.m * cfg.n * cfg.p + cfg.m * cfg.n * (cfg.n + 1.0)) if (cfg.m and do_gram) else 0.0) + \
        (cfg.p * cfg.n * (cfg.n + 1.0) if do_phi else 0.0)


def cpu_baseline_measure(cfg, cfg_idx):
    """The oracle as it stands (SURVEY.md §8(d) "Oracle timing"): fp64 NumPy on the host cores at all threads and at
    one thread, each on a principal sample of the workload, plus the full-matrix time extrapolated from the
    all-core rate (labelled as such: the oracle is never run at full size)."""
    S = ORACLE_SAMPLE[cfg_idx]
    S1 = ORACLE_SAMPLE_1T[cfg_idx]
    oracle_sample(cfg, 128)                                    # warm the caches / BLAS pool
    with blas_threads(None):
        t_all, f_all = oracle_sample(cfg, S, seed=1)
    with blas_threads(1):
        t_1, f_1 = oracle_sample(cfg, S1, seed=2)
    r_all, r_1 = f_all / t_all, f_1 / t_1
    full = workload_flops(cfg)
    return {"value": r_all / 1e12, "unit": "TFLOP/s", "cores": cores_used(), "kind": "oracle",
            "sample": f"|S|={S} random rows of configs[{cfg_idx}]: G_SS (σ(W x_i) over all m={cfg.m}) + Φ_SS by the "
                      f"18-term EQ1, fp64 NumPy, {t_all:.1f} s",
            "threads_all": {"value": r_all / 1e12, "threads": cores_used(), "seconds": t_all, "sample_rows": S},
            "threads_1": {"value": r_1 / 1e12, "threads": 1, "seconds": t_1, "sample_rows": S1},
            "extrapolated_full_s": full / r_all,
            "extrapolated_full_s_1thread": full / r_1,
            "extrapolation": "full-matrix oracle time = algorithmic flops of the whole workload / the measured rate "
                             "(an estimate: the oracle is only ever run on the sample)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synthetic
    cfg = synthetic.CONFIGS[args.config]
    size = ORACLE_SAMPLE[args.config]
    for _ in range(max(args.warmup, 0)):
        oracle_sample(cfg, 128)
    tot_t, tot_f = 0.0, 0.0
    for k in range(args.steps):
        t, f = oracle_sample(cfg, size, seed=k)
        tot_t += t
        tot_f += f
    v = tot_f / tot_t / 1e12
    sample = (f"|S|={size} random rows of configs[{args.config}] per step (the cpu_baseline sample): G_SS (σ(W x_i) "
              f"over all m) + Φ_SS, fp64 NumPy")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json configs)",
            "config": {"workload": f"configs[{args.config}] {cfg.name} (oracle sample)"},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores_used(), "kind": "oracle", "sample": sample,
                             "extrapolated_full_s": workload_flops(cfg) / (v * 1e12)},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ our arm
class ClockSampler:
    def __init__(self, gpus):
        self.proc = None
        self.path = os.path.join("/tmp", f"rf_clocks_{os.getpid()}.csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(str(g) for g in gpus),
                 "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    s, m = float(f[1]), float(f[2])
                except ValueError:
                    continue
                sm.append(s)
                mx.append(m)
                try:
                    pw.append(float(f[3]))
                except ValueError:
                    pass
                for nm, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        except Exception:
            return None
        if not sm:
            return None
        sm.sort()
        pw.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_min_mhz": sm[0], "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_median": pw[len(pw) // 2] if pw else None,
                "power_w_max": pw[-1] if pw else None}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2110_01899_b200 as rf
    import synthetic
    from paper_2110_01899_b200 import collective

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if args.same_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 with torch.distributed.run")
    if args.same_gpu and args.g5 != "peers":
        raise SystemExit("--same-gpu runs the peer G5 only (NCCL needs one GPU per rank)")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    gloo = args.same_gpu
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
    assert rf.rf_device_supported(local), "not an sm_100 device"

    cfg = synthetic.CONFIGS[args.config]
    prec = args.prec or cfg.modes[0]
    tdt = {"bf16": torch.bfloat16, "fp32": torch.float32, "3xtf32": torch.float32, "tf32": torch.float32,
           "fp64": torch.float64}[prec]
    do_gram = cfg.gram
    do_phi = (not args.no_phi)
    n, p, m = cfg.n, cfg.p, cfg.m
    stream = torch.cuda.current_stream()

    # ---------------- inputs (host → pinned → device); W sharded over m (rank r owns rows [m0, m1))
    # BF16 mode: the data are fp32 on the host and step G1 (rf_round_bf16, round to nearest even) runs on the
    # device inside every step, so the timed step covers all of §8(a); the other modes take their dtype as is.
    g1 = prec == "bf16"
    hdt = torch.float32 if g1 else tdt
    X_host = torch.from_numpy(synthetic.make_X(cfg)).to(hdt).pin_memory()
    X_in = X_host.to(device)
    Xd = torch.empty(X_in.shape, dtype=tdt, device=device) if g1 else X_in
    if g1:
        rf.rf_round_bf16(X_in, out=Xd)
    if do_gram:
        if m % world:
            raise SystemExit("m must be divisible by the number of GPUs")
        m_local = m // world
        m0 = rank * m_local
        W_host = torch.from_numpy(synthetic.make_W(cfg, rows=np.arange(m0, m0 + m_local))).to(hdt).pin_memory()
        W_in = W_host.to(device)
        Wd = torch.empty(W_in.shape, dtype=tdt, device=device) if g1 else W_in
        if g1:
            rf.rf_round_bf16(W_in, out=Wd)
        if world == 1:
            G = torch.empty((n, n), dtype=torch.float64 if prec == "fp64" else torch.float32, device=device)
            ws_g = torch.empty(rf.rf_gram_workspace_size(p, n, m_local, prec), dtype=torch.uint8, device=device)
            G_own = G
        else:
            # G5 inside the library's collective rf_gram: peers = K4's epilogue stores each owned tile into the
            # owner's staging buffer over NVLink (CUDA-IPC peer memory), device epoch flags order the owner-side sums;
            # nccl = packed send buffer + per-chunk counters + chunked reduce-scatter on the context's comm stream
            mode = args.g5 if prec in ("bf16", "tf32") else "nccl"
            rs = collective.GramCollective(n, p, m_local, m, cfg.act, prec, mode=mode, device=device)
            G_own = rs.recv
    if do_phi:
        rb, re_ = rf.rf_phi_row_split(n, world, rank)
        Phi = torch.empty((n, n), dtype=torch.float64 if prec == "fp64" else torch.float32, device=device)
        ws_p = torch.empty(rf.rf_phi_workspace_size(p, n, prec), dtype=torch.uint8, device=device)
    launches = [0]

    def round_inputs():
        k = 0
        if g1:
            rf.rf_round_bf16(X_in, out=Xd)
            k += rf.rf_last_launch_count()
            if do_gram:
                rf.rf_round_bf16(W_in, out=Wd)
                k += rf.rf_last_launch_count()
        return k

    def step():
        launches[0] += round_inputs()
        if do_gram:
            if world == 1:
                rf.rf_gram(Xd, Wd, act=cfg.act, prec=prec, out="upper", m_total=m, G=G, ws=ws_g)
            else:
                rs(Xd, Wd)
            launches[0] += rf.rf_last_launch_count()
        if do_phi:
            rf.rf_phi_closed_form(Xd, act=cfg.act, tau=0.0, prec=prec, out="upper", row_begin=rb, row_end=re_,
                                  Phi=Phi, ws=ws_p)
            launches[0] += rf.rf_last_launch_count()

    def barrier():
        if world > 1:
            dist.barrier() if gloo else dist.barrier(device_ids=[local])

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cpu" if gloo else device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    clocks = ClockSampler(list(range(world))) if rank == 0 else None
    time.sleep(0.3 if clocks else 0)
    rf.rf_profile_read()          # drop warm-up records
    rf.rf_profile_enable(True)
    launches[0] = 0
    torch.cuda.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    rf.rf_profile_enable(False)
    recs = rf.rf_profile_read()
    clk = clocks.stop() if clocks else None
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms / args.steps

    # ---------------- algorithmic work of one step (whole job)
    g_flops = (2.0 * m * n * p + m * n * (n + 1.0)) if do_gram else 0.0
    phi_flops = p * n * (n + 1.0) if do_phi else 0.0
    tri = n * (n + 1) / 2.0
    value = (g_flops + phi_flops) / (ms_step * 1e-3) / 1e12
    entries = ((tri if do_gram else 0) + (tri if do_phi else 0)) / (ms_step * 1e-3)

    # ---------------- per-kernel device times (rank-local launches)
    pk = peaks()
    kstat = {}
    for name, t in recs:
        s = kstat.setdefault(name, [0, 0.0])
        s[0] += 1
        s[1] += t
    rows_local = (re_ - rb) if do_phi else 0
    phi_entries_local = (sum(n - i for i in range(rb, re_)) if do_phi else 0)
    per_launch_alg = {
        "K3_gemm_sigma": ("tensor", 2.0 * (m // world if do_gram else 0) * n * p),
        "K4_syrk": ("tensor", (m // world if do_gram else 0) * n * (n + 1.0)),
        "K4_syrk_packed": ("tensor", (m // world if do_gram else 0) * n * (n + 1.0)),
        "K5_xtx_eq1": ("tensor", 2.0 * p * phi_entries_local),
    }
    tf32_like = prec in ("tf32", "3xtf32")
    peak_tensor = pk["bf16_tflops_sustained"] * (0.5 if tf32_like else 1.0)
    if tf32_like:
        pk["tf32_tflops_measured_burst"] = tf32_peak_tflops(device)
    kernels = {}
    for name, (cnt, tot) in kstat.items():
        avg = tot / cnt
        d = {"launches": cnt, "avg_ms": avg, "share_of_step": tot / ms}
        if name in per_launch_alg:
            kind, fl = per_launch_alg[name]
            d["achieved_tflops"] = fl / (avg * 1e-3) / 1e12
            d["frac_of_tensor_peak"] = d["achieved_tflops"] / peak_tensor
        if name == "K5_xtx_eq1":
            by = 4.0 * phi_entries_local + (2 if prec == "bf16" else 4) * n * p
            d["achieved_hbm_gbs"] = by / (avg * 1e-3) / 1e9
            d["frac_of_hbm_peak"] = d["achieved_hbm_gbs"] / pk["hbm_gbs"]
        kernels[name] = d
    dom = max(kernels, key=lambda k: kernels[k]["avg_ms"] * kernels[k]["launches"]) if kernels else None
    traffic, traffic_source = None, {"sources_sha": source_hash(), "record": None}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(traffic_source["sources_sha"], {})
        key = f"configs[{args.config}]:{prec}:w{world}:{dom}"
        traffic = tr.get(key)
        if traffic is not None:
            traffic_source["record"] = key
    except Exception:
        pass
    roof = None
    if dom in per_launch_alg:
        d = kernels[dom]
        roof = {"bound": "tensor", "kernel": dom, "achieved": d["achieved_tflops"], "peak": peak_tensor,
                "unit": "TFLOP/s", "frac": d["achieved_tflops"] / peak_tensor, "traffic": traffic,
                "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                "traffic_source": traffic_source,
                "peak_source": pk["source"] + (" sustained bf16" + (" × 0.5 (tf32 nominal ratio)" if tf32_like else "")),
                "frac_of_burst_peak": d["achieved_tflops"] / (pk["bf16_tflops"] * (0.5 if tf32_like else 1.0))}
        if tf32_like:
            roof["frac_of_measured_tf32_burst"] = d["achieved_tflops"] / pk["tf32_tflops_measured_burst"]

    # ---------------- e2e through the public API with host buffers.  Every step: H2D of X (and this rank's W) from
    # pinned memory, the step, and a D2H read of its results into pinned memory — G (world 1: the packed upper
    # triangle, RF_OUT_PACKED_TRI; world > 1: the rank's owned packed tiles) and the rank's rows of Φ (packed
    # triangle tile rows).  The D2H of step k runs on a copy stream while step k + 1 computes (device result
    # buffers double-buffered); the timed region ends when the last step's results are on the host.
    e2e = None
    if not args.no_e2e:
        h2d = X_host.numel() * X_host.element_size() + ((W_host.numel() * W_host.element_size()) if do_gram else 0)
        T = (n + 255) // 256
        tri_off = lambda I: 65536 * (I * T - I * (I - 1) // 2)   # noqa: E731  packed offset of tile row I
        packed = prec not in ("fp32", "fp64")            # the SIMT modes write dense n × n (include/rf.h)
        out_mode = "packed_tri" if packed else "upper"
        odt = torch.float64 if prec == "fp64" else torch.float32
        dev_bufs = [dict(), dict()]
        host = {}
        if do_gram:
            if world == 1:
                shp = (rf.rf_packed_tri_elems(n),) if packed else (n, n)
                for b in dev_bufs:
                    b["G"] = torch.empty(shp, dtype=odt, device=device)
                host["G"] = torch.empty(shp, dtype=odt, pin_memory=True)
            else:
                host["G"] = torch.empty(G_own.shape, dtype=torch.float32, pin_memory=True)
        if do_phi:
            po0, po1 = (tri_off(rb // 256), tri_off(-(-re_ // 256))) if packed else (rb, re_)
            for b in dev_bufs:
                b["P"] = torch.empty((rf.rf_packed_tri_elems(n),) if packed else (n, n), dtype=odt, device=device)
            host["P"] = torch.empty((po1 - po0,) if packed else (re_ - rb, n), dtype=odt, pin_memory=True)
        d2h = sum(h.numel() * h.element_size() for h in host.values())
        copy_stream = torch.cuda.Stream(device=device)
        done = [None, None]
        e2e_launches = [0]                               # D2H-finished event of each device buffer

        chunk = 64 << 20                                  # 256-MB D2H pieces: ≈ 56 GB/s vs ≈ 52 for one 8-GB copy

        def read_back(dst, src, after):
            copy_stream.wait_event(after)
            dst, src = dst.reshape(-1), src.reshape(-1)
            with torch.cuda.stream(copy_stream):
                for o in range(0, src.numel(), chunk):
                    dst[o:o + chunk].copy_(src[o:o + chunk], non_blocking=True)

        def e2e_step(k):
            # Φ first: its D2H starts ≈ 5 ms into the step and hides G's compute; G's D2H follows.
            b = dev_bufs[k & 1]
            if done[k & 1] is not None:
                stream.wait_event(done[k & 1])            # buffer k&1 is free once its previous D2H finished
            X_in.copy_(X_host, non_blocking=True)
            if do_gram:
                W_in.copy_(W_host, non_blocking=True)
            e2e_launches[0] += round_inputs()
            if do_phi:
                rf.rf_phi_closed_form(Xd, act=cfg.act, tau=0.0, prec=prec, out=out_mode, row_begin=rb,
                                      row_end=re_, Phi=b["P"], ws=ws_p)
                e2e_launches[0] += rf.rf_last_launch_count()
                ep = torch.cuda.Event()
                ep.record(stream)
                read_back(host["P"], b["P"][po0:po1], ep)
            if do_gram:
                if world == 1:
                    rf.rf_gram(Xd, Wd, act=cfg.act, prec=prec, out=out_mode, m_total=m, G=b["G"], ws=ws_g)
                else:
                    rs(Xd, Wd)
                e2e_launches[0] += rf.rf_last_launch_count()
                eg = torch.cuda.Event()
                eg.record(stream)
                read_back(host["G"], b["G"] if world == 1 else G_own, eg)
                if world > 1:
                    eg2 = torch.cuda.Event()
                    eg2.record(copy_stream)
                    stream.wait_event(eg2)                # the next rs() rewrites rs.recv
            ev = torch.cuda.Event()
            ev.record(copy_stream)
            done[k & 1] = ev

        e2e_step(0)
        e2e_step(1)
        torch.cuda.synchronize()
        barrier()
        e2e_launches[0] = 0
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for k in range(args.steps):
            e2e_step(k)
        stream.wait_stream(copy_stream)                   # the last step's results are on the host
        eb.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(ea.elapsed_time(eb))
        e2e = {"value": (g_flops + phi_flops) / (ems / args.steps * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
               "ms_per_step": ems / args.steps,
               "d2h_gbs": d2h / (ems / args.steps * 1e-3) / 1e9, "gpu_launches": e2e_launches[0],
               "layout": ("G and Φ read back as packed upper-triangle tiles (RF_OUT_PACKED_TRI)" if packed else
                          "G and Φ read back dense (the SIMT precision modes have no packed layout)")
                         + ", D2H of step k overlapped with step k+1 on a copy stream"}
        del dev_bufs, host

    # ---------------- NEXT-1 (Ternary Random Features) on the same shapes: reported beside the headline
    trf_line = None
    if do_gram and not args.no_trf:
        eps = 0.9
        T_host = torch.from_numpy(synthetic.make_T(cfg, eps, rows=np.arange(m0, m0 + m_local))).to(torch.bfloat16)
        Td = T_host.to(device)
        Xt = Xd if Xd.dtype == torch.bfloat16 else Xd.to(torch.bfloat16)   # TRF takes bf16 X (include/rf.h)
        tau_t = rf.rf_estimate_tau(Xt)
        sm, sp = rf.rf_trf_thresholds_for(cfg.act, tau_t)
        G_t = G if world == 1 and G.dtype == torch.float32 else torch.empty((n, n), dtype=torch.float32, device=device)
        ws_t = torch.empty(rf.rf_gram_ter_workspace_size(p, n, m_local), dtype=torch.uint8, device=device)
        for _ in range(args.warmup):
            rf.rf_gram_ter(Xt, Td, eps, sm, sp, m_total=m, G=G_t, ws=ws_t)
        torch.cuda.synchronize()
        barrier()
        rf.rf_profile_read()
        rf.rf_profile_enable(True)
        ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ta.record(stream)
        for _ in range(args.steps):
            rf.rf_gram_ter(Xt, Td, eps, sm, sp, m_total=m, G=G_t, ws=ws_t)
        tb.record(stream)
        torch.cuda.synchronize()
        rf.rf_profile_enable(False)
        trec = rf.rf_profile_read()
        tms = ta.elapsed_time(tb) / args.steps
        tk = {}
        for name, t in trec:
            tk.setdefault(name, []).append(t)
        k3t = sum(tk.get("K3_ter_features", [0])) / max(1, len(tk.get("K3_ter_features", [])))
        k4t = sum(tk.get("K4_ter_syrk", [0])) / max(1, len(tk.get("K4_ter_syrk", [])))
        fl_t = 2.0 * m_local * n * p + m_local * n * (n + 1.0)
        fp8_meas = fp8_peak_tflops(device)
        fp8_peak = fp8_meas if fp8_meas else 2.0 * pk["bf16_tflops"]
        trf_line = {"what": "G^ter (Algorithm 1 step 4) on the same X, W^ter sparsity eps=0.9, σ^ter matched to "
                            f"{cfg.act} at the Lemma-1 tau (s-={sm:.4f}, s+={sp:.4f}); per rank",
                    "ms_per_step": tms, "tflops": fl_t / (tms * 1e-3) / 1e12,
                    "K3_ter_ms": k3t, "K3_ter_tflops_bf16": 2.0 * m_local * n * p / (k3t * 1e-3) / 1e12 if k3t else None,
                    "K4_ter_ms": k4t, "K4_ter_tflops_fp8": m_local * n * (n + 1.0) / (k4t * 1e-3) / 1e12 if k4t else None,
                    "K4_ter_frac_fp8_peak": (m_local * n * (n + 1.0) / (k4t * 1e-3) / 1e12) / fp8_peak if k4t else None,
                    "fp8_peak": fp8_peak,
                    "fp8_peak_source": ("measured in this run: cuBLASLt fp8 e4m3 8192^3 (torch._scaled_mm), burst, "
                                        "random operands" if fp8_meas else
                                        "2 × measured burst bf16 (nominal fp8/bf16 ratio; _scaled_mm unavailable)"),
                    "K4_ter_frac_fp8_nominal_4500": (m_local * n * (n + 1.0) / (k4t * 1e-3) / 1e12) / 4500.0 if k4t else None,
                    "speedup_vs_gaussian_G": ((kernels.get("K3_gemm_sigma", {}).get("avg_ms", 0.0) +
                                               kernels.get("K4_syrk", {}).get("avg_ms", 0.0)) / (k3t + k4t)
                                              if (k3t + k4t) > 0 else None)}
        del Td, ws_t

    # ---------------- configs[4] (closed-form Φ only, p = 512, n = 131072): the HBM-write-heavy Φ pass the north star
    # reports in GB/s; rows split over ranks by equal triangle area, no collective.  Reported beside the headline.
    phi4_line = None
    # at N > 1 every rank runs its row block (rf_phi_row_split) and the time is the max over ranks (not on --same-gpu:
    # N dense 68.7-GB Φ buffers on one GPU)
    if (args.config == 3 or args.phi4_n > 0) and not args.no_phi4 and (not args.same_gpu or args.phi4_n > 0):
        if do_phi:
            del Phi, ws_p
        if do_gram and world == 1:   # (N > 1: the collective's receive buffer is G_own)
            del G, ws_g
        torch.cuda.empty_cache()
        c4 = synthetic.CONFIGS[4]
        n4, p4 = (args.phi4_n or c4.n), c4.p
        X4f = torch.from_numpy(synthetic.make_X(c4, n=n4) if args.phi4_n else synthetic.make_X(c4)).to(torch.float32)
        X4f = X4f.to(device)
        Phi4 = torch.empty((n4, n4), dtype=torch.float32, device=device)
        tri4 = n4 * (n4 + 1) / 2.0
        rb4, re4 = rf.rf_phi_row_split(n4, world, rank)

        def phi4_mode(mode, steps):
            """Time rf_phi_closed_form at configs[4] in one precision mode (bf16-stored X is
            the headline; TF32 / 3×TF32 on fp32 X are reported alongside)."""
            X4 = X4f.to(torch.bfloat16) if mode == "bf16" else X4f
            ws4 = torch.empty(rf.rf_phi_workspace_size(p4, n4, mode), dtype=torch.uint8, device=device)
            tau4 = rf.rf_estimate_tau(X4)
            mom4 = rf.rf_moments(c4.act, tau4)
            def phi4_call():
                rf.rf_phi_closed_form(X4, act=c4.act, tau=tau4, mom=mom4, prec=mode, row_begin=rb4, row_end=re4,
                                      Phi=Phi4, ws=ws4)
            for _ in range(args.warmup):
                phi4_call()
            torch.cuda.synchronize()
            barrier()
            rf.rf_profile_read()
            rf.rf_profile_enable(True)
            pa, pb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            pa.record(stream)
            for _ in range(steps):
                phi4_call()
            pb.record(stream)
            torch.cuda.synchronize()
            barrier()
            rf.rf_profile_enable(False)
            ks = [t for nm, t in rf.rf_profile_read() if nm.startswith("K5")]
            k5ms = max_over_ranks(sum(ks) / max(1, len(ks)))
            pms = max_over_ranks(pa.elapsed_time(pb)) / steps
            by4 = 4.0 * tri4 + X4.numel() * X4.element_size() + 4.0 * n4    # Φ triangle + X + row norms
            d = {"ms_per_step": pms, "entries_per_s": tri4 / (pms * 1e-3),
                 "tflops": p4 * n4 * (n4 + 1.0) / (pms * 1e-3) / 1e12,
                 "K5_ms": k5ms, "K5_hbm_gbs": by4 / (k5ms * 1e-3) / 1e9 if k5ms else None,
                 "K5_frac_hbm": by4 / (k5ms * 1e-3) / 1e9 / (pk["hbm_gbs"] * world) if k5ms else None,
                 "K5_tflops": p4 * n4 * (n4 + 1.0) / (k5ms * 1e-3) / 1e12 if k5ms else None}
            if k5ms:
                # K5's two roofline floors (DESIGN.md §7 "K5's roofline"): the 2p-flop upper-triangle contraction on
                # the tensor pipe at the sustained rate of its dtype, and its compulsory bytes at the measured HBM
                # copy rate; at p = 512 the intensity 2p / 4 B = 256 flop/B is above the ridge, so the tensor floor
                # binds.  frac_roofline = max(floors) / K5 time.
                ptc = pk["bf16_tflops_sustained"] * (1.0 if mode == "bf16" else 0.5) / (3.0 if mode == "3xtf32" else 1.0)
                t_tc = p4 * n4 * (n4 + 1.0) / (ptc * 1e12) * 1e3 / world     # each rank: 1/world of the triangle
                t_hbm = by4 / (pk["hbm_gbs"] * 1e9) * 1e3 / world
                d.update({"K5_floor_tensor_ms": t_tc, "K5_floor_hbm_ms": t_hbm,
                          "K5_bound": "tensor" if t_tc >= t_hbm else "hbm",
                          "K5_frac_tensor_sustained": t_tc / k5ms,
                          "K5_frac_roofline": max(t_tc, t_hbm) / k5ms})
            del ws4
            return d

        phi4_line = {"what": f"configs[4] {c4.name}: Φ by EQ1, fp32 upper triangle; headline = bf16-stored X "
                             "(bf16 products exact in fp32)"
                             + (f"; {world} ranks, row blocks of equal triangle area, no collective, max over ranks; "
                                "K5 roofline floors are whole-job figures divided by the ranks" if world > 1 else ""),
                     **phi4_mode("bf16", args.steps)}
        if world == 1:
            phi4_line["tf32"] = phi4_mode("tf32", max(2, args.steps // 2))
            phi4_line["3xtf32"] = phi4_mode("3xtf32", max(2, args.steps // 2))
        del Phi4, X4f
        torch.cuda.empty_cache()

    # ---------------- CPU baseline (oracle, rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_measure(cfg, args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": prec if prec != "3xtf32" else "f32(3xtf32)",
            "data": "synthetic (seeded PCG64 draws of BASELINE.json configs; no dataset)",
            "config": {"workload": f"configs[{args.config}] {cfg.name}" + (" + Φ on the same X" if do_phi and do_gram else ""),
                       "p": p, "n": n, "m": m, "act": cfg.act, "prec": prec,
                       "parallelism": (f"G: W sharded over m ({world} ranks); G5 = "
                                       + ("K4 epilogue storing packed triangle tiles into the owners' buffers over "
                                          "NVLink peer memory + owner-side sum, ordered by device epoch flags"
                                          if args.g5 == "peers" else
                                          "chunked NCCL reduce-scatter of packed triangle tiles overlapped with K4")
                                       + (" [--same-gpu test run: all ranks on one GPU]" if args.same_gpu else "")
                                       + "; "
                                       f"Φ: row blocks, no collective") if world > 1 else "single GPU",
                       "inputs": ("fp32 X, W rounded to bf16 on the device every step (G1, rf_round_bf16)" if g1
                                  else f"{prec} X, W as given"),
                       "l2": "no flush: inputs/workspace/outputs per step ≫ 126 MB L2"},
            "entries_per_s": entries, "pct_tensor_peak_sustained": (roof or {}).get("frac"),
            "roofline": roof, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches[0], "clocks": clk, "peaks": pk, "trf": trf_line, "phi_configs4": phi4_line,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
