"""Host-link probe: pinned D2H bandwidth of an 8-GB copy with the pinned buffer first-touched on each NUMA node's
CPUs (the GPU's own node vs the other), to see whether the e2e leg's read-back depends on host-memory placement.
Prints the GPU's NUMA affinity (nvidia-smi topo) and GB/s per placement (experiment, not product code)."""
import os
import subprocess
import sys
import time

import torch


def node_cpus():
    out = {}
    base = "/sys/devices/system/node"
    for d in sorted(os.listdir(base)) if os.path.isdir(base) else []:
        if d.startswith("node") and d[4:].isdigit():
            s = open(os.path.join(base, d, "cpulist")).read().strip()
            cpus = set()
            for part in s.split(","):
                if "-" in part:
                    a, b = part.split("-")
                    cpus.update(range(int(a), int(b) + 1))
                elif part:
                    cpus.add(int(part))
            out[int(d[4:])] = cpus
    return out


def main():
    print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout, flush=True)
    print("cpu count", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), flush=True)
    dev = torch.device("cuda", 0)
    nbytes = 8 << 30
    src = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    nodes = node_cpus()
    print("nodes", {k: len(v) for k, v in nodes.items()}, flush=True)
    allc = os.sched_getaffinity(0)
    for node, cpus in nodes.items():
        if not cpus:
            continue
        os.sched_setaffinity(0, cpus)
        dst = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ce = (256 << 20) // 4
            for off in range(0, src.numel(), ce):
                dst[off:off + ce].copy_(src[off:off + ce], non_blocking=True)
            torch.cuda.synchronize()
            gbs = nbytes / (time.perf_counter() - t0) / 1e9
            if rep:
                print(f"node {node}: D2H {gbs:.1f} GB/s", flush=True)
        del dst
        os.sched_setaffinity(0, allc)


if __name__ == "__main__":
    main()
