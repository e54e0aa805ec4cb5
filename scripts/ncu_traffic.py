"""Turn an ncu launch list of one bench step into the DRAM-traffic records bench.py reports as `roofline.traffic`.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/traffic.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-trf --no-phi4 \
        --no-cpu-baseline
    python scripts/ncu_traffic.py gpurun_out/traffic.csv --config 3 --prec bf16 --world 1

Launches are attributed to the library's trace names by their epilogue type (EpiSigma → K3_gemm_sigma, EpiSyrk →
K4_syrk, EpiSyrkPacked → K4_syrk_packed, EpiEq1 → K5_xtx_eq1; the hybrid K3/K4 are two kernels per call, summed);
the bytes per call are those of the LAST call of each (the timed step, after the warm-up).  Records are keyed by the
sha256 of the library sources (bench.source_hash), so a kernel change leaves no stale record behind.
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KINDS = [("EpiSyrkPacked", "K4_syrk_packed"), ("EpiSyrk", "K4_syrk"), ("EpiSigma<", "K3_gemm_sigma"),
         ("EpiEq1", "K5_xtx_eq1")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--prec", default="bf16")
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--calls-per-step", type=int, default=1)
    a = ap.parse_args()
    import bench
    rows = [r for r in csv.reader(open(a.csv)) if r and r[0].isdigit()]
    # columns: ID, PID, Process, Host, Port?, Kernel Name, Context, Stream, Block, Grid, Device, CC, Section, Metric,
    # Unit, Value — find them from the header
    hdr = next(r for r in csv.reader(open(a.csv)) if r and r[0] == "ID")
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    launches = {}
    for r in rows:
        d = launches.setdefault(int(r[0]), {"name": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    per_kind = {}
    for lid in sorted(launches):
        d = launches[lid]
        for tag, kind in KINDS:
            if tag in d["name"]:
                by = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
                per_kind.setdefault(kind, []).append(by)
                break
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    allrec = json.load(open(out_path)) if os.path.exists(out_path) else {}
    allrec = {k: v for k, v in allrec.items() if not k.startswith("configs[")}   # drop the r01 config-keyed records
    sha = bench.source_hash()
    rec = allrec.setdefault(sha, {})
    for kind, bys in per_kind.items():
        parts = 2 if kind in ("K3_gemm_sigma", "K4_syrk", "K4_syrk_packed") and len(bys) % 2 == 0 else 1
        last = sum(bys[-parts:]) if len(bys) >= parts else sum(bys)
        rec[f"configs[{a.config}]:{a.prec}:w{a.world}:{kind}"] = int(last)
    rec["_source"] = f"{os.path.relpath(a.csv, ROOT)}: dram__bytes_read.sum + dram__bytes_write.sum of the last call"
    json.dump(allrec, open(out_path, "w"), indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
