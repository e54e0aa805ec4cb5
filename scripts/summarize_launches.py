"""Summarise an ncu launch list (gpu__time_duration + DRAM bytes per launch) by kernel configuration.

  python scripts/summarize_launches.py gpurun_out/launches.csv > profiles/<round>/ncu_launches_summary.txt
"""
import collections
import csv
import io
import re
import sys


def short(name):
    if "tc_gemm_kernel" in name:
        epi = re.search(r"Epi(\w+)", name)
        cfg = re.search(r"TcCfg<([^>]*)>", name)
        return f"tc_gemm<{cfg.group(1) if cfg else ''}>,{epi.group(0) if epi else ''}"
    return name.split("(")[0][:60]


def main(path):
    lines = [l for l in open(path).read().splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    iname, imet, ival, iid, iunit = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID",
                                                          "Metric Unit"))
    per, names = collections.defaultdict(dict), {}
    for r in rows[1:]:
        per[r[iid]][r[imet]] = (float(r[ival].replace(",", "")), r[iunit])
        names[r[iid]] = r[iname]
    agg = collections.OrderedDict()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for i, d in per.items():
        a = agg.setdefault(short(names[i]), [0, 0.0, 0.0, 0.0])
        t, u = d["gpu__time_duration.sum"]
        a[0] += 1
        a[1] += t / 1e6 if u == "ns" else (t / 1e3 if u == "us" else t)
        for key, idx in (("dram__bytes_read.sum", 2), ("dram__bytes_write.sum", 3)):
            if key in d:
                v, u = d[key]
                a[idx] += v * scale.get(u, 1)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':60s} {'n':>3s} {'total ms':>10s} {'share':>6s} {'avg ms':>9s} {'DRAM rd GB/launch':>18s} "
          f"{'DRAM wr GB/launch':>18s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {a[0]:3d} {a[1]:10.3f} {100 * a[1] / tot:5.1f}% {a[1] / a[0]:9.3f} "
              f"{a[2] / a[0] / 1e9:18.3f} {a[3] / a[0] / 1e9:18.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
