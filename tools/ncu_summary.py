"""Summarize ncu evidence for profiles/: `--set full` reports (per-kernel
duration, DRAM traffic, throughputs, occupancy) and a launch-list CSV
(kernel shares). Usage:
  python tools/ncu_summary.py full <report.ncu-rep> [label]
  python tools/ncu_summary.py launches <launches.csv>
  python tools/ncu_summary.py traffic <report.ncu-rep> <workload>   (-> profiles/ncu_traffic.json)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict

WANT = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 (LTS) %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
])
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1,
         "msecond": 1e3}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {}
        for k in ["Kernel Name"] + list(WANT):
            if k in hdr:
                i = hdr.index(k)
                v = r[i]
                u = units[i]
                if k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    v = float(v.replace(",", "")) * SCALE.get(u, 1)
                elif k == "gpu__time_duration.sum":
                    v = float(v.replace(",", "")) * SCALE.get(u, 1)  # -> microseconds
                d[k] = v
        yield d


def short(name):
    name = name.replace("void ", "")
    for ns in ("cclp_cu::", "(anonymous namespace)::", "<unnamed>::", "unnamed>::"):
        name = name.replace(ns, "")
    return name.split("(")[0]


def full(rep, label):
    print(f"### {label}: `ncu --set full` ({os.path.basename(rep)})\n")
    print("| kernel | " + " | ".join(WANT.values()) + " |")
    print("|---|" + "---|" * len(WANT))
    for d in raw_rows(rep):
        cells = []
        for k in WANT:
            v = d.get(k, "")
            if k == "gpu__time_duration.sum":
                v = f"{v:.1f} us"
            elif k.startswith("dram__bytes"):
                v = f"{v/1e6:.1f} MB"
            cells.append(str(v))
        print(f"| `{short(d['Kernel Name'])}` | " + " | ".join(cells) + " |")
    print()


def traffic(rep, workload):
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_traffic.json")
    try:
        data = json.load(open(path))
    except Exception:
        data = {}
    per = defaultdict(list)
    for d in raw_rows(rep):
        per[short(d["Kernel Name"]).split("<")[0]].append(
            d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"])
    data[workload] = {k: sum(v) / len(v) for k, v in per.items()}
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(data[workload], indent=1))


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        t = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += t
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | avg per launch (us) | share of all |")
    print("|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {t/c:.2f} | {100*t/tot:.1f}% |")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[2])
    elif mode == "launches":
        launches(sys.argv[2])
    elif mode == "traffic":
        traffic(sys.argv[2], sys.argv[3])
