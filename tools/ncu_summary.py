"""Summarise ncu outputs into profiles/: the launch list (per-kernel share of
device time) and the key metrics of a `--set full` capture.

    python tools/ncu_summary.py LAUNCHES.csv REPORT.ncu-rep OUT_PREFIX [workload]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            d[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = []
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k[:120], "launches": len(v), "total_us": round(sum(v) / 1e3, 2),
                    "mean_us": round(sum(v) / len(v) / 1e3, 3), "share": round(sum(v) / tot, 4)})
    return out


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        rec = {"kernel": r[h.index("Kernel Name")][:120]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                rec[m] = f"{r[i]} {units[i]}".strip()
        res.append(rec)
    return res


def main():
    lpath, rpath, prefix = sys.argv[1:4]
    workload = sys.argv[4] if len(sys.argv) > 4 else None
    summary = {"launch_list": launches(lpath), "full_capture": full(rpath)}
    with open(prefix + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    if workload:
        cap = summary["full_capture"][0]

        def gb(s):
            v, u = s.split()
            return float(v) * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}[u]

        traffic = (gb(cap["dram__bytes_read.sum"]) + gb(cap["dram__bytes_write.sum"])) * 1e9
        try:
            tr = json.load(open("profiles/ncu_traffic.json"))
        except OSError:
            tr = {}
        tr[workload] = int(traffic)
        json.dump(tr, open("profiles/ncu_traffic.json", "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
