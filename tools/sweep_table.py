"""Markdown tables from tools/sweep.py JSONL (algbw GB/s per implementation).
    python tools/sweep_table.py profiles/r01_sweep_n4.jsonl"""
import json
import sys
from collections import defaultdict

IMPLS = ["forestcoll", "forestcoll_nvls", "nccl", "nccl_ring", "nccl_nvls"]


def fmt_size(b):
    for unit, s in (("GiB", 1 << 30), ("MiB", 1 << 20), ("KiB", 1 << 10)):
        if b >= s:
            v = b / s
            return f"{v:g} {unit}"
    return f"{b} B"


def main(path):
    rows = [json.loads(line) for line in open(path)]
    n = rows[0]["n"]
    t = defaultdict(dict)
    for r in rows:
        t[(r["collective"], r["dtype"], r["M_bytes"])][r["impl"]] = r
    print(f"N={n}: algbw GB/s (frac of T* for forestcoll); best NCCL variant marked\n")
    print("| collective | dtype | M | forestcoll (proto) | frac T\\* | forest NVLS | NCCL default | NCCL Ring | NCCL NVLS | ours / best NCCL |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for k in sorted(t, key=lambda k: (k[0], k[1], k[2])):
        d = t[k]
        f = d.get("forestcoll")
        if not f:
            continue
        best = max((d[i]["algbw_GBps"] for i in IMPLS[2:] if i in d), default=None)
        cells = []
        for i in IMPLS[1:]:
            cells.append(f"{d[i]['algbw_GBps']:.1f}" if i in d else "—")
        ratio = f"{f['algbw_GBps'] / best:.2f}" if best else "—"
        print(f"| {k[0]} | {k[1]} | {fmt_size(k[2])} | {f['algbw_GBps']:.1f} ({f.get('proto', '')}) | "
              f"{f['frac_of_t_star']:.3f} | " + " | ".join(cells) + f" | {ratio} |")


if __name__ == "__main__":
    main(sys.argv[1])
