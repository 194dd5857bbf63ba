"""Summarise executor item traces (ForestCollComm/VirtualComm.read_trace()).

Per rank and task kind: items, mean wait / move time, and the busy fraction
of the workers over the traced launch window.
"""
from __future__ import annotations

import numpy as np

from paper_2402_06787_b200.compiler import KIND_NAMES


def report(rec: np.ndarray, plan, launch=None) -> str:
    if launch is not None:
        rec = rec[rec["launch"] == (launch & 0xFFFF)]
    if rec.size == 0:
        return "no records"
    lines = []
    t0 = rec["t_start"].min()
    t1 = rec["t_end"].max()
    span = (t1 - t0) / 1e3
    lines.append(f"window {span:.1f} us, {rec.size} items")
    for r in np.unique(rec["rank"]):
        rr = rec[rec["rank"] == r]
        workers = np.unique(rr["worker"]).size
        busy = (rr["t_end"] - rr["t_start"]).sum() / 1e3
        wait = rr["t_wait"].sum() / 1e3
        first = (rr["t_start"].min() - t0) / 1e3
        last = (rr["t_end"].max() - t0) / 1e3
        lines.append(f" rank {r}: {rr.size} items, {workers} workers, span {first:.1f}..{last:.1f} us, "
                     f"busy {busy / max(workers, 1) / span:.2f}, waiting {wait / max(busy, 1e-9):.2f} of busy")
        tasks = plan.tasks[int(r)]
        for ti in np.unique(rr["task"]):
            x = rr[rr["task"] == ti]
            kind = KIND_NAMES[tasks[int(ti)].kind]
            dur = (x["t_end"] - x["t_start"]) / 1e3
            pub = dur - x["t_wait"] / 1e3 - x["t_move"] / 1e3
            lines.append(f"    task {ti:2d} {kind:8s} tree {tasks[int(ti)].tree:2d} n={x.size:4d} "
                         f"mean {dur.mean():7.2f} us (wait {x['t_wait'].mean() / 1e3:6.2f} "
                         f"move {x['t_move'].mean() / 1e3:6.2f} pub {pub.mean():5.2f}) "
                         f"first {(x['t_start'].min() - t0) / 1e3:7.1f} last {(x['t_end'].max() - t0) / 1e3:7.1f}")
    return "\n".join(lines)
