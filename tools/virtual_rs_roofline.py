"""HBM roofline of the chunk-flag REDUCTION path on one B200 (virtual ranks).

    python tools/virtual_rs_roofline.py [--n 8] [--mib 64] [--dtype bfloat16] [--iters 20]

Runs the nvswitch(n) reduce-scatter forest with all n ranks as virtual ranks
on cuda:0 through the chunk-flag protocol (the large-message reduction path
of the multi-GPU executor: bulk (TMA) loads of the own slice and the
children's partials into the smem ring, fp32 accumulation in tree order,
16-byte stores to the parent's scratch).  Prints ms, the algorithmic HBM
bytes of one launch (plan_bytes_rs) and achieved GB/s against
MEASURED_PEAKS.json.  Used under `ncu --set full` for profiles/.
"""

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from bench import MIB, gbs, hbm_peak, timed  # noqa: E402
from paper_2402_06787_b200 import VirtualComm  # noqa: E402
from paper_2402_06787_b200 import compiler as C  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def plan_bytes_rs(plan, slice_unit_bytes):
    """HBM bytes one virtual-rank reduce-scatter moves: every task reads its
    own input slice and each child's partial; an rs_fwd task writes its
    partial into the parent's scratch, an rs_root task its output."""
    reads = writes = 0
    for v in range(plan.nranks):
        for t in plan.tasks[v]:
            if t.kind not in (C.K_RS_FWD, C.K_RS_ROOT):
                continue
            sl = slice_unit_bytes * (t.mhi - t.mlo)
            reads += sl * (1 + len(t.rs_children))
            writes += sl
    return reads + writes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--mib", type=int, default=64, help="output shard MiB per rank")
    ap.add_argument("--dtype", default="bfloat16")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--opt", action="append", default=[], help="option=value")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    n = args.n
    opts = {"proto": 0}
    for o in args.opt:
        k, v = o.split("=")
        opts[k] = int(v)
    comm = VirtualComm(nvswitch_doc(n), device=0, options=opts)
    dt = getattr(torch, args.dtype)
    es = torch.tensor([], dtype=dt).element_size()
    S = args.mib * MIB // es
    ins = [torch.randn(n * S, device=dev).to(dt) for _ in range(n)]
    outs = [torch.empty(S, device=dev, dtype=dt) for _ in range(n)]
    fn = lambda: comm.reduce_scatter(outs, ins)  # noqa: E731
    ms = timed(fn, args.iters, args.warmup)
    comm.check()
    plan = comm.plan("reduce_scatter")
    nbytes = plan_bytes_rs(plan, S * es // plan.k)
    peak, kind = hbm_peak()
    info = comm.last_call_info()
    print(json.dumps({"workload": f"nvs{n}-forest-reduce_scatter-virtual{n}-{args.dtype}-{args.mib}MiB",
                      "ms": round(ms, 4), "algorithmic_bytes_per_launch": nbytes,
                      "achieved_GBps": round(gbs(nbytes, ms), 1), "peak_GBps": peak,
                      "peak_kind": kind, "frac": round(gbs(nbytes, ms) / peak, 4),
                      "proto": info["proto"], "launches": info["launches"],
                      "grid": info["grid"], "options": opts}), flush=True)
    comm.close()


if __name__ == "__main__":
    main()
