"""Command line: topology ingestion, schedule cache,
plan inspection and a single-GPU run of any forest.

    python -m paper_2402_06787_b200 topology --nvswitch 8 [--multicast] | --nvml
    python -m paper_2402_06787_b200 schedule -t topo.json --collective allgather [-o s.json]
    python -m paper_2402_06787_b200 describe -s s.json
    python -m paper_2402_06787_b200 run -t topo.json --collective allreduce --mib 64 [--steps 20]
    python -m paper_2402_06787_b200 run -s schedule.json --collective allgather   # wire format in
    torchrun --nproc-per-node N -m paper_2402_06787_b200 run -t topo.json ...     # one rank per GPU

Exit codes follow the reference CLI (pkg/src/collsched/cli.py:8-10): 0 ok,
1 usage, 2 invalid input, 3 schedule failed validation.
"""

from __future__ import annotations

import argparse
import json
import sys

from .errors import CollschedError, PlanError


def _load(path):
    with open(path) as f:
        return json.load(f)


def cmd_topology(a):
    from . import topology as T

    if a.nvml:
        doc = T.discover_nvml()
    elif a.groups:
        doc = T.groups_switch_doc(a.groups, n=a.n)
    else:
        doc = T.nvswitch_doc(a.nvswitch, multicast=a.multicast)
    text = json.dumps(doc, indent=2) + "\n"
    (open(a.output, "w").write(text) if a.output else sys.stdout.write(text))
    return 0


def cmd_schedule(a):
    from .generator import get_schedule
    from .schedule_io import export_json

    s = get_schedule(_load(a.topology), a.collective, prune=not a.no_prune)
    text = export_json(s)
    (open(a.output, "w").write(text) if a.output else sys.stdout.write(text))
    return 0


def cmd_describe(a):
    from .compiler import describe, lower
    from .schedule_io import load_schedule

    print(describe(lower(load_schedule(a.schedule))))
    return 0


def cmd_run(a):
    """Time one collective.  One process: every rank of the forest as virtual
    ranks on one GPU.  Under torchrun (WORLD_SIZE > 1): one rank per GPU over
    NVLink, the topology's compute count equal to the world size.  The forest
    comes from the topology (reference generate(), cached) or, with -s, from a
    schedule JSON in the reference wire format (parse_schedule)."""
    import os

    import torch

    from .executor import ForestCollComm, VirtualComm
    from .schedule_io import load_schedule

    doc = _load(a.topology) if a.topology else None
    schedules = {a.collective: load_schedule(a.schedule)} if a.schedule else None
    world = int(os.environ.get("WORLD_SIZE", "1"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        comm = ForestCollComm(doc, schedules=schedules, device=local)
        dev = torch.device(f"cuda:{local}")
    else:
        comm = VirtualComm(doc, schedules=schedules, device=a.device)
        dev = torch.device(f"cuda:{a.device}")
    n = comm.nranks
    M = a.mib << 20
    ranks = 1 if world > 1 else n  # buffers this process holds
    if a.collective == "allgather":
        S = M // n // 4
        ins = [torch.randn(S, device=dev) for _ in range(ranks)]
        outs = [torch.empty(n * S, device=dev) for _ in range(ranks)]
        fn = (lambda: comm.all_gather(outs[0], ins[0])) if world > 1 else (lambda: comm.all_gather(outs, ins))
    elif a.collective == "reduce_scatter":
        S = M // n // 4
        ins = [torch.randn(n * S, device=dev) for _ in range(ranks)]
        outs = [torch.empty(S, device=dev) for _ in range(ranks)]
        fn = (lambda: comm.reduce_scatter(outs[0], ins[0])) if world > 1 else (
            lambda: comm.reduce_scatter(outs, ins))
    else:
        bufs = [torch.randn(M // 4, device=dev) for _ in range(ranks)]
        fn = (lambda: comm.all_reduce(bufs[0])) if world > 1 else (lambda: comm.all_reduce(bufs))
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(a.steps):
        fn()
    t1.record()
    torch.cuda.synchronize()
    comm.check()
    ms = t0.elapsed_time(t1) / a.steps
    if dist is not None:
        x = torch.tensor([ms], device=dev)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        ms = float(x.item())
    rec = {"collective": a.collective, "ranks": n, "M_bytes": M, "ms": round(ms, 4),
           "algbw_GBps": round(M / ms / 1e6, 2), "info": comm.last_call_info(),
           "mode": (f"{n} ranks, one per GPU" if world > 1 else f"{n} virtual ranks on cuda:{a.device}")}
    if doc is not None:  # T* is a property of the declared graph
        rec["frac_of_t_star"] = round(comm.t_star(a.collective, M) * 1e3 / ms, 4)
    if dist is None or dist.get_rank() == 0:
        print(json.dumps(rec))
    comm.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2402_06787_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    t = sub.add_parser("topology")
    g = t.add_mutually_exclusive_group()
    g.add_argument("--nvswitch", type=int, default=8)
    g.add_argument("--groups", type=int, help="sparse two-group topology with bridge bandwidth beta")
    g.add_argument("--nvml", action="store_true")
    t.add_argument("--multicast", action="store_true")
    t.add_argument("-n", type=int, default=8, help="GPUs of the --groups topology (even, >= 4)")
    t.add_argument("-o", "--output")
    s = sub.add_parser("schedule")
    s.add_argument("-t", "--topology", required=True)
    s.add_argument("--collective", default="allgather",
                   choices=["allgather", "reduce_scatter", "allreduce"])
    s.add_argument("--no-prune", action="store_true")
    s.add_argument("-o", "--output")
    d = sub.add_parser("describe")
    d.add_argument("-s", "--schedule", required=True)
    r = sub.add_parser("run")
    r.add_argument("-t", "--topology", help="topology JSON (the reference format)")
    r.add_argument("-s", "--schedule", help="schedule JSON (reference wire format) to execute")
    r.add_argument("--collective", default="allgather",
                   choices=["allgather", "reduce_scatter", "allreduce"])
    r.add_argument("--mib", type=int, default=64)
    r.add_argument("--steps", type=int, default=20)
    r.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        return {"topology": cmd_topology, "schedule": cmd_schedule, "describe": cmd_describe,
                "run": cmd_run}[a.cmd](a)
    except PlanError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    except (CollschedError, OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
