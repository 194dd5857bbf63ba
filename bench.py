"""Benchmark: ForestColl collectives executed by the B200-native forest kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Metric (BASELINE.json): collective algbw (GB/s, 1 GB = 1e9 B, M/T as in
nccl-tests) and the fraction of ForestColl's optimal time T* (SURVEY.md §8d).

* N >= 2 (one process per GPU, torchrun): allgather of M = 1 GiB total output
  on the nvswitch(N) forest (NVML-discovered topology, nominal fallback),
  inputs resident in HBM; NCCL all_gather_into_tensor on the same buffers
  and reduce-scatter / allreduce points are reported beside it.
* N = 1: the same kernel executes the 8-GPU NVSwitch forest (configs[0]'s
  topology) with all 8 ranks as virtual ranks on one B200 (HBM-bound; the
  per-rank "peer" stores land in local HBM), at M = 512 MiB per rank; the
  1-GPU local-copy sanity point and configs[0]'s 8 x 1 MiB case are attached.
* --impl reference: the CPU executor (oracle/, a restatement: the reference
  ships no executor) timed on the host on a bounded sample.

Timing: W warm-up steps, then K steps between a barrier + synchronize on both
sides, CUDA events on the launching stream, max over ranks.  Inputs are
larger than L2 (126 MB), so no flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

GIB = 1 << 30
MIB = 1 << 20
NVLINK_PEAK_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction (nominal 900)
NVLINK_NOMINAL_GBS = 900.0


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def hbm_peak():
    pk = measured_peaks()
    if "hbm_gbs" in pk:
        return float(pk["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(workload):
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "window": "1 s warm-up soak + timed region"}


# ---------------------------------------------------------------------------
# timing helpers
# ---------------------------------------------------------------------------
def timed(fn, steps, warmup, dist=None, soak_s=0.0):
    """Mean ms per step over `steps` calls (CUDA events on the current stream,
    barrier + synchronize on both sides, max over ranks).  `soak_s` adds an
    untimed warm-up soak of about that many seconds so clock sampling covers
    the kernel under steady load."""
    import torch

    for _ in range(warmup):
        fn()
    if soak_s > 0:
        torch.cuda.synchronize()
        t_end = time.perf_counter() + soak_s
        while time.perf_counter() < t_end:
            for _ in range(8):
                fn()
            torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(s)
    for _ in range(steps):
        fn()
    t1.record(s)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    if dist is not None:
        x = torch.tensor([ms], device="cuda")
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        ms = float(x.item())
    return ms


def pipelined_e2e(h_ins, h_outs, d_sets, collective, steps, warmup, dist=None):
    """End-to-end steps through the public API with host buffers: upload the
    step's inputs from pinned host memory, run the collective, download every
    output to pinned host memory.  Two device buffer sets alternate, so step
    i+1's uploads overlap step i's downloads (PCIe is full duplex) while each
    step still moves all of its bytes.  Returns ms per step (CUDA events,
    barrier + synchronize on both sides, max over ranks)."""
    import torch

    up, comp, down = torch.cuda.Stream(), torch.cuda.current_stream(), torch.cuda.Stream()
    ev_up = [torch.cuda.Event() for _ in d_sets]
    ev_comp = [torch.cuda.Event() for _ in d_sets]
    ev_down = [torch.cuda.Event() for _ in d_sets]
    for e in ev_comp + ev_down:
        e.record(comp)

    def step(i):
        k = i % len(d_sets)
        d_in, d_out = d_sets[k]
        up.wait_event(ev_comp[k])              # inputs of set k no longer read
        with torch.cuda.stream(up):
            for h, d in zip(h_ins, d_in):
                d.copy_(h, non_blocking=True)
        ev_up[k].record(up)
        comp.wait_event(ev_up[k])
        comp.wait_event(ev_down[k])            # outputs of set k already downloaded
        collective(d_out, d_in)
        ev_comp[k].record(comp)
        down.wait_event(ev_comp[k])
        with torch.cuda.stream(down):
            for h, d in zip(h_outs, d_out):
                h.copy_(d, non_blocking=True)
        ev_down[k].record(down)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(comp)
    for i in range(steps):
        step(warmup + i)
    comp.wait_stream(down)
    t1.record(comp)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    if dist is not None:
        x = torch.tensor([ms], device="cuda")
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        ms = float(x.item())
    return ms


def gbs(nbytes, ms):
    return nbytes / (ms * 1e-3) / 1e9


def cpu_allgather_timer(schedule, shard_bytes, threads=None):
    """The CPU restatement executor (oracle/forest_oracle.c, OpenMP over
    trees) on N host buffers; returns (seconds per call, threads, sample)."""
    import numpy as np

    from oracle import c_oracle

    threads = threads or os.cpu_count() or 1
    ff = c_oracle.FlatForest(schedule)
    n = ff.n
    S = shard_bytes // 4
    sends = [np.random.default_rng(r).standard_normal(S).astype(np.float32) for r in range(n)]
    recvs = [np.ones(n * S, dtype=np.float32) for _ in range(n)]  # first touch outside timing

    def step():
        c_oracle.allgather(ff, sends, recvs, threads)

    sample = (f"oracle/forest_oracle.c allgather of the nvswitch({n}) forest, {n} ranks x "
              f"{shard_bytes // MIB} MiB shards in host memory, OpenMP over trees")
    return step, threads, sample


def cpu_baseline_allgather(schedule, shard_bytes, budget_s=10.0):
    """Bounded CPU-baseline sample for the N=1 bench line (rank 0 only)."""
    step, threads, sample = cpu_allgather_timer(schedule, shard_bytes)
    step()
    reps, t0 = 0, time.perf_counter()
    while True:
        step()
        reps += 1
        el = time.perf_counter() - t0
        if el > budget_s or reps >= 2000:
            break
    per = el / reps
    M = schedule.num_compute * shard_bytes
    return {"value": round(gbs(M, per * 1e3), 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"{sample}; {reps} reps in {el:.1f}s (host os.cpu_count()={os.cpu_count()})"}


# ---------------------------------------------------------------------------
# N = 1: virtual ranks on one device
# ---------------------------------------------------------------------------
def plan_bytes_ag(plan, S_bytes):
    """HBM bytes one virtual-rank allgather must move (writes + reads)."""
    n = plan.nranks
    fwd_units = sum(t.mhi - t.mlo for v in range(n) for t in plan.tasks[v] if t.kind == 2)
    writes = n * n * S_bytes  # every rank's output, once
    reads = n * S_bytes + fwd_units * S_bytes // plan.k  # root inputs + forwarded slices
    return writes + reads


def run_single(args):
    import torch

    from paper_2402_06787_b200 import VirtualComm
    from paper_2402_06787_b200.topology import nvswitch_doc

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    n = 8
    comm = VirtualComm(nvswitch_doc(n), device=0)
    S_bytes = args.shard_mib * MIB
    S = S_bytes // 4
    M = n * S_bytes
    sends = [torch.randn(S, device=dev) for _ in range(n)]
    outs = [torch.empty(n * S, device=dev) for _ in range(n)]
    plan = comm.plan("allgather")
    fn = lambda: comm.all_gather(outs, sends)  # noqa: E731
    with Clocks(0) as clk:
        time.sleep(0.3)
        ms = timed(fn, args.steps, args.warmup, soak_s=1.0)
    comm.check()
    info = comm.last_call_info()
    tstar = comm.t_star("allgather", M)
    alg = gbs(M, ms)
    hbm_bytes = plan_bytes_ag(plan, S_bytes)
    peak, peak_kind = hbm_peak()
    achieved = gbs(hbm_bytes, ms)
    workload = f"nvs8-forest-allgather-virtual8-{args.shard_mib}MiBx8"

    # e2e through the public API: every rank's input uploaded from pinned host
    # memory, the collective, and rank 0's whole output read back.  In an
    # N-GPU job each rank's process reads its own output over its own PCIe
    # link; the 8 virtual ranks share one, so one rank's output is the
    # per-process read (downloading all 8 would time 8 links' traffic on one).
    host_in = [torch.empty(S, dtype=torch.float32, pin_memory=True).copy_(x.cpu()) for x in sends]
    host_out = [torch.empty(n * S, dtype=torch.float32, pin_memory=True)]
    d_sets = [(sends, outs), ([torch.empty_like(x) for x in sends], [torch.empty_like(x) for x in outs])]
    e2e_ms = pipelined_e2e(host_in, host_out, d_sets, lambda o, i: comm.all_gather(o, i),
                           max(3, min(args.steps, 10)), 2)
    assert torch.equal(host_out[0].view(n, S), torch.stack(host_in)), "e2e output mismatch"

    # configs[0] case (8 x 1 MiB fp32 shards) and the 1-GPU local-copy sanity point
    small_s = [torch.randn(MIB // 4, device=dev) for _ in range(n)]
    small_o = [torch.empty(n * MIB // 4, device=dev) for _ in range(n)]
    small_ms = timed(lambda: comm.all_gather(small_o, small_s), 50, 10)
    lc_src = torch.randn(S, device=dev)
    lc_dst = torch.empty(S, device=dev)
    from paper_2402_06787_b200 import executor as ex

    single = _local_copy_comm(ex, dev)
    lc_ms = timed(lambda: single.all_gather([lc_dst], [lc_src]), args.steps, args.warmup)

    line = {
        "metric": "collective algbw GB/s (ForestColl allgather, M = total output bytes per rank)",
        "value": round(alg, 2),
        "unit": "GB/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8 (fp32 payload, byte copy)",
        "data": "synthetic torch.randn fp32 shards",
        "config": {"workload": workload, "topology": "nvswitch(8) forest from collsched.generate",
                   "ranks": "8 virtual ranks on cuda:0", "M_bytes": M, "shard_bytes": S_bytes,
                   "l2": "inputs+outputs (4.5 GiB) larger than L2; no flush",
                   "chunks_per_tree": info["nchunks"], "ctas_per_rank": comm.get_option("ctas_per_rank"),
                   "path": info["proto"]},
        "t_star_ms_nvlink_model": round(tstar * 1e3, 4),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": hbm_bytes,
                     "traffic": ncu_traffic(workload)},
        "e2e": {"value": round(gbs(M, e2e_ms), 3), "unit": "GB/s",
                "h2d_bytes_per_step": n * S_bytes, "d2h_bytes_per_step": M,
                "ms_per_step": round(e2e_ms, 3),
                "what": "all 8 ranks' inputs uploaded, rank 0's output (M bytes) read back and "
                        "checked, every step",
                "pipelining": "two device buffer sets: step i+1 uploads overlap step i downloads"},
        "gpu_launches": args.steps * info["launches"],
        "clocks": clk.summary(),
        "configs0_8x1MiB": {"ms": round(small_ms, 4), "algbw_GBps": round(gbs(8 * MIB, small_ms), 2)},
        "local_copy_sanity": {"bytes": S_bytes, "ms": round(lc_ms, 4),
                              "hbm_GBps_rw": round(gbs(2 * S_bytes, lc_ms), 1)},
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_allgather(comm.schedule("allgather"), 16 * MIB)
        try:
            line["cpu_baseline"]["reference_generate"] = generate_timings()
        except Exception as exc:  # noqa: BLE001  (supplementary)
            line["cpu_baseline"]["reference_generate_error"] = f"{type(exc).__name__}: {exc}"[:200]
    comm.close()
    print(json.dumps(line), flush=True)


def _local_copy_comm(ex, dev):
    """1-rank forest (N=1 is outside the reference's API, topology.py:263-266):
    the root task copies send -> recv; the HBM sanity point."""
    from fractions import Fraction

    from paper_2402_06787_b200._refpath import require_collsched

    cs = require_collsched()
    RootTrees, Schedule, ScheduleBatch = cs.RootTrees, cs.Schedule, cs.ScheduleBatch

    s = Schedule(collective="allgather", num_compute=1, k=1, U=Fraction(1), y=Fraction(1),
                 inv_x_star=Fraction(0), roots=(RootTrees("g0", (ScheduleBatch(1, ()),)),))
    return ex.VirtualComm(schedules={"allgather": s}, device=dev.index)


# ---------------------------------------------------------------------------
# N >= 2: one process per GPU
# ---------------------------------------------------------------------------
def run_multi(args):
    import torch
    import torch.distributed as dist

    from paper_2402_06787_b200 import ForestCollComm
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(None, rank=rank, world_size=n, device=local)
    topo_kind = comm.topology_source
    M = args.msg_mib * MIB
    S = M // n // 4
    M = S * 4 * n
    inp = torch.randn(S, device=dev)
    out = comm.empty(n * S, dtype=torch.float32)
    fn = lambda: comm.all_gather(out, inp)  # noqa: E731
    with Clocks(local) as clk:
        time.sleep(0.3)
        ms = timed(fn, args.steps, args.warmup, dist, soak_s=1.0)
    comm.check()
    info = comm.last_call_info()
    tstar = comm.t_star("allgather", M)
    alg = gbs(M, ms)
    ingress = (n - 1) * M // n
    achieved = gbs(ingress, ms)
    # the SM kernel on the same call when the copy engine carried the headline
    sm_alt = None
    if info["proto"] == "ce":
        comm.set_option("ce_min", 0)
        ms_sm = timed(fn, args.steps, args.warmup, dist)
        sm_alt = {"path": comm.last_call_info()["proto"], "ms": round(ms_sm, 4),
                  "algbw_GBps": round(gbs(M, ms_sm), 2),
                  "frac_of_t_star": round(tstar * 1e3 / ms_sm, 4)}
        comm.set_option("ce_min", 24 << 20)
    # kernel-issued peer bytes of one call (the NVLink traffic evidence)
    issued, tinfo = issued_peer_bytes(comm, fn, dist)
    if tinfo and tinfo["proto"] == "ce":
        issued = S * 4 + 16  # one copy-engine transfer of the shard (+ two flag words)
    # NCCL on the same buffers
    nccl_out = torch.empty_like(out)
    nccl_ms = timed(lambda: dist.all_gather_into_tensor(nccl_out, inp), args.steps, args.warmup, dist)
    ok = bool(torch.equal(out, nccl_out))

    # e2e: pinned host input -> device, collective, output -> host
    h_in = torch.empty(S, pin_memory=True).copy_(inp.cpu())
    h_out = torch.empty(n * S, pin_memory=True)
    d_sets = [([inp], [out]), ([torch.empty_like(inp)], [comm.empty(n * S, dtype=torch.float32)])]
    e2e_ms = pipelined_e2e([h_in], [h_out], d_sets, lambda o, i: comm.all_gather(o[0], i[0]),
                           max(2, min(args.steps, 5)), 1, dist)
    assert torch.equal(h_out.view(n, S)[rank], h_in), "e2e output mismatch"

    extra = {}
    if not args.quick:
        try:
            extra = sweep_multi(comm, dist, n, dev, args)
        except Exception as exc:  # the sweep is supplementary: never lose the headline line
            extra = {"sweep_error": f"{type(exc).__name__}: {exc}"[:300]}
    if rank == 0:
        line = {
            "metric": "collective algbw GB/s (ForestColl allgather, M = total output bytes per rank)",
            "value": round(alg, 2),
            "unit": "GB/s",
            "n_gpus": n,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "u8 (fp32 payload, byte copy)",
            "data": "synthetic torch.randn fp32 shards",
            "config": {"workload": f"nvs{n}-forest-allgather-{args.msg_mib}MiB",
                       "topology": f"nvswitch({n}) from {topo_kind} ingestion, collsched forest",
                       "M_bytes": M, "shard_bytes": S * 4, "parallelism": f"{n} ranks, 1 per GPU",
                       "l2": "M larger than L2; no flush", "chunks_per_tree": info["nchunks"],
                       "path": info["proto"] + (" (copy engine moves each tree edge; SM kernels "
                                                "synchronise and place the own shard)"
                                                if info["proto"] == "ce" else ""),
                       "ctas_per_rank": comm.get_option("ctas_per_rank")},
            "frac_of_t_star": round(tstar * 1e3 / ms, 4),
            "t_star_ms": round(tstar * 1e3, 4),
            "busbw_GBps": round(alg * (n - 1) / n, 2),
            "roofline": {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_PEAK_GBS,
                         "unit": "GB/s", "frac": round(achieved / NVLINK_PEAK_GBS, 4),
                         "peak_kind": "fallback: B200_PROFILING.md measured peer copy per direction",
                         "nominal": NVLINK_NOMINAL_GBS,
                         "algorithmic_bytes_per_launch": ingress,
                         "traffic": None,
                         "traffic_note": ("NVML NVLink byte counters are NOT_SUPPORTED on this "
                                          "pool and ncu must not wrap a multi-rank run; "
                                          "issued_peer_bytes_per_launch is the executor's own "
                                          "count of bytes stored into peers (item trace)"),
                         "issued_peer_bytes_per_launch": issued,
                         "issued_over_algorithmic": round(issued / ingress, 4)},
            "e2e": {"value": round(gbs(M, e2e_ms), 3), "unit": "GB/s",
                    "h2d_bytes_per_step": S * 4, "d2h_bytes_per_step": M,
                    "ms_per_step": round(e2e_ms, 3),
                    "pipelining": "two device buffer sets: step i+1 uploads overlap step i downloads"},
            "gpu_launches": args.steps * info["launches"],
            "clocks": clk.summary(),
            "nccl": {"ms": round(nccl_ms, 4), "algbw_GBps": round(gbs(M, nccl_ms), 2),
                     "bitexact_vs_forestcoll": ok},
        }
        if sm_alt is not None:
            line["sm_kernel_path"] = sm_alt
        line.update(extra)
        print(json.dumps(line), flush=True)
    comm.close()
    dist.destroy_process_group()


def issued_peer_bytes(comm, fn, dist):
    """Bytes the kernels of one call store into other ranks' memory (payload,
    LL128 line tags, flag words), from the executor's item trace (the
    trace's per-item peer_bytes); max over ranks.  The copy-engine path runs
    no items: its bytes are the shard the copy engine moves.  NVML's NVLink
    byte counters are NOT_SUPPORTED on this pool (profiles/
    r02_nvlink_counters.md), so this software count stands in for them."""
    import torch

    info = None
    comm.enable_trace(1 << 20)
    try:
        comm.reset_trace()
        dist.barrier()
        torch.cuda.synchronize()
        fn()
        torch.cuda.synchronize()
        info = comm.last_call_info()
        rec = comm.read_trace()
        nb = int(rec["peer_bytes"].astype("int64").sum()) if rec.size else 0
    finally:
        comm.disable_trace()
    x = torch.tensor([nb], dtype=torch.int64, device="cuda")
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return int(x.item()), info


def nccl_group(dist, algo):
    """A separate NCCL communicator with NCCL_ALGO pinned (read at comm init)."""
    import torch

    old = os.environ.get("NCCL_ALGO")
    os.environ["NCCL_ALGO"] = algo
    try:
        g = dist.new_group(backend="nccl")
        x = torch.ones(1024, device="cuda")
        dist.all_reduce(x, group=g)  # create the communicator now, under this NCCL_ALGO
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("NCCL_ALGO", None)
        else:
            os.environ["NCCL_ALGO"] = old
    return g


def steps_for(M, floor):
    """>= ~25 ms of device time per measurement: short windows let host jitter
    (GC, page faults) drain the launch queue of small calls."""
    est = 20e-6 + M / 600e9
    return max(floor, min(2000, int(25e-3 / est)))


def sweep_multi(comm, dist, n, dev, args):
    import torch

    res = {"sweep": []}
    warm = 3
    groups = {"nccl": None}
    for algo in ("Ring", "NVLS"):  # NCCL ring and NVLS beside the default
        try:
            groups[f"nccl_{algo.lower()}"] = nccl_group(dist, algo)
        except Exception as exc:  # noqa: BLE001
            res[f"nccl_{algo.lower()}_error"] = f"{type(exc).__name__}: {exc}"[:200]

    def rec(coll, M, ms, dtype, fn_nccl, fn_ours=None):
        t = comm.t_star(coll, M)
        r = {"collective": coll, "M_bytes": M, "dtype": dtype, "ms": round(ms, 4),
             "algbw_GBps": round(gbs(M, ms), 2), "frac_of_t_star": round(t * 1e3 / ms, 4),
             "proto": comm.last_call_info()["proto"]}
        if fn_ours is not None and r["proto"] != "ce":
            alg = (n - 1) * M // n * (2 if coll == "allreduce" else 1)
            if r["proto"] == "oneshot":  # no item trace: LL128 lines of the input to every peer
                src = M // n if coll == "allgather" else M
                issued = -(-src // 120) * 128 * (n - 1)
            else:
                issued, _ = issued_peer_bytes(comm, fn_ours, dist)
            r["issued_peer_bytes"] = issued
            r["issued_over_algorithmic"] = round(issued / alg, 4)
        for name, g in groups.items():
            try:
                nm = timed(lambda: fn_nccl(g), steps_for(M, max(5, args.steps)), warm, dist)
                r[f"{name}_ms"] = round(nm, 4)
                r[f"{name}_algbw_GBps"] = round(gbs(M, nm), 2)
            except Exception as exc:  # noqa: BLE001
                r[f"{name}_error"] = f"{type(exc).__name__}: {exc}"[:120]
        res["sweep"].append(r)

    for mib in (1, 64, 1024):
        M = mib * MIB
        S = M // n // 4
        inp = torch.randn(S, device=dev)
        out = comm.empty(n * S, dtype=torch.float32)
        o2 = torch.empty_like(out)
        ms = timed(lambda: comm.all_gather(out, inp), steps_for(M, max(5, args.steps)), warm, dist)
        rec("allgather", S * 4 * n, ms, "float32",
            lambda g: dist.all_gather_into_tensor(o2, inp, group=g),
            lambda: comm.all_gather(out, inp))
        comm.deregister(out)
    for mib, dt in ((256, torch.float32), (256, torch.bfloat16)):
        M = mib * MIB
        R = M // n // torch.tensor([], dtype=dt).element_size()
        inp = torch.randn(R * n, device=dev).to(dt)
        out = torch.empty(R, device=dev, dtype=dt)
        ms = timed(lambda: comm.reduce_scatter(out, inp), steps_for(M, max(5, args.steps)), warm, dist)
        rec("reduce_scatter", M, ms, str(dt).split(".")[-1],
            lambda g: dist.reduce_scatter_tensor(out, inp, group=g),
            lambda: comm.reduce_scatter(out, inp))
    for mib in (25, 1024):
        M = mib * MIB
        cnt = M // 2
        buf = comm.empty(cnt, dtype=torch.bfloat16)
        buf.normal_()
        ms = timed(lambda: comm.all_reduce(buf), steps_for(M, max(5, args.steps)), warm, dist)
        rec("allreduce", M, ms, "bfloat16", lambda g: dist.all_reduce(buf, group=g),
            lambda: comm.all_reduce(buf))
        comm.deregister(buf)
    comm.check()
    try:
        res["nvls"] = nvls_points(dist, dev, n, args)
    except Exception as exc:
        res["nvls_error"] = f"{type(exc).__name__}: {exc}"[:300]
    if n in (4, 8):
        try:
            res["sparse_stress"] = sparse_stress(dist, dev, n, args)
        except Exception as exc:
            res["sparse_stress_error"] = f"{type(exc).__name__}: {exc}"[:300]
    return res


def nvls_points(dist, dev, n, args):
    """The forest pruned for a multicast/aggregation NVSwitch
    (schedule.py:237-306), executed by the NVLS engine: small allgathers as LL
    over multicast (one switch hop), allreduce with multimem.ld_reduce/st."""
    import torch

    from paper_2402_06787_b200 import ForestCollComm
    from paper_2402_06787_b200.topology import nvswitch_doc

    c = ForestCollComm(nvswitch_doc(n, multicast=True), rank=dist.get_rank(), world_size=n,
                       device=dev.index, scratch_bytes=64 << 20, nvls_bytes=1100 << 20,
                       reduction_order="switch")
    if not c.nvls_enabled:
        c.close()
        return {"skipped": "no NVSwitch multicast support"}
    out = []
    # small allgathers: LL over multicast (one switch hop), ordinary buffers
    for kib in (64, 1024):
        M = kib * 1024
        S = M // n // 4
        inp = torch.randn(S, device=dev)
        o = torch.empty(n * S, device=dev)
        ms = timed(lambda: c.all_gather(o, inp), steps_for(M, max(5, args.steps)), 3, dist)
        t = c.t_star("allgather", M)
        out.append({"collective": "allgather", "engine": c.last_call_info()["proto"],
                    "M_bytes": M, "dtype": "float32", "ms": round(ms, 4),
                    "algbw_GBps": round(gbs(M, ms), 2), "frac_of_t_star": round(t * 1e3 / ms, 4)})
    # tiny allreduce: LL multicast of every input + local in-tree evaluation
    M = 256 * 1024
    small = torch.randn(M // 2, device=dev).to(torch.bfloat16)
    ms = timed(lambda: c.all_reduce(small), steps_for(M, max(5, args.steps)), 3, dist)
    out.append({"collective": "allreduce", "engine": c.last_call_info()["proto"], "M_bytes": M,
                "dtype": "bfloat16", "ms": round(ms, 4), "algbw_GBps": round(gbs(M, ms), 2),
                "frac_of_t_star": round(c.t_star("allreduce", M) * 1e3 / ms, 4)})
    for mib in (25, 1000):
        M = mib * MIB
        buf = c.nvls_empty(M // 2, torch.bfloat16)
        buf.normal_()
        ms = timed(lambda: c.all_reduce(buf), steps_for(M, max(5, args.steps)), 3, dist)
        t = c.t_star("allreduce", M)
        out.append({"collective": "allreduce", "engine": c.last_call_info()["proto"],
                    "M_bytes": M, "dtype": "bfloat16", "ms": round(ms, 4),
                    "algbw_GBps": round(gbs(M, ms), 2), "frac_of_t_star": round(t * 1e3 / ms, 4)})
    c.check()
    c.close()
    return out


def sparse_stress(dist, dev, n, args):
    """BASELINE configs[4]: two groups of n/2 GPUs joined only by two bridge
    pairs (n = 8, and its 4-GPU analogue at n = 4).
    The forest is the reference's packing for that graph (k up to 3, paths
    through both switches and the bridges); it runs on the physical NVSwitch,
    so achieved bandwidth can exceed the declared graph's T* when the graph
    is slower than the box (small beta)."""
    import torch

    from paper_2402_06787_b200 import ForestCollComm
    from paper_2402_06787_b200.topology import groups_switch_doc

    out = []
    rank = dist.get_rank()
    for beta in (450, 300, 100):
        c = ForestCollComm(groups_switch_doc(beta, n=n), rank=rank, world_size=n,
                           device=dev.index, scratch_bytes=1 << 30)
        for coll in ("allgather", "allreduce"):
            M = args.msg_mib * MIB
            if coll == "allgather":
                S = M // n // 4
                inp = torch.randn(S, device=dev)
                o = c.empty(n * S, dtype=torch.float32)
                fn = lambda: c.all_gather(o, inp)  # noqa: E731
            else:
                o = c.empty(M // 2, dtype=torch.bfloat16)
                o.normal_()
                fn = lambda: c.all_reduce(o)  # noqa: E731
            ms = timed(fn, max(5, args.steps), 3, dist)
            t = c.t_star(coll, M)
            out.append({"topology": f"groups_switch({beta}, n={n})", "k": c.schedule(coll).k,
                        "collective": coll, "M_bytes": M, "ms": round(ms, 4),
                        "proto": c.last_call_info()["proto"],
                        "algbw_GBps": round(gbs(M, ms), 2), "graph_t_star_ms": round(t * 1e3, 4),
                        "frac_of_graph_t_star": round(t * 1e3 / ms, 4)})
            c.deregister(o)
            del o
        c.check()
        c.close()
    return out


# ---------------------------------------------------------------------------
# reference arm: CPU executor on the host
# ---------------------------------------------------------------------------
def generate_timings(reps=5):
    """Single-threaded wall time of the reference's own CPU path,
    ``collsched.generate()`` (pipeline.py:43-78; cli.py:4-6), per topology:
    parse_topology + bottleneck search + splitting + tree packing + pruning.
    SURVEY.md §8d(i) / BASELINE.md §4."""
    from paper_2402_06787_b200._refpath import require_collsched
    from paper_2402_06787_b200.topology import canonical_json, groups_switch_doc, nvswitch_doc

    cs = require_collsched()
    out = {}
    docs = [(f"nvswitch({n})", nvswitch_doc(n)) for n in (2, 4, 8)]
    docs += [(f"groups_switch({b})", groups_switch_doc(b)) for b in (450, 300, 100)]
    for name, doc in docs:
        text = canonical_json(doc)
        row = {}
        for coll in ("allgather", "reduce_scatter", "allreduce"):
            best = None
            for _ in range(reps):
                t0 = time.perf_counter()
                cs.generate(cs.parse_topology(text), coll)
                el = time.perf_counter() - t0
                best = el if best is None else min(best, el)
            row[coll] = round(best * 1e3, 3)
        out[name] = row
    return {"unit": "ms (min of %d, 1 thread)" % reps, "per_topology": out,
            "what": "collsched.generate(parse_topology(doc), collective) wall time"}


def run_reference(args):
    """The reference arm on the host: the reference's CPU data path for this
    workload.  The reference ships no executor, so
    its tree executor is the oracle's C restatement (oracle/forest_oracle.c,
    OpenMP over trees) run on the SAME workload as our arm: N=1 -> the
    nvswitch(8) forest, 8 ranks x --shard-mib shards; N>=2 -> the nvswitch(N)
    forest, M = --msg-mib total output.  The reference's own CPU path
    (collsched.generate) is timed beside it."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    from paper_2402_06787_b200.generator import get_schedule
    from paper_2402_06787_b200.topology import nvswitch_doc

    n = 8 if args.gpus <= 1 else args.gpus
    s = get_schedule(nvswitch_doc(n), "allgather", validate=False)
    if args.gpus <= 1:
        shard_bytes = args.shard_mib * MIB
        wl = f"nvs8-forest-allgather-virtual8-{args.shard_mib}MiBx8"
    else:
        shard_bytes = (args.msg_mib * MIB // n) // 4 * 4
        wl = f"nvs{n}-forest-allgather-{args.msg_mib}MiB"
    step, threads, sample = cpu_allgather_timer(s, shard_bytes)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = (time.perf_counter() - t0) / args.steps
    M = n * shard_bytes
    v = round(gbs(M, el * 1e3), 3)
    line = {
        "impl": "reference",
        "metric": "collective algbw GB/s (ForestColl allgather, M = total output bytes per rank)",
        "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(el * 1e3, 3), "higher_is_better": True,
        "scaling": "weak" if args.gpus <= 1 else "strong", "vs_baseline": None,
        "dtype": "u8 (fp32 payload, byte copy)", "data": "synthetic numpy fp32 shards",
        "config": {"workload": wl, "M_bytes": M, "shard_bytes": shard_bytes},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{sample}; the full workload every step (the reference ships "
                                   f"no executor; this is its CPU restatement; host "
                                   f"os.cpu_count()={os.cpu_count()})"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        line["cpu_baseline"]["reference_generate"] = generate_timings()
    except Exception as exc:  # noqa: BLE001  (supplementary)
        line["cpu_baseline"]["reference_generate_error"] = f"{type(exc).__name__}: {exc}"[:200]
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--msg-mib", type=int, default=1024, help="N>=2: allgather total output")
    ap.add_argument("--shard-mib", type=int, default=64, help="N=1: per virtual rank shard")
    ap.add_argument("--quick", action="store_true", help="skip the RS/AR/size sweep")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        run_multi(args)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
