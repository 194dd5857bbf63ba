"""Calibrate the NVML NVLink byte counters against known traffic.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nvlink_probe.py

For NCCL's and ForestColl's allgather / reduce-scatter / allreduce at a few
sizes: NVLink TX / RX bytes per call on this rank's GPU (tools/
nvlink_counters.py) next to the algorithmic ingress (N-1)/N * M (AR: 2x).
"""

import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from tools.nvlink_counters import NvlinkCounters  # noqa: E402

MIB = 1 << 20


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    from paper_2402_06787_b200 import ForestCollComm

    comm = ForestCollComm(None, rank=rank, world_size=n, device=local)
    ctr = NvlinkCounters(local)
    if rank == 0:
        print(json.dumps({"counters": ctr.describe(), "links": ctr.links}), flush=True)

    def count(fn, reps):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        time.sleep(0.2)
        a = ctr.read()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        dist.barrier()
        time.sleep(0.2)
        b = ctr.read()
        if a is None or b is None:
            return None
        return {"tx_per_call": (b[0] - a[0]) / reps, "rx_per_call": (b[1] - a[1]) / reps,
                "ms_wall": el / reps * 1e3}

    rows = []
    for mib in (64, 1024):
        M = mib * MIB
        S = M // n // 4
        inp = torch.randn(S, device=dev)
        out = comm.empty(n * S, dtype=torch.float32)
        alg = (n - 1) * M // n
        reps = 20
        rows.append({"coll": "allgather", "impl": "nccl", "M": M, "alg_ingress": alg,
                     **(count(lambda: dist.all_gather_into_tensor(out, inp), reps) or {})})
        rows.append({"coll": "allgather", "impl": "forestcoll", "M": M, "alg_ingress": alg,
                     "proto": None, **(count(lambda: comm.all_gather(out, inp), reps) or {})})
        rows[-1]["proto"] = comm.last_call_info()["proto"]
        comm.deregister(out)
        del out
        R = M // n // 2
        rin = torch.randn(R * n, device=dev).to(torch.bfloat16)
        rout = torch.empty(R, device=dev, dtype=torch.bfloat16)
        rows.append({"coll": "reduce_scatter", "impl": "nccl", "M": M, "alg_ingress": alg,
                     **(count(lambda: dist.reduce_scatter_tensor(rout, rin), reps) or {})})
        rows.append({"coll": "reduce_scatter", "impl": "forestcoll", "M": M, "alg_ingress": alg,
                     **(count(lambda: comm.reduce_scatter(rout, rin), reps) or {})})
        rows[-1]["proto"] = comm.last_call_info()["proto"]
        buf = comm.empty(M // 2, dtype=torch.bfloat16)
        buf.normal_()
        rows.append({"coll": "allreduce", "impl": "nccl", "M": M, "alg_ingress": 2 * alg,
                     **(count(lambda: dist.all_reduce(buf), reps) or {})})
        rows.append({"coll": "allreduce", "impl": "forestcoll", "M": M, "alg_ingress": 2 * alg,
                     **(count(lambda: comm.all_reduce(buf), reps) or {})})
        rows[-1]["proto"] = comm.last_call_info()["proto"]
        comm.deregister(buf)
    for r in rows:
        if "tx_per_call" in r:
            r["tx_over_alg"] = round(r["tx_per_call"] / r["alg_ingress"], 4)
            r["rx_over_alg"] = round(r["rx_per_call"] / r["alg_ingress"], 4)
        r["rank"] = rank
    allrows = [None] * n
    dist.all_gather_object(allrows, rows)
    if rank == 0:
        for rr in allrows:
            for r in rr:
                print(json.dumps(r), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
