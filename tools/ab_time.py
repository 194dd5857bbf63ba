"""A/B timing of one tree's executor (torchrun, N ranks): device time per call
for a list of (collective, MiB, dtype, proto) points.  Uses only the API
present in every round, so it runs in old checkouts too.

    torchrun --nproc-per-node N tools/ab_time.py ag:64:f32:-1 ar:25:bf16:-1 ar:25+1:bf16:-1 ...
(MiB+k: k extra elements per shard / buffer, for odd counts)
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402

MIB = 1 << 20
DT = {"f32": torch.float32, "bf16": torch.bfloat16}


def dev_time(fn, k):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(k):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    x = torch.tensor([e0.elapsed_time(e1) / k], device="cuda")
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return float(x.item())


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    for spec in sys.argv[1:]:
        coll, mib, dt, proto, *opts = spec.split(":")
        for o in opts:  # name=value options (absent in old trees: skipped there)
            k, v = o.split("=")
            try:
                comm.set_option(k, int(v))
            except Exception:  # noqa: BLE001
                pass
        mib, _, extra = mib.partition("+")  # "25+1": 25 MiB plus one element (odd counts)
        dt = DT[dt]
        es = torch.tensor([], dtype=dt).element_size()
        M = int(mib) * MIB + int(extra or 0) * es * (1 if coll == "ar" else n)
        comm.set_option("proto", int(proto))
        if coll == "ag":
            S = M // n // es
            inp = torch.randn(S, device=dev).to(dt)
            out = comm.empty(n * S, dtype=dt)
            fn = lambda: comm.all_gather(out, inp)  # noqa: E731
        elif coll == "rs":
            R = M // n // es
            inp = torch.randn(R * n, device=dev).to(dt)
            out = torch.empty(R, device=dev, dtype=dt)
            fn = lambda: comm.reduce_scatter(out, inp)  # noqa: E731
        else:
            buf = comm.empty(M // es, dtype=dt)
            buf.normal_()
            fn = lambda: comm.all_reduce(buf)  # noqa: E731
        k = max(5, min(200, int(0.03 / (20e-6 + M / 500e9))))
        ms = dev_time(fn, k)
        if rank == 0:
            print(f"{spec:32s} {ms * 1e3:9.1f} us  {M / ms / 1e6:8.1f} GB/s  proto={comm.last_call_info()['proto']}",
                  flush=True)
        for o in opts:
            k, _ = o.split("=")
            try:
                comm.set_option(k, {"ce_min": 24 << 20, "twohop_max": 12 << 20, "oneshot_ag_max": 16 << 20,
                                    "ctas_per_rank": 128, "ll_worker_warps": 4,
                                    "ll_chunk_max": 64 << 10, "lag": 64, "worker_warps": 8,
                                    "copy_mode": 1, "pdl": 1}.get(k, -1))
            except Exception:  # noqa: BLE001
                pass
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
