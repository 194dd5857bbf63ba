"""Message-size sweep (BASELINE.json configs[1..3]): ForestColl forest kernel,
the NVLS engine on the multicast-pruned forest, and NCCL default / Ring / NVLS
on the same box, same buffers, same timing (bench.timed: CUDA events, barrier
+ synchronize on both sides, max over ranks).

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
      --master-addr 127.0.0.1 --master-port 29613 tools/sweep.py --out gpurun_out/sweep_nN.jsonl

M convention: AG M = output bytes, RS M = per-rank input
bytes, AR M = buffer bytes.  One JSON record per (collective, M, impl)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import gbs, nccl_group, steps_for, timed  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402

KIB, MIB = 1 << 10, 1 << 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.jsonl")
    ap.add_argument("--ag-max-mib", type=int, default=4096)
    ap.add_argument("--nvls-max-mib", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    pool = 2 * args.nvls_max_mib * MIB + 64 * MIB
    nv = ForestCollComm(nvswitch_doc(n, multicast=True), rank=rank, world_size=n, device=local,
                        scratch_bytes=64 << 20, nvls_bytes=pool, reduction_order="switch")
    groups = {"nccl": None}
    for algo in ("Ring", "NVLS"):
        try:
            groups[f"nccl_{algo.lower()}"] = nccl_group(dist, algo)
        except Exception as exc:  # noqa: BLE001
            if rank == 0:
                print(f"# NCCL_ALGO={algo} unavailable: {exc}", flush=True)
    recs = []

    def emit(coll, M, impl, ms, dtype, **kw):
        t = comm.t_star(coll, M) * 1e3
        r = {"n": n, "collective": coll, "M_bytes": M, "dtype": dtype, "impl": impl,
             "ms": round(ms, 5), "algbw_GBps": round(gbs(M, ms), 2),
             "frac_of_t_star": round(t / ms, 4), **kw}
        recs.append(r)
        if rank == 0:
            print(json.dumps(r), flush=True)

    def steps(M):
        return steps_for(M, args.iters)

    def run_nccl(coll, M, dtype, fn):
        for name, g in groups.items():
            try:
                ms = timed(lambda: fn(g), steps(M), 3, dist)
                emit(coll, M, name, ms, dtype)
            except Exception as exc:  # noqa: BLE001
                if rank == 0:
                    print(f"# {name} {coll} {M}: {type(exc).__name__}: {str(exc)[:120]}", flush=True)

    # --- allgather sweep 1 KiB .. ag_max (x2) ---
    M = KIB
    while M <= args.ag_max_mib * MIB:
        S = max(1, M // n // 4)
        Mb = S * 4 * n
        inp = torch.randn(S, device=dev)
        out = comm.empty(n * S)
        ms = timed(lambda: comm.all_gather(out, inp), steps(Mb), 3, dist)
        emit("allgather", Mb, "forestcoll", ms, "float32", proto=comm.last_call_info()["proto"])
        ref = out.clone()
        comm.deregister(out)
        del out
        if nv.nvls_enabled and Mb <= args.nvls_max_mib * MIB:
            nv._nvls_next = 0
            o3 = nv.nvls_empty(n * S)
            ms = timed(lambda: nv.all_gather(o3, inp), steps(Mb), 3, dist)
            assert torch.equal(o3, ref), "NVLS allgather mismatch"
            emit("allgather", Mb, "forestcoll_nvls", ms, "float32")
            del o3
        o2 = torch.empty(n * S, device=dev)
        run_nccl("allgather", Mb, "float32",
                 lambda g: dist.all_gather_into_tensor(o2, inp, group=g))
        assert torch.equal(o2, ref), "NCCL allgather differs from ours"
        del o2, inp, ref
        M *= 2
    comm.check()

    # --- reduce-scatter 256 MiB .. 4 GiB per rank, fp32 / bf16 ---
    for dt in (torch.float32, torch.bfloat16):
        es = torch.tensor([], dtype=dt).element_size()
        for mib in (256, 512, 1024, 2048, 4096):
            M = mib * MIB
            R = M // n // es
            inp = torch.randn(R * n, device=dev).to(dt)
            out = torch.empty(R, device=dev, dtype=dt)
            ms = timed(lambda: comm.reduce_scatter(out, inp), steps(M), 3, dist)
            emit("reduce_scatter", M, "forestcoll", ms, str(dt)[6:], proto=comm.last_call_info()["proto"])
            if nv.nvls_enabled and M <= args.nvls_max_mib * MIB:
                nv._nvls_next = 0
                i3 = nv.nvls_empty(R * n, dt)
                i3.copy_(inp)
                ms = timed(lambda: nv.reduce_scatter(out, i3), steps(M), 3, dist)
                emit("reduce_scatter", M, "forestcoll_nvls", ms, str(dt)[6:])
                del i3
            run_nccl("reduce_scatter", M, str(dt)[6:],
                     lambda g: dist.reduce_scatter_tensor(out, inp, group=g))
            del inp, out
    comm.check()

    # --- small reductions (bf16): tree engine vs NVLS LL multicast vs NCCL ---
    for kib in (64, 256, 1024, 4096):
        M = kib * KIB
        R = M // n // 2
        inp = torch.randn(R * n, device=dev).to(torch.bfloat16)
        out = torch.empty(R, device=dev, dtype=torch.bfloat16)
        ms = timed(lambda: comm.reduce_scatter(out, inp), steps(M), 3, dist)
        emit("reduce_scatter", M, "forestcoll", ms, "bfloat16", proto=comm.last_call_info()["proto"])
        if nv.nvls_enabled:
            ms = timed(lambda: nv.reduce_scatter(out, inp), steps(M), 3, dist)
            emit("reduce_scatter", M, "forestcoll_nvls", ms, "bfloat16", proto=nv.last_call_info()["proto"])
        run_nccl("reduce_scatter", M, "bfloat16", lambda g: dist.reduce_scatter_tensor(out, inp, group=g))
        buf = comm.empty(M // 2, dtype=torch.bfloat16)
        buf.normal_()
        ms = timed(lambda: comm.all_reduce(buf), steps(M), 3, dist)
        emit("allreduce", M, "forestcoll", ms, "bfloat16", proto=comm.last_call_info()["proto"])
        comm.deregister(buf)
        if nv.nvls_enabled:
            b2 = torch.randn(M // 2, device=dev).to(torch.bfloat16)
            ms = timed(lambda: nv.all_reduce(b2), steps(M), 3, dist)
            emit("allreduce", M, "forestcoll_nvls", ms, "bfloat16", proto=nv.last_call_info()["proto"])
        b3 = torch.randn(M // 2, device=dev).to(torch.bfloat16)
        run_nccl("allreduce", M, "bfloat16", lambda g: dist.all_reduce(b3, group=g))
    comm.check()

    # --- allreduce bf16: DDP bucket and 1 GiB ---
    for mib in (25, 1024):
        M = mib * MIB
        buf = comm.empty(M // 2, dtype=torch.bfloat16)
        buf.normal_()
        ms = timed(lambda: comm.all_reduce(buf), steps(M), 3, dist)
        emit("allreduce", M, "forestcoll", ms, "bfloat16", proto=comm.last_call_info()["proto"])
        comm.deregister(buf)
        if nv.nvls_enabled and M <= args.nvls_max_mib * MIB:
            nv._nvls_next = 0
            b3 = nv.nvls_empty(M // 2, torch.bfloat16)
            b3.normal_()
            ms = timed(lambda: nv.all_reduce(b3), steps(M), 3, dist)
            emit("allreduce", M, "forestcoll_nvls", ms, "bfloat16")
            del b3
        run_nccl("allreduce", M, "bfloat16", lambda g: dist.all_reduce(buf, group=g))
        del buf
    comm.check()
    nv.check()
    if rank == 0:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        with open(args.out, "w") as f:
            for r in recs:
                f.write(json.dumps(r) + "\n")
    nv.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
