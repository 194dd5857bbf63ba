"""torchrun worker: randomized soak of back-to-back collectives (mixed
collective, size, dtype, protocol, buffer reuse) checked against closed
forms — allgather = concatenation, reductions = exact sums (int32 wrapping;
bf16 / fp32 on small integers, exact in any order).  Catches
races in the epoch / entry-barrier / flag protocol that single calls miss."""

import os
import random
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from _common import init  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1234
    local = init()
    dev = torch.device(f"cuda:{local}")
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local,
                          scratch_bytes=256 << 20, options={"timeout_ms": 20000})
    rng = random.Random(seed)  # same sequence on every rank
    # a few persistent (registered) output buffers, reused across calls
    pools = {dt: comm.empty(n * (1 << 22), dtype=dt) for dt in (torch.float32, torch.int32, torch.bfloat16)}
    fails = 0
    for it in range(iters):
        coll = rng.choice(["allgather", "reduce_scatter", "allreduce"])
        proto = rng.choice([-1, 0])
        comm.set_option("proto", proto)
        comm.set_option("chunk_max", rng.choice([16 << 10, 64 << 10, 256 << 10]))
        # up to the copy-engine (N=2, >= 24 MiB output) and two-hop (2-12 MiB) ranges
        S = rng.choice([1, 17, 256, 4096, 4097, 65536 + 8, 1 << 18, (1 << 18) + 3, 1 << 20, (1 << 21) - 4,
                        (1 << 21) + 1, 1 << 22])
        g = torch.Generator().manual_seed(it)
        if coll == "allgather":
            allin = torch.randint(-2**31, 2**31 - 1, (n, S), generator=g, dtype=torch.int32)
            out = pools[torch.float32][: n * S].view(torch.int32)
            comm.all_gather(out, allin[rank].to(dev))
            ok = torch.equal(out.cpu(), allin.reshape(-1))
        else:
            # int32 wraps exactly; bf16 / fp32 get small integers, so every
            # partial sum is exact in any order and the result is closed-form
            dt = rng.choice([torch.int32, torch.bfloat16, torch.float32])
            lim = 2**20 if dt == torch.int32 else 9
            allin = torch.randint(-lim, lim, (n, n * S), generator=g, dtype=torch.int32)
            want = allin.sum(0, dtype=torch.int64).to(dt)
            src = allin[rank].to(dt).to(dev)
            if coll == "reduce_scatter":
                out = torch.empty(S, dtype=dt, device=dev)
                comm.reduce_scatter(out, src)
                ok = torch.equal(out.cpu(), want[rank * S:(rank + 1) * S])
            else:
                out = pools[dt][: n * S]
                out.copy_(src)
                comm.all_reduce(out)
                ok = torch.equal(out.cpu(), want)
        if not ok:
            fails += 1
            print(f"rank {rank} iter {it} {coll} S={S} proto={proto} {out.dtype} MISMATCH", flush=True)
    # bursts: several collectives queued back to back with no host sync, on two
    # alternating streams, each into its own output, verified only at the end.
    # Exercises launch-to-launch reuse of staging / scratch / flags (LL128
    # has no entry handshake) and the cross-stream ordering of one comm.
    streams = [torch.cuda.current_stream(), torch.cuda.Stream()]
    bufs = [comm.empty(n * (1 << 18), dtype=torch.int32) for _ in range(8)]
    for burst in range(max(1, iters // 20)):
        pending = []
        for j in range(8):
            coll = rng.choice(["allgather", "reduce_scatter", "allreduce"])
            comm.set_option("proto", rng.choice([-1, 0]))
            S = rng.choice([3, 256, 4096, 65536 + 8, 1 << 18])
            g = torch.Generator().manual_seed(100000 + 8 * burst + j)
            allin = torch.randint(-2**20, 2**20, (n, n * S if coll != "allgather" else S),
                                  generator=g, dtype=torch.int32)
            src = allin[rank].to(dev)
            s = streams[j % 2]
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                if coll == "allgather":
                    out = bufs[j][: n * S]
                    comm.all_gather(out, src)
                    want = allin.reshape(-1)
                elif coll == "reduce_scatter":
                    out = torch.empty(S, dtype=torch.int32, device=dev)
                    comm.reduce_scatter(out, src)
                    want = allin.sum(0, dtype=torch.int64).to(torch.int32)[rank * S:(rank + 1) * S]
                else:
                    out = bufs[j][: n * S]
                    out.copy_(src)
                    comm.all_reduce(out)
                    want = allin.sum(0, dtype=torch.int64).to(torch.int32)
            pending.append((coll, S, out, want, src))
        torch.cuda.synchronize()
        for coll, S, out, want, _ in pending:
            if not torch.equal(out.cpu(), want):
                fails += 1
                print(f"rank {rank} burst {burst} {coll} S={S} MISMATCH", flush=True)
    comm.check()
    print(f"STRESS rank {rank} {'OK' if not fails else f'FAIL {fails}'} ({iters} calls + bursts)",
          flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
