"""Chain forest vs star forest on one NVSwitch (torchrun, N ranks).

On a single switch a star (root -> every peer) loads every link exactly as
the reference's chain forest does (FC_PLAN_ONEHOP): does the depth-1 tree
move large messages faster through the chunk-flag kernel?  Builds the star
as a reference Schedule and times both with tools/ab_time.py's method."""
import os
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import MIB, gbs, timed  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200._refpath import require_collsched  # noqa: E402
from paper_2402_06787_b200.generator import get_schedule  # noqa: E402
from paper_2402_06787_b200.topology import compute_ids, nvswitch_doc  # noqa: E402


def star_allgather(doc, ref):
    cs = require_collsched()
    ids = compute_ids(doc)
    roots = []
    for r in ids:
        edges = tuple(cs.ScheduleEdge(r, d, (cs.PathUse((r, "nvs", d), 1),)) for d in ids if d != r)
        roots.append(cs.RootTrees(r, (cs.ScheduleBatch(1, edges),)))
    return cs.Schedule(collective="allgather", num_compute=ref.num_compute, k=1, U=ref.U, y=ref.y,
                       inv_x_star=ref.inv_x_star, roots=tuple(roots), exact=ref.exact)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    doc = nvswitch_doc(n)
    chain = get_schedule(doc, "allgather", validate=False)
    star = star_allgather(doc, chain)
    cs = require_collsched()
    import json

    t = cs.parse_topology(json.dumps(doc))
    _, meta = cs.generate(t, "allgather")
    rep = cs.validate_schedule(star, t, meta)
    if rank == 0:
        print(f"star valid: {rep.ok} {[v.kind for v in rep.violations][:3]}", flush=True)
    import collsched.schedule as CS

    star_rs = CS.reverse_for_reduce_scatter(star)
    star_ar = CS.combine_allreduce(star_rs, star)
    if "--ar" in sys.argv:  # allreduce / reduce-scatter, star vs chain, LL128
        for name, scheds in (("chain", {"allreduce": get_schedule(doc, "allreduce", validate=False),
                                        "reduce_scatter": get_schedule(doc, "reduce_scatter",
                                                                       validate=False)}),
                             ("star", {"allreduce": star_ar, "reduce_scatter": star_rs})):
            comm = ForestCollComm(doc, schedules=scheds, device=local,
                                  options={"oneshot_max": 0, "twohop_max": 0})
            for mib in (4, 8, 16, 25, 64, 256):
                M = mib * MIB
                buf = comm.empty(M // 2, dtype=torch.bfloat16)
                buf.normal_()
                ms = timed(lambda: comm.all_reduce(buf), max(5, int(0.03 / (M / 3e11))), 3, dist)
                rin = torch.randn(M // 2, device=dev).to(torch.bfloat16)
                rout = torch.empty(M // 2 // n, device=dev, dtype=torch.bfloat16)
                ms2 = timed(lambda: comm.reduce_scatter(rout, rin), max(5, int(0.03 / (M / 6e11))), 3, dist)
                if rank == 0:
                    print(f"{name:5s} AR {mib:4d} MiB {comm.last_call_info()['proto']:6s} "
                          f"{gbs(M, ms):7.1f} GB/s | RS {gbs(M, ms2):7.1f} GB/s", flush=True)
                comm.deregister(buf)
            comm.close()
        dist.destroy_process_group()
        return
    for name, sched in (("chain", chain), ("star", star)):
        comm = ForestCollComm(doc, schedules={"allgather": sched}, device=local,
                              options={"oneshot_ag_max": 0, "ce_min": 0})
        for mib, proto in ((64, 1), (256, 1), (1024, 0), (4096, 0)):
            comm.set_option("proto", proto)
            M = mib * MIB
            S = M // n // 4
            inp = torch.randn(S, device=dev)
            out = comm.empty(n * S, dtype=torch.float32)
            ms = timed(lambda: comm.all_gather(out, inp), max(5, int(0.03 / (M / 6e11))), 3, dist)
            if rank == 0:
                print(f"{name:5s} AG {mib:5d} MiB proto={comm.last_call_info()['proto']:6s} "
                      f"{gbs(M, ms):8.1f} GB/s  frac T* {comm.t_star('allgather', M) * 1e3 / ms:.3f}",
                      flush=True)
            comm.deregister(out)
            del out, inp
        comm.check()
        comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
