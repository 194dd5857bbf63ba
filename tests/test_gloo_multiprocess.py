"""World-size-2 host-side logic over gloo on CPU: every rank must derive the
same forest, the same plan tables and exchange handle blobs correctly."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2402_06787_b200 import compiler, generator
    from paper_2402_06787_b200.executor import ForestCollComm
    from paper_2402_06787_b200.topology import nvswitch_doc

    doc = nvswitch_doc(world)
    tables = {}
    for coll in ("allgather", "reduce_scatter", "allreduce"):
        s = generator.get_schedule(doc, coll, validate=False, write_cache=False)
        tables[coll] = compiler.lower(s).table.tobytes()
    gathered = [None] * world
    dist.all_gather_object(gathered, tables)
    same = all(g == gathered[0] for g in gathered)
    # the handle-exchange helper used by ForestCollComm (no CUDA needed)
    fake = ForestCollComm.__new__(ForestCollComm)
    fake._group = dist.new_group(backend="gloo")
    fake.nranks = world
    blobs = fake._allgather_obj(bytes([rank]) * 192)
    ok_blobs = [b[0] for b in blobs] == list(range(world))
    q.put((rank, same, ok_blobs))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_agree_on_plans(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(same and ok for _, same, ok in res)
