"""Schedule compiler: lowering invariants and tamper detection."""

import dataclasses

import numpy as np
import pytest

from conftest import golden_names, load_golden
from paper_2402_06787_b200 import compiler as C
from paper_2402_06787_b200.errors import PlanError
from paper_2402_06787_b200._refpath import require_collsched

_cs = require_collsched()
ScheduleBatch, ScheduleEdge = _cs.ScheduleBatch, _cs.ScheduleEdge


@pytest.mark.parametrize("name", golden_names())
def test_lowering_invariants(name):
    s = load_golden(name)
    p = C.lower(s)
    n = p.nranks
    t = p.table
    assert t[0] == C.MAGIC and t[3] == n and t[4] == s.k and t[5] == len(p.trees)
    assert t.size == C.HEADER_WORDS + n * C.RANKDESC_WORDS + sum(map(len, p.tasks)) * C.TASK_WORDS
    # one role per (tree, rank); two for allreduce non-roots
    for v in range(n):
        per_tree = {}
        for task in p.tasks[v]:
            per_tree.setdefault(task.tree, []).append(task.kind)
        assert set(per_tree) == {tr.index for tr in p.trees}
        for tr in p.trees:
            want = 1 if (s.collective != "allreduce" or tr.root == v) else 2
            assert len(per_tree[tr.index]) == want
        # active tasks sorted by stage, waits last
        act = p.tasks[v][: p.nactive[v]]
        assert [x.stage for x in act] == sorted(x.stage for x in act)
        assert all(x.kind == C.K_WAIT_AG for x in p.tasks[v][p.nactive[v]:])
    # every dependency has a strictly smaller stage (progress argument)
    by = {(v, task.tree, task.kind): task for v in range(n) for task in p.tasks[v]}
    for v in range(n):
        for task in p.tasks[v]:
            tr = p.trees[task.tree]
            if task.kind in (C.K_AG_FWD, C.K_WAIT_AG):
                par = tr.parent[v]
                deps = [x for x in p.tasks[par] if x.tree == task.tree and x.kind in
                        (C.K_AG_ROOT, C.K_AG_FWD, C.K_AR_ROOT)]
                assert len(deps) == 1 and deps[0].stage < task.stage
            if task.kind in (C.K_RS_FWD, C.K_RS_ROOT, C.K_AR_ROOT):
                for x in tr.children[v]:
                    deps = [d for d in p.tasks[x] if d.tree == task.tree and d.kind == C.K_RS_FWD]
                    assert len(deps) == 1 and deps[0].stage < task.stage
    # reduction slots: unique per receiving rank, prefixes consistent
    if s.collective != "allgather":
        for v in range(n):
            slots = {}
            for x in range(n):
                for task in p.tasks[x]:
                    if task.kind == C.K_RS_FWD and task.rs_parent == v:
                        slots[task.rs_pslot] = (task.rs_pprefix, task.mhi - task.mlo)
            assert sorted(slots) == list(range(p.nslots[v]))
            pre = 0
            for sl in range(p.nslots[v]):
                assert slots[sl][0] == pre
                pre += slots[sl][1]
            assert pre == p.slot_units[v]


@pytest.mark.parametrize("base", ["nvs8", "groups300", "fig3a", "nvs2"])
def test_reduce_scatter_lowers_to_reversed_allgather_forest(base):
    ag = C.lower(load_golden(base + "_allgather"))
    rs = C.lower(load_golden(base + "_reduce_scatter"))
    assert C._skeleton(ag.trees) == C._skeleton(rs.trees)
    assert ag.send_units() == rs.send_units()


def _tamper(s, root_i, batch_i, edges):
    rts = list(s.roots)
    rt = rts[root_i]
    bs = list(rt.batches)
    bs[batch_i] = dataclasses.replace(bs[batch_i], edges=tuple(edges))
    rts[root_i] = dataclasses.replace(rt, batches=tuple(bs))
    return dataclasses.replace(s, roots=tuple(rts))


def _edge(a, b):
    return ScheduleEdge(a, b, ())


def test_tampered_forests_are_rejected():
    s = load_golden("nvs4_allgather")
    edges = list(s.roots[0].batches[0].edges)
    with pytest.raises(PlanError, match="two parents"):
        C.lower(_tamper(s, 0, 0, edges + [_edge("g1", edges[-1].dst)]))
    with pytest.raises(PlanError, match="no edge reaches"):
        C.lower(_tamper(s, 0, 0, edges[:-1]))
    with pytest.raises(PlanError, match="root receives"):
        C.lower(_tamper(s, 0, 0, edges + [_edge("g1", "g0")]))
    with pytest.raises(PlanError, match="leaves the compute set"):
        C.lower(_tamper(s, 0, 0, edges[:-1] + [_edge("g0", "nvs")]))
    # cycle: g1->g2, g2->g3, g3->g1 with g0 isolated from them
    cyc = [_edge("g1", "g2"), _edge("g2", "g3"), _edge("g3", "g1")]
    with pytest.raises(PlanError):
        C.lower(_tamper(s, 0, 0, cyc))
    with pytest.raises(PlanError, match="expected"):
        C.lower(dataclasses.replace(s, k=2))
    with pytest.raises(PlanError, match="appears twice"):
        C.lower(dataclasses.replace(s, roots=s.roots + (s.roots[0],)), ranks=("g0", "g1", "g2", "g3"))


def test_allreduce_phase_mismatch_rejected():
    ar = load_golden("nvs4_allreduce")
    other = load_golden("groups450_reduce_scatter")
    with pytest.raises(PlanError):
        C.lower(dataclasses.replace(ar, phases=(other, ar.phases[1])))
    with pytest.raises(PlanError):
        C.lower(dataclasses.replace(ar, phases=(ar.phases[1], ar.phases[0])))


def test_multibatch_slices():
    s = load_golden("random1_allgather")  # k = 7, 6 batches (pkg/tests/test_packing.py:128-142)
    p = C.lower(s)
    assert p.k == 7 and len(p.trees) == 6
    for r in range(p.nranks):
        ts = [t for t in p.trees if t.root == r]
        assert ts[0].mlo == 0 and ts[-1].mhi == 7
        assert all(a.mhi == b.mlo for a, b in zip(ts, ts[1:]))
    assert any(t.multiplicity < p.k for t in p.trees)


def test_table_roundtrip_fields():
    p = C.lower(load_golden("nvs8_allreduce"))
    t = p.table
    task0 = C.HEADER_WORDS + p.nranks * C.RANKDESC_WORDS
    row = t[task0:task0 + C.TASK_WORDS]
    first = p.tasks[0][0]
    assert row[C.TW_KIND] == first.kind and row[C.TW_TREE] == first.tree
    assert row[C.TW_N_RS_CHILD] == len(first.rs_children)
    assert t.dtype == np.int32
