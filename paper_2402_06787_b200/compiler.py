"""Schedule compiler: a reference ``Schedule`` forest -> per-rank executor tables.

Input contract (pkg/src/collsched/schedule.py:31-81):

* ``roots``: one ``RootTrees`` per compute node, in ``compute_ids`` order
  (schedule.py:98); rank r is the r-th compute id in lexicographic order
  (topology.py:126-128).
* each root holds ``batches`` of ``multiplicity`` identical trees; the
  multiplicities of one root sum to ``k`` (checked like verify.py:442-449).
* allgather edges are out-tree arcs parent->child (schedule.py:88-129);
  reduce-scatter edges are the same arcs reversed (schedule.py:136-174);
  allreduce is ``phases=(rs, ag)`` over one forest (schedule.py:177-211).
* physical ``paths`` and ``pruned`` hops do not change delivery
  (schedule.py:281-290: pruning keeps "delivery and the congestion bottleneck"
  untouched) — on one NVSwitch every logical edge is a direct peer store.

Lowering: batch j of root r becomes one *tree* that
carries elements [floor(S*lo_j/k), floor(S*hi_j/k)) of shard r, lo_j/hi_j the
cumulative multiplicities before/through batch j in schedule order.  Each rank
gets one *task* per tree (root / interior / leaf role), sorted by a stage key
so that every dependency points to a strictly smaller (chunk, stage) key —
the property the kernel's dynamic work claiming relies on for progress.

The table layout is documented in csrc/fc_internal.h and DESIGN.md §3.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .errors import PlanError, Unsupported
from .schedule_io import ALLGATHER, ALLREDUCE, REDUCE_SCATTER

FC_MAXR = 16
MAGIC = 0x50434C46
VERSION = 1
HEADER_WORDS = 16
RANKDESC_WORDS = 8
TASK_WORDS = 128
COLLECTIVE_CODE = {ALLGATHER: 0, REDUCE_SCATTER: 1, ALLREDUCE: 2}

K_AG_ROOT, K_AG_FWD, K_RS_FWD, K_RS_ROOT, K_AR_ROOT, K_WAIT_AG = 1, 2, 3, 4, 5, 6
KIND_NAMES = {K_AG_ROOT: "ag_root", K_AG_FWD: "ag_fwd", K_RS_FWD: "rs_fwd",
              K_RS_ROOT: "rs_root", K_AR_ROOT: "ar_root", K_WAIT_AG: "wait_ag"}
AR_ROOT_STAGE = FC_MAXR
PLAN_ONEHOP = 1  # TH_FLAGS bit (fc_internal.h FC_PLAN_ONEHOP)

# task word offsets (fc_internal.h)
TW_KIND, TW_TREE, TW_STAGE, TW_ROOT, TW_MLO, TW_MHI = 0, 1, 2, 3, 4, 5
TW_AG_PARENT, TW_N_AG_CHILD, TW_AG_CHILD = 6, 7, 8
TW_RS_PARENT, TW_RS_PSLOT, TW_RS_PPREFIX, TW_N_RS_CHILD = 24, 25, 26, 27
TW_RS_CHILD, TW_RS_CSLOT, TW_RS_CPREFIX = 28, 44, 60
TW_LAG, TW_AG_LEAFMASK = 76, 77
TW_AG_MYSLOT, TW_AG_MYPREFIX, TW_AG_CSLOT, TW_AG_CPREFIX = 78, 79, 80, 96


@dataclass
class Tree:
    """One broadcast out-tree (AG orientation) carrying a 1/k-unit slice."""

    index: int
    root: int
    mlo: int
    mhi: int
    parent: list  # parent[v] (-1 at the root)
    children: list = field(default_factory=list)  # ascending ranks
    depth: list = field(default_factory=list)
    height: list = field(default_factory=list)

    @property
    def multiplicity(self) -> int:
        return self.mhi - self.mlo


@dataclass
class Task:
    kind: int
    tree: int
    stage: int
    root: int
    mlo: int
    mhi: int
    ag_parent: int = -1
    ag_children: tuple = ()
    rs_parent: int = -1
    rs_pslot: int = -1
    rs_pprefix: int = 0
    rs_children: tuple = ()
    rs_cslots: tuple = ()
    rs_cprefix: tuple = ()
    lag: int = 0  # dense stage index (claim-order skew), set by lower()
    leafmask: int = 0  # bit j: ag_children[j] is a leaf of this tree
    ag_myslot: int = -1  # LL staging slot receiving this tree's broadcast here
    ag_myprefix: int = 0
    ag_cslots: tuple = ()  # the children's staging slots for this tree
    ag_cprefix: tuple = ()


@dataclass
class Plan:
    collective: str
    nranks: int
    k: int
    ranks: tuple  # compute ids in rank order
    trees: list
    tasks: list  # per rank: list[Task] (active sorted by stage, then waits)
    nactive: list
    nwait: list
    slot_units: list
    nslots: list
    table: np.ndarray
    ag_slot_units: list = field(default_factory=list)
    ag_nslots: list = field(default_factory=list)
    flags: int = 0  # TH_FLAGS: PLAN_ONEHOP

    @property
    def onehop(self) -> bool:
        return bool(self.flags & PLAN_ONEHOP)

    @property
    def max_depth(self) -> int:
        return max(max(t.depth) for t in self.trees)

    def send_units(self) -> list:
        """Tree-multiplicity units each rank sends per collective phase."""
        out = [0] * self.nranks
        for t in self.trees:
            for v in range(self.nranks):
                out[v] += len(t.children[v]) * t.multiplicity
        return out


def _rank_map(schedule, ranks):
    if ranks is None:
        roots = schedule.phases[1].roots if schedule.collective == ALLREDUCE else schedule.roots
        ranks = sorted(rt.root for rt in roots)
    ranks = tuple(ranks)
    if len(set(ranks)) != len(ranks):
        raise PlanError("duplicate compute ids in the rank map")
    return ranks, {r: i for i, r in enumerate(ranks)}


def forest_of(schedule, ranks=None, reverse: bool | None = None):
    """Out-trees (AG orientation) of an allgather or reduce-scatter schedule.

    Checks the structure the executor depends on: every root present once,
    batch multiplicities summing to k per root, each batch a spanning
    arborescence over the compute ranks (verify.py:301-331 checks the same
    shape; repeated here because a malformed forest would deadlock the
    kernel rather than merely under-perform).
    """
    ranks, idx = _rank_map(schedule, ranks)
    n = len(ranks)
    if schedule.num_compute != n:
        raise PlanError(f"schedule has {schedule.num_compute} compute nodes, rank map {n}")
    if n > FC_MAXR:
        raise Unsupported(f"{n} ranks exceed the executor's limit of {FC_MAXR}")
    if reverse is None:
        reverse = schedule.collective == REDUCE_SCATTER
    k = int(schedule.k)
    seen = set()
    trees = []
    for rt in schedule.roots:
        if rt.root not in idx:
            raise PlanError(f"root {rt.root!r} is not a compute rank")
        if rt.root in seen:
            raise PlanError(f"root {rt.root!r} appears twice")
        seen.add(rt.root)
        r = idx[rt.root]
        lo = 0
        for batch in rt.batches:
            m = int(batch.multiplicity)
            if m < 1:
                raise PlanError(f"batch of root {rt.root} has multiplicity {m}")
            parent = [None] * n
            parent[r] = -1
            for e in batch.edges:
                src, dst = (e.dst, e.src) if reverse else (e.src, e.dst)
                if src not in idx or dst not in idx:
                    raise PlanError(f"edge {e.src}->{e.dst} leaves the compute set")
                u, v = idx[src], idx[dst]
                if v == r:
                    raise PlanError(f"tree of root {rt.root}: root receives an edge")
                if parent[v] is not None:
                    raise PlanError(f"tree of root {rt.root}: {dst} has two parents")
                parent[v] = u
            missing = [ranks[v] for v in range(n) if parent[v] is None]
            if missing:
                raise PlanError(f"tree of root {rt.root}: no edge reaches {', '.join(missing)}")
            t = Tree(index=len(trees), root=r, mlo=lo, mhi=lo + m, parent=parent)
            _finish_tree(t, n, rt.root)
            trees.append(t)
            lo += m
        if lo != k:
            raise PlanError(f"root {rt.root} has {lo} trees, expected {k}")
    if seen != set(ranks):
        raise PlanError(f"roots {sorted(seen)} differ from compute ranks {list(ranks)}")
    return ranks, k, trees


def _finish_tree(t: Tree, n: int, root_id: str) -> None:
    t.children = [[] for _ in range(n)]
    for v, p in enumerate(t.parent):
        if p >= 0:
            t.children[p].append(v)
    for c in t.children:
        c.sort()
    t.depth = [-1] * n
    t.depth[t.root] = 0
    q = deque([t.root])
    order = []
    while q:
        u = q.popleft()
        order.append(u)
        for c in t.children[u]:
            t.depth[c] = t.depth[u] + 1
            q.append(c)
    if len(order) != n:
        raise PlanError(f"tree of root {root_id}: edges contain a cycle")
    t.height = [0] * n
    for u in reversed(order):
        if t.children[u]:
            t.height[u] = 1 + max(t.height[c] for c in t.children[u])


def _skeleton(trees):
    return [(t.root, t.mlo, t.mhi, tuple(t.parent)) for t in trees]


def lower(schedule, ranks=None, collective: str | None = None) -> Plan:
    """Lower a schedule to the executor's int32 plan table."""
    coll = collective or schedule.collective
    if coll == ALLREDUCE:
        if schedule.collective != ALLREDUCE or len(schedule.phases) != 2:
            raise PlanError("allreduce needs a schedule with (reduce_scatter, allgather) phases")
        rs, ag = schedule.phases
        if rs.collective != REDUCE_SCATTER or ag.collective != ALLGATHER:
            raise PlanError("allreduce phases must be reduce_scatter then allgather")
        ranks, k, trees = forest_of(ag, ranks, reverse=False)
        _, k_rs, rs_trees = forest_of(rs, ranks, reverse=True)
        if k_rs != k or _skeleton(rs_trees) != _skeleton(trees):
            # combine_allreduce (schedule.py:188-200) requires the same forest
            raise PlanError("allreduce phases do not reverse the same tree forest")
    else:
        if schedule.collective != coll:
            raise PlanError(f"schedule is for {schedule.collective}, not {coll}")
        ranks, k, trees = forest_of(schedule, ranks)
    n = len(ranks)

    # reduce-scatter slots: one per (tree, child) in-edge at each rank
    slot_of = {}
    slot_units = [0] * n
    nslots = [0] * n
    if coll in (REDUCE_SCATTER, ALLREDUCE):
        for t in trees:
            for v in range(n):
                for x in t.children[v]:
                    slot_of[(t.index, x)] = (nslots[v], slot_units[v])
                    nslots[v] += 1
                    slot_units[v] += t.multiplicity

    tasks = [[] for _ in range(n)]
    for t in trees:
        for v in range(n):
            base = dict(tree=t.index, root=t.root, mlo=t.mlo, mhi=t.mhi)
            kids = tuple(t.children[v])
            rs_kw = {}
            if coll in (REDUCE_SCATTER, ALLREDUCE):
                rs_kw = dict(
                    rs_children=kids,
                    rs_cslots=tuple(slot_of[(t.index, x)][0] for x in kids),
                    rs_cprefix=tuple(slot_of[(t.index, x)][1] for x in kids),
                )
                if v != t.root:
                    ps, pp = slot_of[(t.index, v)]
                    rs_kw.update(rs_parent=t.parent[v], rs_pslot=ps, rs_pprefix=pp)
            if coll == ALLGATHER:
                if v == t.root:
                    tasks[v].append(Task(K_AG_ROOT, stage=0, ag_children=kids, **base))
                elif kids:
                    tasks[v].append(Task(K_AG_FWD, stage=t.depth[v], ag_parent=t.parent[v],
                                         ag_children=kids, **base))
                else:
                    tasks[v].append(Task(K_WAIT_AG, stage=t.depth[v], ag_parent=t.parent[v],
                                         **base))
            elif coll == REDUCE_SCATTER:
                kind = K_RS_ROOT if v == t.root else K_RS_FWD
                tasks[v].append(Task(kind, stage=t.height[v], **base, **rs_kw))
            else:
                if v == t.root:
                    tasks[v].append(Task(K_AR_ROOT, stage=AR_ROOT_STAGE, ag_children=kids,
                                         **base, **rs_kw))
                else:
                    tasks[v].append(Task(K_RS_FWD, stage=t.height[v], **base, **rs_kw))
                    kw = dict(stage=AR_ROOT_STAGE + t.depth[v], ag_parent=t.parent[v], **base)
                    if kids:
                        tasks[v].append(Task(K_AG_FWD, ag_children=kids, **kw))
                    else:
                        tasks[v].append(Task(K_WAIT_AG, **kw))

    # broadcast staging slots (fenceless LL protocol): one per (tree, non-root rank)
    ag_slot_of = {}
    ag_units = [0] * n
    ag_nslots = [0] * n
    if coll in (ALLGATHER, ALLREDUCE):
        for t in trees:
            for v in range(n):
                if v != t.root:
                    ag_slot_of[(t.index, v)] = (ag_nslots[v], ag_units[v])
                    ag_nslots[v] += 1
                    ag_units[v] += t.multiplicity
        for v in range(n):
            for x in tasks[v]:
                if x.kind in (K_AG_ROOT, K_AG_FWD, K_AR_ROOT, K_WAIT_AG):
                    if x.kind in (K_AG_FWD, K_WAIT_AG):
                        x.ag_myslot, x.ag_myprefix = ag_slot_of[(x.tree, v)]
                    x.ag_cslots = tuple(ag_slot_of[(x.tree, ch)][0] for ch in x.ag_children)
                    x.ag_cprefix = tuple(ag_slot_of[(x.tree, ch)][1] for ch in x.ag_children)
    # dense stage index, global over ranks: the kernel claims item (c, task)
    # at diagonal c + lag * index, so dependencies stay at smaller diagonals
    dense = {st: i for i, st in enumerate(sorted({x.stage for ts in tasks for x in ts}))}
    for ts in tasks:
        for x in ts:
            x.lag = dense[x.stage]
            tr = trees[x.tree]
            x.leafmask = sum(1 << j for j, ch in enumerate(x.ag_children) if not tr.children[ch])
    nactive, nwait = [], []
    for v in range(n):
        act = sorted((x for x in tasks[v] if x.kind != K_WAIT_AG), key=lambda x: (x.stage, x.tree))
        wai = sorted((x for x in tasks[v] if x.kind == K_WAIT_AG), key=lambda x: (x.stage, x.tree))
        tasks[v] = act + wai
        nactive.append(len(act))
        nwait.append(len(wai))
    flags = PLAN_ONEHOP if onehop_equivalent(schedule, ranks, trees, k) else 0
    table = encode(coll, n, k, trees, tasks, nactive, nwait, slot_units, nslots, ag_units,
                   ag_nslots, flags)
    return Plan(coll, n, k, ranks, trees, tasks, nactive, nwait, slot_units, nslots, table,
                ag_units, ag_nslots, flags)


def onehop_equivalent(schedule, ranks, trees, k) -> bool:
    """May a depth-1 all-to-all replace this forest without changing any
    link's load (so T*, ``congestion_time`` verify.py:537-562, is unchanged)?

    True when (1) every logical edge of every tree is a single physical path
    ``[src, sw, dst]`` through one and the same switch ``sw`` (paths partition
    an edge's copies, schedule.py:3-7; path interiors are switches,
    verify.py:350-353) -- every GPU then has an uplink and a downlink to
    ``sw``, so every pair has the path ``[i, sw, j]`` -- and (2) every rank
    sends exactly (N-1)*k tree units, the one-hop scheme's uplink load
    (downlink loads are (N-1)*k for any spanning forest).  Derived from the
    schedule alone, so a plan table carries it (FC_PLAN_ONEHOP) to the C ABI.
    """
    n = len(ranks)
    rankset = set(ranks)
    phases = schedule.phases if schedule.collective == ALLREDUCE else (schedule,)
    switch = None
    for ph in phases:
        for rt in ph.roots:
            for batch in rt.batches:
                for e in batch.edges:
                    if len(e.paths) != 1:
                        return False
                    path = tuple(e.paths[0].path)
                    if len(path) != 3 or path[1] in rankset or {path[0], path[2]} != {e.src, e.dst}:
                        return False
                    if switch is None:
                        switch = path[1]
                    elif path[1] != switch:
                        return False
    if switch is None:
        return False
    units = [0] * n
    for t in trees:
        for v in range(n):
            units[v] += len(t.children[v]) * t.multiplicity
    return all(u == (n - 1) * k for u in units)


def encode(coll, n, k, trees, tasks, nactive, nwait, slot_units, nslots, ag_units=None,
           ag_nslots=None, flags=0) -> np.ndarray:
    ntasks = sum(len(t) for t in tasks)
    words = HEADER_WORDS + n * RANKDESC_WORDS + ntasks * TASK_WORDS
    a = np.zeros(words, dtype=np.int32)
    ag_units = ag_units or [0]
    ag_nslots = ag_nslots or [0]
    a[0:12] = [MAGIC, VERSION, COLLECTIVE_CODE[coll], n, k, len(trees), ntasks, TASK_WORDS,
               max(slot_units) if slot_units else 0, max(nslots) if nslots else 0,
               max(ag_units), max(ag_nslots)]
    a[12] = flags  # TH_FLAGS
    first = 0
    pos = HEADER_WORDS + n * RANKDESC_WORDS
    for v in range(n):
        d = HEADER_WORDS + v * RANKDESC_WORDS
        a[d:d + 5] = [first, nactive[v], nwait[v], slot_units[v], nslots[v]]
        first += len(tasks[v])
        for t in tasks[v]:
            row = a[pos:pos + TASK_WORDS]
            row[:] = 0
            row[[TW_KIND, TW_TREE, TW_STAGE, TW_ROOT, TW_MLO, TW_MHI]] = [
                t.kind, t.tree, t.stage, t.root, t.mlo, t.mhi]
            row[TW_AG_PARENT] = t.ag_parent
            row[TW_N_AG_CHILD] = len(t.ag_children)
            row[TW_AG_CHILD:TW_AG_CHILD + len(t.ag_children)] = t.ag_children
            row[TW_RS_PARENT] = t.rs_parent
            row[TW_RS_PSLOT] = t.rs_pslot
            row[TW_RS_PPREFIX] = t.rs_pprefix
            row[TW_N_RS_CHILD] = len(t.rs_children)
            m = len(t.rs_children)
            row[TW_RS_CHILD:TW_RS_CHILD + m] = t.rs_children
            row[TW_RS_CSLOT:TW_RS_CSLOT + m] = t.rs_cslots
            row[TW_RS_CPREFIX:TW_RS_CPREFIX + m] = t.rs_cprefix
            row[TW_LAG] = t.lag
            row[TW_AG_LEAFMASK] = t.leafmask
            row[TW_AG_MYSLOT] = t.ag_myslot
            row[TW_AG_MYPREFIX] = t.ag_myprefix
            g = len(t.ag_cslots)
            row[TW_AG_CSLOT:TW_AG_CSLOT + g] = t.ag_cslots
            row[TW_AG_CPREFIX:TW_AG_CPREFIX + g] = t.ag_cprefix
            pos += TASK_WORDS
    return a


def describe(plan: Plan) -> str:
    lines = [f"{plan.collective}: N={plan.nranks} k={plan.k} trees={len(plan.trees)} "
             f"max_depth={plan.max_depth} send_units={plan.send_units()}"]
    for v in range(plan.nranks):
        parts = [f"{KIND_NAMES[t.kind]}(t{t.tree},s{t.stage})" for t in plan.tasks[v]]
        lines.append(f"  rank {v}: " + " ".join(parts))
    return "\n".join(lines)
