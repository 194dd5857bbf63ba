"""CPU restatement oracle of the ForestColl executor — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product path (paper_2402_06787_b200) never calls
it and has no CPU fallback.

Why a restatement: the reference (``collsched`` 0.1.0) generates schedules
but ships no executor (pkg/tests/test_acceptance.py:
159-163 skips the hardware criterion).  This oracle executes a reference
``Schedule`` on N host buffers with the semantics the reference documents:

* allgather — "a 1/k shard of data is broadcast along each out-tree"
  (PAPER.md:478).  Root r's batches (schedule.py:55-65) split shard r in
  schedule order: batch j carries elements [floor(S*lo/k), floor(S*hi/k)),
  lo/hi the cumulative multiplicities before/through j.
  Every edge u->v copies that slice from u's output into v's output at
  offset r*S; roots copy their own input in.  Edges are replayed in BFS
  order from the root (verify.py:266-283), which is delivery order.
* reduce-scatter — the in-trees are the reversed out-trees
  (schedule.py:166-174).  At node v of root r's tree:
  partial_v = own_v[slice] (+) partials of v's children in ascending rank
  order, accumulated in fp32 for fp32/bf16/fp16 and in wrapping int32 for
  int32, rounded to the buffer dtype once per hop; a node without children
  forwards its own slice unchanged.  The root's partial is its output.
  op "avg" (floating-point dtypes): the root multiplies its fp32 sum by the
  fp32 value 1/N once, before its final rounding (include/forestcoll.h
  FC_AVG; NCCL-shaped ncclAvg, used by FSDP / DDP gradient averaging).
* allreduce — reduce-scatter then allgather over one forest
  (schedule.py:177-211, combine_allreduce); the buffer of `count` elements
  is split into N root shards of S = align_up(ceil(count/N), 128 B / esize)
  elements (the last shards may be short or empty).

Parity status: allgather and integer reductions are pinned by closed forms
(concatenation; exact sum) that the tests assert on reference-generated
forests.  fp32/bf16/fp16 reduction *order* is not defined anywhere in the
reference, so floating-point parity is pinned only against this stated
contract ("parity unpinned" w.r.t. the reference).
"""

from __future__ import annotations

from collections import deque
from fractions import Fraction

import numpy as np

ALIGN_BYTES = 128


# ---------------------------------------------------------------------------
# dtype helpers.  bf16 buffers are numpy uint16 bit patterns.
# ---------------------------------------------------------------------------

def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16(f32: np.ndarray) -> np.ndarray:
    """IEEE round-to-nearest-even (denormals kept); every NaN becomes the
    canonical 0x7FFF.  This is sm_100's cvt.rn.bf16x2.f32, which the kernel
    uses (csrc/fc_device.cuh Red<FC_BFLOAT16>; measured by tools/cvt_probe.cu)."""
    u = np.ascontiguousarray(f32, dtype=np.float32).view(np.uint32)
    nan = (u & np.uint32(0x7FFFFFFF)) > np.uint32(0x7F800000)
    rounded = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return np.where(nan, np.uint32(0x7FFF), rounded).astype(np.uint16)


def _to_acc(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "float32":
        return x.astype(np.float32, copy=True)
    if dtype == "bfloat16":
        return bf16_to_f32(x)
    if dtype == "float16":
        return x.astype(np.float32)
    if dtype in ("int32", "uint32"):
        return x.view(np.uint32).astype(np.uint32, copy=True)
    raise ValueError(f"dtype {dtype} cannot be reduced")


def _from_acc(a: np.ndarray, dtype: str, like: np.ndarray) -> np.ndarray:
    if dtype == "float32":
        return a.astype(np.float32)
    if dtype == "bfloat16":
        return f32_to_bf16(a)
    if dtype == "float16":
        return a.astype(np.float16)
    return a.astype(np.uint32).view(like.dtype)


def _add(a: np.ndarray, b: np.ndarray, dtype: str) -> np.ndarray:
    # float32 + float32 in numpy is one IEEE round-to-nearest add (no FMA)
    return a + b


# ---------------------------------------------------------------------------
# Forest walking, straight from the reference Schedule fields.
# ---------------------------------------------------------------------------

def rank_order(schedule) -> list[str]:
    sched = schedule.phases[1] if schedule.collective == "allreduce" else schedule
    return sorted(rt.root for rt in sched.roots)


def trees(schedule, reverse: bool):
    """Yield (root_id, lo, hi, children) per batch; children maps a node to its
    out-tree children (AG orientation), ascending by rank."""
    ids = rank_order(schedule)
    pos = {x: i for i, x in enumerate(ids)}
    for rt in schedule.roots:
        lo = 0
        for b in rt.batches:
            kids: dict[str, list[str]] = {}
            for e in b.edges:
                u, v = (e.dst, e.src) if reverse else (e.src, e.dst)
                kids.setdefault(u, []).append(v)
            for u in kids:
                kids[u].sort(key=pos.__getitem__)
            yield rt.root, lo, lo + b.multiplicity, kids
            lo += b.multiplicity


def _bfs(root, kids):
    order, q = [], deque([root])
    while q:
        u = q.popleft()
        order.append(u)
        q.extend(kids.get(u, ()))
    return order


def slice_bounds(S: int, k: int, lo: int, hi: int) -> tuple[int, int]:
    return (S * lo) // k, (S * hi) // k


# ---------------------------------------------------------------------------
# Collectives
# ---------------------------------------------------------------------------

def allgather(schedule, sends: list[np.ndarray]) -> list[np.ndarray]:
    """sends[r]: rank r's shard (any dtype, S elements) -> outputs (N*S)."""
    ids = rank_order(schedule)
    n = len(ids)
    pos = {x: i for i, x in enumerate(ids)}
    S = sends[0].size
    k = schedule.k
    outs = [np.zeros(n * S, dtype=sends[0].dtype) for _ in range(n)]
    covered = [np.zeros(n * S, dtype=bool) for _ in range(n)]
    for root, lo, hi, kids in trees(schedule, reverse=False):
        r = pos[root]
        a, b = slice_bounds(S, k, lo, hi)
        off = r * S
        outs[r][off + a:off + b] = sends[r][a:b]
        covered[r][off + a:off + b] = True
        for u in _bfs(root, kids):
            for v in kids.get(u, ()):
                iu, iv = pos[u], pos[v]
                outs[iv][off + a:off + b] = outs[iu][off + a:off + b]
                covered[iv][off + a:off + b] = True
    for r in range(n):
        if not covered[r].all():
            raise AssertionError(f"allgather oracle: rank {r} not fully delivered")
    return outs


def _root_scale(op: str, n: int, dtype: str):
    if op == "sum":
        return None
    if op != "avg" or dtype not in ("float32", "bfloat16", "float16"):
        raise ValueError(f"op {op!r} is not defined for dtype {dtype}")
    return np.float32(1.0) / np.float32(n)


def _reduce_tree(root, kids, get_own, dtype, pos, scale=None):
    """Post-order in-tree reduction; returns the root's partial (scaled in
    fp32 by `scale` before its rounding when given)."""
    order = _bfs(root, kids)
    partial = {}
    for v in reversed(order):
        own = get_own(pos[v])
        ch = kids.get(v, ())
        if not ch:
            partial[v] = own.copy()
            continue
        acc = _to_acc(own, dtype)
        for c in ch:  # ascending rank order
            acc = _add(acc, _to_acc(partial[c], dtype), dtype)
        if scale is not None and v == root:
            acc = acc * scale  # float32 x float32: one IEEE round-to-nearest multiply
        partial[v] = _from_acc(acc, dtype, own)
    return partial[root]


def reduce_scatter(schedule, inputs: list[np.ndarray], dtype: str, op: str = "sum") -> list[np.ndarray]:
    """inputs[r]: N*S elements -> outputs[r]: S elements (sum over ranks of
    inputs[*][r*S:(r+1)*S], tree order per the contract above)."""
    ids = rank_order(schedule)
    n = len(ids)
    pos = {x: i for i, x in enumerate(ids)}
    S = inputs[0].size // n
    k = schedule.k
    scale = _root_scale(op, n, dtype)
    outs = [np.zeros(S, dtype=inputs[0].dtype) for _ in range(n)]
    for root, lo, hi, kids in trees(schedule, reverse=True):
        r = pos[root]
        a, b = slice_bounds(S, k, lo, hi)
        off = r * S
        outs[r][a:b] = _reduce_tree(root, kids, lambda i: inputs[i][off + a:off + b], dtype, pos,
                                    scale)
    return outs


def allreduce_shard(count: int, n: int, esize: int) -> int:
    a = ALIGN_BYTES // esize
    s = -(-count // n)
    return -(-s // a) * a


def allreduce(schedule, inputs: list[np.ndarray], dtype: str, op: str = "sum") -> list[np.ndarray]:
    rs, ag = schedule.phases
    ids = rank_order(schedule)
    n = len(ids)
    pos = {x: i for i, x in enumerate(ids)}
    count = inputs[0].size
    S = allreduce_shard(count, n, inputs[0].itemsize)
    k = schedule.k
    scale = _root_scale(op, n, dtype)
    outs = [np.zeros(count, dtype=inputs[0].dtype) for _ in range(n)]
    reduced = {}
    for root, lo, hi, kids in trees(rs, reverse=True):
        r = pos[root]
        sr = max(0, min(S, count - r * S))
        a, b = slice_bounds(sr, k, lo, hi)
        off = r * S
        reduced[(root, lo)] = _reduce_tree(root, kids, lambda i: inputs[i][off + a:off + b],
                                           dtype, pos, scale)
    for root, lo, hi, kids in trees(ag, reverse=False):
        r = pos[root]
        sr = max(0, min(S, count - r * S))
        a, b = slice_bounds(sr, k, lo, hi)
        off = r * S
        for v in _bfs(root, kids):
            outs[pos[v]][off + a:off + b] = reduced[(root, lo)]
    return outs


def t_star(schedule, message_bytes: int) -> float:
    """T* (seconds) per SURVEY.md §8d: (M/N)*inv_x_star, doubled for AR."""
    phases = 2 if schedule.collective == "allreduce" else 1
    return phases * float(Fraction(schedule.inv_x_star)) / schedule.num_compute * message_bytes / 1e9
