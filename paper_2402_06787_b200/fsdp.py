"""PyTorch FSDP2 integration (the paper's FSDP consumer,
PAPER.md:1275-1281).

FSDP2 (``torch.distributed.fsdp.fully_shard``) lets a module replace its
parameter all-gather and gradient reduce-scatter (``set_custom_all_gather`` /
``set_custom_reduce_scatter``), including where the all-gather output is
allocated.  These adapters route both through the ForestColl forest kernel:

    comm = ForestCollComm()
    ag = ForestCollAllGather(comm, pool_bytes=2 << 30)
    rs = ForestCollReduceScatter(comm)
    for m in model.modules():
        if isinstance(m, FSDPModule):
            m.set_custom_all_gather(ag)
            m.set_custom_reduce_scatter(rs)

All-gather outputs must be peer-mapped.  ``SymmetricPool`` is one registered
buffer, sub-allocated identically on every rank, so an output lands at the
same pool offset everywhere and needs no per-call registration.  SPMD
programs such as FSDP allocate and free in the same order on every rank.  If
a program breaks that, the forest kernel's buffer tag check raises
``DeviceError`` ("different output buffer") instead of misplacing data.
Reduce-scatter needs no registration: peers write only into the library's own
scratch.  ``ReduceOp.AVG``, which FSDP uses for fp32/bf16 gradients, runs
fused in the kernel: each tree root scales its fp32 sum by 1/N once.
"""

from __future__ import annotations

import bisect

import torch

from .errors import InvalidArgument, Unsupported

try:  # FSDP2's comm interfaces (torch >= 2.8)
    from torch.distributed.fsdp._fully_shard._fsdp_api import AllGather as _AllGatherBase
    from torch.distributed.fsdp._fully_shard._fsdp_api import ReduceScatter as _ReduceScatterBase
except Exception:  # pragma: no cover - older torch: duck-typed adapters still work
    _AllGatherBase = object
    _ReduceScatterBase = object


class _Block:
    """`__cuda_array_interface__` holder for one pool block.  The tensor
    built on it keeps it alive: torch releases it only when the last view of
    that storage dies, and only then does the block return to the pool."""

    def __init__(self, pool, off, nbytes, ptr):
        self._pool, self._off, self._nbytes = pool, off, nbytes
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}

    def __del__(self):
        pool = self._pool
        if pool is not None:
            self._pool = None
            pool._release(self._off, self._nbytes)


class Extents:
    """Free-extent bookkeeping of a SymmetricPool (host-only, deterministic):
    best fit, lowest offset on ties, neighbours coalesced on release."""

    def __init__(self, nbytes: int):
        self.nbytes = nbytes
        self._off = [0]          # sorted offsets of free extents
        self._len = {0: nbytes}  # offset -> length

    def alloc(self, need: int) -> int | None:
        best = None
        for off in self._off:
            ln = self._len[off]
            if ln >= need and (best is None or ln < self._len[best]):
                best = off
        if best is None:
            return None
        ln = self._len.pop(best)
        self._off.remove(best)
        if ln > need:
            bisect.insort(self._off, best + need)
            self._len[best + need] = ln - need
        return best

    def release(self, off: int, nbytes: int) -> None:
        i = bisect.bisect_left(self._off, off)
        if i < len(self._off) and self._off[i] == off + nbytes:
            nbytes += self._len.pop(self._off.pop(i))
        if i > 0:
            prev = self._off[i - 1]
            if prev + self._len[prev] == off:
                self._len[prev] += nbytes
                return
        self._off.insert(i, off)
        self._len[off] = nbytes

    @property
    def free_bytes(self) -> int:
        return sum(self._len.values())

    def extents(self):
        return [(o, self._len[o]) for o in self._off]


class SymmetricPool:
    """One peer-registered buffer, sub-allocated the same way on every rank.

    * Best fit, lowest offset on ties.  The placement depends only on the
      sequence of ``empty`` calls and block releases, which SPMD programs
      repeat identically on every rank.
    * A released block records an event on the stream current at release.
      The next allocation that overlaps it makes its own stream wait for
      that event, like the caching allocator's stream semantics.
    * Peers never write into a block before its owner's kernel has entered
      the collective: the forest kernel's entry barrier guards reuse.
    """

    def __init__(self, comm, nbytes: int, align: int = 4096):
        if nbytes <= 0:
            raise InvalidArgument("pool size must be positive")
        self._comm = comm
        self._align = align
        nbytes = (nbytes + align - 1) // align * align
        self._base_t = comm.empty(nbytes, dtype=torch.uint8)  # collective registration
        self._base = self._base_t.data_ptr()
        self.nbytes = nbytes
        self._ext = Extents(nbytes)
        self._pending = []            # (off, nbytes, event) recorded at release
        self.device = self._base_t.device

    # -- allocation ---------------------------------------------------------
    def empty(self, numel: int, dtype=torch.float32) -> torch.Tensor | None:
        """A 1-D tensor in the pool, or None if no free extent fits."""
        es = torch.tensor([], dtype=dtype).element_size()
        need = max(self._align, (numel * es + self._align - 1) // self._align * self._align)
        best = self._ext.alloc(need)
        if best is None:
            return None
        self._wait_pending(best, need)
        holder = _Block(self, best, need, self._base + best)
        t = torch.as_tensor(holder, device=self.device)
        return t[: numel * es].view(dtype)

    def _wait_pending(self, off, nbytes):
        keep = []
        stream = torch.cuda.current_stream(self.device)
        for o, n, ev in self._pending:
            if o < off + nbytes and off < o + n:
                stream.wait_event(ev)
            elif not ev.query():
                keep.append((o, n, ev))
        self._pending = keep

    def _release(self, off, nbytes):
        try:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            self._pending.append((off, nbytes, ev))
        except Exception:  # interpreter shutdown: nothing left to order against
            pass
        self._ext.release(off, nbytes)

    @property
    def free_bytes(self) -> int:
        return self._ext.free_bytes

    def contains(self, t: torch.Tensor) -> bool:
        a = t.data_ptr()
        return self._base <= a and a + t.numel() * t.element_size() <= self._base + self.nbytes


def _check_group(comm, group):
    if group is not None and group.size() != comm.nranks:
        raise InvalidArgument(f"process group has {group.size()} ranks, communicator {comm.nranks}")


class ForestCollAllGather(_AllGatherBase):
    """FSDP2 ``AllGather``: outputs come from ``SymmetricPool`` segments.
    When no segment has room, a new segment of at least ``pool_bytes`` is
    registered.  Registration is collective, and the pool state is identical
    on every rank, so every rank grows at the same call.  Segments are reused
    and never leak per-call buffers."""

    def __init__(self, comm, pool_bytes: int = 1 << 30, pool: SymmetricPool | None = None):
        self.comm = comm
        self.pool_bytes = int(pool_bytes)
        self.pools = [pool if pool is not None else SymmetricPool(comm, self.pool_bytes)]

    @property
    def pool(self) -> SymmetricPool:
        return self.pools[0]

    def allocate(self, size, *, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
        numel = 1
        for s in size:
            numel *= int(s)
        for p in self.pools:
            t = p.empty(numel, dtype)
            if t is not None:
                break
        else:
            es = torch.tensor([], dtype=dtype).element_size()
            self.pools.append(SymmetricPool(self.comm, max(self.pool_bytes, 2 * numel * es)))
            t = self.pools[-1].empty(numel, dtype)
        return t.view(*[int(s) for s in size])

    def __call__(self, output_tensor, input_tensor, group=None, async_op: bool = False):
        _check_group(self.comm, group)
        self.comm.all_gather(output_tensor.view(-1), input_tensor.view(-1))
        return None  # stream-ordered: FSDP synchronises on its all-gather event


class ForestCollReduceScatter(_ReduceScatterBase):
    """FSDP2 ``ReduceScatter``: sum or average over the ForestColl in-trees.
    Plain allocations suffice because peers write only into the library's
    scratch."""

    def __init__(self, comm):
        self.comm = comm

    def allocate(self, size, *, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
        return torch.empty(*[int(s) for s in size], dtype=dtype, device=device)

    def __call__(self, output_tensor, input_tensor, group=None, op=None, async_op: bool = False):
        _check_group(self.comm, group)
        name = "sum" if op is None else str(getattr(op, "name", op)).rsplit(".", 1)[-1].lower()
        if name not in ("sum", "avg"):
            raise Unsupported(f"FSDP reduce op {op!r}: only SUM and AVG run on the forest")
        self.comm.reduce_scatter(output_tensor.view(-1), input_tensor.view(-1), op=name)
        return None
