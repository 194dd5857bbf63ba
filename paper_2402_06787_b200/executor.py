"""PyTorch-facing executor for ForestColl schedules.

``ForestCollComm`` is one communicator per rank process (torchrun, one GPU
per rank): NCCL-shaped ``all_gather`` / ``reduce_scatter`` / ``all_reduce``
on CUDA tensors, executed by the persistent sm_100a kernel through the C ABI.
``VirtualComm`` runs all N ranks of a forest inside one grid on one GPU (the
single-device test mode).  ``Executor`` is the §8b surface:
one schedule (object, JSON text or path) plus its topology.

Schedules come from the reference generator (``collsched.generate``,
pipeline.py:43-78) through generator.get_schedule; pre-flight follows the
reference CLI (validate before use, cli.py:186-195); errors derive from
``CollschedError`` (errors.py:10-11).  torch is plumbing here — device
memory, streams and the host-side handle exchange — not the data path.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from .compiler import lower
from .errors import InvalidArgument, Unsupported
from .generator import get_schedule, preflight
from .schedule_io import ALLGATHER, ALLREDUCE, COLLECTIVES, REDUCE_SCATTER, load_schedule, \
    parse_schedule_json, t_star_seconds
from .topology import compute_ids, discover_for_torch, nvswitch_doc

COLL_CODE = {ALLGATHER: 0, REDUCE_SCATTER: 1, ALLREDUCE: 2}
DTYPE_CODE = {
    torch.int8: 0, torch.uint8: 1, torch.int32: 2, torch.int64: 4, torch.float16: 6,
    torch.float32: 7, torch.float64: 8, torch.bfloat16: 9,
}
for _name, _code in (("uint32", 3), ("uint64", 5)):
    if hasattr(torch, _name):
        DTYPE_CODE[getattr(torch, _name)] = _code
REDUCIBLE = {torch.int32, torch.float16, torch.float32, torch.bfloat16}
if hasattr(torch, "uint32"):
    REDUCIBLE.add(torch.uint32)
OPS = {"sum": 0, "avg": 4}  # ncclRedOp_t numbering (include/forestcoll.h)
# Per-rank workspace: two regions of scratch_bytes (reduction scratch and the
# LL128 staging).  ForestCollComm starts at INITIAL_SCRATCH (enough for the
# one-hop / one-shot paths) and grows on demand, collectively, up to
# MAX_SCRATCH (fc_call_scratch / fc_comm_grow); an explicit scratch_bytes
# fixes the size.
INITIAL_SCRATCH = 64 << 20
MAX_SCRATCH = 2 << 30
DEFAULT_SCRATCH = None
VIRTUAL_SCRATCH = 1 << 30


# raw cudaStream_t of the current stream without building a torch.cuda.Stream
# object per call (host overhead matters for small collectives)
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
if _raw_stream is None:  # pragma: no cover
    def _raw_stream(device):
        return torch.cuda.current_stream(device).cuda_stream


def _dtype_args(t: torch.Tensor, count: int):
    code = DTYPE_CODE.get(t.dtype)
    if code is None:  # opaque dtype: move bytes (allgather only)
        return count * t.element_size(), 1
    return count, code


def _pci_bus_id(device: int):
    p = torch.cuda.get_device_properties(device)
    try:
        return f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    except AttributeError:
        return None


def _op_code(op) -> int:
    """'sum' / 'avg' or torch.distributed.ReduceOp.SUM / .AVG."""
    if not isinstance(op, str):
        name = str(getattr(op, "name", op)).rsplit(".", 1)[-1].lower()
        op = name if name in OPS else op
    if op not in OPS:
        raise Unsupported(f"reduction op {op!r} is not supported (only 'sum' and 'avg')")
    return OPS[op]


def _as_doc(topology):
    if topology is None:
        return None
    if isinstance(topology, dict):
        return topology
    if isinstance(topology, str):
        import json

        return json.loads(topology)
    # reference Topology object: serialize through the reference
    from ._refpath import import_collsched
    import json

    cs = import_collsched()
    return json.loads(cs.serialize_topology(topology))


def _aligned(t: torch.Tensor) -> torch.Tensor:
    """`t`, or an aligned copy of it when its address is not 16-byte aligned
    (the LL-multicast kernels move 8/16-byte units).  Only the local buffer's
    placement decides this, never the engine choice."""
    if t.data_ptr() % 16 == 0:
        return t
    return t.clone()


class _CommBase:
    """Shared plan management for real and virtual communicators."""

    def __init__(self, topology_doc, nranks, schedules=None, validate=True, prune=True):
        self.topology = topology_doc
        self.nranks = nranks
        self._validate = validate
        self._prune = prune
        self._schedules = dict(schedules or {})
        self._plans = {}
        self._capable = {}  # switch capability -> bool (cached: checked on every call)
        self._comm = None
        self._lib = _lib.load()
        if topology_doc is not None and len(compute_ids(topology_doc)) != nranks:
            raise InvalidArgument(
                f"topology has {len(compute_ids(topology_doc))} compute nodes, comm {nranks} ranks")

    # -- schedules and plans ------------------------------------------------
    def schedule(self, collective: str):
        if collective not in COLLECTIVES:
            raise InvalidArgument(f"unknown collective {collective!r}")
        s = self._schedules.get(collective)
        if s is None:
            if self.topology is None:
                raise InvalidArgument(f"no schedule for {collective} and no topology to generate one")
            s = get_schedule(self.topology, collective, prune=self._prune, validate=self._validate)
            self._schedules[collective] = s
        return s

    def plan(self, collective: str):
        p = self._plans.get(collective)
        if p is None:
            s = self.schedule(collective)
            ranks = compute_ids(self.topology) if self.topology is not None else None
            p = lower(s, ranks=ranks, collective=collective)
            if p.nranks != self.nranks:
                raise InvalidArgument(f"schedule has {p.nranks} ranks, comm {self.nranks}")
            tbl = np.ascontiguousarray(p.table, dtype=np.int32)
            _lib.check(
                self._lib.fc_plan_load(self._comm, COLL_CODE[collective],
                                       tbl.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                       tbl.size),
                self._comm, f"plan_load({collective})")
            self._plans[collective] = p
        return p

    def t_star(self, collective: str, message_bytes: int) -> float:
        """ForestColl optimal time (seconds) for M bytes."""
        return t_star_seconds(self.schedule(collective), message_bytes, collective, self.topology)

    # -- options / status ---------------------------------------------------
    def set_option(self, name: str, value: int) -> None:
        _lib.check(self._lib.fc_comm_set_option(self._comm, _lib.OPTIONS[name], int(value)),
                   self._comm, f"set_option({name})")
        if hasattr(self, "_scratch_ok"):
            self._scratch_ok.clear()  # options change paths (and their workspace needs)
        if hasattr(self, "_paths"):
            self._paths.clear()
        if name == "nvls_ll_max":
            self._nvls_ll_max = int(value)
        if name == "nvls_ll_red_max":
            self._nvls_ll_red_max = int(value)

    def get_option(self, name: str) -> int:
        v = ctypes.c_longlong()
        _lib.check(self._lib.fc_comm_get_option(self._comm, _lib.OPTIONS[name], ctypes.byref(v)),
                   self._comm, f"get_option({name})")
        return v.value

    def check(self) -> None:
        """Synchronize and raise DeviceError if a device-side wait failed."""
        err = ctypes.c_int()
        _lib.check(self._lib.fc_comm_check(self._comm, ctypes.byref(err)), self._comm, "check")

    def last_call_info(self) -> dict:
        buf = (ctypes.c_longlong * 8)()
        self._lib.fc_last_call_info(self._comm, buf, 8)
        info = {"launches": buf[0], "nchunks": buf[1], "window": buf[2], "grid": buf[3],
                "unit_bytes": buf[4],
                "proto": {0: "flags", 1: "ll128", 2: "nvls", 3: "nvls_ll", 4: "oneshot",
                          5: "ce", 6: "local", 7: "twohop"}[buf[5]]}
        # floating-point summation order of the last reduction: "tree" (the
        # forest's order, bit-exact vs the oracle) or "switch" (in-NVSwitch)
        info["order"] = getattr(self, "_last_order", None)
        return info

    # -- tracing ------------------------------------------------------------
    TRACE_DTYPE = np.dtype([("t_start", "<u8"), ("t_end", "<u8"), ("t_wait", "<u4"),
                            ("t_move", "<u4"), ("chunk", "<i4"), ("rank", "<i2"),
                            ("task", "<i2"), ("worker", "<i2"), ("launch", "<u2"),
                            ("peer_bytes", "<u4")])

    def enable_trace(self, capacity: int = 1 << 20) -> None:
        """Record one (start, end, rank, task, chunk, worker, launch) row per
        executed item into device memory (fc_comm_set_trace)."""
        dev = f"cuda:{self.device}"
        self._trace_buf = torch.zeros(capacity * self.TRACE_DTYPE.itemsize, dtype=torch.uint8,
                                      device=dev)
        self._trace_cnt = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(self._lib.fc_comm_set_trace(self._comm, self._trace_buf.data_ptr(),
                                               self._trace_cnt.data_ptr(), capacity),
                   self._comm, "set_trace")
        self._trace_cap = capacity

    def disable_trace(self) -> None:
        self._lib.fc_comm_set_trace(self._comm, None, None, 0)

    def reset_trace(self) -> None:
        self._trace_cnt.zero_()

    def read_trace(self) -> np.ndarray:
        torch.cuda.synchronize(self.device)
        n = min(int(self._trace_cnt.item()), self._trace_cap)
        raw = self._trace_buf[: n * self.TRACE_DTYPE.itemsize].cpu().numpy()
        return raw.view(self.TRACE_DTYPE)

    def close(self) -> None:
        if self._comm is not None:
            self._lib.fc_comm_destroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _check_tensor(t, device, name):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise InvalidArgument(f"{name} must be a CUDA tensor")
        if t.get_device() != device:
            raise InvalidArgument(f"{name} is on {t.device}, communicator on cuda:{device}")
        if not t.is_contiguous():
            raise InvalidArgument(f"{name} must be contiguous")


class ForestCollComm(_CommBase):
    """One rank of a ForestColl communicator (one process per GPU)."""

    def __init__(self, topology=None, *, rank=None, world_size=None, device=None, group=None,
                 scratch_bytes=DEFAULT_SCRATCH, schedules=None, validate=True, prune=True,
                 options=None, nvls_bytes=0, reduction_order="tree",
                 max_scratch_bytes=MAX_SCRATCH):
        import torch.distributed as dist

        if reduction_order not in ("tree", "switch"):
            raise InvalidArgument("reduction_order must be 'tree' or 'switch'")
        # "tree": every floating-point sum in the forest's order (bit-exact vs
        # the oracle, whatever the buffer); "switch": tensors in the NVLS pool
        # are reduced inside the NVSwitch (multimem.ld_reduce), in its order
        self.reduction_order = reduction_order
        self._last_order = None

        if rank is None or world_size is None:
            if not dist.is_initialized():
                raise InvalidArgument("rank/world_size not given and torch.distributed is not initialized")
            rank = dist.get_rank() if rank is None else rank
            world_size = dist.get_world_size() if world_size is None else world_size
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", torch.cuda.current_device()))
        self.rank, self.device = rank, device
        self._prune_default = prune
        self._group = None
        if world_size > 1:
            self._group = group if group is not None else dist.new_group(backend="gloo")
        self.nranks = world_size
        self.topology_source = "given"
        doc = _as_doc(topology)
        if doc is None and not schedules:
            buses = self._allgather_obj(_pci_bus_id(device))
            doc, self.topology_source = discover_for_torch(world_size,
                                                           None if None in buses else buses)
        if self.topology_source == "nvml" and not schedules:
            doc = self._usable_topology(doc, world_size)
        super().__init__(doc, world_size, schedules, validate, prune)
        # workspace: fixed when scratch_bytes is given, else grown on demand
        self._grow = scratch_bytes is None
        self._max_scratch = int(max_scratch_bytes)
        self._scratch_ok = set()  # (collective, count, dtype) needing no growth
        self._paths = {}  # (collective, count, dtype) -> fc_call_path
        comm = ctypes.c_void_p()
        init = INITIAL_SCRATCH if scratch_bytes is None else int(scratch_bytes)
        _lib.check(self._lib.fc_comm_init(rank, world_size, device, init, ctypes.byref(comm)),
                   None, "fc_comm_init")
        self._comm = comm
        for name, value in (options or {}).items():
            self.set_option(name, value)
        self._connect()
        self._nvls_base = None
        self._nvls_bytes = 0
        self._nvls_next = 0
        if nvls_bytes and world_size > 1:
            self._setup_nvls(int(nvls_bytes))

    def _connect(self):
        """Exchange workspace handles and map the peers' (collective)."""
        if self.nranks == 1:
            return
        hb = self._lib.fc_handle_bytes()
        mine = ctypes.create_string_buffer(hb)
        _lib.check(self._lib.fc_comm_export(self._comm, mine), self._comm, "comm_export")
        allh = self._allgather_obj(mine.raw)
        blob = ctypes.create_string_buffer(b"".join(allh), hb * self.nranks)
        _lib.check(self._lib.fc_comm_connect(self._comm, blob), self._comm, "comm_connect")

    @property
    def scratch_bytes(self) -> int:
        """Current workspace region size (reduction scratch = LL128 staging)."""
        return int(self._lib.fc_comm_scratch_bytes(self._comm))

    def _ensure_scratch(self, collective: str, count: int, code: int) -> None:
        """Grow the workspace (collectively) when this call's path wants more
        than it holds.  The need depends only on rank-uniform values (size,
        dtype, plan, options), so every rank grows at the same call."""
        key = (collective, count, code)
        if not self._grow or key in self._scratch_ok:
            return
        self.plan(collective)
        need = ctypes.c_size_t()
        _lib.check(self._lib.fc_call_scratch(self._comm, COLL_CODE[collective], count, code,
                                             self._max_scratch, ctypes.byref(need)),
                   self._comm, "call_scratch")
        have = self.scratch_bytes
        if need.value > have:
            if torch.cuda.is_current_stream_capturing():
                raise InvalidArgument(
                    f"{collective} of {count} elements needs a {need.value}-byte workspace "
                    f"(have {have}): run it once outside CUDA-graph capture first")
            target = have
            while target < need.value:
                target *= 2
            self._grow_to(min(target, self._max_scratch))
        if len(self._scratch_ok) > 4096:  # many distinct sizes: keep the memo bounded
            self._scratch_ok.clear()
        self._scratch_ok.add(key)

    def _grow_to(self, nbytes: int) -> None:
        """Collective: every rank's collectives on this communicator have
        completed (device sync + barrier) before the workspaces are
        re-allocated, then handles are exchanged again."""
        import torch.distributed as dist

        torch.cuda.synchronize(self.device)
        self.check()  # a sticky device error must surface, not vanish with the old workspace
        if self._group is not None:
            dist.barrier(group=self._group)
        _lib.check(self._lib.fc_comm_grow(self._comm, int(nbytes)), self._comm, "comm_grow")
        self._paths.clear()  # staging-dependent choices may change with the size
        self._connect()

    # -- NVLS (multicast) engine ----------------------------------------------
    def _setup_nvls(self, nbytes):
        """Collective: bind a symmetric pool to an NVSwitch multicast object.
        Every rank must call with the same size; falls back (pool disabled) on
        all ranks together when any rank lacks multicast support."""
        import torch.distributed as dist

        ok = bool(self._lib.fc_nvls_supported(self.device))
        if not all(self._allgather_obj(ok)):
            return
        import socket
        import struct
        import uuid

        hb = self._lib.fc_handle_bytes()
        blob = ctypes.create_string_buffer(hb)
        srv = None
        if self.rank == 0:
            _lib.check(self._lib.fc_nvls_create(self._comm, nbytes, blob), self._comm, "nvls_create")
            addr = f"\0forestcoll-nvls-{uuid.uuid4().hex}"
            srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            srv.bind(addr)
            srv.listen(self.nranks)
        else:
            addr = None
        blob0, addr = self._allgather_obj((blob.raw, addr))[0]
        h = ctypes.create_string_buffer(blob0, hb)
        # the multicast object travels as a POSIX fd (SCM_RIGHTS over a unix socket)
        if self.rank == 0:
            fd = struct.unpack_from("<i", blob0, 4)[0]
            for _ in range(self.nranks - 1):
                conn, _ = srv.accept()
                socket.send_fds(conn, [b"f"], [fd])
                conn.close()
            srv.close()
        else:
            cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            cli.connect(addr)
            _, fds, _, _ = socket.recv_fds(cli, 1, 1)
            cli.close()
            struct.pack_into("<i", h, 4, fds[0])
        _lib.check(self._lib.fc_nvls_attach(self._comm, h), self._comm, "nvls_attach")
        dist.barrier(group=self._group)
        base = ctypes.c_void_p()
        _lib.check(self._lib.fc_nvls_bind(self._comm, ctypes.byref(base)), self._comm, "nvls_bind")
        dist.barrier(group=self._group)
        self._nvls_base = base.value
        # the top 2 x nvls_ll_half bytes hold the LL multicast staging
        self._nvls_ll_half = self.get_option("nvls_ll_half")
        self._nvls_ll_max = self.get_option("nvls_ll_max")
        self._nvls_ll_red_max = self.get_option("nvls_ll_red_max")
        self._nvls_bytes = nbytes - 2 * self._nvls_ll_half

    @property
    def nvls_enabled(self) -> bool:
        return self._nvls_base is not None

    def nvls_empty(self, numel: int, dtype=torch.float32) -> torch.Tensor:
        """A tensor in the symmetric NVLS pool (bump-allocated: every rank must
        allocate the same sequence of sizes).  Valid while the comm lives."""
        if not self.nvls_enabled:
            raise Unsupported("NVLS pool is not set up (nvls_bytes=0 or no multicast support)")
        es = torch.tensor([], dtype=dtype).element_size()
        off = (self._nvls_next + 4095) // 4096 * 4096
        if off + numel * es > self._nvls_bytes:
            raise InvalidArgument("NVLS pool exhausted")
        self._nvls_next = off + numel * es
        typestr = {1: "|u1", 2: "<i2", 4: "<i4", 8: "<i8"}[es]

        class _CAI:
            pass

        holder = _CAI()
        holder.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr,
                                           "data": (self._nvls_base + off, False), "version": 3}
        t = torch.as_tensor(holder, device=f"cuda:{self.device}")
        return t.view(dtype)

    def _nvls_ll(self, out: torch.Tensor, inp: torch.Tensor) -> bool:
        """Small allgather the NVLS engine runs as LL over multicast (any buffers)."""
        nb = out.numel() * out.element_size()
        sb = inp.numel() * inp.element_size()
        # sizes only (equal on every rank): local pointer alignment must not
        # pick the engine, or ranks could run different kernels
        return (self.nvls_enabled and nb <= self._nvls_ll_max and sb % 8 == 0
                and 2 * nb <= self._nvls_ll_half)

    def _nvls_ll_red(self, inp: torch.Tensor, out: torch.Tensor) -> bool:
        """Small reduce-scatter / allreduce the NVLS engine runs as one LL
        multicast of each input plus a local evaluation of the in-trees."""
        if not self.nvls_enabled:
            return False
        nb = inp.numel() * inp.element_size()
        lim = self._nvls_ll_red_max if out is inp else self._nvls_ll_red_max // self.nranks
        return (nb <= lim and nb % 8 == 0
                and (out.numel() * out.element_size()) % 8 == 0
                and 2 * nb * self.nranks <= self._nvls_ll_half)

    def _in_pool(self, t) -> bool:
        if not self.nvls_enabled:
            return False
        a = t.data_ptr()
        return self._nvls_base <= a and a + t.numel() * t.element_size() <= self._nvls_base + self._nvls_bytes

    def _switch_capable(self, capability: str) -> bool:
        """The topology routes every pair through one switch that declares
        `capability` (multicast / aggregation): the pruned forest then sends
        each shard into the switch once (schedule.py:237-306)."""
        hit = self._capable.get(capability)
        if hit is None:
            sws = [] if self.topology is None else \
                [n for n in self.topology["nodes"] if n["kind"] == "switch"]
            hit = self._capable[capability] = len(sws) == 1 and bool(sws[0].get(capability, False))
        return hit

    def _usable_topology(self, doc, world_size):
        """An NVML topology whose schedule is neither cached nor generatable
        here (no reference generator on this machine) falls back, on every
        rank alike, to the nominal NVSwitch model when NVML shows a single
        switch (the forest shape of a uniform NVSwitch does not depend on
        the bandwidth value)."""
        from .generator import cache_key, _cache_paths
        from ._refpath import import_collsched

        cached = any(os.path.exists(p) for p in _cache_paths(cache_key(doc, ALLGATHER, self._prune_default)))
        ok = cached or import_collsched() is not None
        if all(self._allgather_obj(ok)):
            return doc
        nominal = nvswitch_doc(world_size)
        switches = [n for n in doc["nodes"] if n["kind"] == "switch"]
        if len(switches) == 1:
            self.topology_source = "nvml->nominal (schedule not cached, no generator)"
            return nominal
        return doc

    def _allgather_obj(self, obj):
        import torch.distributed as dist

        if self._group is None:
            return [obj]
        out = [None] * self.nranks
        dist.all_gather_object(out, obj, group=self._group)
        return out

    # -- buffers ------------------------------------------------------------
    def register(self, t: torch.Tensor) -> None:
        """Map the allocation (cudaMalloc segment) holding `t` into every peer.
        Collective: all ranks call together.  Nothing is pinned: the
        registration is keyed by the driver's buffer id and tracks the
        segment, so the caching allocator's reuse of it costs nothing and a
        freed-and-reused address range is recognised as new."""
        if self.nranks == 1:
            return
        nbytes = t.numel() * t.element_size()
        hb = self._lib.fc_handle_bytes()
        mine = ctypes.create_string_buffer(hb)
        _lib.check(self._lib.fc_buffer_export(self._comm, t.data_ptr(), nbytes, mine), self._comm,
                   "buffer_export")
        allh = self._allgather_obj(mine.raw)
        blob = ctypes.create_string_buffer(b"".join(allh), hb * self.nranks)
        _lib.check(self._lib.fc_buffer_register(self._comm, t.data_ptr(), nbytes, blob), self._comm,
                   "buffer_register")

    def _ensure_registered(self, collective: str, out: torch.Tensor, count: int, code: int) -> None:
        """Register `out`'s allocation when this call takes the chunk-flag
        path, the only one that stores into peers' outputs (fc_call_path; the
        one-hop, one-shot and LL128 paths write only the library's staging).
        The path is the same on every rank; registration is per allocator
        segment, so it happens once per segment, not per call."""
        if self.nranks == 1 or self._call_path(collective, count, code) not in (0, 5):
            return
        have = ctypes.c_int()
        _lib.check(self._lib.fc_buffer_query(self._comm, out.data_ptr(),
                                             out.numel() * out.element_size(), ctypes.byref(have)),
                   self._comm, "buffer_query")
        # Registered here: SPMD programs allocate outputs in the same order on
        # every rank, so every rank finds its own (equally placed) output
        # registered and no host round trip is spent per call.  A rank that
        # passes a differently placed buffer fails the device tag check.
        if not have.value:
            self.register(out)  # collective: SPMD ranks all reach this call together

    def _call_path(self, collective: str, count: int, code: int) -> int:
        """fc_call_path: 0 chunk flags, 1 LL128, 4 one-hop / one-shot, 5 copy
        engine, 7 two-hop, -1 empty.  Memoised per (collective, count, dtype):
        the answer changes only with the options or the workspace size, which
        clear the memo."""
        key = (collective, count, code)
        path = self._paths.get(key)
        if path is not None:
            return path
        self.plan(collective)
        out = ctypes.c_int()
        _lib.check(self._lib.fc_call_path(self._comm, COLL_CODE[collective], count, code,
                                          ctypes.byref(out)), self._comm, "call_path")
        if len(self._paths) > 4096:
            self._paths.clear()
        self._paths[key] = out.value
        return out.value

    def _switch_order(self, order) -> bool:
        order = self.reduction_order if order is None else order
        if order not in ("tree", "switch"):
            raise InvalidArgument("order must be 'tree' or 'switch'")
        return order == "switch"

    def registration_count(self) -> int:
        """Live peer registrations (one per allocator segment, never per tensor)."""
        return int(self._lib.fc_buffer_count(self._comm))

    def deregister(self, t: torch.Tensor) -> None:
        """Drop the peer mapping of the allocation holding `t` (local)."""
        self._lib.fc_buffer_deregister(self._comm, t.data_ptr())

    def empty(self, *shape, dtype=torch.float32) -> torch.Tensor:
        t = torch.empty(*shape, dtype=dtype, device=f"cuda:{self.device}")
        self.register(t)
        return t

    def _stream(self):
        return _raw_stream(self.device)

    # -- collectives --------------------------------------------------------
    def all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> torch.Tensor:
        """out[r*S:(r+1)*S] = inp of rank r (NCCL all_gather_into_tensor)."""
        self._check_tensor(inp, self.device, "input")
        self._check_tensor(out, self.device, "output")
        if out.dtype != inp.dtype or out.numel() != inp.numel() * self.nranks:
            raise InvalidArgument("output must hold world_size x input elements of the same dtype")
        count, code = _dtype_args(inp, inp.numel())
        if (self._in_pool(out) or self._nvls_ll(out, inp)) and self._switch_capable("multicast"):
            self.schedule(ALLGATHER)
            src, dst = _aligned(inp), _aligned(out)
            _lib.check(self._lib.fc_nvls_allgather(self._comm, src.data_ptr(), dst.data_ptr(),
                                                   count, code, self._stream()),
                       self._comm, "nvls_allgather")
            if dst is not out:
                out.copy_(dst)
            return out
        self.plan(ALLGATHER)
        self._ensure_scratch(ALLGATHER, count, code)
        self._ensure_registered(ALLGATHER, out, count, code)
        _lib.check(self._lib.fc_allgather(self._comm, inp.data_ptr(), out.data_ptr(), count, code,
                                          self._stream()), self._comm, "allgather")
        return out

    all_gather_into_tensor = all_gather

    def reduce_scatter(self, out: torch.Tensor, inp: torch.Tensor, op="sum",
                       order=None) -> torch.Tensor:
        """out = sum over ranks of inp[rank*S:(rank+1)*S] (reduce_scatter_tensor).

        `order` ("tree" / "switch", default the communicator's
        reduction_order): "switch" lets an input in the NVLS pool be reduced
        inside the NVSwitch, in the switch's summation order."""
        self._check_tensor(inp, self.device, "input")
        self._check_tensor(out, self.device, "output")
        if out.dtype != inp.dtype or inp.numel() != out.numel() * self.nranks:
            raise InvalidArgument("input must hold world_size x output elements of the same dtype")
        if inp.dtype not in REDUCIBLE:
            raise Unsupported(f"dtype {inp.dtype} cannot be reduced")
        switch = self._switch_order(order) and self._in_pool(inp)
        if (switch or self._nvls_ll_red(inp, out)) and self._switch_capable("aggregation"):
            self.plan(REDUCE_SCATTER)  # the LL path evaluates the plan's in-trees
            src, dst = (inp, out) if switch else (_aligned(inp), _aligned(out))
            _lib.check(self._lib.fc_nvls_reduce_scatter(
                self._comm, src.data_ptr(), dst.data_ptr(), out.numel(), DTYPE_CODE[inp.dtype],
                _op_code(op), self._stream()), self._comm, "nvls_reduce_scatter")
            if dst is not out:
                out.copy_(dst)
            self._last_order = "switch" if switch else "tree"
            return out
        self._last_order = "tree"
        self.plan(REDUCE_SCATTER)
        self._ensure_scratch(REDUCE_SCATTER, out.numel(), DTYPE_CODE[inp.dtype])
        _lib.check(self._lib.fc_reduce_scatter(self._comm, inp.data_ptr(), out.data_ptr(),
                                               out.numel(), DTYPE_CODE[inp.dtype], _op_code(op),
                                               self._stream()), self._comm, "reduce_scatter")
        return out

    reduce_scatter_tensor = reduce_scatter

    def all_reduce(self, buf: torch.Tensor, op="sum", out: torch.Tensor | None = None,
                   order=None) -> torch.Tensor:
        """In-place (or into `out`) sum over ranks.  `order` as in
        reduce_scatter: "switch" (opt-in) reduces NVLS-pool buffers inside
        the NVSwitch; "tree" (default) keeps the forest's order everywhere."""
        out = buf if out is None else out
        self._check_tensor(buf, self.device, "buffer")
        self._check_tensor(out, self.device, "output")
        if out.dtype != buf.dtype or out.numel() != buf.numel():
            raise InvalidArgument("output must match the buffer")
        if buf.dtype not in REDUCIBLE:
            raise Unsupported(f"dtype {buf.dtype} cannot be reduced")
        switch = self._switch_order(order) and self._in_pool(buf)
        if (out is buf and (switch or self._nvls_ll_red(buf, buf))
                and self._switch_capable("multicast") and self._switch_capable("aggregation")):
            self.plan(ALLREDUCE)  # the LL path evaluates the plan's in-trees
            b2 = buf if switch else _aligned(buf)
            _lib.check(self._lib.fc_nvls_allreduce(self._comm, b2.data_ptr(), buf.numel(),
                                                   DTYPE_CODE[buf.dtype], _op_code(op),
                                                   self._stream()), self._comm, "nvls_allreduce")
            if b2 is not buf:
                buf.copy_(b2)
            self._last_order = "switch" if switch else "tree"
            return out
        self._last_order = "tree"
        if self._in_pool(out) and self._call_path(ALLREDUCE, buf.numel(), DTYPE_CODE[buf.dtype]) == 0:
            # tree order on a pool tensor at chunk-flag sizes: peers store into
            # the output, which must be IPC-registrable (the pool's VMM memory
            # is not) -- run into an ordinary buffer and copy back
            tmp = torch.empty_like(out)
            self.all_reduce(buf, op=op, out=tmp, order="tree")
            out.copy_(tmp)
            return out
        self.plan(ALLREDUCE)
        self._ensure_scratch(ALLREDUCE, buf.numel(), DTYPE_CODE[buf.dtype])
        self._ensure_registered(ALLREDUCE, out, buf.numel(), DTYPE_CODE[buf.dtype])
        _lib.check(self._lib.fc_allreduce(self._comm, buf.data_ptr(), out.data_ptr(), buf.numel(),
                                          DTYPE_CODE[buf.dtype], _op_code(op), self._stream()),
                   self._comm, "allreduce")
        return out


class VirtualComm(_CommBase):
    """All N ranks of a forest executed by one cooperative grid on one GPU.

    Rank r's buffers are ordinary tensors on the same device; "peer" stores
    land in local HBM.  Same kernel, tables, flags and chunking as the
    multi-GPU path (SURVEY.md §4 "virtual ranks" mode).
    """

    def __init__(self, topology=None, *, nranks=None, device=0, scratch_bytes=VIRTUAL_SCRATCH,
                 schedules=None, validate=True, prune=True, options=None):
        doc = _as_doc(topology)
        if doc is None:
            if schedules:
                any_s = next(iter(schedules.values()))
                nranks = any_s.num_compute
            elif nranks is not None:
                doc = nvswitch_doc(nranks)
            else:
                raise InvalidArgument("need a topology, schedules or nranks")
        if doc is not None:
            nranks = len(compute_ids(doc))
        self.device = device
        super().__init__(doc, nranks, schedules, validate, prune)
        comm = ctypes.c_void_p()
        _lib.check(self._lib.fc_comm_init_virtual(nranks, device, int(scratch_bytes),
                                                  ctypes.byref(comm)), None, "fc_comm_init_virtual")
        self._comm = comm
        for name, value in (options or {}).items():
            self.set_option(name, value)

    def _ptrs(self, ts, name):
        if len(ts) != self.nranks:
            raise InvalidArgument(f"need {self.nranks} {name} tensors, got {len(ts)}")
        for t in ts:
            self._check_tensor(t, self.device, name)
        arr = (ctypes.c_void_p * self.nranks)(*[t.data_ptr() for t in ts])
        return arr

    def _stream(self):
        return _raw_stream(self.device)

    def all_gather(self, outs, inps):
        for o, i in zip(outs, inps):
            if o.dtype != i.dtype or o.numel() != i.numel() * self.nranks or i.numel() != inps[0].numel():
                raise InvalidArgument("each output must hold nranks x input elements")
        self.plan(ALLGATHER)
        count, code = _dtype_args(inps[0], inps[0].numel())
        _lib.check(self._lib.fc_allgather_multi(self._comm, self._ptrs(inps, "input"),
                                                self._ptrs(outs, "output"), count, code,
                                                self._stream()), self._comm, "allgather")
        return outs

    def reduce_scatter(self, outs, inps, op="sum"):
        self._last_order = "tree"
        for o, i in zip(outs, inps):
            if o.dtype != i.dtype or i.numel() != o.numel() * self.nranks or o.numel() != outs[0].numel():
                raise InvalidArgument("each input must hold nranks x output elements")
        if inps[0].dtype not in REDUCIBLE:
            raise Unsupported(f"dtype {inps[0].dtype} cannot be reduced")
        self.plan(REDUCE_SCATTER)
        _lib.check(self._lib.fc_reduce_scatter_multi(
            self._comm, self._ptrs(inps, "input"), self._ptrs(outs, "output"), outs[0].numel(),
            DTYPE_CODE[inps[0].dtype], _op_code(op), self._stream()), self._comm, "reduce_scatter")
        return outs

    def all_reduce(self, bufs, op="sum", outs=None):
        self._last_order = "tree"
        outs = bufs if outs is None else outs
        for o, b in zip(outs, bufs):
            if o.dtype != b.dtype or o.numel() != b.numel() or b.numel() != bufs[0].numel():
                raise InvalidArgument("buffers must all have the same size and dtype")
        if bufs[0].dtype not in REDUCIBLE:
            raise Unsupported(f"dtype {bufs[0].dtype} cannot be reduced")
        self.plan(ALLREDUCE)
        _lib.check(self._lib.fc_allreduce_multi(
            self._comm, self._ptrs(bufs, "buffer"), self._ptrs(outs, "output"), bufs[0].numel(),
            DTYPE_CODE[bufs[0].dtype], _op_code(op), self._stream()), self._comm, "allreduce")
        return outs


class MultiRankComm(_CommBase):
    """Several ranks of one forest per process / GPU (one cooperative grid),
    connected over NVLink to the ranks of other processes.

    Used to run forests with more ranks than GPUs (e.g. the 8-GPU NVSwitch
    forest on 4 GPUs, 2 ranks each) through real peer memory.  Collectives
    take one tensor per local rank, like VirtualComm.
    """

    def __init__(self, topology, *, local_ranks, world_size, device=None, group=None,
                 scratch_bytes=VIRTUAL_SCRATCH, schedules=None, validate=True, prune=True,
                 options=None):
        import torch.distributed as dist

        doc = _as_doc(topology)
        self.device = int(os.environ.get("LOCAL_RANK", 0)) if device is None else device
        self.local_ranks = tuple(local_ranks)
        self.nranks = world_size
        self._group = group if group is not None else dist.new_group(backend="gloo")
        super().__init__(doc, world_size, schedules, validate, prune)
        comm = ctypes.c_void_p()
        arr = (ctypes.c_int * len(self.local_ranks))(*self.local_ranks)
        _lib.check(self._lib.fc_comm_init_ranks(arr, len(self.local_ranks), world_size,
                                                self.device, int(scratch_bytes),
                                                ctypes.byref(comm)), None, "fc_comm_init_ranks")
        self._comm = comm
        for name, value in (options or {}).items():
            self.set_option(name, value)
        hb = self._lib.fc_handle_bytes()
        mine = ctypes.create_string_buffer(hb * len(self.local_ranks))
        _lib.check(self._lib.fc_comm_export(self._comm, mine), self._comm, "comm_export")
        blobs = self._gather_by_rank(mine.raw, hb)
        _lib.check(self._lib.fc_comm_connect(self._comm, ctypes.create_string_buffer(blobs, len(blobs))),
                   self._comm, "comm_connect")

    def _gather_by_rank(self, raw, hb):
        import torch.distributed as dist

        out = [None] * dist.get_world_size(self._group)
        dist.all_gather_object(out, (self.local_ranks, raw), group=self._group)
        per = {}
        for ranks, blob in out:
            for i, r in enumerate(ranks):
                per[r] = blob[i * hb:(i + 1) * hb]
        return b"".join(per[r] for r in range(self.nranks))

    def _register(self, outs, collective, count, code):
        """Register the local ranks' output allocations when the call takes the
        chunk-flag path (see ForestCollComm._ensure_registered)."""
        path = ctypes.c_int()
        _lib.check(self._lib.fc_call_path(self._comm, COLL_CODE[collective], count, code,
                                          ctypes.byref(path)), self._comm, "call_path")
        if path.value != 0:
            return
        nbytes = outs[0].numel() * outs[0].element_size()
        have = ctypes.c_int(1)
        for t in outs:
            h = ctypes.c_int()
            _lib.check(self._lib.fc_buffer_query(self._comm, t.data_ptr(), nbytes, ctypes.byref(h)),
                       self._comm, "buffer_query")
            have.value &= h.value
        import torch.distributed as dist

        flags = [None] * dist.get_world_size(self._group)
        dist.all_gather_object(flags, not have.value, group=self._group)
        if not any(flags):
            return
        hb = self._lib.fc_handle_bytes()
        ptrs = (ctypes.c_void_p * len(outs))(*[t.data_ptr() for t in outs])
        mine = ctypes.create_string_buffer(hb * len(outs))
        _lib.check(self._lib.fc_buffer_export_multi(self._comm, ptrs, nbytes, mine), self._comm,
                   "buffer_export")
        blobs = self._gather_by_rank(mine.raw, hb)
        _lib.check(self._lib.fc_buffer_register_multi(self._comm, ptrs, nbytes,
                                                      ctypes.create_string_buffer(blobs, len(blobs))),
                   self._comm, "buffer_register")

    def _ptrs(self, ts, name):
        if len(ts) != len(self.local_ranks):
            raise InvalidArgument(f"need {len(self.local_ranks)} {name} tensors, got {len(ts)}")
        for t in ts:
            self._check_tensor(t, self.device, name)
        return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])

    def _stream(self):
        return _raw_stream(self.device)

    def all_gather(self, outs, inps):
        self.plan(ALLGATHER)
        count, code = _dtype_args(inps[0], inps[0].numel())
        self._register(outs, ALLGATHER, count, code)
        _lib.check(self._lib.fc_allgather_multi(self._comm, self._ptrs(inps, "input"),
                                                self._ptrs(outs, "output"), count, code,
                                                self._stream()), self._comm, "allgather")
        return outs

    def reduce_scatter(self, outs, inps, op="sum"):
        self._last_order = "tree"
        self.plan(REDUCE_SCATTER)
        _lib.check(self._lib.fc_reduce_scatter_multi(
            self._comm, self._ptrs(inps, "input"), self._ptrs(outs, "output"), outs[0].numel(),
            DTYPE_CODE[inps[0].dtype], _op_code(op), self._stream()), self._comm, "reduce_scatter")
        return outs

    def all_reduce(self, bufs, op="sum"):
        self._last_order = "tree"
        self.plan(ALLREDUCE)
        self._register(bufs, ALLREDUCE, bufs[0].numel(), DTYPE_CODE[bufs[0].dtype])
        _lib.check(self._lib.fc_allreduce_multi(
            self._comm, self._ptrs(bufs, "buffer"), self._ptrs(bufs, "buffer"), bufs[0].numel(),
            DTYPE_CODE[bufs[0].dtype], _op_code(op), self._stream()), self._comm, "allreduce")
        return bufs


class Executor:
    """§8b surface: ``Executor(schedule_or_path, topology, rank, world, device)``.

    Accepts a reference ``Schedule``, its JSON text, or a path to the JSON
    (``parse_schedule``, schedule.py:439-448); with a topology it validates
    the schedule against it (``validate_schedule``, verify.py:478-534) before
    lowering, as the reference CLI does.  ``virtual=True`` executes all ranks
    on one device; other keywords (options, reduction_order, ...) go to the
    communicator.
    """

    def __init__(self, schedule_or_path, topology=None, rank=None, world=None, device=None,
                 virtual=False, **kw):
        s = schedule_or_path
        if isinstance(s, str):
            s = load_schedule(s) if os.path.exists(s) else parse_schedule_json(s)
        doc = _as_doc(topology)
        if doc is not None and kw.get("validate", True):
            preflight(s, doc)
        scheds = {s.collective: s}
        self.collective = s.collective
        if virtual:
            self.comm = VirtualComm(doc, device=device or 0, schedules=scheds, **kw)
        else:
            self.comm = ForestCollComm(doc, rank=rank, world_size=world, device=device,
                                       schedules=scheds, **kw)

    def all_gather(self, out, inp):
        return self.comm.all_gather(out, inp)

    def reduce_scatter(self, out, inp, op="sum"):
        return self.comm.reduce_scatter(out, inp, op)

    def all_reduce(self, buf, op="sum"):
        return self.comm.all_reduce(buf, op)

    def close(self):
        self.comm.close()
