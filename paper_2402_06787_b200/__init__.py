"""B200-native executor for ForestColl schedules (arxiv 2402.06787).

The reference ``collsched`` package generates throughput-optimal spanning-tree
forests; this package executes them on GPU buffers with a persistent sm_100a
kernel.  Public surface:

* ``ForestCollComm`` — one rank per process: ``all_gather``,
  ``reduce_scatter``, ``all_reduce`` on CUDA tensors.
* ``VirtualComm`` — all ranks of a forest on one GPU (testing / benchmarks).
* ``Executor`` — schedule-in, collectives-out wrapper.
* ``topology`` — NVML ingestion and the reference-format builders.
"""

from .errors import (  # noqa: F401
    CollschedError, DeviceError, ExecutorError, InvalidArgument, NativeLibraryMissing,
    NotRegistered, PlanError, Unsupported,
)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent classes load lazily so the host-side modules (topology,
    # compiler, generator) import without torch or a GPU.
    if name in ("ForestCollComm", "VirtualComm", "MultiRankComm", "Executor"):
        from . import executor

        return getattr(executor, name)
    raise AttributeError(name)
