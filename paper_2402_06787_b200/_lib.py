"""ctypes binding of the C ABI (include/forestcoll.h).

The library is built in-tree (``paper_2402_06787_b200/lib/libforestcoll.so``,
see build.py).  There is no fallback: if it is missing every collective
raises ``NativeLibraryMissing``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import FC_CODES, DeviceError, NativeLibraryMissing

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.path.join(LIB_DIR, "libforestcoll.so")

FC_ALLGATHER, FC_REDUCE_SCATTER, FC_ALLREDUCE = 0, 1, 2
FC_SUM = 0
OPT_CTAS_PER_RANK, OPT_CHUNK_MAX, OPT_CHUNK_MIN, OPT_ITEMS_PER_WORKER, OPT_TIMEOUT_MS = 1, 2, 3, 4, 5
OPT_LAG, OPT_COPY_MODE, OPT_DMA_ROOT_COPY, OPT_WORKER_WARPS = 6, 7, 8, 9
OPT_PROTO, OPT_LL_MAX, OPT_LL_CHUNK_MAX, OPT_LL_WORKER_WARPS, OPT_NVLS_CTAS = 10, 11, 12, 13, 14
OPT_PDL, OPT_CHUNK_TAIL, OPT_NVLS_LL_MAX, OPT_NVLS_LL_HALF, OPT_NVLS_LL_RED_MAX = 15, 16, 17, 18, 19
OPT_ONESHOT_MAX, OPT_ONESHOT_AG_MAX, OPT_MAX_CTAS_PER_RANK = 20, 21, 22
OPT_CE_MIN, OPT_TWOHOP_MAX = 23, 25
OPTIONS = {
    "ctas_per_rank": OPT_CTAS_PER_RANK,
    "chunk_max": OPT_CHUNK_MAX,
    "chunk_min": OPT_CHUNK_MIN,
    "items_per_worker": OPT_ITEMS_PER_WORKER,
    "timeout_ms": OPT_TIMEOUT_MS,
    "lag": OPT_LAG,
    "copy_mode": OPT_COPY_MODE,
    "dma_root_copy": OPT_DMA_ROOT_COPY,
    "worker_warps": OPT_WORKER_WARPS,
    "proto": OPT_PROTO,
    "ll_max": OPT_LL_MAX,
    "ll_chunk_max": OPT_LL_CHUNK_MAX,
    "ll_worker_warps": OPT_LL_WORKER_WARPS,
    "nvls_ctas": OPT_NVLS_CTAS,
    "pdl": OPT_PDL,
    "chunk_tail": OPT_CHUNK_TAIL,
    "nvls_ll_max": OPT_NVLS_LL_MAX,
    "nvls_ll_half": OPT_NVLS_LL_HALF,
    "nvls_ll_red_max": OPT_NVLS_LL_RED_MAX,
    "oneshot_max": OPT_ONESHOT_MAX,
    "oneshot_ag_max": OPT_ONESHOT_AG_MAX,
    "max_ctas_per_rank": OPT_MAX_CTAS_PER_RANK,
    "ce_min": OPT_CE_MIN,
    "twohop_max": OPT_TWOHOP_MAX,
}

# symbol -> (restype, argtypes)
_P = ctypes.c_void_p
_I = ctypes.c_int
_SZ = ctypes.c_size_t
_LL = ctypes.c_longlong
SIGNATURES = {
    "fc_version": (ctypes.c_char_p, []),
    "fc_handle_bytes": (_SZ, []),
    "fc_comm_init": (_I, [_I, _I, _I, _SZ, ctypes.POINTER(_P)]),
    "fc_comm_init_virtual": (_I, [_I, _I, _SZ, ctypes.POINTER(_P)]),
    "fc_comm_init_ranks": (_I, [_P, _I, _I, _I, _SZ, ctypes.POINTER(_P)]),
    "fc_buffer_export_multi": (_I, [_P, _P, _SZ, _P]),
    "fc_buffer_register_multi": (_I, [_P, _P, _SZ, _P]),
    "fc_comm_export": (_I, [_P, _P]),
    "fc_comm_connect": (_I, [_P, _P]),
    "fc_comm_set_option": (_I, [_P, _I, _LL]),
    "fc_comm_get_option": (_I, [_P, _I, ctypes.POINTER(_LL)]),
    "fc_comm_check": (_I, [_P, ctypes.POINTER(_I)]),
    "fc_comm_destroy": (_I, [_P]),
    "fc_last_error": (ctypes.c_char_p, [_P]),
    "fc_buffer_export": (_I, [_P, _P, _SZ, _P]),
    "fc_buffer_register": (_I, [_P, _P, _SZ, _P]),
    "fc_buffer_deregister": (_I, [_P, _P]),
    "fc_buffer_query": (_I, [_P, _P, _SZ, ctypes.POINTER(_I)]),
    "fc_buffer_count": (_I, [_P]),
    "fc_call_path": (_I, [_P, _I, _SZ, _I, ctypes.POINTER(_I)]),
    "fc_call_scratch": (_I, [_P, _I, _SZ, _I, _SZ, ctypes.POINTER(_SZ)]),
    "fc_comm_scratch_bytes": (_SZ, [_P]),
    "fc_comm_grow": (_I, [_P, _SZ]),
    "fc_plan_load": (_I, [_P, _I, ctypes.POINTER(ctypes.c_int32), _SZ]),
    "fc_allgather": (_I, [_P, _P, _P, _SZ, _I, _P]),
    "fc_reduce_scatter": (_I, [_P, _P, _P, _SZ, _I, _I, _P]),
    "fc_allreduce": (_I, [_P, _P, _P, _SZ, _I, _I, _P]),
    "fc_allgather_multi": (_I, [_P, _P, _P, _SZ, _I, _P]),
    "fc_reduce_scatter_multi": (_I, [_P, _P, _P, _SZ, _I, _I, _P]),
    "fc_allreduce_multi": (_I, [_P, _P, _P, _SZ, _I, _I, _P]),
    "fc_last_call_info": (_I, [_P, ctypes.POINTER(_LL), _I]),
    "fc_comm_set_trace": (_I, [_P, _P, _P, ctypes.c_uint]),
    "fc_nvls_supported": (_I, [_I]),
    "fc_nvls_create": (_I, [_P, _SZ, _P]),
    "fc_nvls_attach": (_I, [_P, _P]),
    "fc_nvls_bind": (_I, [_P, ctypes.POINTER(_P)]),
    "fc_nvls_allgather": (_I, [_P, _P, _P, _SZ, _I, _P]),
    "fc_nvls_reduce_scatter": (_I, [_P, _P, _P, _SZ, _I, _I, _P]),
    "fc_nvls_allreduce": (_I, [_P, _P, _SZ, _I, _I, _P]),
}

_LIB = []


def load():
    """Load (once) and return the ctypes library handle."""
    if _LIB:
        return _LIB[0]
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (the executor has no CPU or eager fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB.append(lib)
    return lib


def check(code: int, comm=None, what: str = "") -> None:
    if code == 0:
        return
    lib = load()
    msg = lib.fc_last_error(comm).decode() if comm else ""
    exc = FC_CODES.get(code, DeviceError)
    raise exc(f"{what}: {msg}" if what else msg)
