"""ctypes front-end of oracle/forest_oracle.c (test infrastructure only).

Flattens a reference ``Schedule`` into per-tree arrays by walking its own
fields (roots -> batches -> edges), independently of the product compiler.
"""

from __future__ import annotations

import ctypes
import os
from collections import deque

import numpy as np

from . import build as _build
from .forest_oracle import rank_order, trees

_LIB = []


def lib():
    if not _LIB:
        path = _build.build()
        L = ctypes.CDLL(path)
        P = ctypes.c_void_p
        L.fo_allgather.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P, P, P, P,
                                   ctypes.c_longlong, ctypes.c_int, ctypes.c_int]
        _LIB.append(L)
    return _LIB[0]


class FlatForest:
    def __init__(self, schedule):
        ids = rank_order(schedule)
        pos = {x: i for i, x in enumerate(ids)}
        n = len(ids)
        rows = list(trees(schedule, reverse=False))
        self.n, self.k, self.ntrees = n, schedule.k, len(rows)
        self.root = np.array([pos[r] for r, _, _, _ in rows], dtype=np.int32)
        self.mlo = np.array([lo for _, lo, _, _ in rows], dtype=np.int32)
        self.mhi = np.array([hi for _, _, hi, _ in rows], dtype=np.int32)
        self.parent = np.full((len(rows), n), -1, dtype=np.int32)
        self.order = np.zeros((len(rows), n), dtype=np.int32)
        for t, (r, _, _, kids) in enumerate(rows):
            q, seen = deque([r]), []
            while q:
                u = q.popleft()
                seen.append(pos[u])
                for v in kids.get(u, ()):
                    self.parent[t, pos[v]] = pos[u]
                    q.append(v)
            self.order[t] = seen


def allgather(forest: FlatForest, sends, recvs, threads=None):
    """sends / recvs: lists of numpy arrays (any dtype), recvs preallocated."""
    threads = threads or os.cpu_count() or 1
    n = forest.n
    sp = (ctypes.c_void_p * n)(*[s.ctypes.data for s in sends])
    rp = (ctypes.c_void_p * n)(*[r.ctypes.data for r in recvs])
    lib().fo_allgather(n, forest.ntrees, forest.k, forest.root.ctypes.data,
                       forest.mlo.ctypes.data, forest.mhi.ctypes.data, forest.order.ctypes.data,
                       forest.parent.ctypes.data, sp, rp, sends[0].size, sends[0].itemsize,
                       threads)
    return recvs
