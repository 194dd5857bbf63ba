"""Locate the reference generator package (`collsched`) without vendoring it.

The generator stays the reference's own Python (BASELINE.json north_star
item 1).  It is imported, never copied: from the interpreter path, from the
offline install under ``<repo>/baseline/_ref``, or from a
directory named by ``FORESTCOLL_REF_PATH``.  Returns None when absent; callers
then work from cached schedule JSON (generator.py).
"""

from __future__ import annotations

import importlib
import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CACHED = []


def candidate_paths() -> list[str]:
    paths = []
    env = os.environ.get("FORESTCOLL_REF_PATH")
    if env:
        paths.append(env)
    paths.append(os.path.join(_REPO, "baseline", "_ref"))
    return paths


def import_collsched():
    if _CACHED:
        return _CACHED[0]
    mod = None
    try:
        mod = importlib.import_module("collsched")
    except ImportError:
        for p in candidate_paths():
            if os.path.isdir(os.path.join(p, "collsched")):
                sys.path.insert(0, p)
                try:
                    mod = importlib.import_module("collsched")
                    break
                except ImportError:
                    sys.path.remove(p)
    _CACHED.append(mod)
    return mod


def require_collsched():
    """The reference package, or ``ReferenceMissing``.  Schedules are always
    the reference's own objects (parse_schedule / export, schedule.py:439-482):
    there is no private reader to fall back to."""
    mod = import_collsched()
    if mod is None:
        from .errors import ReferenceMissing

        raise ReferenceMissing(
            "the reference package `collsched` is not importable: install it with "
            "`python -m pip install --no-index --no-build-isolation --find-links "
            "/opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>` "
            "or point FORESTCOLL_REF_PATH at it"
        )
    return mod
