"""Shared fixtures.  `gpu` marks tests that need a B200 (run with -m gpu)."""

import glob
import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    """A hung device wait must not hang the run: every GPU test gets a
    generous wall-clock limit (pytest-timeout) unless it sets its own; the
    kernels' own flag-wait timeouts fire well before it."""
    if not config.pluginmanager.hasplugin("timeout"):
        return
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(1800))


def golden_names(collective=None):
    names = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "schedules", "*.json"))):
        name = os.path.basename(p)[:-5]
        if collective is None or name.endswith("_" + collective):
            names.append(name)
    return names


def load_golden(name):
    """Golden schedule, parsed by the reference's own parse_schedule
    (schedule.py:439-448) from the baseline/_ref install."""
    from paper_2402_06787_b200.schedule_io import load_schedule

    return load_schedule(os.path.join(GOLDEN, "schedules", name + ".json"))


def load_golden_topology(name):
    with open(os.path.join(GOLDEN, "topologies", name + ".json")) as f:
        return json.load(f)


def reference_collsched():
    """The reference package for CPU-only cross checks (None if absent)."""
    try:
        import collsched  # noqa: F401

        return collsched
    except ImportError:
        pass
    for p in ("/root/reference/pkg/src", os.path.join(REPO, "baseline", "_ref")):
        if os.path.isdir(os.path.join(p, "collsched")):
            sys.path.insert(0, p)
            import collsched

            return collsched
    return None
