"""The C-ABI library builds for sm_100a, loads without a GPU and exports
every entry point include/forestcoll.h declares.  No compute calls here."""

import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "forestcoll.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2402_06787_b200 import _lib, build

    build.build()
    return _lib.load()


def declared():
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|size_t|int)\s+(fc_\w+)\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for required in ("fc_comm_init", "fc_comm_connect", "fc_plan_load", "fc_allgather",
                     "fc_reduce_scatter", "fc_allreduce", "fc_comm_destroy", "fc_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared():
        assert hasattr(lib, name), name
    from paper_2402_06787_b200 import _lib

    assert set(declared()) == set(_lib.SIGNATURES)


def test_version_and_handle_size(lib):
    assert b"sm_100a" in lib.fc_version()
    assert lib.fc_handle_bytes() >= 64 + 64


def test_sass_is_sm100a():
    from paper_2402_06787_b200 import build

    import shutil
    import subprocess

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    out = subprocess.run(["cuobjdump", "--list-elf", build.OUT], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_arguments_are_rejected_without_gpu(lib):
    assert lib.fc_allgather(None, None, None, 0, 7, None) != 0
    assert lib.fc_comm_destroy(None) == 0
    assert lib.fc_last_error(None) == b"null communicator"


def test_error_codes_map_to_collsched_errors():
    from paper_2402_06787_b200 import _lib, errors

    assert issubclass(errors.ExecutorError, errors.CollschedError)
    with pytest.raises(errors.NotRegistered):
        _lib.check(4, None, "x")
    with pytest.raises(errors.PlanError):
        _lib.check(5, None, "x")


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(REPO, "paper_2402_06787_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                with open(os.path.join(root, f)) as fh:
                    src = fh.read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f


def test_python_option_and_op_codes_match_the_header():
    """Option numbers, reduction-op codes and dtype codes in the ctypes binding
    and the executor are the ones include/forestcoll.h defines."""
    from paper_2402_06787_b200 import _lib
    from paper_2402_06787_b200.executor import DTYPE_CODE, OPS

    with open(HEADER) as f:
        text = f.read()
    defs = {k: int(v) for k, v in re.findall(r"^#define (FC_\w+) (\d+)", text, re.M)}
    opts = {k[len("FC_OPT_"):].lower(): v for k, v in defs.items() if k.startswith("FC_OPT_")}
    assert opts == _lib.OPTIONS
    assert OPS == {"sum": defs["FC_SUM"], "avg": defs["FC_AVG"]}
    names = {"int8": "FC_INT8", "uint8": "FC_UINT8", "int32": "FC_INT32", "int64": "FC_INT64",
             "float16": "FC_FLOAT16", "float32": "FC_FLOAT32", "float64": "FC_FLOAT64",
             "bfloat16": "FC_BFLOAT16"}
    for dt, code in DTYPE_CODE.items():
        name = str(dt).split(".")[-1]
        if name in names:
            assert code == defs[names[name]], name
