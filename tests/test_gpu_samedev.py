"""The production (one process per rank) path on a single B200.

Two rank processes share cuda:0, each with its own CUDA context, so the
communicator runs exactly as on two GPUs: CUDA IPC workspace and output
mappings opened from another process, the entry barrier with the
output-buffer tag check, PDL, registration only on the chunk-flag path,
and the one-hop / one-shot kernels outside virtual mode.  Results are
compared bit-for-bit with the CPU oracle (tests/mp/samedev_worker.py).
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def _launch(mode, n=2, port=29650, timeout=600):
    if not _have_gpu():
        pytest.skip("no CUDA device")
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(HERE, "mp", "samedev_worker.py"), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    return r.returncode, r.stdout + r.stderr


def test_two_processes_one_gpu_parity():
    rc, out = _launch("parity", port=29651)
    assert rc == 0 and out.count(" OK") >= 2, out[-4000:]


def test_fresh_outputs_do_not_grow_registrations():
    rc, out = _launch("fresh_outputs", port=29652)
    assert rc == 0 and out.count(" OK") >= 2, out[-4000:]


def test_mismatched_outputs_fail_loudly_copy_engine_one_gpu():
    rc, out = _launch("mismatch_ce", port=29655)
    assert rc == 0 and out.count(" OK") >= 2, out[-4000:]
    assert "different output buffer" in out, out[-4000:]


def test_peer_stores_stay_inside_outputs_one_gpu():
    rc, out = _launch("guards", port=29656)
    assert rc == 0 and out.count(" OK") >= 2, out[-4000:]


def test_workspace_grows_on_demand_one_gpu():
    rc, out = _launch("grow", port=29654)
    assert rc == 0 and out.count(" OK") >= 2, out[-4000:]


def test_mismatched_outputs_fail_loudly_one_gpu():
    rc, out = _launch("mismatch", port=29653)
    assert rc == 0 and out.count(" OK") >= 2, out[-4000:]
    assert "different output buffer" in out or "timed out" in out, out[-4000:]


def _launch_worker(script, args=(), n=2, port=29660, timeout=900):
    """A multi-GPU worker (tests/mp/*) with every rank on cuda:0 (FC_SAMEDEV)."""
    if not _have_gpu():
        pytest.skip("no CUDA device")
    env = dict(os.environ, FC_SAMEDEV="1",
               CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(HERE, "mp", script), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    return r.returncode, r.stdout + r.stderr


def test_production_parity_worker_one_gpu():
    """The multi-GPU parity worker (one-hop / one-shot, forest LL128, chunk
    flags; fp32 / bf16 / int32; odd sizes and raw bit patterns) with 2 rank
    processes on one B200."""
    rc, out = _launch_worker("parity_worker.py", port=29661)
    assert rc == 0 and out.count(" OK") >= 2, out[-4000:]


def test_ddp_comm_hook_one_gpu():
    """§8f-2: DDP with the ForestColl all-reduce hook (fused AVG) matches
    DDP's default all-reduce."""
    rc, out = _launch_worker("ddp_worker.py", port=29662)
    assert rc == 0 and out.count(" OK") >= 2, out[-4000:]


def test_fsdp2_custom_collectives_one_gpu():
    """§8f-2: FSDP2 with ForestColl all-gather (symmetric pool) and
    reduce-scatter matches stock FSDP2, fp32 and bf16 mixed precision."""
    rc, out = _launch_worker("fsdp_worker.py", port=29663)
    assert rc == 0 and out.count(" OK") >= 2, out[-4000:]


def test_randomized_soak_one_gpu():
    rc, out = _launch_worker("stress_worker.py", args=("40",), port=29664)
    assert rc == 0 and out.count("STRESS") >= 2, out[-4000:]
