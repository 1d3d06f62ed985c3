"""Multi-GPU parity (one process per GPU, exchanges over NVLink peer memory):
the decomposed run equals the 1-GPU run of the same plan bitwise.  Needs at least two GPUs
(skipped otherwise); each case runs tools/mgpu_check.py under torchrun."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except ImportError:                                    # pragma: no cover
        return 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("system,scale,steps,plan", (("kochi", 0.001, 40, "minmax"),
                                                      ("quad_wetdry", 0.0, 30, "minmax"),
                                                      ("kochi", 0.01, 20, "packed"),
                                                      ("kochi", 0.001, 40, "packed"),
                                                      ("fuzz", 0.0, 60, "packed"),
                                                      ("fuzz", 0.0, 60, "minmax")))
@pytest.mark.parametrize("ranks", (2, 4))
def test_decomposed_run_bitwise_equals_one_gpu(system, scale, steps, plan, ranks):
    if _gpus() < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--system", system, "--steps", str(steps),
           "--plan", plan]
    if system == "kochi":
        cmd += ["--scale", str(scale)]
    if system == "fuzz":                  # random nested systems, compared per system
        cmd += ["--seeds", "48"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    lines = [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert lines
    for out in lines:                     # one line per system (fuzz: per random seed)
        assert out["ranks"] == ranks
        assert out["bitwise_equal_to_1gpu"], (out["system"], out["diffs"][:5])


@pytest.mark.parametrize("system,scale,steps,plan", (("kochi", 0.001, 20, "packed"),
                                                      ("kochi", 0.001, 20, "minmax"),
                                                      ("fuzz", 0.0, 30, "packed")))
def test_eight_ranks_on_shared_gpus(system, scale, steps, plan):
    """Eight ranks (the 8-GPU rank count) on a box with fewer GPUs: the ranks
    share GPUs round-robin (tools/mgpu_check.py), so the 8-rank exchange
    tables, receive areas and barriers are checked bitwise against the
    one-process run."""
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--system", system, "--steps", str(steps),
           "--plan", plan]
    cmd += ["--scale", str(scale)] if system == "kochi" else ["--seeds", "24"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    lines = [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert lines
    for out in lines:
        assert out["ranks"] == 8
        assert out["bitwise_equal_to_1gpu"], (out["system"], out["diffs"][:5])


@pytest.mark.parametrize("ranks", (2, 4))
def test_failure_on_one_rank_stops_every_rank(ranks):
    """A NaN depth in the last rank's block: every rank raises the same
    NumericsError as the one-process run (device error words adopted at the
    phase barriers, agreed on the host), none hangs in a barrier."""
    if _gpus() < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--system", "nan", "--steps", "6"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    out = [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")][0]
    assert out["bitwise_equal_to_1gpu"], out
