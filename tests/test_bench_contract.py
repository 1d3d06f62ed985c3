"""bench.py output contract on CPU: the reference arm (the oracle port on the
host cores) prints exactly one JSON line on stdout, whatever else the
process writes to file descriptor 1, with the keys the driver reads."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=300, env=env)


def test_reference_arm_prints_one_json_line():
    r = _bench("--impl", "reference", "--steps", "2", "--warmup", "3", "--scale", "0.01")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["metric"] == "Gcell-updates/s" and line["unit"] == "Gcell/s"
    assert line["warmup"] >= 3 and line["steps"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_native_stdout_writes_go_to_stderr():
    # what native libraries print on fd 1 (NCCL's version line) must not
    # reach stdout: simulate it with a raw write to fd 1 before the arm runs
    code = ("import os, sys\n"
            "import bench\n"
            "orig = bench.run_reference\n"
            "def noisy(args):\n"
            "    os.write(1, b'NCCL version 0.0.0\\n')\n"
            "    orig(args)\n"
            "bench.run_reference = noisy\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--scale', '0.01']\n"
            "bench.main()\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert len(r.stdout.splitlines()) == 1 and r.stdout.startswith("{"), r.stdout
    assert "NCCL version 0.0.0" in r.stderr
