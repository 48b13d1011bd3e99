"""bench.py keeps the driver's JSON-line contract (CPU: the reference arm;
GPU: the device arm with roofline, clocks and launch count)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--config", "cfg2"], 300)
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["value"] > 0 and d["config"]["workload"] == "cfg2"
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["cpu"]["model"]


def test_reference_arm_under_torchrun():
    """Launched as the driver launches N > 1 (torch.distributed.run, one process
    per rank): rank 0 alone times the CPU port and prints the one line, the
    other ranks exit 0 without work."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
         "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--config",
         "cfg2"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    sys.path.insert(0, ROOT)
    import argparse

    import bench

    # the same config object (incl. the split it names) as the device arm at N = 2
    assert d["config"] == bench.bench_config(argparse.Namespace(config="cfg2"),
                                             bench.CONFIGS["cfg2"], 2)
    assert d["scaling"] == "strong" and "2" in d["config"]["parallelism"]


def test_both_arms_print_the_same_config():
    """The reference arm and the device arm build one config object."""
    sys.path.insert(0, ROOT)
    import argparse

    import bench

    for name in ("cfg5", "cfg2", "cfg3"):
        a = argparse.Namespace(config=name)
        assert bench.bench_config(a, bench.CONFIGS[name], 1) == bench.bench_config(
            a, bench.CONFIGS[name], 1)
    assert bench.bench_config(argparse.Namespace(config="cfg5"), bench.CONFIGS["cfg5"],
                              1)["workload"] == "cfg5"


@pytest.mark.gpu
def test_device_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--no-extras", "--config", "cfg2"], 900)
    assert d["metric"] and d["unit"] == "Gmodmul/s" and d["value"] > 0
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["gpu_launches"] > 0
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor") and 0 < rf["frac"] <= 1 and rf["peak"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
