"""The bench.py JSON contract, checkable without a GPU: the reference (oracle) arm's line and
the fields the driver compares across arms (metric, unit, config, higher_is_better)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    # stdout carries exactly the one JSON line (library banners go to stderr)
    assert len(out.stdout.strip().splitlines()) == 1, out.stdout[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC
    # one unit string in both arms (the driver divides only like units)
    assert d["unit"] == bench.UNIT == "TFLOP/s"
    assert d["e2e"]["unit"] == d["unit"] and d["cpu_baseline"]["unit"] == d["unit"]
    assert d["higher_is_better"] is True and d["value"] > 0
    # the config is the same workload naming the GPU arm prints
    import argparse
    name, N, heads, hd, causal = bench.workload(argparse.Namespace(workload="gpt", seq=0), 1)
    assert d["config"] == bench.config_of(name, N, heads, hd, causal, 1)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


def test_result_line_survives_fd1_writers():
    """Anything a library writes to file descriptor 1 after _keep_stdout_for_result() lands on
    stderr; emit() still reaches the original stdout."""
    code = ("import os, sys; sys.path.insert(0, %r); import bench; bench._keep_stdout_for_result(); "
            "os.write(1, b'NCCL version banner\\n'); print('python print'); bench.emit({'k': 1})") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().splitlines() == ['{"k": 1}']
    assert "NCCL version banner" in out.stderr and "python print" in out.stderr


def test_workloads_are_baseline_shapes():
    import argparse
    a = argparse.Namespace(workload="gpt", seq=0)
    assert bench.workload(a, 1)[1:] == (32768, 32, 128, True)        # configs[1]
    assert bench.workload(a, 8)[1:] == (131072, 32, 128, True)       # configs[2]
    assert bench.workload(a, 1, "dit")[1:] == (65536, 16, 72, False)  # configs[3]
