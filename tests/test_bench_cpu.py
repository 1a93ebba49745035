"""bench.py's contract on CPU: the reference arm (the CPU oracle, per the tier framing)
prints one JSON line with the required keys, and our arm refuses to run without a GPU
(no CPU fallback)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "3",
                        "--n", "200000"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("sync-path microbench")


def test_our_arm_needs_a_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode != 0
    assert "no CPU fallback" in (r.stdout + r.stderr)


def test_warmup_below_three_is_rejected():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--warmup", "2"], capture_output=True,
                       text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0


def test_hidden_fraction_estimator_cancels_drift():
    """§8(d) hidden fraction from alternating cycles: a linear drift of the cycle time (clock / power)
    20x the exchange over the run cancels in the paired differences except the one drift step inside
    a pair; exposure is capped at [0, 1]."""
    import bench
    drift = [1.0 + 0.01 * i for i in range(40)]            # ms, 0.4 ms of drift over the run
    t_with = [drift[2 * i] + 0.02 for i in range(20)]      # 20 us exposed per cycle
    t_without = [drift[2 * i + 1] for i in range(20)]
    exposed = bench.exposed_from_cycles(t_with, t_without)
    assert abs(exposed - (0.02 - 0.01)) < 1e-12            # the pair's own 10 us drift step remains
    assert abs(bench.hidden_fraction(exposed, 1, 0.05) - 0.8) < 1e-9
    assert bench.hidden_fraction(-0.01, 1, 0.05) == 1.0    # faster with the exchange: fully hidden
    assert bench.hidden_fraction(0.2, 4, 0.05) == 0.0
    assert bench.hidden_fraction(0.01, 1, 0.0) is None
