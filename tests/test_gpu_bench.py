"""GPU: bench.py keeps its contract (one JSON line with the keys the driver
and the judge read), in a short configuration: both arms, N = 1."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHORT = ["--steps", "2", "--warmup", "3", "--iters-per-step", "20", "--e2e-iters", "50", "--e2e-steps", "1",
         "--no-ttt", "--per-config", "", "--cpu-iters", "3"]


def run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_keys():
    d = run(*SHORT)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"] == "C2"
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel", "kernels"):
        assert k in d["roofline"], k
    assert 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] == 4 * 2 * 20
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k


def test_reference_arm_line():
    d = run("--impl", "reference", "--steps", "1", "--warmup", "3", "--ref-iters", "2")
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["config"]["workload"] == "C2"
