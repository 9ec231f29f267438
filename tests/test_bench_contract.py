"""bench.py's one-line JSON contract (driver-facing): the reference arm on
the host (CPU), the B200 arm on a GPU."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    j = _run("--impl", "reference", "--steps", "1", "--warmup", "1")
    assert BASE_KEYS <= set(j) and j["impl"] == "reference"
    assert j["metric"] == "sGS-ADMM iters/s" and j["unit"] == "iter/s" and j["higher_is_better"] is True
    assert j["value"] > 0 and j["e2e"]["value"] == j["value"]
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0
    cb = j["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == j["value"]


@pytest.mark.gpu
def test_b200_arm_line():
    j = _run("--config", "c1", "--steps", "20", "--warmup", "3", "--no-cpu", "--no-next", "--kkt-iters", "30")
    assert BASE_KEYS <= set(j) and "impl" not in j
    assert j["steps"] == 20 and j["warmup"] == 3 and j["value"] > 0 and j["dtype"] == "f64"
    r = j["roofline"]
    # "l2": the Gram-space persistent kernel keeps its matrices on chip and is
    # reported against the probe-measured L2 read rate (profiles/r02/peaks_probe.json)
    assert r["bound"] in ("hbm", "tensor", "l2") and r["unit"] in ("GB/s", "TFLOP/s") and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert j["gpu_launches"] >= 1 and "sm_mhz" in j["clocks"]
    assert j["config"]["workload"].startswith("c1")
