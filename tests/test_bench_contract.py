"""bench.py's output contract (the driver parses it): one JSON line on stdout
with the keys the task's bench contract names, for the reference arm (CPU,
runs here) and for our arm (GPU)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(args, timeout=600):
    env = dict(os.environ, NCCL_DEBUG="VERSION")  # the image's default: must stay off stdout
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


COMMON = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
          "higher_is_better", "scaling", "vs_baseline", "dtype", "config")


def test_reference_arm_contract():
    if not (ROOT / "baseline" / "_ref" / "mehdg").is_dir():
        pytest.skip("reference not installed into baseline/_ref (__graft_entry__.build())")
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3"])
    for k in COMMON:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["steps"] == 2 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] == "reference" and cb["cores"] >= 1
    # the arm runs the unmodified reference and never loads this package
    assert d["product_loaded"] is False and cb["extrapolated"] is False
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_contract(gpu):
    d = _run(["--config", "c1", "--steps", "20", "--warmup", "3", "--no-cpu-baseline", "--no-mb",
              "--no-asm"])
    for k in COMMON:
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3
    assert d["dtype"] == "f64" and "workload" in d["config"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert rf["achieved"] > 0 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 2 * d["steps"]
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["solve"]["converged"]
