"""bench.py keeps the driver's JSON contract.

* CPU: the reference arm (`--impl reference`, the CPU oracle decoder) on the tiny
  model prints one JSON line with the contract's keys;
* GPU: the B200 arm on a truncated Llama-3-shape run prints the full line --
  device value, e2e (host copies inside the timed region), roofline, launches,
  clocks -- with self-consistent numbers.
"""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def run_bench(*args, timeout=600):
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-3000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--model", "tiny-llama", "--batch", "4", "--prompt", "32",
                  "--decode", "4", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "tok/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_b200_arm_contract():
    d = run_bench("--layers", "2", "--batch", "8", "--prompt", "64", "--decode", "8", "--steps", "3",
                  "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["value"] <= d["value"] * 1.05          # host copies only add time
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * 64 * 8 and d["e2e"]["d2h_bytes_per_step"] == 8 * 8 * 8
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["gpu_launches"] > 100
    assert d["cpu_baseline"] is None and d["vs_baseline"] is None
    assert "workload" in d["config"] and d["dtype"] == "bf16"
