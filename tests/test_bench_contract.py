"""bench.py's JSON line (the driver's contract): the reference arm (the oracle on the host
cores, CPU) and the GPU arm (one tiny run through the C ABI)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line(cfgdata):
    cfgdata("C1")
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0", "--ref-seconds", "1"])
    assert BASE_KEYS <= set(d), set(d) ^ BASE_KEYS
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C1")


@pytest.mark.gpu
def test_gpu_arm_line(cfgdata):
    cfgdata("C1")
    d = _run(["--config", "C1", "--nrhs", "1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d), set(d) ^ BASE_KEYS
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "alu", "tensor") and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 16 * d["config"]["N"]
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert "flushed" in d["config"]["l2"] or "written before every timed step" in d["config"]["l2"]
