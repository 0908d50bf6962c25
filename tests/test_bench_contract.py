"""bench.py's output contract: one JSON line with the keys the driver reads.  The reference arm
(the CPU oracle on a bounded sample) runs here on CPU; our arm needs the GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--nx", "16", "--steps", "1", "--warmup", "1"])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["config"]["workload"] == "cfg3"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_contract():
    d = _run(["--nx", "128", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "roofline_flux", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    r = d["roofline"]
    assert r["kernel"] in ("k_dual_mma", "k_dual_group") and 0 < r["frac"] < 1 and 0 < r["algorithmic"]["frac"] < 1
    assert r["bound"] == "alu" and r["unit"] == "TFLOP/s"
    assert d["roofline_flux"]["bound"] == "hbm" and 0 < d["roofline_flux"]["frac"] < 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["n_gpus"] == 1 and d["config"]["workload"] == "cfg3"
