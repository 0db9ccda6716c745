"""bench.py keeps the driver's JSON-line contract (one line on rank 0).

The reference arm runs the oracle port on host cores, so it is checked here on
CPU; the product arm needs a B200 (``-m gpu``)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    env = dict(os.environ, ICCL_BENCH_NO_CLOCKS="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--bytes", str(4 << 20)])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_product_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--bytes", str(64 << 20), "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] <= 1.1 and r["peak"] > 0
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 64 << 20 and e["d2h_bytes_per_step"] == 64 << 20
    assert e["bit_exact"] and e["value"] > 0 and e["bound"]["value"] > 0
    assert "gpu_launches" in d and d["copy_engine_copies"] >= 3
