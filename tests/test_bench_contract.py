"""bench.py's JSON-line contract, checked on CPU through the reference arm
(`--impl reference` runs the unmodified reference from baseline/_ref -- or,
absent that, the oracle port -- on host cores; the
GPU arm has the same keys plus roofline/clocks/gpu_launches and is exercised
on the B200 by scripts/gpu_bench.sh)."""

from __future__ import annotations

import json
import subprocess
import sys

import pytest

from tests.conftest import ROOT


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--ref-rows-per-core", "1"], capture_output=True, text=True, timeout=600,
                         check=True).stdout.strip().splitlines()
    assert len(out) == 1, out  # exactly one JSON line
    d = json.loads(out[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["metric"].startswith("G pair-tests/s at N=2^20")
    assert set(d["cpu_baseline"]) >= {"value", "unit", "cores", "kind", "sample"}
    # the unmodified reference when baseline/_ref holds it (pip install --target), else the oracle port
    want_kind = "reference" if (ROOT / "baseline" / "_ref" / "paircount" / "spi_engine.py").exists() else "port"
    assert d["cpu_baseline"]["kind"] == want_kind and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """The GPU arm's line on the B200: the base contract plus roofline (the dominant kernel's bound,
    achieved / peak / frac, traffic), e2e through the public API with its copy bytes, clocks and
    gpu_launches; the headline's count is the oracle's."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3", "--no-secondary",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=900,
                         check=True).stdout.strip().splitlines()
    assert len(out) == 1, out
    d = json.loads(out[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["contacts"] == 521266  # tests/golden/golden_full.json cfg3
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm", "fp32 FMA pipe") and 0 < r["frac"] <= 1.0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and r["unit"] == "TFLOP/s"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2**20 * 12 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
