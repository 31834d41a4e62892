"""bench.py's JSON-line contract, checked on CPU through the reference arm
(`--impl reference` runs the unmodified reference from baseline/_ref -- or,
absent that, the oracle port -- on host cores; the
GPU arm has the same keys plus roofline/clocks/gpu_launches and is exercised
on the B200 by scripts/gpu_bench.sh)."""

from __future__ import annotations

import json
import subprocess
import sys

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
