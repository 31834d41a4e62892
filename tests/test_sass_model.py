"""The per-loop FMA-pipe costs bench.py's roofline uses (profiles/sass_model.json)
must describe the shipped kernels: recompute them from the built library's
SASS (cuobjdump, no GPU needed) and compare."""

from __future__ import annotations

import json
import shutil

import pytest

from tests.conftest import ROOT


def test_sass_model_matches_shipped_library():
    lib = ROOT / "paper_1901_11204_b200" / "libpaircount.so"
    if not lib.exists() or not shutil.which("cuobjdump"):
        pytest.skip("libpaircount.so not built or cuobjdump missing")
    import importlib.util

    spec = importlib.util.spec_from_file_location("sass_model", ROOT / "scripts" / "sass_model.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    got = mod.model(lib)["kernels"]
    want = json.loads((ROOT / "profiles" / "sass_model.json").read_text())["kernels"]
    for kern, loops in want.items():
        for loop, v in loops.items():
            assert got[kern][loop]["fma_cycles_per_pair"] == pytest.approx(v["fma_cycles_per_pair"]), (kern, loop)
    # the loops the roofline needs are all found
    assert {"gram", "near", "direct"} <= set(got["sorted_sum"])
    assert got["sorted_sum"]["gram"]["fma_cycles_per_pair"] < got["sorted_sum"]["direct"]["fma_cycles_per_pair"]
