"""Headline-size parity against the full-size oracle totals (tests/golden/golden_full.json).

The reference's whole-triangle result at 2^20 / 2^22 points is out of its CPU
reach; golden_full.json holds the C oracle's float64 totals over every pair
(tests/golden/make_full_totals.py, pinned to the reference's own row samples).
Every GPU path that computes a whole-triangle result is checked against them:
counts bit-exact, sums within 1e-6 relative (north_star allows 1e-5):
  * the drop-in calls (spi_balanced / spi_standard / spi_parallel);
  * the sorted sum kernel (PC_TILE_AUTO), the input-order sum (PC_TILE_FLAT),
    the FFMA2 Gram count, the tensor-core count, the naive standard schedule;
  * the multi-GPU splits: 2/4/8 contiguous slabs of the sorted order and
    2/4/8 round-robin tile parts -- their partials must add up to the total.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from paper_1901_11204_b200 import _lib
from paper_1901_11204_b200 import spi_engine as se
from paper_1901_11204_b200.distributed import row_slabs
from tests.helpers import config_input, digest

pytestmark = pytest.mark.gpu

FULL = json.loads((Path(__file__).parent / "golden" / "golden_full.json").read_text())
REL = 1e-6


def _golden(name):
    if name not in FULL:
        pytest.skip(f"{name} full total not generated yet (tests/golden/make_full_totals.py)")
    return FULL[name]


@pytest.fixture(scope="module")
def inputs(golden_configs):
    cache = {}

    def get(name):
        if name not in cache:
            x = config_input(golden_configs, name)
            assert digest(x) == FULL.get(name, {}).get("sha256", digest(x)), name
            cache[name] = x
        return cache[name]

    return get


def _host(x, interaction, sched, tiling=_lib.PC_TILE_AUTO, bounds=None):
    (r,) = _lib.pairs_host(x, interaction, sched, bounds or [0, len(x)], tiling=tiling)
    assert r.error == 0
    return r


@pytest.mark.parametrize("name", ["cfg3", "cfg4u", "cfg4c"])
def test_full_totals_every_path(inputs, name):
    g = _golden(name)
    x = inputs(name)
    n = len(x)
    assert n == g["n"]
    # drop-in API
    assert se.spi_balanced(x, se.collision_indicator).total == g["count"]
    s = se.spi_balanced(x, se.inverse_square).total
    assert abs(s - g["inv_sum"]) <= REL * g["inv_sum"], (s, g["inv_sum"])
    # the sorted kernel (what spi_balanced takes) counts contacts exactly in the same pass
    r = _host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED)
    assert r.count == g["count"] and r.sum == s and r.pairs == g["pairs"]
    prof = _lib.last_profile()
    # the sorted FFMA kernel plus the tensor-core Gram chunks (kernel 10; 3 with PAIRCOUNT_TCSUM=0)
    assert prof.kernel in (3, 10) and prof.f64_taken == 0 and prof.chunks_gram + prof.chunks_tc > 0
    assert (prof.chunks_tc > 0) == (prof.kernel == 10)
    # input-order sum kernel
    r = _host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, _lib.PC_TILE_FLAT)
    assert r.count == g["count"] and abs(r.sum - g["inv_sum"]) <= REL * g["inv_sum"]
    # counts: FFMA2 Gram filter, tensor cores, the naive standard schedule
    assert _host(x, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_FLAT).count == g["count"]
    assert _host(x, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_TC).count == g["count"]
    assert _host(x, _lib.PC_COLLISION, _lib.PC_STANDARD, _lib.PC_TILE_PER_ROW_TILE).count == g["count"]


@pytest.mark.parametrize("name", ["cfg3", "cfg4c"])
def test_full_totals_multi_gpu_splits(inputs, name):
    """The shares one GPU of a G-GPU job computes, each run alone here: their
    partials add up to the oracle total (counts exactly)."""
    g = _golden(name)
    x = inputs(name)
    n = len(x)
    for world in (2, 4, 8):
        # contiguous slabs of the sorted order
        rs = [_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, _lib.PC_TILE_SORTED, [lo, hi])
              for lo, hi in row_slabs(n, world, "balanced")]
        assert sum(r.count for r in rs) == g["count"]
        assert abs(sum(r.sum for r in rs) - g["inv_sum"]) <= REL * g["inv_sum"]
        assert sum(r.pairs for r in rs) == g["pairs"]
        # round-robin tile parts (what bench.py and spi_distributed run at N > 1)
        for interaction, tiling in ((_lib.PC_COLLISION_INVSQ, _lib.PC_TILE_SORTED),
                                    (_lib.PC_COLLISION, _lib.PC_TILE_FLAT)):
            parts = [_lib.pairs_part_host(x, interaction, _lib.PC_BALANCED, 0, n, k, world, tiling)
                     for k in range(world)]
            assert all(p.error == 0 for p in parts)
            assert sum(p.count for p in parts) == g["count"], (world, interaction)
            assert sum(p.pairs for p in parts) == g["pairs"]
            if interaction == _lib.PC_COLLISION_INVSQ:
                assert abs(sum(p.sum for p in parts) - g["inv_sum"]) <= REL * g["inv_sum"]


def test_full_size_sums_bit_reproducible(inputs):
    """Float sums are fixed-association (per-claim float64 partials added in
    claim order), so repeated calls agree bitwise -- sorted, input-order and
    tile-part paths alike."""
    x = inputs("cfg3")
    n = len(x)
    for tiling in (_lib.PC_TILE_AUTO, _lib.PC_TILE_FLAT):
        a = _host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, tiling).sum
        for _ in range(2):
            assert _host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, tiling).sum == a
    p = [_lib.pairs_part_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, 0, n, 1, 4, _lib.PC_TILE_SORTED).sum
         for _ in range(3)]
    assert p[0] == p[1] == p[2]
