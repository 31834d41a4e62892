"""Parity of the tensor-core count kernel (csrc/pairs_tc.cuh) with the oracle.

PC_TILE_TC forces the kernel at any size, so the ragged shapes (n not a
multiple of the 8-point operand groups, the 128-row tiles or the 256-column
chunks; odd and even n) and the adversarial inputs are covered at sizes the C
oracle finishes in well under a second.  Counts must be bit-exact: the tensor
cores only filter, every candidate is re-checked with the reference's own
predicate."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1901_11204_b200 as pc
from paper_1901_11204_b200 import _lib
from paper_1901_11204_b200 import generators as gen
from paper_1901_11204_b200 import spi_engine as se
from oracle import c_oracle

pytestmark = pytest.mark.gpu


def _tc(arr, interaction=_lib.PC_COLLISION):
    (r,) = _lib.pairs_host(np.ascontiguousarray(arr), interaction, _lib.PC_BALANCED, [0, len(arr)],
                           tiling=_lib.PC_TILE_TC)
    return r


@pytest.mark.parametrize("n", [2, 3, 7, 8, 9, 127, 128, 129, 255, 256, 257, 1000, 1001, 4097, 9000])
def test_tc_count_matches_oracle_ragged_sizes(n):
    # box side chosen for ~n/2 contacts, so most tiles hold candidates
    pts = gen.random_spheres(n, max(1.0, (4.18879 * n / 1.0) ** (1 / 3) / 1.26), 100 + n)
    for arr in (pts, pts.astype(np.float32)):
        want, _, pairs = c_oracle.rows(arr, 0, n, "balanced")
        r = _tc(arr)
        assert (r.count, r.pairs, r.error) == (want, pairs, 0)


def test_tc_count_dense_cluster_and_tangent_pairs():
    # every pair a candidate in a tight cluster; a lattice of exactly tangent
    # spheres (d = 1: not a contact) with neighbours 1 ulp inside and outside
    rng = np.random.default_rng(5)
    dense = rng.random((3000, 3)) * 4.0
    g = np.stack(np.meshgrid(np.arange(16.0), np.arange(16.0), np.arange(12.0), indexing="ij"), -1).reshape(-1, 3)
    inside = g[::7] + np.array([np.nextafter(1.0, 0.0), 0.0, 0.0])
    outside = g[3::11] + np.array([0.0, np.nextafter(1.0, 2.0), 0.0])
    tangent = np.concatenate([g, inside, outside])
    for arr in (dense, tangent, tangent.astype(np.float32)):
        want, _, _ = c_oracle.rows(arr, 0, len(arr), "balanced")
        assert _tc(arr).count == want


def test_tc_count_far_from_origin_and_wide_spans():
    # centring keeps M small for a far cluster; two clusters 1e6 apart make M
    # large (wide band, many exact re-checks); spans near 1e16 force every pair
    # through the exact path (M >= 1e30)
    rng = np.random.default_rng(6)
    c1 = rng.random((2000, 3)) * 12.0 + 1e4
    c2 = np.concatenate([rng.random((1500, 3)) * 10.0, rng.random((1500, 3)) * 10.0 + 1e6])
    c3 = np.concatenate([rng.random((300, 3)) * 3.0, rng.random((300, 3)) * 3.0 + 1e16])
    for arr in (c1, c2, c3):
        want, _, _ = c_oracle.rows(arr, 0, len(arr), "balanced")
        assert _tc(arr).count == want


@pytest.mark.parametrize("seed", [0, 1])
def test_tc_integer_predicates(seed):
    beads = gen.random_chain(6000, seed)[0]
    beads[::13] = beads[0]
    col, con = c_oracle.int_pairs(beads)
    for arr in (beads, beads.astype(np.int32)):
        assert _tc(arr, _lib.PC_COINCIDE).count == col
        assert _tc(arr, _lib.PC_MANHATTAN1).count == con


def test_tc_auto_dispatch_at_config2_size(golden_configs):
    # PC_TILE_AUTO sends balanced counts with 2^14 <= n < 2^21 over row ranges covering >= n/8 rows
    # to the tensor cores (spi_parallel's workers here; a whole-range fp32 call from 2^15 points
    # takes the pruned sorted count): config 2 keeps its golden count on every path, and so does
    # the FFMA kernel forced with PC_TILE_FLAT
    from tests.helpers import config_input

    pts = config_input(golden_configs, "cfg2")
    want = golden_configs["cfg2"]["balanced"]["total"]
    assert se.spi_balanced(pts, se.collision_indicator).total == want
    assert sum(se.spi_parallel(pts, se.collision_indicator, workers=3, schedule="balanced").partials) == want
    assert _lib.last_profile().kernel == 5  # the tensor cores took the workers' ranges
    (flat,) = _lib.pairs_host(np.ascontiguousarray(pts), _lib.PC_COLLISION, _lib.PC_BALANCED, [0, len(pts)],
                              tiling=_lib.PC_TILE_FLAT)
    assert flat.count == want


def test_tc_argument_errors():
    pts = gen.random_spheres(500, 6.0, 1)
    with pytest.raises(Exception, match="PC_TILE_TC"):
        _tc(pts, _lib.PC_COLLISION_INVSQ)
    with pytest.raises(Exception, match="PC_TILE_TC"):
        _lib.pairs_host(pts, _lib.PC_COLLISION, _lib.PC_STANDARD, [0, 500], tiling=_lib.PC_TILE_TC)


@pytest.mark.parametrize("n", [1000, 4099])
def test_tc_row_ranges_match_oracle_partials(n):
    # row ranges (spi_parallel partials, spi_rows) on the tensor cores: tiles start at the
    # range's 8-point group, rows outside the range masked; empty ranges give zero
    pts = gen.random_spheres(n, (4.18879 * n) ** (1 / 3) / 1.26, 7).astype(np.float32)
    bounds = [0, 13, 13, 500, 777, 778, n - 3, n]
    res = _lib.pairs_host(pts, _lib.PC_COLLISION, _lib.PC_BALANCED, bounds, tiling=_lib.PC_TILE_TC)
    for (lo, hi), r in zip(zip(bounds[:-1], bounds[1:]), res):
        want, _, pairs = c_oracle.rows(pts, lo, hi, "balanced")
        assert (r.count, r.pairs, r.error) == (want, pairs, 0), (lo, hi)
    beads = gen.random_chain(n, 3)[0]
    col, con = c_oracle.int_pairs(beads)
    for inter, want in ((_lib.PC_COINCIDE, col), (_lib.PC_MANHATTAN1, con)):
        res = _lib.pairs_host(beads, inter, _lib.PC_BALANCED, [0, 5, 333, n], tiling=_lib.PC_TILE_TC)
        assert sum(r.count for r in res) == want


def test_tc_auto_for_spi_parallel_partials():
    # workers' ranges together cover n rows: PC_TILE_AUTO takes the tensor cores, and the
    # partials equal the oracle's per-worker counts
    pts = gen.random_spheres(40_000, 30.0, 11).astype(np.float32)
    r = se.spi_parallel(pts, se.collision_indicator, workers=5, schedule="balanced")
    for b, got in zip(se._partition(len(pts), 5), r.partials):
        assert got == c_oracle.rows(pts, b.start, b.stop, "balanced")[0]


def test_tc_exposed_through_the_drop_in_api():
    # spi_balanced at 2^14 <= n < 2^21 goes through the tensor cores; same total as the
    # FFMA kernel on the same input
    pts = gen.random_spheres(40_000, 30.0, 9).astype(np.float32)
    tot = pc.spi_balanced(pts, se.collision_indicator).total
    (flat,) = _lib.pairs_host(pts, _lib.PC_COLLISION, _lib.PC_BALANCED, [0, len(pts)], tiling=_lib.PC_TILE_FLAT)
    assert tot == flat.count == c_oracle.rows(pts, 0, len(pts), "balanced")[0]
