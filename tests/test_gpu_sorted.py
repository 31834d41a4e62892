"""Parity of the sorted inverse-square path (whole-range fp32 sums from 2^15 points:
Morton sort + tile-local Gram chunks, csrc/pairs_kernel.cuh SORTED) with the C oracle.

The sort permutes the points, so counts must stay bit-exact and sums within the
north_star's 1e-5 -- held here to 1e-6, the path's own per-term bound being 2e-6.
Distributions that stress the chunk test: uniform, clustered, two clusters far
apart, far from the origin, a thin slab, and lattice points at exact distance 1."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1901_11204_b200 import _lib
from paper_1901_11204_b200 import generators as gen
from paper_1901_11204_b200 import spi_engine as se
from oracle import c_oracle

pytestmark = pytest.mark.gpu


def _inputs(n, seed):
    rng = np.random.default_rng(seed)
    box = (4.18879 * n) ** (1 / 3) / 1.26
    k = 48
    cent = rng.random((k, 3)) * box * 3
    far = rng.random((n, 3)) * 15.0
    far[n // 2:] += 5e3
    lat = rng.integers(0, int(box) + 1, size=(n, 3)).astype(np.float64)
    return {
        "uniform": gen.random_spheres(n, box, seed),
        "clustered": cent[rng.integers(0, k, n)] + rng.normal(size=(n, 3)) * 1.5,
        "two far clusters": far,
        "offset 3e4": rng.random((n, 3)) * box + 3e4,
        "thin slab": rng.random((n, 3)) * np.array([box * 6, box * 6, 0.8]),
        "lattice": lat,
    }


@pytest.mark.parametrize("n", [32768, 40001, 65537])
def test_sorted_sum_matches_oracle(n):
    for name, pts in _inputs(n, n).items():
        pts = pts.astype(np.float32)
        want_c, want_s, pairs = c_oracle.rows(pts, 0, n, "balanced")
        (r,) = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])  # AUTO: sorted
        assert (r.count, r.pairs, r.error) == (want_c, pairs, 0), name
        assert abs(r.sum - want_s) <= 1e-6 * want_s, (name, r.sum, want_s)
        res = se.spi_balanced(pts, se.inverse_square)
        assert abs(res.total - want_s) <= 1e-6 * want_s, name


@pytest.mark.parametrize("n", [32768, 40001, 65537])
def test_sorted_sum_float64_points(n):
    """Float64 points on the sorted path (round 2): Morton sort of the float64 array, the
    compensated hi + lo staging, Gram chunks formed from b = (hi - o) + lo."""
    for name, pts in _inputs(n, n + 1).items():
        want_c, want_s, pairs = c_oracle.rows(pts, 0, n, "balanced")
        (r,) = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])  # AUTO: sorted
        prof = _lib.last_profile()
        # 9: the compensated sorted kernel alone; 11: with the tensor-core Gram chunks beside it
        assert prof.kernel in (9, 11) and prof.chunks_gram + prof.chunks_tc > 0, name
        assert (r.count, r.pairs, r.error) == (want_c, pairs, 0), name
        assert abs(r.sum - want_s) <= 1e-6 * want_s, (name, r.sum, want_s)
        assert se.spi_balanced(pts, se.inverse_square).total == r.sum, name
    # far from the origin and two clusters 1e6 apart: the centred hi + lo keeps separations exact
    rng = np.random.default_rng(n)
    for name, pts in (("offset 1e6", rng.random((n, 3)) * 40 + 1e6),
                      ("clusters 1e6 apart", np.concatenate([rng.random((n // 2, 3)) * 20,
                                                             rng.random((n - n // 2, 3)) * 20 + 1e6]))):
        want_c, want_s, _ = c_oracle.rows(pts, 0, n, "balanced")
        (r,) = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
        assert r.count == want_c and abs(r.sum - want_s) <= 1e-6 * want_s, (name, r.sum, want_s)


def test_sorted_ranges_are_partials_of_the_total():
    # PC_TILE_SORTED row ranges index the sorted order (the multi-GPU slabs): each is a
    # partial of the same total, not the reference's _run_outer over those input rows
    n = 50_000
    pts = gen.random_spheres(n, 30.0, 5).astype(np.float32)
    want_c, want_s, _ = c_oracle.rows(pts, 0, n, "balanced")
    res = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, 7, 12_501, 33_333, n],
                          tiling=_lib.PC_TILE_SORTED)
    assert sum(r.count for r in res) == want_c
    assert abs(sum(r.sum for r in res) - want_s) <= 1e-6 * want_s
    # the plain kernel on the input order keeps the reference's per-range meaning
    flat = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, 7, 12_501, 33_333, n],
                           tiling=_lib.PC_TILE_FLAT)
    for (lo, hi), r in zip(((0, 7), (7, 12_501), (12_501, 33_333), (33_333, n)), flat):
        c, s, _ = c_oracle.rows(pts, lo, hi, "balanced")
        assert r.count == c and abs(r.sum - s) <= 1e-6 * s


def test_sorted_argument_errors():
    pts = gen.random_spheres(40_000, 30.0, 1)
    # fp32 contact counts take the sorted order too (the pruned count, round 2)
    (r,) = _lib.pairs_host(pts.astype(np.float32), _lib.PC_COLLISION, _lib.PC_BALANCED, [0, 40_000],
                           tiling=_lib.PC_TILE_SORTED)
    assert r.count == c_oracle.rows(pts.astype(np.float32), 0, 40_000, "balanced")[0]
    with pytest.raises(Exception, match="PC_TILE_SORTED"):
        _lib.pairs_host(pts.astype(np.int64), _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, 40_000],
                        tiling=_lib.PC_TILE_SORTED)
    with pytest.raises(Exception, match="PC_TILE_SORTED"):
        _lib.pairs_host(pts.astype(np.float32), _lib.PC_COLLISION, _lib.PC_STANDARD, [0, 40_000],
                        tiling=_lib.PC_TILE_SORTED)


def test_sorted_path_non_finite_and_degenerate_inputs():
    # Non-finite coordinates, reference semantics (spi_engine.py:84-99): the sum's terms are
    # evaluated in float64 by the device (pairs_f64_kernel), so an isolated inf adds
    # 1/(1+inf) = 0 terms and the total matches the oracle; a NaN term (a NaN coordinate, or
    # the same inf on one axis of both points) is AccumulationError naming the first pair in
    # the reference's order; collision_indicator raises InteractionDomainError.  Points on a
    # line (a flat bounding box: zero Morton scale on two axes) stay exact.
    n = 40_000
    pts = gen.random_spheres(n, 30.0, 2).astype(np.float32)
    for bad in (np.inf, -np.inf):
        p = pts.copy()
        p[31_337, 1] = bad
        want_c, want_s, _ = c_oracle.rows(p, 0, n, "balanced")
        (r,) = _lib.pairs_host(p, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
        assert r.error == 0 and r.count == want_c and abs(r.sum - want_s) <= 1e-12 * want_s
        assert se.spi_balanced(p, se.inverse_square).total == r.sum
        assert _lib.last_profile().f64_taken == 1
        with pytest.raises(se.InteractionDomainError):
            se.spi_balanced(p, se.collision_indicator)
    p = pts.copy()
    p[31_337, 1] = np.nan
    (r,) = _lib.pairs_host(p, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    assert r.error == _lib.PC_ERR_DOMAIN
    with pytest.raises(se.AccumulationError, match=r"\(11337, 31337\)"):
        se.spi_balanced(p, se.inverse_square)
    p = pts.copy()
    p[100, 2] = p[7000, 2] = np.inf  # inf - inf on the same axis: NaN term
    with pytest.raises(se.AccumulationError, match=r"\(100, 7000\)"):
        se.spi_balanced(p, se.inverse_square)
    line = np.zeros((n, 3), np.float32)
    line[:, 0] = np.arange(n, dtype=np.float32) * 0.75
    want_c, want_s, _ = c_oracle.rows(line, 0, n, "balanced")
    (r,) = _lib.pairs_host(line, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    assert r.count == want_c and abs(r.sum - want_s) <= 1e-6 * want_s
