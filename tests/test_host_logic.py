"""Host-side logic of the drop-in that runs before any device call: argument
validation order, n < 2 short-circuits, interaction mapping, typed errors
(spi_engine.py:32-41,76-81,139-144,179-204; lattice_counter.py:52-59,118-122)."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1901_11204_b200 as pc
from paper_1901_11204_b200 import _lib
from paper_1901_11204_b200 import lattice_counter as lc
from paper_1901_11204_b200 import spi_engine as se


def test_public_names_match_reference():
    ref_names = {"CountReport", "LatticeSpace", "Sphere", "SpiResult", "collision_indicator", "count_collisions",
                 "count_contacts", "first_violation_step", "new_space", "oracle_collisions", "oracle_contacts",
                 "pairs", "pairs_array", "reach", "reached", "reset_sparse", "spi_balanced", "spi_parallel",
                 "spi_standard", "steps_for"}
    assert ref_names <= set(pc.__all__)
    for name in ("_depth", "_partition", "SCHEDULES", "InteractionDomainError", "AccumulationError",
                 "SymmetryViolationError", "as_object_array"):
        assert hasattr(se, name)
    for name in ("contact_accumulator", "interior_cell_count", "NEIGHBOR_OFFSETS", "CoordinateRangeError",
                 "OccupancyOverflowError", "SpaceSizeError", "as_bead_array"):
        assert hasattr(lc, name)


def test_collision_indicator_scalar_semantics():
    assert se.collision_indicator((0, 0, 0), (0, 0, 0)) == 1
    assert se.collision_indicator((0, 0, 0), (1.0, 0, 0)) == 0
    assert se.collision_indicator((0, 0, 0), (0.6, 0, 0)) == 1
    with pytest.raises(se.InteractionDomainError):
        se.collision_indicator((0, 0, float("nan")), (0, 0, 0))


def test_indicator_golden(golden_small):
    for case in golden_small["indicator_cases"]:
        pts = np.asarray(case["points"])
        got = [int(se.collision_indicator(a, b)) for a, b in zip(pts[0::2], pts[1::2])]
        assert got == case["values"]


def test_empty_and_singleton_need_no_device():
    for objs in ([], [se.Sphere(0, 0, 0)]):
        r = se.spi_standard(objs, se.collision_indicator)
        assert r.total == 0 and r.pairs_evaluated == 0 and r.depth_per_worker == 0
        r = se.spi_parallel(objs, lambda a, b: 1, 3, "standard")
        assert r.partials == (0, 0, 0) and r.worker_pairs == (0, 0, 0)


def test_parallel_validation_order():
    with pytest.raises(ValueError):
        se.spi_parallel([], lambda a, b: 1, 0)
    with pytest.raises(ValueError):
        se.spi_parallel([], lambda a, b: 1, 1, "diagonal")


def test_unsupported_interaction_raises_type_error():
    with pytest.raises(TypeError):
        se.spi_standard(np.arange(5), lambda a, b: 1)
    with pytest.raises(TypeError):
        se.spi_balanced(np.zeros((4, 3)), lambda a, b: 1)


def _brute_first_bad(xyz, schedule, ranges, nan_only):
    """The reference's evaluation order, pair by pair (spi_engine.py:102-120)."""
    n = len(xyz)
    for k, (lo, hi) in enumerate(ranges):
        for i in range(lo, hi):
            if schedule == "standard":
                js = range(i + 1, n)
            else:
                steps = n // 2 if (n % 2 or i < n // 2) else n // 2 - 1
                js = [(i + s) % n for s in range(1, steps + 1)]
            for j in js:
                a, b = xyz[i].astype(np.float64), xyz[j].astype(np.float64)
                if nan_only:
                    with np.errstate(all="ignore"):
                        bad = not np.isfinite(1.0 / (1.0 + ((a - b) ** 2).sum()))
                else:
                    bad = not (np.isfinite(a).all() and np.isfinite(b).all())
                if bad:
                    return k, i, j
    return None


def test_first_bad_pair_matches_reference_order():
    """Error-path locator (no interaction evaluated on the host) against a
    pair-by-pair walk: NaN terms (NaN coordinate, same infinity on one axis)
    for the inverse-square sum, any non-finite point for the count."""
    rng = np.random.default_rng(5)
    specials = [np.nan, np.inf, -np.inf]
    for trial in range(300):
        n = int(rng.integers(2, 40))
        xyz = rng.normal(size=(n, 3))
        for _ in range(int(rng.integers(1, 4))):
            xyz[rng.integers(0, n), rng.integers(0, 3)] = specials[int(rng.integers(0, 3))]
        sched = ("standard", "balanced")[trial % 2]
        w = int(rng.integers(1, 5))
        ranges = [(b.start, b.stop) for b in se._partition(n, w)]
        for nan_only in (True, False):
            assert se._first_bad_pair(xyz, sched, ranges, nan_only) == \
                _brute_first_bad(xyz, sched, ranges, nan_only), (trial, nan_only)


def test_resolve_domain_maps_reference_errors():
    """PC_ERR_DOMAIN from the device -> the reference's exception (host logic
    only: the device results are stand-ins)."""
    class R:
        def __init__(self, error):
            self.error, self.count, self.sum, self.pairs = error, 0, 0.0, 0

    pts = np.zeros((4, 3))
    pts[2, 1] = np.nan
    with pytest.raises(se.AccumulationError, match=r"\(0, 2\)"):
        se._resolve_domain(pts, _lib.PC_COLLISION_INVSQ, "standard", [(0, 4)], [R(_lib.PC_ERR_DOMAIN)], None)
    with pytest.raises(se.InteractionDomainError):
        se._resolve_domain(pts, _lib.PC_COLLISION, "balanced", [(0, 4)], [R(_lib.PC_ERR_DOMAIN)], None)
    # rows [3, 4) of the standard schedule own no pair: the bad point is never evaluated, so the
    # call is rerun with it zeroed instead of raising (the reference returns 0 there)
    seen = []
    out = se._resolve_domain(pts, _lib.PC_COLLISION, "standard", [(3, 4)], [R(_lib.PC_ERR_DOMAIN)],
                             lambda x: seen.append(x.copy()) or [R(0)])
    assert out[0].error == 0 and np.isfinite(seen[0]).all()
    ok = [R(0)]
    assert se._resolve_domain(pts, _lib.PC_COLLISION, "standard", [(0, 4)], ok, None) is ok


def test_symmetry_audit_runs_on_host():
    with pytest.raises(se.SymmetryViolationError):
        se.spi_standard(np.arange(10), lambda a, b: int(a) - int(b), audit_symmetry=True)


def test_depth_and_partition():
    for n in (3, 4, 5, 100, 101, 10_001):
        assert se._depth(n, "standard") == n - 1
        assert se._depth(n, "balanced") == math.ceil((n - 1) / 2)
    assert [len(b) for b in se._partition(10, 3)] == [4, 3, 3]
    assert se._partition(0, 2) == [range(0, 0), range(0, 0)]


def test_object_conversion():
    arr = se.as_object_array([se.Sphere(1, 2, 3), se.Sphere(4, 5, 6)])
    assert arr.dtype == np.float64 and arr.shape == (2, 3)
    x = np.arange(6, dtype=np.float32).reshape(3, 2)
    d = se._device_coords(x)
    assert d.shape == (3, 3) and d.dtype == np.float32 and (d[:, 2] == 0).all()
    assert se._device_coords(np.ones((2, 3), np.float16)).dtype == np.float64
    with pytest.raises(TypeError):
        se._device_coords(np.ones((2, 4)))
    with pytest.raises(np.exceptions.AxisError):  # as the reference's scalar fallback
        se.spi_standard(np.arange(4.0), se.collision_indicator)


def test_lattice_host_helpers():
    assert lc.interior_cell_count(960) == 1921**3
    with pytest.raises(ValueError):
        lc.interior_cell_count(-1)
    with pytest.raises(ValueError):
        lc.as_bead_array([(1, 2)])
    assert lc.as_bead_array([]).shape == (0, 3)
    assert lc.oracle_collisions([]) == 0 and lc.oracle_contacts([(1, 1, 1)]) == 0
    assert lc.count_collisions([], None).count == 0
