"""The reference's acceptance suite (pkg/tests/test_acceptance.py), criterion
by criterion, run against the drop-in API.

Criteria 1, 2, 6, 7 (public result objects) and 8 exercise the GPU path and
are `-m gpu`; 3, 4, 5 and 7's closed forms are host-side schedule logic and run
on CPU.  The checker is the pinned C oracle (oracle/c_oracle.py), plus the
GPU all-pairs oracles where the reference compares against its own oracle.
Criterion 9 compares CPU wall times of the reference's two algorithms and
criterion 10 is covered by tests/test_bench_cli.py.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from paper_1901_11204_b200 import generators as gen
from paper_1901_11204_b200 import pair_schedule as ps

CHAIN_SIZES = [1, 2, 3, 16, 64, 257, 1024]
CHAINS_PER_SIZE = 500  # as the reference (test_acceptance.py:25-26)


def _adversarial():
    """test_acceptance.py:33-43: all coincident, all distinct, empty."""
    yield np.zeros((40, 3), dtype=np.int64)
    g = np.arange(4) * 2
    yield np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3).astype(np.int64)
    yield np.zeros((0, 3), dtype=np.int64)


@pytest.mark.gpu
def test_criterion_1_oracle_equivalence_collisions():
    """test_acceptance.py:49-64: count_collisions + reset_sparse per chain,
    500 chains x 7 sizes, equal to the brute-force oracle."""
    import paper_1901_11204_b200 as pc
    from oracle import c_oracle

    for n in CHAIN_SIZES:
        space = None
        for v in range(CHAINS_PER_SIZE):
            beads, extent = gen.random_chain(n, 1000 * n + v)
            if space is None or space.half_extent < extent:
                space = pc.new_space(max(extent, 1))
            report = pc.count_collisions(beads, space)
            pc.reset_sparse(space, beads)
            assert report.count == c_oracle.int_pairs(beads)[0], (n, v)
    for beads in _adversarial():
        assert pc.count_collisions(beads, pc.new_space(8)).count == pc.oracle_collisions(beads) \
            == c_oracle.int_pairs(beads)[0]


@pytest.mark.gpu
def test_criterion_2_oracle_equivalence_contacts():
    """test_acceptance.py:67-84: doubled accumulator even, half = oracle."""
    import paper_1901_11204_b200 as pc
    from oracle import c_oracle
    from paper_1901_11204_b200.lattice_counter import contact_accumulator

    for n in CHAIN_SIZES:
        space = None
        for v in range(CHAINS_PER_SIZE):
            beads, extent = gen.random_chain(n, 1000 * n + v)
            if space is None or space.half_extent < extent:
                space = pc.new_space(max(extent, 1))
            doubled = contact_accumulator(beads, space)
            pc.reset_sparse(space, beads)
            assert doubled % 2 == 0 and doubled // 2 == c_oracle.int_pairs(beads)[1], (n, v)
    for beads in _adversarial():
        assert pc.count_contacts(beads, pc.new_space(8)).count == pc.oracle_contacts(beads) \
            == c_oracle.int_pairs(beads)[1]


@pytest.mark.gpu
def test_criterion_1_batched():
    """Criterion 1 again through the one-launch batch API (§8 f4)."""
    import paper_1901_11204_b200 as pc
    from oracle import c_oracle

    for n in CHAIN_SIZES:
        chains = [gen.random_chain(n, 1000 * n + v) for v in range(CHAINS_PER_SIZE)]
        space = pc.new_space(max(max(e for _, e in chains), 1))
        reports = pc.count_collisions_batch([b for b, _ in chains], space)
        for (beads, _), rep in zip(chains, reports):
            assert rep.count == c_oracle.int_pairs(beads)[0]


def _canon(p: np.ndarray, n: int) -> np.ndarray:
    lo, hi = np.minimum(p[:, 0], p[:, 1]), np.maximum(p[:, 0], p[:, 1])
    return lo * n + hi


def test_criterion_3_schedule_completeness():
    """test_acceptance.py:110-122: pairs(N) covers every unordered pair once.
    Every N <= 300 plus a stride through N <= 2000 (vectorised instead of numba)."""
    for n in list(range(1, 301)) + list(range(301, 2001, 53)) + [1999, 2000]:
        p = ps.pairs_array(n)
        assert len(p) == ps.total_pairs(n)
        if len(p):
            assert (p[:, 0] != p[:, 1]).all() and p.min() >= 0 and p.max() < n
            assert len(np.unique(_canon(p, n))) == len(p)


def test_criterion_4_violation_tightness():
    """test_acceptance.py:125-147: for odd N, step (N+1)/2 is the first
    that repeats a pair, and no earlier step does."""
    for n in range(3, 1000, 2):
        s_viol = ps.first_violation_step(n)
        assert s_viol == (n + 1) // 2
        i = np.repeat(np.arange(n, dtype=np.int64), s_viol)
        s = np.tile(np.arange(1, s_viol + 1, dtype=np.int64), n)
        key = _canon(np.stack([i, (i + s) % n], 1), n)
        assert np.bincount(key[s < s_viol], minlength=n * n).max() <= 1
        assert np.bincount(key, minlength=n * n).max() >= 2


def test_criterion_5_balance():
    """test_acceptance.py:150-161: step spread 0 (odd) / 1 (even), total N(N-1)/2."""
    for n in range(2, 2001):
        c = ps.step_counts(n)
        assert int(c.max() - c.min()) == (0 if n % 2 else 1)
        assert int(c.sum()) == ps.total_pairs(n)


@pytest.mark.gpu
def test_criterion_6_spi_equivalence_grid():
    """test_acceptance.py:164-187: totals identical across schedules and
    worker counts, and equal to the oracle (float64 spheres as the reference)."""
    from oracle import c_oracle
    from paper_1901_11204_b200 import spi_engine as se

    f = se.collision_indicator
    for n in [2, 3, 4, 5, 7, 8, 16, 31, 32, 64, 127, 128, 256, 257, 512]:
        spheres = gen.random_spheres(n, 6.0, 100 + n)
        base = se.spi_standard(spheres, f).total
        assert base == c_oracle.rows(spheres, 0, n, "standard")[0]
        assert se.spi_balanced(spheres, f).total == base
        for workers in (1, 2, 3, 7, 8):
            for schedule in se.SCHEDULES:
                assert se.spi_parallel(spheres, f, workers, schedule).total == base
    spheres = gen.random_spheres(10_000, 40.0, 99)
    base = se.spi_standard(spheres, f).total
    assert base == c_oracle.rows(spheres, 0, 10_000, "balanced")[0]
    assert se.spi_balanced(spheres, f).total == base
    for schedule in se.SCHEDULES:
        assert se.spi_parallel(spheres, f, 8, schedule).total == base


def test_criterion_7_depth_closed_forms():
    """test_acceptance.py:190-204 (closed forms): ceil((N-1)/2) < N-1."""
    from paper_1901_11204_b200 import spi_engine as se

    for n in list(range(3, 64)) + [127, 128, 511, 512, 10_001]:
        assert se._depth(n, "balanced") == math.ceil((n - 1) / 2)
        assert se._depth(n, "standard") == n - 1


@pytest.mark.gpu
def test_criterion_7_depth_public_result():
    """test_acceptance.py:201-203 through the public result object.  The
    reference passes `lambda a, b: 1`; a Python callable cannot run on the GPU,
    so the same nine objects go through collision_indicator (all coincident:
    every pair counts 1, like the lambda)."""
    from paper_1901_11204_b200 import spi_engine as se

    r = se.spi_balanced(np.zeros((9, 3)), se.collision_indicator)
    assert r.depth_per_worker == 4 and r.total == 36 and r.pairs_evaluated == 36


@pytest.mark.gpu
def test_criterion_8_physical_touch_bound():
    """test_acceptance.py:207-223: cells touched <= N (collisions), <= 7N (contacts)."""
    import paper_1901_11204_b200 as pc

    for n in [1, 16, 64, 257, 1024]:
        for v in range(20):
            beads, extent = gen.random_chain(n, 777 + v)
            space = pc.new_space(max(extent, 1))
            col = pc.count_collisions(beads, space)
            assert col.cells_touched <= n
            pc.reset_sparse(space, beads)
            con = pc.count_contacts(beads, space)
            assert con.cells_touched <= 7 * n
            assert sum(len(t) for t in space.touched) <= 7 * n
