"""pair_schedule mirror: the reference's schedule tests (test_pair_schedule.py)
plus the golden step counts / pair arrays recorded from the reference."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1901_11204_b200 import pair_schedule as ps
from tests.helpers import digest


def brute(n):
    return {(i, j) for i in range(n) for j in range(i + 1, n)}


def unordered(seq):
    return [(min(i, j), max(i, j)) for i, j in seq]


def test_examples():
    assert (ps.reach(5, 1, 1), ps.reach(5, 4, 1), ps.reach(7, 3, 3)) == (2, 0, 6)
    assert (ps.reached(5, 1, 1), ps.reached(5, 1, 2), ps.reached(3, 0, 1)) == (0, 4, 2)
    assert [ps.steps_for(4, i) for i in range(4)] == [2, 2, 1, 1]
    assert ps.steps_for(1, 0) == 0
    assert (ps.first_violation_step(5), ps.first_violation_step(3), ps.first_violation_step(7)) == (3, 2, 4)
    with pytest.raises(IndexError):
        ps.reach(5, 5, 1)
    with pytest.raises(ValueError):
        ps.reach(5, 0, 0)
    with pytest.raises(ValueError):
        ps.reached(0, 0, 1)
    with pytest.raises(ValueError):
        ps.steps_for(0, 0)
    with pytest.raises(ValueError):
        ps.first_violation_step(4)


def test_golden_schedules(golden_small):
    for case in golden_small["schedule_cases"]:
        n = case["n"]
        assert ps.step_counts(n).tolist() == case["steps"]
        assert digest(ps.pairs_array(n)) == case["pairs_sha256"]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 16, 17, 100, 101, 256, 257])
def test_cover_once(n):
    got = unordered(ps.pairs(n))
    assert len(got) == len(set(got)) == ps.total_pairs(n)
    assert set(got) == brute(n)
    assert [tuple(r) for r in ps.pairs_array(n)] == list(ps.pairs(n))


def test_balance_and_row_pairs():
    for n in range(1, 200):
        c = ps.step_counts(n)
        assert int(c.sum()) == ps.total_pairs(n)
        if n >= 2:
            assert int(c.max() - c.min()) == (0 if n % 2 else 1)
        for lo in range(0, n + 1, max(1, n // 5)):
            for hi in range(lo, n + 1, max(1, n // 4)):
                assert ps.row_pairs(n, lo, hi, "balanced") == int(c[lo:hi].sum())
                assert ps.row_pairs(n, lo, hi, "standard") == sum(n - 1 - i for i in range(lo, hi))


@pytest.mark.parametrize("n", [3, 5, 7, 11, 25])
def test_reciprocity(n):
    owner = {}
    for i, j in ps.pairs(n):
        owner[(min(i, j), max(i, j))] = i
    for i in range(n):
        for j in range(i + 1, n):
            assert owner[(i, j)] == (i if j - i <= (n - 1) // 2 else j)


def test_violation_introduces_duplicates():
    for n in (3, 5, 7, 9, 21, 99, 101):
        s = ps.first_violation_step(n)
        emitted = unordered(ps.pairs(n))
        ext = emitted + [tuple(sorted((i, (i + s) % n))) for i in range(n)]
        assert len(set(ext)) < len(ext)
