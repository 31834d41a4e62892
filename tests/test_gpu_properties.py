"""Property tests on the GPU path, restating the reference's hypothesis suites
(test_lattice_counter.py:79-141, test_spi_engine.py:52-102) against the
drop-in API, with the pinned C oracle as the checker."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1901_11204_b200 as pc
from oracle import c_oracle
from paper_1901_11204_b200 import lattice_counter as lc
from paper_1901_11204_b200 import spi_engine as se

pytestmark = pytest.mark.gpu

coord = st.integers(min_value=-8, max_value=8)
bead_lists = st.lists(st.tuples(coord, coord, coord), max_size=64)


@given(bead_lists)
@settings(max_examples=150, deadline=None)
def test_collisions_and_contacts_match_oracle(beads):
    col, con = c_oracle.int_pairs(np.asarray(beads, dtype=np.int64).reshape(-1, 3)) if beads else (0, 0)
    sp = pc.new_space(8)
    assert pc.count_collisions(beads, sp).count == col == pc.oracle_collisions(beads)
    pc.reset_sparse(sp, beads)
    assert pc.count_contacts(beads, sp).count == con == pc.oracle_contacts(beads)


@given(bead_lists, st.randoms(use_true_random=False))
@settings(max_examples=60, deadline=None)
def test_permutation_invariance(beads, rnd):
    shuffled = list(beads)
    rnd.shuffle(shuffled)
    sp = pc.new_space(8)
    col = pc.count_collisions(beads, sp).count
    pc.reset_sparse(sp, beads)
    assert pc.count_collisions(shuffled, sp).count == col
    pc.reset_sparse(sp, shuffled)
    con = pc.count_contacts(beads, sp).count
    pc.reset_sparse(sp, beads)
    assert pc.count_contacts(shuffled, sp).count == con


@given(bead_lists, st.tuples(coord, coord, coord))
@settings(max_examples=60, deadline=None)
def test_translation_invariance(beads, offset):
    sp = pc.new_space(16)
    col = pc.count_collisions(beads, sp).count
    pc.reset_sparse(sp, beads)
    con = pc.count_contacts(beads, sp).count
    pc.reset_sparse(sp, beads)
    shifted = [(x + offset[0], y + offset[1], z + offset[2]) for x, y, z in beads]
    assert pc.count_collisions(shifted, sp).count == col
    pc.reset_sparse(sp, shifted)
    assert pc.count_contacts(shifted, sp).count == con
    pc.reset_sparse(sp, shifted)
    assert sp.is_zero()


@given(bead_lists)
@settings(max_examples=60, deadline=None)
def test_contact_accumulator_parity(beads):
    sp = pc.new_space(8)
    doubled = lc.contact_accumulator(beads, sp)
    assert doubled % 2 == 0
    pc.reset_sparse(sp, beads)
    assert pc.count_contacts(beads, sp).count == doubled // 2


sphere_sets = st.integers(min_value=0, max_value=400).flatmap(
    lambda n: st.tuples(st.just(n), st.floats(min_value=0.5, max_value=20.0), st.integers(0, 2**31 - 1)))


@given(sphere_sets, st.sampled_from(["float32", "float64"]), st.integers(min_value=1, max_value=9))
@settings(max_examples=60, deadline=None)
def test_spi_schedules_and_workers_agree(spec, dtype, workers):
    n, box, seed = spec
    objs = np.random.default_rng(seed).random((n, 3)) * box
    objs = objs.astype(dtype)
    want, _, _ = c_oracle.rows(objs, 0, n, "standard") if n else (0, 0.0, 0)
    for sched in se.SCHEDULES:
        r = se.spi_parallel(objs, se.collision_indicator, workers, sched)
        assert r.total == want and sum(r.partials) == want
        blocks = se._partition(n, workers)
        for b, part in zip(blocks, r.partials):
            assert part == c_oracle.rows(objs, b.start, b.stop, sched)[0] if n else part == 0
    assert se.spi_standard(objs, se.collision_indicator).total == want
    assert se.spi_balanced(objs, se.collision_indicator).total == want
