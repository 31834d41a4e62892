"""The repo's generator restatement reproduces the reference's inputs bit-for-bit
(digests recorded from the reference by tests/golden/make_golden.py), plus
the reference's own generator tests (tests/test_generators.py:12-74)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1901_11204_b200 import generators as gen
from tests.helpers import digest


def test_digests_match_reference(golden_small):
    for rec in golden_small["generator_digests"]:
        fn, args = rec["fn"], rec["args"]
        if fn == "random_chain":
            beads, ext = gen.random_chain(*args)
            assert ext == rec["extent"]
            got = beads
        elif fn == "normal_cloud":
            got = gen.normal_cloud(*args)
        elif fn == "random_spheres":
            got = gen.random_spheres(*args)
        else:
            seed, stream, n = args
            got = gen._box_muller(gen._rng(seed, stream), n)
        assert digest(got) == rec["sha256"], (fn, args)


def test_chain_unit_steps_and_determinism():
    for seed in (0, 1, 42):
        beads, extent = gen.random_chain(200, seed)
        assert (np.abs(np.diff(beads, axis=0)).sum(axis=1) == 1).all()
        assert beads[0].tolist() == [0, 0, 0]
        assert extent >= np.abs(beads).max()
    a, _ = gen.random_chain(500, 7)
    b, _ = gen.random_chain(500, 7)
    assert (a == b).all()
    assert gen.random_chain(1, 0)[0].tolist() == [[0, 0, 0]]


def test_cloud_and_spheres():
    assert (gen.normal_cloud(50, 1e-9, 4, 0) == 0).all()
    wide = gen.normal_cloud(1000, 500.0, 10, 2)
    assert np.abs(wide).max() == 10
    s = gen.random_spheres(100, 6.5, 5)
    assert s.shape == (100, 3) and s.min() >= 0 and s.max() <= 6.5


def test_parameter_validation():
    with pytest.raises(ValueError):
        gen.random_chain(0, 0)
    with pytest.raises(ValueError):
        gen.normal_cloud(10, 0.0, 4, 0)
    with pytest.raises(ValueError):
        gen.random_spheres(10, -1.0, 0)


def test_benchmark_recipes(golden_configs):
    assert gen.contact_box_edge(65536) == golden_configs["cfg2"]["args"][1]
    assert gen.contact_box_edge(2**20) == golden_configs["cfg3"]["args"][1]
    c = gen.clustered_spheres(2**22).astype(np.float32)
    assert digest(c) == golden_configs["cfg4c"]["sha256"]
