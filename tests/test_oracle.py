"""Pin the CPU oracle (test infrastructure) to the reference's own outputs.

The golden JSON was produced by running the unmodified reference
(tests/golden/make_golden.py); the oracle is trusted by the GPU parity
tests only because these checks pass.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import c_oracle, numpy_port as npo
from tests.helpers import config_input, digest, lattice_input, spi_input


def _f(name):
    return npo.collision_indicator if name == "collision" else npo.inverse_square


def test_numpy_port_matches_reference_spi(golden_small):
    for case in golden_small["spi_cases"]:
        if case["n"] > 2100:
            continue
        objs = spi_input(case)
        assert digest(objs) == case["input_sha256"], case["tag"]
        f = _f(case["f"])
        for entry in case["parallel"]:
            total, partials, worker_pairs = npo.spi_partials(objs, f, entry["workers"], entry["schedule"])
            assert list(worker_pairs) == entry["worker_pairs"], case["tag"]
            if case["f"] == "collision":
                assert list(partials) == entry["partials"], case["tag"]
                assert total == entry["total"]
            else:
                # float64 per-row numpy sums in the same order: ulp-identical
                assert partials == pytest.approx(entry["partials"], rel=1e-14, abs=1e-300), case["tag"]


def test_c_oracle_matches_reference_spi(golden_small):
    for case in golden_small["spi_cases"]:
        objs = spi_input(case)
        for entry in case["parallel"]:
            n = case["n"]
            bounds = npo.partition(n, entry["workers"])
            for (lo, hi), want, wp in zip(bounds, entry["partials"], entry["worker_pairs"]):
                c, s, p = c_oracle.rows(objs, lo, hi, entry["schedule"])
                assert p == wp
                if case["f"] == "collision":
                    assert c == want, (case["tag"], lo, hi)
                else:
                    assert s == pytest.approx(want, rel=1e-12), (case["tag"], lo, hi)


def test_schedule_cover_and_depth_port():
    for n in range(1, 60):
        for sched in ("standard", "balanced"):
            seen = set()
            for i in range(n):
                for j in npo.partners(n, i, sched):
                    key = (min(i, int(j)), max(i, int(j)))
                    assert key not in seen
                    seen.add(key)
            assert len(seen) == n * (n - 1) // 2
            for lo in range(0, n + 1, 7):
                for hi in range(lo, n + 1, 5):
                    assert npo.row_pairs(n, lo, hi, sched) == sum(len(npo.partners(n, i, sched)) for i in range(lo, hi))


def test_indicator_port(golden_small):
    for case in golden_small["indicator_cases"]:
        pts = np.asarray(case["points"], dtype=np.float64)
        got = [int(npo.collision_indicator(a, b)) for a, b in zip(pts[0::2], pts[1::2])]
        assert got == case["values"], case["name"]


def test_lattice_port(golden_small):
    for case in golden_small["lattice_cases"]:
        beads = lattice_input(case)
        assert npo.oracle_collisions(beads) == case["oracle_collisions"], case["tag"]
        assert npo.oracle_contacts(beads) == case["oracle_contacts"], case["tag"]
        col, con = c_oracle.int_pairs(beads)
        assert (col, con) == (case["oracle_collisions"], case["oracle_contacts"]), case["tag"]
        # the row-range integer oracle: any partition of the rows adds up, under both schedules
        n = len(beads)
        for sched in ("standard", "balanced"):
            parts = [c_oracle.int_rows(beads, lo, hi, sched) for lo, hi in npo.partition(n, 3)]
            assert (sum(p[0] for p in parts), sum(p[1] for p in parts)) == (col, con), case["tag"]
        if "count_collisions" in case:
            assert list(npo.count_collisions(beads, case["half_extent"])) == case["count_collisions"], case["tag"]
            cells = npo.new_dense_space(case["half_extent"])
            assert list(npo.count_collisions_dense(beads, cells, case["half_extent"])) == case["count_collisions"]
            assert not cells.any()  # left clean by the sparse reset
            assert list(npo.count_contacts(beads, case["half_extent"])) == case["count_contacts"], case["tag"]


def test_config1_port(golden_configs):
    g = golden_configs["cfg1"]
    for name, key in (("cfg1_cloud", "cloud"), ("cfg1_chain", "chain")):
        beads = config_input(golden_configs, name)
        assert digest(beads) == g[key]["sha256"]
        assert c_oracle.int_pairs(beads) == (g[key]["oracle_collisions"], g[key]["oracle_contacts"])


@pytest.mark.slow
def test_config_row_samples_c_oracle(golden_configs):
    for name in ("cfg2", "cfg3", "cfg4u", "cfg4c"):
        objs = config_input(golden_configs, name)
        assert digest(objs) == golden_configs[name]["sha256"], name
        for smp in golden_configs[name]["samples"]:
            lo, hi = smp["rows"]
            c, s, p = c_oracle.rows(objs, lo, hi, smp["schedule"])
            assert (c, p) == (smp["count"], smp["pairs"]), (name, smp)
            assert s == pytest.approx(smp["inv_sum"], rel=1e-12), (name, smp)


@pytest.mark.slow
def test_config2_full_totals_c_oracle(golden_configs):
    objs = config_input(golden_configs, "cfg2")
    n = len(objs)
    for sched in ("standard", "balanced"):
        c, _, p = c_oracle.rows(objs, 0, n, sched)
        assert c == golden_configs["cfg2"][sched]["total"] == 32178
        assert p == golden_configs["cfg2"][sched]["pairs"]


@pytest.mark.slow
def test_config5_counting_array_port(golden_configs):
    pts = config_input(golden_configs, "cfg5")
    g = golden_configs["cfg5"]
    assert digest(pts) == g["sha256"]
    count, n, touched = npo.count_collisions(pts, 512)
    assert (count, n, touched) == (g["count"], g["beads_processed"], g["cells_touched"])
