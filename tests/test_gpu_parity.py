"""GPU parity: the drop-in API (ctypes -> libpaircount.so on the B200) against
the reference's outputs (golden fixtures) and the pinned CPU oracle.

Bars (BASELINE.json north_star): integer counts bit-exact; the float
inverse-square sum within REL_TOL = 1e-5 relative of the float64 reference.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_1901_11204_b200 as pc
from paper_1901_11204_b200 import _lib
from paper_1901_11204_b200 import generators as gen
from paper_1901_11204_b200 import lattice_counter as lc
from paper_1901_11204_b200 import spi_engine as se
from oracle import c_oracle
from tests.helpers import config_input, digest, lattice_input, spi_input

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5  # fp32 interaction sum vs float64 reference (north_star)


def _f(name):
    return se.collision_indicator if name == "collision" else se.inverse_square


def _close(got, want):
    return got == pytest.approx(want, rel=REL_TOL, abs=1e-9)


# ------------------------------------------------------------------ SPI --

def test_spi_golden_cases(golden_small):
    for case in golden_small["spi_cases"]:
        objs = spi_input(case)
        assert digest(objs) == case["input_sha256"], case["tag"]
        f = _f(case["f"])
        for name, fn in (("standard", se.spi_standard), ("balanced", se.spi_balanced)):
            if name not in case:
                continue
            r = fn(objs, f)
            want = case[name]
            assert r.pairs_evaluated == want["pairs"] and r.depth_per_worker == want["depth"], case["tag"]
            if case["f"] == "collision":
                assert r.total == want["total"] and isinstance(r.total, int), (case["tag"], name)
            else:
                assert isinstance(r.total, float) and _close(r.total, want["total"]), (case["tag"], name)
        for entry in case["parallel"]:
            r = se.spi_parallel(objs, f, entry["workers"], entry["schedule"])
            assert list(r.worker_pairs) == entry["worker_pairs"], case["tag"]
            assert r.depth_per_worker == entry["depth"]
            if case["f"] == "collision":
                assert list(r.partials) == entry["partials"], (case["tag"], entry["workers"], entry["schedule"])
                assert r.total == entry["total"]
            else:
                for got, want in zip(r.partials, entry["partials"]):
                    assert _close(got, want), (case["tag"], entry)


def test_reference_unit_cases():
    # test_spi_engine.py:32-49 with GPU-supported interactions
    assert se.spi_standard([se.Sphere(0.0, 0.0, 0.0)] * 3, se.collision_indicator).total == 3
    assert se.spi_balanced([se.Sphere(0.0, 0.0, 0.0)] * 3, se.collision_indicator).total == 3
    spheres = gen.random_spheres(100, 4.0, 3)
    for sched, seq in (("standard", se.spi_standard), ("balanced", se.spi_balanced)):
        assert se.spi_parallel(spheres, se.collision_indicator, 1, sched).total == seq(spheres, se.collision_indicator).total
    runs = {se.spi_parallel(gen.random_spheres(200, 3.0, 9), se.collision_indicator, 4, "balanced").total for _ in range(3)}
    assert len(runs) == 1
    # (n, 1) / (n, 2) objects are padded with zero coordinates
    line = np.array([0.0, 0.5, 2.0, 2.9, 10.0])[:, None]
    assert se.spi_standard(line, se.collision_indicator).total == 2
    ints = np.array([[0, 0, 0], [0, 0, 0], [1, 0, 0]], dtype=np.int64)
    assert se.spi_balanced(ints, se.collision_indicator).total == 1


def test_near_boundary_exactness():
    # pairs at d^2 = 1 +- ulp far from the origin, where fp32 Gram arithmetic is coarsest
    rng = np.random.default_rng(5)
    for base in (0.0, 100.0, 1000.0, 1.0e5):
        a = base + rng.random((500, 3)) * 50
        d = rng.normal(size=(500, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        b = a + d * np.where(rng.random((500, 1)) < 0.5, np.nextafter(1.0, 0.0), np.nextafter(1.0, 2.0))
        pts = np.empty((1000, 3))
        pts[0::2], pts[1::2] = a, b
        for arr in (pts, pts.astype(np.float32)):
            want, _, _ = c_oracle.rows(arr, 0, len(arr), "balanced")
            assert se.spi_balanced(arr, se.collision_indicator).total == want
            assert se.spi_standard(arr, se.collision_indicator).total == want


@pytest.mark.parametrize("n", [2, 3, 63, 64, 65, 127, 129, 1023, 1024, 1025, 4095, 16383, 16384, 16385, 20001])
def test_sizes_vs_c_oracle(n):
    # tile-boundary sizes on both kernel configurations (small < 16384 <= big)
    box = max(2.0, (n / 2.0) ** (1 / 3) * 1.6)
    objs = gen.random_spheres(n, box, n).astype(np.float32)
    for sched in ("standard", "balanced"):
        for workers in (1, 3):
            blocks = se._partition(n, workers)
            r = se.spi_parallel(objs, se.collision_indicator, workers, sched)
            for b, got in zip(blocks, r.partials):
                c, _, _ = c_oracle.rows(objs, b.start, b.stop, sched)
                assert got == c, (n, sched, workers)
        r = se.spi_parallel(objs, se.inverse_square, 2, sched)
        for b, got in zip(se._partition(n, 2), r.partials):
            _, s, _ = c_oracle.rows(objs, b.start, b.stop, sched)
            assert _close(got, s), (n, sched)


def test_dense_every_pair_in_contact():
    objs = gen.random_spheres(3000, 0.5, 1)
    assert se.spi_balanced(objs, se.collision_indicator).total == 3000 * 2999 // 2
    assert se.spi_standard(objs.astype(np.float32), se.collision_indicator).total == 3000 * 2999 // 2


def test_tilings_agree():
    objs = gen.random_spheres(40_000, 30.0, 4).astype(np.float32)
    n = len(objs)
    want, s_want, _ = c_oracle.rows(objs, 0, n, "balanced")
    for tiling in (_lib.PC_TILE_FLAT, _lib.PC_TILE_PER_ROW_TILE):
        (r,) = _lib.pairs_host(objs, _lib.PC_COLLISION, _lib.PC_BALANCED, [0, n], tiling)
        assert r.count == want
        (r,) = _lib.pairs_host(objs, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n], tiling)
        assert r.count == want and _close(r.sum, s_want)
    with pytest.raises(ValueError):
        _lib.pairs_host(objs, _lib.PC_COLLISION, _lib.PC_STANDARD, [0, n], _lib.PC_TILE_FLAT)


# --------------------------------------------------------- BASELINE configs --

def test_config1_integer_coincidence(golden_configs):
    for name, key in (("cfg1_cloud", "cloud"), ("cfg1_chain", "chain")):
        beads = config_input(golden_configs, name)
        g = golden_configs["cfg1"][key]
        assert pc.oracle_collisions(beads) == g["oracle_collisions"]
        assert pc.oracle_contacts(beads) == g["oracle_contacts"]


def test_config2_naive_and_balanced(golden_configs):
    objs = config_input(golden_configs, "cfg2")
    g = golden_configs["cfg2"]
    for name, fn in (("standard", se.spi_standard), ("balanced", se.spi_balanced)):
        r = fn(objs, se.collision_indicator)
        assert (r.total, r.pairs_evaluated, r.depth_per_worker) == (g[name]["total"], g[name]["pairs"], g[name]["depth"])
    for smp in g["samples"]:
        cnt, pairs = se.spi_rows(objs, se.collision_indicator, tuple(smp["rows"]), smp["schedule"])
        assert (cnt, pairs) == (smp["count"], smp["pairs"])
        s, _ = se.spi_rows(objs, se.inverse_square, tuple(smp["rows"]), smp["schedule"])
        assert _close(s, smp["inv_sum"])


@pytest.mark.parametrize("name", ["cfg3", "cfg4u", "cfg4c"])
def test_large_config_row_samples(golden_configs, name):
    objs = config_input(golden_configs, name)
    assert digest(objs) == golden_configs[name]["sha256"]
    for smp in golden_configs[name]["samples"]:
        rows = tuple(smp["rows"])
        cnt, pairs = se.spi_rows(objs, se.collision_indicator, rows, smp["schedule"])
        assert (cnt, pairs) == (smp["count"], smp["pairs"]), smp
        s, _ = se.spi_rows(objs, se.inverse_square, rows, smp["schedule"])
        assert _close(s, smp["inv_sum"]), smp


def test_config3_full_size_properties(golden_configs):
    """N = 2^20: beyond the CPU oracle; pinned by size-independent properties:
    standard == balanced, 1 range == sum of 8 ranges, count(INVSQ kernel) ==
    count(Gram kernel), determinism."""
    objs = config_input(golden_configs, "cfg3")
    n = len(objs)
    b = se.spi_balanced(objs, se.collision_indicator).total
    s = se.spi_standard(objs, se.collision_indicator).total
    assert b == s
    par = se.spi_parallel(objs, se.collision_indicator, 8, "balanced")
    assert par.total == b and sum(par.partials) == b
    (r,) = _lib.pairs_host(objs, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    assert r.count == b
    (r2,) = _lib.pairs_host(objs, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    assert r2.sum == r.sum  # bitwise deterministic
    (rs,) = _lib.pairs_host(objs, _lib.PC_COLLISION_INVSQ, _lib.PC_STANDARD, [0, n])
    assert rs.count == b and _close(rs.sum, r.sum)


def test_config5_counting_array(golden_configs):
    pts = config_input(golden_configs, "cfg5")
    g = golden_configs["cfg5"]
    sp = pc.new_space(512)
    rep = pc.count_collisions(pts, sp)
    assert (rep.count, rep.beads_processed, rep.cells_touched) == (g["count"], g["beads_processed"], g["cells_touched"])
    pc.reset_sparse(sp)
    assert sp.is_zero()
    # counting array == all-pairs count on a slice (north_star: "checked against the all-pairs count")
    part = pts[:200_000]
    rep = pc.count_collisions(part, sp)
    assert rep.count == pc.oracle_collisions(part)


def _dense_cases():
    rng = np.random.default_rng(21)
    yield 64, rng.integers(-64, 65, size=(2_000_003, 3))                       # uniform, n % 4 != 0
    yield 64, rng.integers(-5, 5, size=(600_000, 3))                            # one heavy region
    yield 64, np.zeros((100_000, 3), dtype=np.int64) + 7                        # a single cell
    yield 150, np.concatenate([rng.integers(-150, -140, size=(300_000, 3)),      # two far clusters
                               rng.integers(140, 151, size=(300_000, 3))])
    yield 64, rng.integers(-64, 65, size=(1_000_000, 3)).astype(np.int32)       # vectorised int32 path
    yield 64, rng.integers(-64, 65, size=(1_000_001, 3)).astype(np.int32)[1:]   # int32, unaligned start


@pytest.mark.parametrize("case", range(6))
def test_dense_regime_counting_array(case):
    # beads > cells/64 on a clean grid: keys + tile sort + segment partition +
    # shared-memory slabs.  Oracle: keys histogram on the host (Alg. 1 result).
    a, beads = list(_dense_cases())[case]
    side = 2 * a + 3
    b64 = beads.astype(np.int64)
    keys = ((b64[:, 0] + a + 1) * side + (b64[:, 1] + a + 1)) * side + (b64[:, 2] + a + 1)
    occ = np.bincount(keys, minlength=side**3)
    sp = pc.new_space(a)
    assert len(beads) * 64 > side**3  # the dense regime
    if beads.dtype == np.int32:  # device-resident int32 beads (bench's layout), aligned or not
        import ctypes

        import torch

        lib = _lib.load()
        full = torch.from_numpy(np.ascontiguousarray(np.concatenate([beads[:1], beads]))).cuda()
        dev = full[1:] if case % 2 else full[:-1]  # 12-byte offset (scalar loads) or 16-byte aligned
        if not case % 2:
            dev.copy_(torch.from_numpy(beads).cuda())
        kbuf = torch.empty(len(beads), dtype=torch.int32, device="cuda")
        r = _lib.LatticeResult()
        _lib.check(lib.pc_lattice_collisions(dev.data_ptr(), _lib.PC_I32, 1, len(beads), a, sp.grid_ptr,
                                             kbuf.data_ptr(), 1, ctypes.byref(r), None))
        assert r.error == 0
        count, touched = int(r.count), int(r.cells_touched)
        torch.cuda.synchronize()
        assert np.array_equal(np.asarray(sp.cells).ravel(), occ.astype(np.uint32))
        _lib.check(lib.pc_lattice_clear(sp.grid_ptr, a, None))
    else:
        rep = pc.count_collisions(beads, sp)
        count, touched = rep.count, rep.cells_touched
        assert np.array_equal(np.asarray(sp.cells).ravel(), occ.astype(np.uint32))
        pc.reset_sparse(sp)
    assert count == int((occ * (occ - 1) // 2).sum())
    assert touched == int(np.count_nonzero(occ))
    assert sp.is_zero()
    # Alg. 2 on the same beads (dense regime: slab histogram + one stencil pass)
    offs = np.array([1, -1, side, -side, side * side, -side * side], dtype=np.int64)
    doubled = int(sum(occ[keys + o].sum(dtype=np.int64) for o in offs))
    touched7 = len(np.unique(np.concatenate([keys] + [keys + o for o in offs])))
    rep = pc.count_contacts(b64, sp)
    assert (rep.count, rep.cells_touched) == (doubled // 2, touched7)
    assert np.array_equal(np.asarray(sp.cells).ravel(), occ.astype(np.uint32))  # left populated
    pc.reset_sparse(sp)
    assert sp.is_zero()


# ------------------------------------------------------------- lattice --

def test_lattice_golden(golden_small):
    for case in golden_small["lattice_cases"]:
        beads = lattice_input(case)
        assert pc.oracle_collisions(beads) == case["oracle_collisions"], case["tag"]
        assert pc.oracle_contacts(beads) == case["oracle_contacts"], case["tag"]
        if "count_collisions" not in case:
            continue
        sp = pc.new_space(case["half_extent"])
        col = pc.count_collisions(beads, sp)
        assert [col.count, col.beads_processed, col.cells_touched] == case["count_collisions"], case["tag"]
        pc.reset_sparse(sp, beads)
        assert sp.is_zero()
        con = pc.count_contacts(beads, sp)
        assert [con.count, con.beads_processed, con.cells_touched] == case["count_contacts"], case["tag"]
        pc.reset_sparse(sp, beads)
        assert lc.contact_accumulator(beads, pc.new_space(case["half_extent"])) == case["contact_accumulator"]


def test_lattice_reference_unit_cases():
    # test_lattice_counter.py:23-76,144-182
    assert pc.new_space(0).interior_cells == 1 and pc.new_space(0).cells.size == 27
    sp = pc.new_space(1)
    assert pc.count_collisions([(0, 0, 0)] * 5, sp).count == 10
    assert sum(len(t) for t in sp.touched) <= 5
    pc.reset_sparse(sp)
    assert sp.is_zero() and not sp.touched
    with pytest.raises(lc.CoordinateRangeError, match="bead 1"):
        pc.count_collisions([(0, 0, 0), (3, 0, 0)], pc.new_space(2))
    sp = pc.new_space(2)
    pc.count_collisions([(1, 1, 0), (0, 0, 0)], sp)
    sp.touched.clear()
    pc.reset_sparse(sp, [(1, 1, 0), (0, 0, 0)])
    assert sp.is_zero()
    sp = pc.new_space(1)
    pc.count_contacts([(1, 1, 1), (-1, -1, -1), (1, -1, 0)], sp)
    cells = sp.cells
    assert cells.sum() == cells[1:-1, 1:-1, 1:-1].sum()


def test_lattice_dirty_space_semantics():
    # counting into a populated space evaluates the reference's formulas exactly
    rng = np.random.default_rng(0)
    first = rng.integers(-3, 4, size=(300, 3))
    second = rng.integers(-3, 4, size=(200, 3))
    import importlib
    npo = importlib.import_module("oracle.numpy_port")
    sp = pc.new_space(4)
    pc.count_collisions(first, sp)
    rep = pc.count_collisions(second, sp)  # no reset in between
    both = np.concatenate([first, second])
    # reference: occ = final occupancy of each second-vector bead's cell
    side = 11
    flat = lambda b: ((b[:, 0] + 5) * side + (b[:, 1] + 5)) * side + (b[:, 2] + 5)
    occ = np.bincount(flat(both), minlength=side**3)[flat(second)]
    assert rep.count == int((occ - 1).sum()) // 2
    assert rep.cells_touched == len(np.unique(flat(second)))
    pc.reset_sparse(sp)
    assert sp.is_zero()
    assert pc.count_collisions(second, sp).count == npo.count_collisions(second, 4)[0]


def test_sparse_reset_soundness_random():
    rng = np.random.default_rng(1)
    reused = pc.new_space(8)
    for _ in range(30):
        first = rng.integers(-8, 9, size=(rng.integers(0, 65), 3))
        second = rng.integers(-8, 9, size=(rng.integers(0, 65), 3))
        pc.count_contacts(first, reused)
        pc.reset_sparse(reused, first)
        fresh = pc.new_space(8)
        assert pc.count_contacts(second, reused).count == pc.count_contacts(second, fresh).count
        pc.reset_sparse(reused, second)
        assert pc.count_collisions(second, reused).count == pc.oracle_collisions(second)
        pc.reset_sparse(reused, second)


def test_chains_vs_oracle():
    # acceptance criterion 1/2 (test_acceptance.py:49-84), 40 chains per size
    for n in (1, 2, 3, 16, 64, 257, 1024):
        for v in range(40):
            beads, ext = gen.random_chain(n, 1000 * n + v)
            sp = pc.new_space(max(ext, 1))
            col = pc.count_collisions(beads, sp)
            pc.reset_sparse(sp, beads)
            doubled = lc.contact_accumulator(beads, sp)
            pc.reset_sparse(sp, beads)
            want_col, want_con = c_oracle.int_pairs(beads)
            assert col.count == want_col == pc.oracle_collisions(beads)
            assert doubled % 2 == 0 and doubled // 2 == want_con == pc.oracle_contacts(beads)


def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


def test_batched_small_vectors():
    # §8(f4): one launch for many vectors == count_collisions + reset_sparse per vector
    vectors = [gen.random_chain(n, 5000 + v)[0] for n in (1, 2, 3, 16, 64, 257, 1024, 4096) for v in range(12)]
    vectors += [np.zeros((40, 3), dtype=np.int64), np.zeros((0, 3), dtype=np.int64), gen.random_chain(6000, 1)[0]]
    ext = max(int(np.abs(v).max()) if len(v) else 0 for v in vectors)
    sp = pc.new_space(ext)
    reps = pc.count_collisions_batch(vectors, sp)
    assert sp.is_zero() and not sp.touched
    for v, rep in zip(vectors, reps):
        want = c_oracle.int_pairs(v)[0] if len(v) else 0
        ref = lc.count_collisions(v, sp)
        pc.reset_sparse(sp)
        assert (rep.count, rep.beads_processed, rep.cells_touched) == (want, len(v), ref.cells_touched)
    with pytest.raises(lc.CoordinateRangeError, match="bead 1"):
        pc.count_collisions_batch([[(0, 0, 0)], [(0, 0, 0), (ext + 1, 0, 0)]], sp)
    # int64 coordinates that would wrap into range if narrowed naively
    for bad in (2**32, 2**32 + 1, -(2**32), 2**62, -(2**63)):
        with pytest.raises(lc.CoordinateRangeError, match="bead 2"):
            pc.count_collisions_batch([[(0, 0, 0)], [(1, 1, 1), (0, 0, 0), (0, bad, 0)]], sp)
    assert sp.is_zero()


def test_batched_all_pairs_oracles():
    # oracle_collisions_batch / oracle_contacts_batch == per-vector oracles (C oracle)
    vectors = [gen.random_chain(n, 9000 + n + v)[0] for n in (1, 2, 3, 16, 64, 257, 1024, 4096) for v in range(6)]
    vectors += [np.zeros((0, 3), dtype=np.int64), np.zeros((40, 3), dtype=np.int64),
                np.array([[2**62, 0, 0], [-(2**62), 0, 0], [1, 0, 0], [0, 0, 0]], dtype=np.int64),  # wrap-around
                gen.random_chain(5000, 3)[0]]                                                    # > 4096: fallback
    cols = pc.oracle_collisions_batch(vectors)
    cons = pc.oracle_contacts_batch(vectors)
    for v, c, m in zip(vectors, cols, cons):
        assert (c, m) == c_oracle.int_pairs(v), len(v)
    # float predicates through the C ABI: exact count, float64 sum
    rng = np.random.default_rng(4)
    objs = [np.ascontiguousarray(rng.random((k, 3)) * (k ** (1 / 3)) * 1.2) for k in (2, 5, 100, 777, 4096)]
    objs.append(np.array([[0.0, 0.0, 0.0], [np.nan, 0.0, 0.0]]))
    for code in (_lib.PC_COLLISION, _lib.PC_COLLISION_INVSQ):
        res = _lib.pairs_batch(objs, code)
        for o, r in zip(objs, res):
            if not np.isfinite(o).all():
                assert r.error == _lib.PC_ERR_DOMAIN
                continue
            want_c, want_s, pairs = c_oracle.rows(o, 0, len(o), "balanced")
            assert (r.error, r.count, r.pairs) == (0, want_c, pairs)
            if code == _lib.PC_COLLISION_INVSQ:
                assert r.sum == pytest.approx(want_s, rel=1e-12)


def test_batch_entry_points_agree():
    # pc_lattice_collisions_vectors (separate host vectors, int32 and int64) ==
    # pc_lattice_collisions_batch (one packed array + offsets)
    import ctypes

    lib = _lib.load()
    vectors = [np.zeros((0, 3), dtype=np.int64)] + [gen.random_chain(n, 800 + n)[0] for n in (1, 5, 300, 2000, 4096, 4097)]
    a = max(int(np.abs(v).max()) for v in vectors if len(v))
    lengths = np.array([len(v) for v in vectors], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    packed = np.ascontiguousarray(np.concatenate(vectors))
    want = (_lib.LatticeResult * len(vectors))()
    _lib.check(lib.pc_lattice_collisions_batch(packed.ctypes.data, _lib.PC_I64, 0, offsets.ctypes.data,
                                               len(vectors), a, ctypes.addressof(want), None))
    for dt, code in ((np.int64, _lib.PC_I64), (np.int32, _lib.PC_I32)):
        arrs = [np.ascontiguousarray(v.astype(dt)) for v in vectors]
        ptrs = np.array([x.__array_interface__["data"][0] for x in arrs], dtype=np.uintp)
        got = (_lib.LatticeResult * len(vectors))()
        _lib.check(lib.pc_lattice_collisions_vectors(ptrs.ctypes.data, lengths.ctypes.data, code, len(vectors), a,
                                                     ctypes.addressof(got), None))
        for v, g, w in zip(vectors, got, want):
            assert (g.count, g.cells_touched, g.error, g.beads_processed) == \
                (w.count, w.cells_touched, w.error, w.beads_processed)
            if len(v) and len(v) <= 4096:
                assert g.error == 0 and g.count == c_oracle.int_pairs(v)[0]
        assert got[-1].error == _lib.PC_ERR_ARG  # > 4096 beads: the caller routes it through the grid


def _invsq_cases():
    rng = np.random.default_rng(11)
    a = rng.random((1500, 3)) * 6.0
    yield "f64 cluster far from the origin", a + 1.0e4
    two = np.concatenate([a, rng.random((1500, 3)) * 6.0 + np.array([1.0e5, 0.0, 0.0])])
    yield "f64 two clusters 1e5 apart", two
    yield "f64 default generator dtype", gen.random_spheres(3000, 80.0, 5)
    yield "f64 huge offset, unit spacing", rng.random((1000, 3)) * 3.0 + 3.0e7
    ints = rng.integers(0, 4, size=(1500, 3)) + np.int64(2**40)
    yield "int64 near 2^40", ints
    yield "int64 two clusters", np.concatenate([ints, ints[:700] - np.int64(2**41)])
    yield "int32 spread", rng.integers(-2**30, 2**30, size=(800, 3)).astype(np.int32)
    # n >= 16384: the big-tile compensated configuration
    yield "f64 big config, offset cluster", rng.random((40_000, 3)) * 34.0 + np.array([5.0e3, -2.0e4, 7.0e2])
    # spans beyond 2^26: the float64 path (pairs_f64_kernel)
    far = rng.random((1200, 3)) * 5.0
    far[600:] += np.array([1.0e10, -3.0e9, 0.0])
    yield "f64 two clusters 1e10 apart", far
    ifar = rng.integers(0, 5, size=(1000, 3)).astype(np.int64)
    ifar[500:] += np.int64(2**50)
    yield "int64 two clusters 2^50 apart", ifar
    big = rng.random((20_000, 3)) * 40.0
    big[::2] += 4.0e8
    yield "f64 big config, span 4e8", big


@pytest.mark.parametrize("case", range(11))
def test_inverse_square_sum_tight_for_non_f32_inputs(case):
    # float64 / integer coordinates: the kernel must not lose the pair separation
    # to fp32 rounding of large coordinates (compensated hi+lo staging, DESIGN.md
    # §3).  Bar: 2e-6 relative, 5x tighter than the north_star's 1e-5.
    name, pts = list(_invsq_cases())[case]
    n = len(pts)
    for sched in ("balanced", "standard"):
        c_want, s_want, _ = c_oracle.rows(pts, 0, n, sched)
        (r,) = _lib.pairs_host(np.ascontiguousarray(pts), _lib.PC_COLLISION_INVSQ,
                               _lib.PC_BALANCED if sched == "balanced" else _lib.PC_STANDARD, [0, n])
        assert r.count == c_want, name
        assert r.sum == pytest.approx(s_want, rel=2e-6), name
    r = se.spi_parallel(pts, se.inverse_square, 3, "balanced")
    for b, got in zip(se._partition(n, 3), r.partials):
        assert got == pytest.approx(c_oracle.rows(pts, b.start, b.stop, "balanced")[1], rel=2e-6), name


def test_filter_bypass_for_huge_spans():
    # spans beyond ~1e15 make the fp32 Gram filter meaningless: every pair takes the exact path
    rng = np.random.default_rng(3)
    pts = rng.random((300, 3)) * 4.0
    pts[::7] += 1e20
    pts[1::7] = pts[::7][: len(pts[1::7])] + 0.3  # near pairs far out
    want, _, _ = c_oracle.rows(pts, 0, len(pts), "balanced")
    assert se.spi_balanced(pts, se.collision_indicator).total == want
    assert se.spi_standard(pts, se.collision_indicator).total == want
    ints = np.array([[2**62, 0, 0], [2**62, 0, 0], [-2**62, 1, 0], [-2**62, 0, 0], [5, 5, 5]], dtype=np.int64)
    assert pc.oracle_collisions(ints) == c_oracle.int_pairs(ints)[0] == 1
    assert pc.oracle_contacts(ints) == c_oracle.int_pairs(ints)[1]
    # |c| >= 1e18 overflows fp32 squares: the float64 kernel evaluates the reference's terms
    huge = np.array([[0.0, 0, 0], [1e19, 0, 0], [1e19 + 2**12, 0.5, 0], [-3e25, 1, 2]])
    _, s_want, _ = c_oracle.rows(huge, 0, len(huge), "balanced")
    assert se.spi_balanced(huge, se.inverse_square).total == pytest.approx(s_want, rel=1e-12)
    assert se.spi_balanced(huge.astype(np.float32), se.inverse_square).total == pytest.approx(
        c_oracle.rows(huge.astype(np.float32), 0, len(huge), "balanced")[1], rel=1e-12)


def test_row_range_api_edges():
    objs = gen.random_spheres(5000, 12.0, 8).astype(np.float32)
    for rows in ((0, 0), (4999, 5000), (2500, 2500), (0, 1), (17, 4000)):
        for sched in se.SCHEDULES:
            got, pairs = se.spi_rows(objs, se.collision_indicator, rows, sched)
            c, _, p = c_oracle.rows(objs, rows[0], rows[1], sched)
            assert (got, pairs) == (c, p)
    with pytest.raises(ValueError):
        se.spi_rows(objs, se.collision_indicator, (10, 5), "balanced")


@pytest.mark.parametrize("trial", range(12))
def test_boundary_stress_random_offsets(trial):
    """Pairs planted at |d|^2 = 1 +- O(1e-7) inside clouds of random offset and
    span (the Gram filter's error grows with the span; its band must too)."""
    rng = np.random.default_rng(100 + trial)
    offset = rng.choice([0.0, 1.0, 37.5, 1e3, 2.5e4, 1e6]) * rng.choice([-1, 1])
    span = rng.choice([2.0, 50.0, 400.0, 3000.0])
    n_bg, n_pair = int(rng.integers(500, 6000)), 400
    bg = offset + rng.random((n_bg, 3)) * span
    a = offset + rng.random((n_pair, 3)) * span
    d = rng.normal(size=(n_pair, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    b = a + d * (1.0 + rng.normal(scale=2e-7, size=(n_pair, 1)))
    pts = np.concatenate([bg, a, b])
    rng.shuffle(pts)
    for arr in (pts, pts.astype(np.float32)):
        want_c, want_s, _ = c_oracle.rows(arr, 0, len(arr), "balanced")
        assert se.spi_balanced(arr, se.collision_indicator).total == want_c
        (r,) = _lib.pairs_host(np.ascontiguousarray(arr), _lib.PC_COLLISION_INVSQ, _lib.PC_STANDARD, [0, len(arr)])
        assert r.count == want_c and _close(r.sum, want_s)


def test_large_host_int64_beads_narrowed_exactly():
    # large int64 host vectors go to the device narrowed to int32 through pinned
    # chunks on host threads (lat_prepare): counts exact in the dense and sparse
    # regimes and for Alg. 2, and a bead beyond int32 or just outside the cube is
    # still reported by its index, whichever chunk it lands in
    rng = np.random.default_rng(8)
    beads = rng.integers(-40, 41, size=(3_000_000, 3))
    sp = pc.new_space(40)
    rep = pc.count_collisions(beads, sp)
    keys = np.ravel_multi_index(tuple((beads + 41).T), (83, 83, 83))
    occ = np.bincount(keys, minlength=83**3)
    assert rep.count == int((occ * (occ - 1) // 2).sum()) and rep.cells_touched == np.count_nonzero(occ)
    pc.reset_sparse(sp)
    assert pc.count_contacts(beads, sp).count == _contacts_by_grid(occ.reshape(83, 83, 83), beads + 41)
    pc.reset_sparse(sp)
    for idx, bad in ((250_001, 2**32 + 5), (2_999_999, -(2**40)), (1_400_000, 41), (0, -41)):
        b2 = beads.copy()
        b2[idx, 1] = bad
        with pytest.raises(lc.CoordinateRangeError, match=f"bead {idx} "):
            pc.count_collisions(b2, sp)
        assert sp.is_zero()
    sparse = rng.integers(-500, 501, size=(600_000, 3))
    sparse[::7] = sparse[0]
    sp2 = pc.new_space(500)
    keys = np.ravel_multi_index(tuple((sparse + 501).T), (1003,) * 3)
    _, cnt = np.unique(keys, return_counts=True)
    rep = pc.count_collisions(sparse, sp2)
    assert (rep.count, rep.cells_touched) == (int((cnt * (cnt - 1) // 2).sum()), len(cnt))
    pc.reset_sparse(sp2)
    assert sp2.is_zero()


def _contacts_by_grid(occ, shifted):
    # sum over beads of the six face-neighbour occupancies (Alg. 2), halved
    pad = np.pad(occ, 1)
    x, y, z = (shifted + 1).T
    tot = 0
    for dx, dy, dz in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
        tot += int(pad[x + dx, y + dy, z + dz].sum())
    assert tot % 2 == 0
    return tot // 2


@pytest.mark.parametrize("devs", [[0], [0, 0], [0, 0, 0, 0, 0]])
def test_counting_array_multi_gpu_slabs(devs):
    # pc_lattice_collisions_multi: x-slab split over a device list (ordinal 0 repeated on
    # the one-GPU box) == the single-grid counting array, dense and sparse regimes
    rng = np.random.default_rng(len(devs))
    for a, n in ((30, 2_000_000), (30, 5_000), (200, 300_000)):
        beads = rng.integers(-a, a + 1, size=(n, 3))
        beads[: n // 10] = beads[0]  # one heavy cell
        side = 2 * a + 3
        keys = np.ravel_multi_index(tuple((beads + a + 1).T), (side,) * 3)
        occ = np.bincount(keys)
        rep = lc.count_collisions_multi_gpu(beads, a, devs)
        assert (rep.count, rep.cells_touched, rep.beads_processed) == \
            (int((occ * (occ - 1) // 2).sum()), int(np.count_nonzero(occ)), n)
    bad = rng.integers(-5, 6, size=(1000, 3))
    bad[777, 2] = 6
    with pytest.raises(lc.CoordinateRangeError, match="bead 777"):
        lc.count_collisions_multi_gpu(bad, 5, devs)
    assert lc.count_collisions_multi_gpu(np.zeros((0, 3), dtype=np.int64), 5, devs).count == 0


def test_abi_argument_errors():
    # every C entry rejects malformed arguments with PC_ERR_ARG (ValueError) and a message
    import ctypes

    lib = _lib.load()
    pts = gen.random_spheres(1000, 10.0, 1).astype(np.float32)
    n = len(pts)
    with pytest.raises(ValueError, match="row range"):
        _lib.pairs_host(pts, _lib.PC_COLLISION, _lib.PC_BALANCED, [0, n + 1])
    with pytest.raises(ValueError, match="row range"):
        _lib.pairs_host(pts, _lib.PC_COLLISION, _lib.PC_BALANCED, [5, 3])
    with pytest.raises(ValueError, match="integer interactions"):
        _lib.pairs_host(pts, _lib.PC_COINCIDE, _lib.PC_BALANCED, [0, n])
    with pytest.raises(ValueError, match="schedule"):
        _lib.pairs_host(pts, _lib.PC_COLLISION, 7, [0, n])
    res = (_lib.PairsResult * 1)()
    b = np.array([0, n], dtype=np.int64)
    ws = _lib.DeviceBuffer(1024)
    d = _lib.DeviceBuffer(pts.nbytes)
    _lib.check(lib.pc_memcpy_h2d(d.ptr, pts.ctypes.data, pts.nbytes, None))
    rc = lib.pc_pairs(d.ptr, _lib.PC_F32, n, _lib.PC_COLLISION, _lib.PC_BALANCED, 0, 1, b.ctypes.data, ws.ptr, 1024,
                      ctypes.addressof(res), None)
    assert rc == _lib.PC_ERR_ARG and b"workspace" in lib.pc_last_error()
    with pytest.raises(ValueError, match="device"):
        _lib.pairs_multi(pts, _lib.PC_COLLISION, _lib.PC_BALANCED, [0, 1000], [0, 500, n])
    with pytest.raises(ValueError, match="cover"):
        _lib.pairs_multi(pts, _lib.PC_COLLISION, _lib.PC_BALANCED, [0, 0], [0, 500, n - 1])
    with pytest.raises(ValueError):
        lc.count_collisions_multi_gpu(np.zeros((4, 3), dtype=np.int64), 5, [1000])
    with pytest.raises(ValueError, match="integer"):
        _lib.pairs_batch([pts], _lib.PC_MANHATTAN1)


def test_spi_totals_batch():
    # many small SPI problems in one launch == spi_balanced per problem (C oracle)
    rng = np.random.default_rng(12)
    objs = [rng.random((k, 3)) * (k ** (1 / 3)) * 1.3 for k in (0, 1, 2, 7, 64, 500, 4096, 5000)]
    objs.append(objs[4].astype(np.float32))
    objs.append(rng.integers(0, 6, size=(300, 3)))
    counts = se.spi_totals_batch(objs, se.collision_indicator)
    sums = se.spi_totals_batch(objs, se.inverse_square)
    for o, c, s in zip(objs, counts, sums):
        if len(o) < 2:
            assert c == 0 and s == 0
            continue
        want_c, want_s, _ = c_oracle.rows(o, 0, len(o), "balanced")
        assert c == want_c and isinstance(c, int)
        assert s == pytest.approx(want_s, rel=1e-12 if len(o) <= 4096 else REL_TOL)
    with pytest.raises(TypeError):
        se.spi_totals_batch(objs[3:5], lambda a, b: 1)


def test_lattice_64bit_keys():
    # a = 820: (2a+3)^3 = 4.4e9 cells > 2^32, so keys are 64-bit (17.7 GB grid); beads near the
    # far corner have keys above 2^32
    a = 820
    assert _lib.load().pc_lattice_key_bytes(a) == 8
    rng = np.random.default_rng(9)
    beads = np.concatenate([rng.integers(a - 3, a + 1, size=(3000, 3)), rng.integers(-a, -a + 4, size=(3000, 3)),
                            rng.integers(-a, a + 1, size=(3000, 3))])
    side = 2 * a + 3
    keys = np.ravel_multi_index(tuple((beads + a + 1).T), (side,) * 3)
    assert keys.max() > 2**32
    _, inv, occ = np.unique(keys, return_inverse=True, return_counts=True)
    sp = pc.new_space(a)
    rep = pc.count_collisions(beads, sp)
    assert (rep.count, rep.cells_touched) == (int((occ * (occ - 1) // 2).sum()), len(occ))
    pc.reset_sparse(sp)
    rep = pc.count_contacts(beads, sp)
    assert rep.count == c_oracle.int_pairs(beads)[1]
    pc.reset_sparse(sp)
    assert sp.is_zero()
    del sp


def test_non_contiguous_inputs():
    # strided views, Fortran order and Sphere lists give the same results as contiguous copies
    pts = gen.random_spheres(6001, 14.0, 5)
    views = [pts[::2], np.asfortranarray(pts), pts.T.copy().T, [se.Sphere(*p) for p in pts[:500]]]
    for v in views:
        ref = np.ascontiguousarray(np.asarray(v if not isinstance(v, list) else [(s.x, s.y, s.z) for s in v], dtype=np.float64))
        want = c_oracle.rows(ref, 0, len(ref), "balanced")
        assert se.spi_balanced(v, se.collision_indicator).total == want[0]
        assert se.spi_balanced(v, se.inverse_square).total == pytest.approx(want[1], rel=REL_TOL)
    beads = gen.random_chain(5000, 4)[0]
    sp = pc.new_space(int(np.abs(beads).max()))
    for v in (beads[::3], np.asfortranarray(beads)):
        rep = pc.count_collisions(v, sp)
        pc.reset_sparse(sp)
        assert rep.count == c_oracle.int_pairs(np.ascontiguousarray(v))[0]


def test_concurrent_callers():
    # the library is thread-safe (per-device arena lock, thread-local errors): the
    # reference's spi_parallel runs its workers on threads, and so may users
    from concurrent.futures import ThreadPoolExecutor

    inputs = [gen.random_spheres(3000 + 17 * k, 12.0, 40 + k) for k in range(8)]
    chains = [gen.random_chain(2000, 60 + k)[0] for k in range(8)]
    want = [c_oracle.rows(p, 0, len(p), "balanced")[0] for p in inputs]
    want_l = [c_oracle.int_pairs(c)[0] for c in chains]

    def job(k):
        sp = pc.new_space(int(np.abs(chains[k]).max()))
        out = []
        for _ in range(5):
            out.append(se.spi_balanced(inputs[k], se.collision_indicator).total)
            out.append(pc.count_collisions(chains[k], sp).count)
            pc.reset_sparse(sp)
        return out

    with ThreadPoolExecutor(max_workers=8) as pool:
        results = list(pool.map(job, range(8)))
    for k, out in enumerate(results):
        assert out[0::2] == [want[k]] * 5 and out[1::2] == [want_l[k]] * 5


def test_concurrent_large_host_bead_vectors():
    # several threads staging large int64 bead vectors at once (pinned chunk pool
    # under the per-device arena lock): every count exact, every space clean after
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(21)
    vecs = [rng.integers(-60, 61, size=(700_000 + 1000 * k, 3)) for k in range(4)]
    want = []
    for v in vecs:
        _, cnt = np.unique(np.ravel_multi_index(tuple((v + 61).T), (123,) * 3), return_counts=True)
        want.append((int((cnt * (cnt - 1) // 2).sum()), len(cnt)))

    def job(k):
        sp = pc.new_space(60)
        out = []
        for _ in range(3):
            rep = pc.count_collisions(vecs[k], sp)
            out.append((rep.count, rep.cells_touched))
            pc.reset_sparse(sp)
        return out, sp.is_zero()

    with ThreadPoolExecutor(max_workers=4) as pool:
        results = list(pool.map(job, range(4)))
    for k, (out, clean) in enumerate(results):
        assert out == [want[k]] * 3 and clean
