"""Round-2 GPU behaviour: tile parts, path profile, fixed-association sums,
non-finite inputs on every sum kernel, the multi-GPU lattice key width, the
NCCL exchange at world size 1, device-count defaults."""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1901_11204_b200 as pc
from oracle import c_oracle
from paper_1901_11204_b200 import _lib
from paper_1901_11204_b200 import distributed as D
from paper_1901_11204_b200 import generators as gen
from paper_1901_11204_b200 import lattice_counter as lc
from paper_1901_11204_b200 import spi_engine as se

pytestmark = pytest.mark.gpu


def _spheres(n, seed, dtype=np.float32, scale=1.0):
    return (gen.random_spheres(n, gen.contact_box_edge(n) * scale, seed)).astype(dtype)


@pytest.mark.parametrize("n", [2, 3, 257, 5000, 16385, 40001, 70000])
def test_tile_parts_add_up(n):
    """pc_pairs_part_*: the row tiles of [lo, hi) dealt over nparts calls add up
    to the [lo, hi) result on every kernel (sorted / input-order / compensated
    sums, FFMA2 count), both schedules, ranges and whole."""
    x = _spheres(n, 11, scale=0.7)
    for sched in ("balanced", "standard"):
        for lo, hi in ((0, n), (n // 3, n - n // 5)):
            c, s, p = c_oracle.rows(x, lo, hi, sched)
            cases = [(_lib.PC_COLLISION, _lib.PC_TILE_AUTO, x), (_lib.PC_COLLISION_INVSQ, _lib.PC_TILE_AUTO, x),
                     (_lib.PC_COLLISION_INVSQ, _lib.PC_TILE_AUTO, x.astype(np.float64))]
            if sched == "balanced" and n >= 2:
                cases.append((_lib.PC_COLLISION_INVSQ, _lib.PC_TILE_FLAT, x))
            for inter, tiling, arr in cases:
                for nparts in (1, 2, 3, 8):
                    parts = [_lib.pairs_part_host(arr, inter, _lib.SCHEDULE_CODES[sched], lo, hi, k, nparts, tiling)
                             for k in range(nparts)]
                    assert all(q.error == 0 for q in parts)
                    assert sum(q.count for q in parts) == c, (sched, lo, hi, inter, tiling, nparts)
                    assert sum(q.pairs for q in parts) == p
                    if inter == _lib.PC_COLLISION_INVSQ and p:
                        assert abs(sum(q.sum for q in parts) - s) <= 1e-6 * s
    with pytest.raises(ValueError, match="part"):
        _lib.pairs_part_host(x, _lib.PC_COLLISION, _lib.PC_BALANCED, 0, n, 2, 2)
    with pytest.raises(ValueError):
        _lib.pairs_part_host(x, _lib.PC_COLLISION, _lib.PC_BALANCED, 0, n, 0, 2, _lib.PC_TILE_TC)


def test_sorted_tile_parts_on_clustered_points():
    n = 65537
    x = (gen.clustered_spheres(n, centres=64, box_edge=40.0)).astype(np.float32)
    c, s, p = c_oracle.rows(x, 0, n, "balanced")
    for nparts in (2, 5, 8):
        parts = [_lib.pairs_part_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, 0, n, k, nparts,
                                      _lib.PC_TILE_SORTED) for k in range(nparts)]
        assert sum(q.count for q in parts) == c and sum(q.pairs for q in parts) == p
        assert abs(sum(q.sum for q in parts) - s) <= 1e-6 * s
        # round-robin tiles: every part holds about 1/nparts of the pairs
        assert max(q.pairs for q in parts) <= 1.2 * p / nparts


def test_profile_accounts_for_every_pair():
    """pc_pairs_profile: the chunks of each inner loop cover the call's pairs;
    the kernel ids follow the dispatch; claims only on FLAT tilings."""
    tcs = os.environ.get("PAIRCOUNT_TCSUM", "1") != "0"
    for n, tiling, inter, kern in ((70000, _lib.PC_TILE_AUTO, _lib.PC_COLLISION_INVSQ, 10 if tcs else 3),
                                   (70000, _lib.PC_TILE_FLAT, _lib.PC_COLLISION_INVSQ, 2),
                                   (70000, _lib.PC_TILE_FLAT, _lib.PC_COLLISION, 1),
                                   (70000, _lib.PC_TILE_TC, _lib.PC_COLLISION, 5),
                                   (70000, _lib.PC_TILE_AUTO, _lib.PC_COLLISION, 8),
                                   (9000, _lib.PC_TILE_PER_ROW_TILE, _lib.PC_COLLISION, 1)):
        x = _spheres(n, 3)
        (r,) = _lib.pairs_host(x, inter, _lib.PC_BALANCED, [0, n], tiling=tiling)
        prof = _lib.last_profile()
        assert prof.kernel == kern and prof.pairs == r.pairs
        assert prof.exact_checks == r.exact_checks
        if kern == 5:
            continue
        chunks = (prof.chunks_gram + prof.chunks_main + prof.chunks_near + prof.chunks_far + prof.chunks_edge +
                   prof.chunks_tc)
        assert chunks * prof.pairs_per_chunk >= r.pairs  # edge chunks are partly masked
        assert (prof.claims > 0) == (tiling != _lib.PC_TILE_PER_ROW_TILE)
        if kern in (3, 10):
            assert prof.chunks_gram + prof.chunks_tc > 0 and prof.chunks_near > 0
            # every (tile, chunk) of the window space evaluated once, by one of the two kernels
            T = W = 256
            tiles = -(-n // T)
            assert chunks == tiles * -(-(T - 1 + n // 2) // W)
        if kern == 10:
            assert prof.chunks_tc > 0
        if kern == 8:  # pruned sorted count: most chunks decided by their boxes
            assert prof.chunks_far > 0.5 * chunks


@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.int64])
def test_sums_are_bit_reproducible(dtype):
    n = 50_000
    x = _spheres(n, 5).astype(dtype) if dtype != np.int64 else gen.normal_cloud(n, 40.0, 200, 1)
    for tiling in (_lib.PC_TILE_AUTO, _lib.PC_TILE_FLAT, _lib.PC_TILE_PER_ROW_TILE):
        sums = {_lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, 7, n - 3, n], tiling)[1].sum
                for _ in range(4)}
        assert len(sums) == 1, (dtype, tiling, sums)


@pytest.mark.parametrize("n,dtype", [(300, np.float32), (5000, np.float32), (5000, np.float64),
                                     (20000, np.float64), (40000, np.float32)])
def test_isolated_infinity_adds_zero_terms(n, dtype):
    """Reference semantics on every sum kernel (small, compensated, sorted):
    1/(1+inf) = 0 is a finite term and is added (spi_engine.py:84-99)."""
    x = _spheres(n, 9, dtype)
    x[n // 3, 0] = np.inf
    x[n // 2, 2] = -np.inf
    for sched in ("balanced", "standard"):
        w = 3
        r = se.spi_parallel(x, se.inverse_square, w, sched)
        for b, got in zip(se._partition(n, w), r.partials):
            want = c_oracle.rows(x, b.start, b.stop, sched)[1]
            assert got == pytest.approx(want, rel=1e-12)
        with pytest.raises(se.InteractionDomainError):
            se.spi_parallel(x, se.collision_indicator, w, sched)


def test_nan_term_names_reference_pair_per_worker():
    n = 3000
    x = _spheres(n, 2, np.float64)
    x[2500, 1] = np.nan
    # balanced, 3 workers: rows [0,1000) own (i, 2500) for i >= 1000 only -> worker 1 row 1000 first
    with pytest.raises(se.AccumulationError, match=r"\(1000, 2500\)"):
        se.spi_parallel(x, se.inverse_square, 3, "balanced")
    with pytest.raises(se.AccumulationError, match=r"\(0, 2500\)"):
        se.spi_standard(x, se.inverse_square)
    # rows that never meet the NaN point are fine, as in the reference
    got, _ = se.spi_rows(x, se.inverse_square, (0, 100), "balanced")
    assert got == pytest.approx(c_oracle.rows(x, 0, 100, "balanced")[1], rel=1e-12)
    got, _ = se.spi_rows(x, se.collision_indicator, (0, 100), "balanced")
    assert got == c_oracle.rows(x, 0, 100, "balanced")[0]


def test_multi_gpu_lattice_keys_beyond_32_bits():
    """a slab grid of >= 2^32 cells needs 8-byte keys.  a = 1100
    on two slabs: slab 0 has 1102 x 2203^2 > 2^32 cells; beads whose slab keys
    differ by exactly 2^32 must not alias."""
    a = 1100
    side = 2 * a + 3
    dx, rem = divmod(2**32, side * side)
    dy, dz = divmod(rem, side)
    beads = np.array([[-a, -a, -a], [-a + dx, -a + dy, -a + dz], [5, 5, 5], [5, 5, 5]], dtype=np.int64)
    for devs in ([0, 0], [0, 0, 0]):
        rep = lc.count_collisions_multi_gpu(beads, a, devs)
        assert (rep.count, rep.cells_touched) == (1, 3), devs


def test_dense_regime_between_2_31_and_2_32_cells():
    """a = 700 has 1403^3 = 2.76e9 cells (2^31 < cells < 2^32);
    dense inputs there must not take the 2^31-cell slab path."""
    a = 700
    cells = (2 * a + 3) ** 3
    k = 357
    ax = np.arange(-a, -a + k, dtype=np.int32)
    g = np.stack(np.meshgrid(ax, ax, ax[:340], indexing="ij"), -1).reshape(-1, 3)  # 43.3M distinct beads
    beads = np.concatenate([g, g[:1000]])
    assert len(beads) * 64 > cells
    space = lc.new_space(a)
    rep = lc.count_collisions(beads, space)
    assert (rep.count, rep.cells_touched) == (1000, len(g))
    lc.reset_sparse(space)
    assert space.is_zero()
    del space


def test_device_count_defaults():
    assert _lib.device_count() >= 1
    x = _spheres(2000, 4)
    want = c_oracle.rows(x, 0, len(x), "balanced")[0]
    assert D.spi_multi_gpu(x, se.collision_indicator)[0] == want
    beads, ext = gen.random_chain(3000, 3)
    assert lc.count_collisions_multi_gpu(beads, ext).count == c_oracle.int_pairs(beads)[0]


def test_nccl_exchange_world_size_1():
    """The NCCL path end to end on one GPU: process group over NCCL, the int64
    slot all-reduce on the device, both splits."""
    import torch
    import torch.distributed as dist

    store = dist.HashStore()
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = _spheres(40_000, 6)
        c, s, p = c_oracle.rows(x, 0, len(x), "balanced")
        for split in ("slabs", "tiles"):
            total, parts, pairs = D.spi_distributed(x, se.inverse_square, split=split, device="cuda")
            assert abs(total - s) <= 1e-6 * s and pairs == (p,)
            total, parts, pairs = D.spi_distributed(x, se.collision_indicator, split=split, device="cuda")
            assert total == c and parts == (c,)
        counts, sums, flags, prs = D.allreduce_partials(7, 0.5, device="cuda", is_float=True, pairs=3)
        assert (counts, sums, flags, prs) == ([7], [0.5], [1], [3])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [2, 3, 191, 192, 193, 5000, 40001, 70000])
def test_int32_key_coincidence_counts(n):
    """PC_TILE_KEY (packed 30-bit keys, INT32 compares) against the oracle, whole
    range and row ranges, and through oracle_collisions (which routes there)."""
    rng = np.random.default_rng(n)
    pts = rng.integers(-6, 7, size=(n, 3)).astype(np.int64) * rng.integers(1, 3) + 300
    want = c_oracle.int_pairs(pts)[0]
    assert pc.oracle_collisions(pts) == want
    assert _lib.last_profile().kernel == 6
    for b in ([0, n], [0, n // 3, n // 2, n]):
        rs = _lib.pairs_host(pts.astype(np.int32), _lib.PC_COINCIDE, _lib.PC_BALANCED, b, tiling=_lib.PC_TILE_KEY)
        for (lo, hi), r in zip(zip(b[:-1], b[1:]), rs):
            assert r.error == 0 and r.count == c_oracle.int_rows(pts, lo, hi, "balanced")[0], (lo, hi)
        assert sum(r.count for r in rs) == want


def test_int32_key_span_limits():
    base = np.zeros((5000, 3), dtype=np.int64)
    base[:, 0] = np.arange(5000) % 1024          # span 1023: keys fit
    base[::7] = base[1::7][: len(base[::7])]      # plant coincidences
    want = c_oracle.int_pairs(base)[0]
    (r,) = _lib.pairs_host(base, _lib.PC_COINCIDE, _lib.PC_BALANCED, [0, 5000], tiling=_lib.PC_TILE_KEY)
    assert r.error == 0 and r.count == want
    wide = base.copy()
    wide[0, 2] = 1024                             # span 1024: the key path refuses, AUTO still exact
    (r,) = _lib.pairs_host(wide, _lib.PC_COINCIDE, _lib.PC_BALANCED, [0, 5000], tiling=_lib.PC_TILE_KEY)
    assert r.error == _lib.PC_ERR_ARG
    assert pc.oracle_collisions(wide) == c_oracle.int_pairs(wide)[0]
    assert _lib.last_profile().kernel != 6
    with pytest.raises(ValueError, match="PC_TILE_KEY"):
        _lib.pairs_host(base, _lib.PC_MANHATTAN1, _lib.PC_BALANCED, [0, 5000], tiling=_lib.PC_TILE_KEY)


@pytest.mark.parametrize("n", [2, 3, 1023, 1024, 1025, 5000, 20001])
def test_paper_thread_row_schemes(n):
    """PC_TILE_THREAD_ROW: the paper's thread-per-row kernels (standard = the
    straightforward scheme, balanced = Alg. 4) against the oracle, whole range
    and row ranges, counts exact and sums within 1e-6."""
    x = _spheres(n, 12, scale=0.8)
    for sched in ("standard", "balanced"):
        for b in ([0, n], [0, n // 3, n - n // 4, n]):
            for inter in (_lib.PC_COLLISION, _lib.PC_COLLISION_INVSQ):
                rs = _lib.pairs_host(x, inter, _lib.SCHEDULE_CODES[sched], b, tiling=_lib.PC_TILE_THREAD_ROW)
                for (lo, hi), r in zip(zip(b[:-1], b[1:]), rs):
                    c, s, p = c_oracle.rows(x, lo, hi, sched)
                    assert r.error == 0 and r.count == c and r.pairs == p, (sched, lo, hi, inter)
                    if inter == _lib.PC_COLLISION_INVSQ and p:
                        assert abs(r.sum - s) <= 1e-6 * s
    assert _lib.last_profile().kernel == 7
    with pytest.raises(ValueError, match="THREAD_ROW"):
        _lib.pairs_host(x.astype(np.float64), _lib.PC_COLLISION, _lib.PC_BALANCED, [0, n],
                        tiling=_lib.PC_TILE_THREAD_ROW)


@pytest.mark.parametrize("n,dtype", [(32768, np.float32), (40001, np.float32), (65537, np.float32),
                                     (40001, np.float64)])
def test_pruned_sorted_count(n, dtype):
    """Whole-range fp32 contact counts (spi_balanced / PC_TILE_AUTO) run on Morton-sorted
    points with box pruning: exact against the oracle on distributions that stress the
    box test (contacts at exactly distance 1 on a lattice, dense clusters, far-apart
    clusters, a thin slab); the profile reports the pruned chunks apart."""
    rng = np.random.default_rng(n)
    box = (4.18879 * n) ** (1 / 3)
    lat = rng.integers(0, int(box) + 1, size=(n, 3)).astype(np.float32)
    cent = rng.random((64, 3)) * box * 2
    cases = {
        "uniform": _spheres(n, 3),
        "lattice (d = 1 exactly)": lat,
        "clustered": (cent[rng.integers(0, 64, n)] + rng.normal(size=(n, 3))).astype(np.float32),
        "two far clusters": np.concatenate([rng.random((n // 2, 3)) * 12, rng.random((n - n // 2, 3)) * 12 + 1e4]
                                           ).astype(np.float32),
        "thin slab": (rng.random((n, 3)) * np.array([box * 6, box * 6, 0.8])).astype(np.float32),
    }
    if dtype == np.float64:  # float64 points: boxes rounded outward, Gram staging from float64
        cases = {k: v.astype(np.float64) + (1e-7 if k != "lattice (d = 1 exactly)" else 0.0)
                 for k, v in cases.items()}
        cases["offset 1e5"] = cases["uniform"] + 1e5
    for name, x in cases.items():
        want = c_oracle.rows(x, 0, n, "balanced")[0]
        assert se.spi_balanced(x, se.collision_indicator).total == want, name
        prof = _lib.last_profile()
        assert prof.kernel == 8 and prof.chunks_far > 0, name
        (r,) = _lib.pairs_host(x, _lib.PC_COLLISION, _lib.PC_BALANCED, [0, n], tiling=_lib.PC_TILE_SORTED)
        assert r.count == want, name
        parts = [_lib.pairs_part_host(x, _lib.PC_COLLISION, _lib.PC_BALANCED, 0, n, k, 3, _lib.PC_TILE_SORTED)
                 for k in range(3)]
        assert sum(q.count for q in parts) == want, name
