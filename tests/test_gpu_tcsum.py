"""The tensor-core Gram chunks of the sorted fp32 sum (csrc/pairs_tcsum.cuh, kernel 10).

A whole-range fp32 inverse-square sum runs the sorted FFMA kernel, which leaves the
dense chunks tcs_takes() accepts alone, then pairs_tcs_kernel over exactly those
chunks (tcgen05.mma kind::f16 on three-way bf16 splits).  Checked here:
  * against the C oracle on distributions that stress the chunk test (counts exact,
    sums within 1e-6 -- north_star allows 1e-5);
  * against the FFMA-only path (PAIRCOUNT_TCSUM=0, a fresh process) on the same inputs;
  * every (tile, chunk) evaluated exactly once, by one of the two kernels;
  * tile parts adding up to the whole, and bit-reproducible sums.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import c_oracle
from paper_1901_11204_b200 import _lib
from paper_1901_11204_b200 import generators as gen

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
TCS = os.environ.get("PAIRCOUNT_TCSUM", "1") != "0"


def _inputs(n, seed):
    rng = np.random.default_rng(seed)
    box = (4.18879 * n) ** (1 / 3) / 1.26
    k = 32
    cent = rng.random((k, 3)) * box * 4
    return {
        "uniform": gen.random_spheres(n, box, seed),
        "sparse uniform": gen.random_spheres(n, box * 6, seed + 1),
        "clustered": cent[rng.integers(0, k, n)] + rng.normal(size=(n, 3)) * 2.0,
        "normal cloud": rng.normal(size=(n, 3)) * box / 3,
        "offset 1e5": rng.random((n, 3)) * box + 1e5,
        "wide span 1e5": rng.random((n, 3)) * 1e5,
    }


def _chunks(prof):
    return (prof.chunks_gram + prof.chunks_main + prof.chunks_near + prof.chunks_far + prof.chunks_edge +
            prof.chunks_tc)


@pytest.mark.parametrize("n", [32768, 40001, 65536])
def test_tcsum_matches_oracle(n):
    for name, pts in _inputs(n, n + 7).items():
        pts = np.ascontiguousarray(pts, dtype=np.float32)
        want_c, want_s, pairs = c_oracle.rows(pts, 0, n, "balanced")
        (r,) = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
        prof = _lib.last_profile()
        assert (r.count, r.pairs, r.error) == (want_c, pairs, 0), name
        assert abs(r.sum - want_s) <= 1e-6 * want_s, (name, r.sum, want_s)
        if TCS:
            assert prof.kernel == 10, name
        # one owner per chunk
        tiles = -(-n // 256)
        assert _chunks(prof) == tiles * -(-(255 + n // 2) // 256), name


@pytest.mark.parametrize("n", [32768, 65537])
def test_tcsum_float64_points_match_oracle(n):
    # float64 points (what the reference's generators return): the compensated sorted kernel beside
    # the tensor-core kernel, which forms a = fl32((q - c) - o) in float64 (kernel 11)
    for name, pts in _inputs(n, n + 11).items():
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        want_c, want_s, pairs = c_oracle.rows(pts, 0, n, "balanced")
        (r,) = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
        prof = _lib.last_profile()
        assert (r.count, r.pairs, r.error) == (want_c, pairs, 0), name
        assert abs(r.sum - want_s) <= 1e-6 * want_s, (name, r.sum, want_s)
        if TCS:
            assert prof.kernel == 11, (name, prof.kernel)
        if not prof.f64_taken:  # (a span beyond the compensated staging goes to the float64 kernel)
            tiles = -(-n // 256)
            assert _chunks(prof) == tiles * -(-(255 + n // 2) // 256), name


def test_tcsum_takes_most_chunks_of_the_headline_shape():
    if not TCS:
        pytest.skip("PAIRCOUNT_TCSUM=0")
    n = 2**18
    x = gen.random_spheres(n, gen.contact_box_edge(n), 3).astype(np.float32)
    (r,) = _lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    prof = _lib.last_profile()
    assert prof.kernel == 10 and prof.chunks_tc > 0.4 * _chunks(prof)  # 80 % at the 2^20 headline
    # the wide-span guard: |a| + |b| beyond 3e4 never reaches the tensor cores
    y = (np.random.default_rng(1).random((n, 3)) * 1e6).astype(np.float32)
    (r2,) = _lib.pairs_host(y, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    assert _lib.last_profile().chunks_tc == 0 and r2.error == 0


_FFMA_ONLY = """
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_1901_11204_b200 import _lib
out = []
for path in sys.argv[1:]:
    x = np.load(path)
    (r,) = _lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, len(x)])
    out.append([r.count, r.sum, _lib.last_profile().kernel, _lib.last_profile().chunks_tc])
print(json.dumps(out))
"""


def test_tcsum_agrees_with_the_ffma_only_path(tmp_path):
    if not TCS:
        pytest.skip("PAIRCOUNT_TCSUM=0")
    n = 2**17 + 3
    files, got = [], []
    for name, pts in _inputs(n, 5).items():
        pts = np.ascontiguousarray(pts, dtype=np.float32)
        f = tmp_path / f"{len(files)}.npy"
        np.save(f, pts)
        files.append(str(f))
        (r,) = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
        got.append((name, r.count, r.sum))
    env = dict(os.environ, PAIRCOUNT_TCSUM="0")
    res = subprocess.run([sys.executable, "-c", _FFMA_ONLY.format(root=str(ROOT)), *files], env=env,
                         capture_output=True, text=True, timeout=600, check=True)
    ref = json.loads(res.stdout.strip().splitlines()[-1])
    for (name, c, s), (c0, s0, kern0, tc0) in zip(got, ref):
        assert kern0 == 3 and tc0 == 0, name
        assert c == c0, name
        assert abs(s - s0) <= 1e-6 * s0, (name, s, s0)


def test_tcsum_in_loop_classification_matches_the_bitmap(tmp_path):
    # beyond the bitmap's size cap (n > ~2^23) both kernels classify every chunk in-loop;
    # PAIRCOUNT_TCS_BITMAP=0 forces that path here: the same chunks, the same total, bit for bit
    if not TCS:
        pytest.skip("PAIRCOUNT_TCSUM=0")
    files, got = [], []
    # n = 2^17 + 5: the general chunk boxes; n = 2^17: the precomputed per-256 ones (tcs_chunk_box_kernel)
    for n, name, pts in [(m, nm, p) for m in (2**17 + 5, 2**17) for nm, p in list(_inputs(m, 21).items())[:4]]:
        for dt in (np.float32, np.float64):
            x = np.ascontiguousarray(pts, dtype=dt)
            f = tmp_path / f"{len(files)}.npy"
            np.save(f, x)
            files.append(str(f))
            (r,) = _lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
            got.append((name, r.count, r.sum, _lib.last_profile().chunks_tc))
    env = dict(os.environ, PAIRCOUNT_TCS_BITMAP="0")
    res = subprocess.run([sys.executable, "-c", _FFMA_ONLY.format(root=str(ROOT)), *files], env=env,
                         capture_output=True, text=True, timeout=600, check=True)
    ref = json.loads(res.stdout.strip().splitlines()[-1])
    for (name, c, s_, tc), (c0, s0, kern0, tc0) in zip(got, ref):
        assert (c, s_, tc) == (c0, s0, tc0), (name, c, s_, tc, c0, s0, tc0)


def test_tcsum_unaligned_ranges_stay_on_the_ffma_kernel():
    # a range starting off a 32-point block boundary: its tiles' boxes differ from the per-32 boxes,
    # so the whole range stays on the FFMA kernel; aligned ranges split as usual
    n = 50_000
    pts = gen.random_spheres(n, 30.0, 5).astype(np.float32)
    want_c, want_s, _ = c_oracle.rows(pts, 0, n, "balanced")
    res = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, 7, 12_512, 33_333, n],
                          tiling=_lib.PC_TILE_SORTED)
    assert sum(r.count for r in res) == want_c
    assert abs(sum(r.sum for r in res) - want_s) <= 1e-6 * want_s


def test_tcsum_tile_parts_and_reproducibility():
    n = 2**17
    x = gen.random_spheres(n, gen.contact_box_edge(n), 9).astype(np.float32)
    (r,) = _lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    (r2,) = _lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    assert r.sum == r2.sum and r.count == r2.count  # fixed association: bitwise equal
    for nparts in (2, 3, 8):
        parts = [_lib.pairs_part_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, 0, n, p, nparts,
                                      tiling=_lib.PC_TILE_SORTED) for p in range(nparts)]
        assert sum(q.count for q in parts) == r.count and sum(q.pairs for q in parts) == r.pairs
        assert abs(sum(q.sum for q in parts) - r.sum) <= 1e-9 * r.sum, nparts


@pytest.mark.parametrize("lo", [12_512, 4_096 + 32])
def test_tcsum_origin_groups_on_offset_ranges_and_parts(lo):
    # a range starting on a 32-point block but not on a 256-point tile: the origin groups are counted
    # from lo; tile parts deal blocks of three tiles (the last block ragged).  PC_TILE_SORTED ranges
    # index the sorted order (include/paircount.h), so [0, lo) + [lo, n) make the oracle's total
    n = 70_001
    x = gen.random_spheres(n, gen.contact_box_edge(n), 17).astype(np.float32)
    want_c, want_s, pairs = c_oracle.rows(x, 0, n, "balanced")
    r0, r = _lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, lo, n], tiling=_lib.PC_TILE_SORTED)
    assert (r0.count + r.count, r0.pairs + r.pairs) == (want_c, pairs)
    assert abs(r0.sum + r.sum - want_s) <= 1e-6 * want_s
    (r1,) = _lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [lo, n], tiling=_lib.PC_TILE_SORTED)
    prof = _lib.last_profile()
    assert (r1.count, r1.pairs) == (r.count, r.pairs) and abs(r1.sum - r.sum) <= 1e-9 * r.sum
    if TCS:
        assert prof.kernel == 10 and prof.chunks_tc > 0
    for nparts in (2, 3, 7):
        parts = [_lib.pairs_part_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, lo, n, p, nparts,
                                      tiling=_lib.PC_TILE_SORTED) for p in range(nparts)]
        assert sum(q.count for q in parts) == r.count and sum(q.pairs for q in parts) == r.pairs, nparts
        assert abs(sum(q.sum for q in parts) - r.sum) <= 1e-9 * r.sum, nparts
