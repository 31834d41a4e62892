"""Randomised parity soak: many random (size, dtype, distribution, schedule, row
ranges, predicate) cases through the drop-in API against the pinned C oracle.

    python scripts/parity_soak.py --minutes 15 [--seed 0]

Prints one summary line per case family and a final tally; exits 1 on any
mismatch.  Counts must match bit-exactly, sums within 1e-5 relative (the
north_star tolerance).  Not part of pytest (it runs for minutes); its log is
kept under profiles/.
"""

from __future__ import annotations

import argparse
import math
import sys
import time
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1901_11204_b200 as pc  # noqa: E402
from oracle import c_oracle  # noqa: E402
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import lattice_counter as lc  # noqa: E402
from paper_1901_11204_b200 import spi_engine as se  # noqa: E402


def random_points(rng, n):
    kind = rng.integers(0, 6)
    dens = rng.uniform(0.05, 2.0)
    box = max(1.0, (n / dens) ** (1 / 3))
    if kind == 0:  # uniform
        p = rng.random((n, 3)) * box
    elif kind == 1:  # clustered
        k = max(1, n // int(rng.integers(5, 200)))
        cent = rng.random((k, 3)) * box
        p = cent[rng.integers(0, k, n)] + rng.normal(size=(n, 3)) * rng.uniform(0.3, 3.0)
    elif kind == 2:  # far from the origin
        p = rng.random((n, 3)) * box + rng.uniform(-1e5, 1e5, size=3)
    elif kind == 3:  # lattice-like: many exact distances 1
        p = rng.integers(0, max(2, int(box)), size=(n, 3)).astype(np.float64)
    elif kind == 4:  # thin slab
        p = rng.random((n, 3)) * np.array([box * 4, box * 4, 1.0])
    else:  # two far clusters
        p = rng.random((n, 3)) * box
        p[n // 2:] += rng.uniform(1e3, 1e6)
    dt = [np.float32, np.float64][int(rng.integers(0, 2))]
    return p.astype(dt), ["uniform", "clustered", "offset", "lattice", "slab", "far-pair"][kind]


def check_spi(rng, stats):
    n = int(rng.choice([2, 3, 17, 64, 257, 1000, 4097, 16384, 16385, 20000, 33333]))
    pts, kind = random_points(rng, n)
    sched = ["standard", "balanced"][int(rng.integers(0, 2))]
    workers = int(rng.integers(1, 6))
    for f, name in ((se.collision_indicator, "count"), (se.inverse_square, "sum")):
        r = se.spi_parallel(pts, f, workers, sched)
        for b, got in zip(se._partition(n, workers), r.partials):
            c, s, _ = c_oracle.rows(pts, b.start, b.stop, sched)
            want = c if name == "count" else s
            ok = got == want if name == "count" else math.isclose(got, want, rel_tol=1e-5, abs_tol=1e-12)
            stats[(f"spi-{name}", ok)] += 1
            if not ok:
                print(f"MISMATCH spi {name} n={n} {kind} {pts.dtype} {sched} w={workers} "
                      f"[{b.start},{b.stop}): got {got} want {want}", flush=True)


def check_sorted(rng, stats):
    # the headline's path: whole-range fp32 sums on Morton-sorted points (n >= 2^15)
    n = int(rng.integers(32768, 70000))
    pts, kind = random_points(rng, n)
    pts = pts.astype(np.float32)
    (r,) = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    want_c, want_s, _ = c_oracle.rows(pts, 0, n, "balanced")
    ok = r.count == want_c and math.isclose(r.sum, want_s, rel_tol=1e-6)
    stats[("sorted-sum", ok)] += 1
    if not ok:
        print(f"MISMATCH sorted-sum n={n} {kind}: got {r.count} {r.sum!r} want {want_c} {want_s!r}", flush=True)


def check_tc(rng, stats):
    # the tensor-core count filter forced at any size (PC_TILE_TC), every distribution,
    # float and integer predicates
    n = int(rng.choice([2, 9, 127, 129, 255, 257, 1000, 4097, 8191, 12345, 20000]))
    pts, kind = random_points(rng, n)
    (r,) = _lib.pairs_host(np.ascontiguousarray(pts), _lib.PC_COLLISION, _lib.PC_BALANCED, [0, n],
                           tiling=_lib.PC_TILE_TC)
    want = c_oracle.rows(pts, 0, n, "balanced")[0]
    ok = r.count == want and r.error == 0
    stats[("tc-count", ok)] += 1
    if not ok:
        print(f"MISMATCH tc-count n={n} {kind} {pts.dtype}: got {r.count} want {want}", flush=True)
    span = int(rng.integers(1, 30))
    beads = rng.integers(-span, span + 1, size=(n, 3))
    if rng.random() < 0.3:
        beads += np.int64(rng.integers(-2**40, 2**40))
    col, con = c_oracle.int_pairs(beads)
    for name, inter, want in (("tc-coincide", _lib.PC_COINCIDE, col), ("tc-manhattan1", _lib.PC_MANHATTAN1, con)):
        (r,) = _lib.pairs_host(beads, inter, _lib.PC_BALANCED, [0, n], tiling=_lib.PC_TILE_TC)
        stats[(name, r.count == want)] += 1
        if r.count != want:
            print(f"MISMATCH {name} n={n} span={span}: got {r.count} want {want}", flush=True)


def check_parts(rng, stats):
    # round 2: tile parts (pc_pairs_part_host) of a random range add up to the oracle's range
    # result on the sorted / direct / Gram paths; sums bit-reproducible across repeats
    n = int(rng.choice([2, 3, 257, 5000, 16385, 40001, 65537]))
    pts, kind = random_points(rng, n)
    pts = pts.astype(np.float32)
    lo = int(rng.integers(0, n))
    hi = int(rng.integers(lo, n + 1))
    if rng.random() < 0.5:
        lo, hi = 0, n
    nparts = int(rng.integers(1, 9))
    want_c, want_s, want_p = c_oracle.rows(pts, lo, hi, "balanced")
    for inter, tiling in ((_lib.PC_COLLISION_INVSQ, _lib.PC_TILE_SORTED if (lo, hi) == (0, n) else _lib.PC_TILE_FLAT),
                          (_lib.PC_COLLISION, _lib.PC_TILE_FLAT)):
        parts = [_lib.pairs_part_host(pts, inter, _lib.PC_BALANCED, lo, hi, k, nparts, tiling) for k in range(nparts)]
        c = sum(q.count for q in parts)
        pr = sum(q.pairs for q in parts)
        ok = c == want_c and pr == want_p and all(q.error == 0 for q in parts)
        if inter == _lib.PC_COLLISION_INVSQ and want_p:
            s = sum(q.sum for q in parts)
            ok = ok and math.isclose(s, want_s, rel_tol=1e-6)
            again = _lib.pairs_part_host(pts, inter, _lib.PC_BALANCED, lo, hi, 0, nparts, tiling)
            ok = ok and again.sum == parts[0].sum
        stats[(f"parts-{'sum' if inter == _lib.PC_COLLISION_INVSQ else 'count'}", ok)] += 1
        if not ok:
            print(f"MISMATCH parts n={n} {kind} [{lo},{hi}) x{nparts} inter={inter}: got {c} want {want_c}",
                  flush=True)


def check_pruned(rng, stats):
    # round 2: whole-range fp32 contact counts take the pruned sorted count (n >= 2^15); the
    # paper's thread-per-row kernels at random sizes
    n = int(rng.integers(32768, 70000))
    pts, kind = random_points(rng, n)
    pts = pts.astype(np.float32)
    want = c_oracle.rows(pts, 0, n, "balanced")[0]
    got = se.spi_balanced(pts, se.collision_indicator).total
    stats[("pruned-count", got == want)] += 1
    if got != want:
        print(f"MISMATCH pruned-count n={n} {kind}: got {got} want {want}", flush=True)
    m = int(rng.integers(2, 6000))
    sched = ("standard", "balanced")[int(rng.integers(0, 2))]
    sub = pts[:m]
    c, s_, p_ = c_oracle.rows(sub, 0, m, sched)
    (r,) = _lib.pairs_host(np.ascontiguousarray(sub), _lib.PC_COLLISION_INVSQ, _lib.SCHEDULE_CODES[sched], [0, m],
                           tiling=_lib.PC_TILE_THREAD_ROW)
    ok = r.count == c and r.pairs == p_ and math.isclose(r.sum, s_, rel_tol=1e-6)
    stats[("thread-row", ok)] += 1
    if not ok:
        print(f"MISMATCH thread-row m={m} {sched}: got {r.count} {r.sum!r} want {c} {s_!r}", flush=True)


def check_int(rng, stats):
    n = int(rng.choice([1, 2, 5, 100, 1000, 4096, 5000, 20000]))
    span = int(rng.integers(1, 40))
    beads = rng.integers(-span, span + 1, size=(n, 3))
    if rng.random() < 0.3:
        beads += np.int64(rng.integers(-2**40, 2**40))
    want_col, want_con = c_oracle.int_pairs(beads)
    for name, got, want in (("oracle_collisions", pc.oracle_collisions(beads), want_col),
                            ("oracle_contacts", pc.oracle_contacts(beads), want_con)):
        stats[(name, got == want)] += 1
        if got != want:
            print(f"MISMATCH {name} n={n} span={span}: got {got} want {want}", flush=True)


def check_lattice(rng, stats):
    a = int(rng.integers(1, 120))
    n = int(rng.choice([1, 10, 1000, 50_000, 400_000]))
    spread = int(rng.integers(0, a + 1))
    beads = rng.integers(-spread, spread + 1, size=(n, 3))
    side = 2 * a + 3
    keys = np.ravel_multi_index(tuple((beads + a + 1).T), (side,) * 3)
    occ = np.bincount(keys)
    want = (int((occ * (occ - 1) // 2).sum()), int(np.count_nonzero(occ)))
    sp = pc.new_space(a)
    rep = pc.count_collisions(beads, sp)
    pc.reset_sparse(sp)
    ok = (rep.count, rep.cells_touched) == want
    stats[("count_collisions", ok)] += 1
    if not ok:
        print(f"MISMATCH count_collisions a={a} n={n} spread={spread}: got {(rep.count, rep.cells_touched)} "
              f"want {want}", flush=True)
    doubled = lc.contact_accumulator(beads, sp)
    pc.reset_sparse(sp)
    if n <= 50_000:
        ok = doubled // 2 == c_oracle.int_pairs(beads)[1]
        stats[("count_contacts", ok)] += 1
        if not ok:
            print(f"MISMATCH contacts a={a} n={n}", flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--minutes", type=float, default=15.0)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--sorted", action="store_true", help="also whole-range fp32 sums on the sorted path (slower)")
    args = p.parse_args()
    rng = np.random.default_rng(args.seed)
    stats: Counter = Counter()
    t_end = time.time() + 60 * args.minutes
    rounds = 0
    while time.time() < t_end:
        check_spi(rng, stats)
        check_int(rng, stats)
        check_lattice(rng, stats)
        check_tc(rng, stats)
        check_parts(rng, stats)
        check_pruned(rng, stats)
        if args.sorted:
            check_sorted(rng, stats)
        rounds += 1
    fams = sorted({k for k, _ in stats})
    bad = 0
    for f in fams:
        print(f"{f:20s} pass {stats[(f, True)]:6d}  fail {stats[(f, False)]:4d}")
        bad += stats[(f, False)]
    print(f"rounds {rounds}, total checks {sum(stats.values())}, failures {bad} (seed {args.seed})")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
