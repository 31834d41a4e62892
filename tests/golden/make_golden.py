"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs only in the dev container, where /root/reference exists; the GPU box
and the test-suite read the committed JSON, never the reference.  The
reference package is loaded read-only under the module name ``paircount_ref``
 so it cannot collide with anything in this repo; run
with ``python -B`` so no bytecode is written next to the reference sources.

    python -B tests/golden/make_golden.py small     # seconds  -> golden_small.json
    python -B tests/golden/make_golden.py configs   # ~15 min  -> golden_configs.json

Every value stored here is produced by a reference function call; the
inputs are produced by the reference generators and recorded as SHA-256
digests so the repo's own generator restatement can be pinned to them.
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import sys
import time
from pathlib import Path

import numpy as np

REF_PKG = Path("/root/reference/pkg/src/paircount")
HERE = Path(__file__).resolve().parent


def load_reference():
    sys.dont_write_bytecode = True
    spec = importlib.util.spec_from_file_location(
        "paircount_ref", REF_PKG / "__init__.py",
        submodule_search_locations=[str(REF_PKG)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["paircount_ref"] = mod
    spec.loader.exec_module(mod)
    import paircount_ref.generators  # noqa: F401
    import paircount_ref.lattice_counter  # noqa: F401
    import paircount_ref.pair_schedule  # noqa: F401
    import paircount_ref.spi_engine  # noqa: F401
    return mod


def digest(arr: np.ndarray) -> str:
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256()
    h.update(str(arr.dtype).encode())
    h.update(str(arr.shape).encode())
    h.update(arr.tobytes())
    return h.hexdigest()


def inv_square(a, b):
    """Softened inverse square 1/(1+|a-b|^2): test_spi_engine.py:108-111."""
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return 1.0 / (1.0 + ((a - b) ** 2).sum(axis=-1))


def near_boundary_spheres():
    """Adversarial pairs whose float64 distance^2 straddles 1.0 by an ulp,
    placed near the origin and far from it (where float32 Gram arithmetic
    loses the most precision)."""
    pts = []
    for base in (0.0, 3.25, 250.0, -180.5, 1000.0):
        for dx in (1.0, np.nextafter(1.0, 0.0), np.nextafter(1.0, 2.0),
                   0.999999, 1.000001, 0.9999999403953552, 1.0000001192092896):
            pts.append((base, base, base))
            pts.append((base + dx, base, base))
        # a diagonal pair at distance^2 ~ 1 in all three axes
        s = np.float64(1.0) / np.sqrt(3.0)
        pts.append((base, -base, base))
        pts.append((base + s, -base + s, base + s))
    return np.asarray(pts, dtype=np.float64)


def small(ref):
    gen, se, lc, ps = ref.generators, ref.spi_engine, ref.lattice_counter, ref.pair_schedule
    out = {"generator_digests": [], "spi_cases": [], "lattice_cases": [],
           "indicator_cases": [], "schedule_cases": []}

    # ---- generator digests -------------------------------------------------
    for n, seed in ((1, 0), (2, 5), (200, 42), (4096, 0), (1000, 1000 * 1000 + 3)):
        beads, ext = gen.random_chain(n, seed)
        out["generator_digests"].append(
            {"fn": "random_chain", "args": [n, seed], "sha256": digest(beads), "extent": ext})
    for args in ((50, 1e-9, 4, 0), (1000, 5.0, 30, 11), (1000, 500.0, 10, 2), (4096, 8.0, 64, 0), (333, 2.5, 9, 7)):
        out["generator_digests"].append(
            {"fn": "normal_cloud", "args": list(args), "sha256": digest(gen.normal_cloud(*args))})
    for args in ((100, 6.5, 5), (1, 1.0, 0), (4097, 16.0, 3), (65536, 64.99094755261542, 0)):
        out["generator_digests"].append(
            {"fn": "random_spheres", "args": list(args), "sha256": digest(gen.random_spheres(*args))})
    for n in (7, 1001):
        out["generator_digests"].append(
            {"fn": "_box_muller", "args": [0, 9, n], "sha256": digest(gen._box_muller(gen._rng(0, 9), n))})

    # ---- collision_indicator scalar/batch cases ------------------------------
    pts = near_boundary_spheres()
    a, b = pts[0::2], pts[1::2]
    vals = [int(se.collision_indicator(x, y)) for x, y in zip(a, b)]
    out["indicator_cases"].append({"name": "near_boundary_pairs", "points": pts.tolist(), "values": vals})
    for name, x, y in (("coincident", (0, 0, 0), (0, 0, 0)), ("tangent", (0, 0, 0), (1.0, 0, 0)),
                       ("inside", (0, 0, 0), (0.6, 0, 0))):
        out["indicator_cases"].append({"name": name, "points": [list(x), list(y)],
                                       "values": [int(se.collision_indicator(x, y))]})

    # ---- SPI cases -----------------------------------------------------------
    def spi_record(tag, objs, fname, f, gen_args=None, workers_list=(1, 2, 3, 7, 8)):
        rec = {"tag": tag, "f": fname, "n": int(len(objs)), "gen": gen_args,
               "dtype": str(objs.dtype), "input_sha256": digest(objs)}
        if gen_args is None:
            rec["points"] = objs.tolist()
        for name, fn in (("standard", se.spi_standard), ("balanced", se.spi_balanced)):
            r = fn(objs, f)
            rec[name] = {"total": r.total, "pairs": r.pairs_evaluated, "depth": r.depth_per_worker}
        rec["parallel"] = []
        for w in workers_list:
            for sched in se.SCHEDULES:
                r = se.spi_parallel(objs, f, w, sched)
                rec["parallel"].append({"workers": w, "schedule": sched, "total": r.total,
                                        "partials": list(r.partials), "worker_pairs": list(r.worker_pairs),
                                        "depth": r.depth_per_worker})
        out["spi_cases"].append(rec)

    grid = [(2, 6.0), (3, 6.0), (4, 6.0), (5, 6.0), (7, 6.0), (8, 6.0), (16, 6.0), (31, 6.0), (32, 6.0),
            (64, 6.0), (100, 4.0), (127, 6.0), (128, 6.0), (150, 3.0), (200, 3.0), (256, 6.0), (257, 6.0),
            (512, 6.0), (1000, 10.0), (2048, 12.0), (2049, 8.0)]
    for n, box in grid:
        seed = 100 + n
        objs = gen.random_spheres(n, box, seed)
        spi_record(f"spheres64_n{n}", objs, "collision", se.collision_indicator,
                   ["random_spheres", n, box, seed, "float64"])
        objs32 = objs.astype(np.float32)
        spi_record(f"spheres32_n{n}", objs32, "collision", se.collision_indicator,
                   ["random_spheres", n, box, seed, "float32"], workers_list=(1, 3, 8))
        if n <= 512 or n == 2048:
            spi_record(f"spheres64_inv_n{n}", objs, "inverse_square", inv_square,
                       ["random_spheres", n, box, seed, "float64"], workers_list=(1, 2, 7))
            spi_record(f"spheres32_inv_n{n}", objs32, "inverse_square", inv_square,
                       ["random_spheres", n, box, seed, "float32"], workers_list=(1, 7))
    # dense and degenerate inputs
    for n in (40, 300):
        dense = gen.random_spheres(n, 0.5, 77)  # every pair in contact
        spi_record(f"dense_n{n}", dense, "collision", se.collision_indicator,
                   ["random_spheres", n, 0.5, 77, "float64"], workers_list=(1, 4))
    spi_record("near_boundary", pts, "collision", se.collision_indicator, None, workers_list=(1, 2, 5))
    spi_record("near_boundary32", pts.astype(np.float32), "collision", se.collision_indicator, None,
               workers_list=(1, 3))
    coincident = np.zeros((3, 3))
    spi_record("three_coincident", coincident, "collision", se.collision_indicator, None)
    # spot check of test_acceptance.py:179-187 (N=10000, box 40, seed 99)
    big = gen.random_spheres(10_000, 40.0, 99)
    rec = {"tag": "acceptance_n10000", "f": "collision", "n": 10_000,
           "gen": ["random_spheres", 10_000, 40.0, 99, "float64"], "dtype": "float64",
           "input_sha256": digest(big)}
    r = se.spi_standard(big, se.collision_indicator)
    rec["standard"] = {"total": r.total, "pairs": r.pairs_evaluated, "depth": r.depth_per_worker}
    r = se.spi_parallel(big, se.collision_indicator, 8, "balanced")
    rec["parallel"] = [{"workers": 8, "schedule": "balanced", "total": r.total, "partials": list(r.partials),
                        "worker_pairs": list(r.worker_pairs), "depth": r.depth_per_worker}]
    out["spi_cases"].append(rec)

    # ---- lattice cases ---------------------------------------------------------
    def lattice_record(tag, beads, a, gen_args):
        beads = np.asarray(beads, dtype=np.int64).reshape(-1, 3)
        rec = {"tag": tag, "n": int(len(beads)), "half_extent": int(a), "gen": gen_args,
               "input_sha256": digest(beads)}
        if gen_args is None:
            rec["beads"] = beads.tolist()
        sp = lc.new_space(a)
        col = lc.count_collisions(beads, sp)
        lc.reset_sparse(sp, beads)
        con = lc.count_contacts(beads, sp)
        lc.reset_sparse(sp, beads)
        rec.update({"oracle_collisions": lc.oracle_collisions(beads), "oracle_contacts": lc.oracle_contacts(beads),
                    "count_collisions": [col.count, col.beads_processed, col.cells_touched],
                    "count_contacts": [con.count, con.beads_processed, con.cells_touched],
                    "contact_accumulator": lc.contact_accumulator(beads, lc.new_space(a))})
        out["lattice_cases"].append(rec)

    for n in (1, 2, 3, 16, 64, 257, 1024, 4096):
        for v in range(3):
            seed = 1000 * n + v
            beads, ext = gen.random_chain(n, seed)
            lattice_record(f"chain_n{n}_v{v}", beads, max(ext, 1), ["random_chain", n, seed])
    for n, sd, a, seed in ((100, 1.0, 8, 5), (1000, 5.0, 30, 11), (4096, 8.0, 64, 0), (2000, 2.0, 8, 3)):
        lattice_record(f"cloud_n{n}_sd{sd}", gen.normal_cloud(n, sd, a, seed), a, ["normal_cloud", n, sd, a, seed])
    lattice_record("all_coincident_40", np.zeros((40, 3)), 8, None)
    grid_pts = [[2 * x, 2 * y, 2 * z] for x in range(4) for y in range(4) for z in range(4)]
    lattice_record("all_distinct_64", grid_pts, 8, None)
    lattice_record("empty", np.zeros((0, 3)), 8, None)
    lattice_record("five_coincident", [(0, 0, 0)] * 5, 1, None)
    lattice_record("star", [(0, 0, 0)] + [tuple(o) for o in lc.NEIGHBOR_OFFSETS], 1, None)
    lattice_record("multiplicity", [(0, 0, 0)] * 2 + [(1, 0, 0)] * 3, 1, None)
    big_coords = np.array([[2**40, -2**40, 7], [2**40, -2**40, 7], [2**40 + 1, -2**40, 7],
                           [-3, 2**35, 0], [-3, 2**35, 1], [-3, 2**35, 0]], dtype=np.int64)
    out["lattice_cases"].append({"tag": "wide_int64", "n": 6, "beads": big_coords.tolist(), "gen": None,
                                 "oracle_collisions": lc.oracle_collisions(big_coords),
                                 "oracle_contacts": lc.oracle_contacts(big_coords)})

    # ---- schedule cases --------------------------------------------------------
    for n in (1, 2, 3, 4, 5, 6, 7, 16, 17, 100, 101):
        out["schedule_cases"].append({"n": n, "steps": ps.step_counts(n).tolist(),
                                      "pairs_sha256": digest(ps.pairs_array(n))})
    return out


def run_outer_sample(ref, objs, rows, schedule):
    se = ref.spi_engine
    cnt, pairs = se._run_outer(objs, se.collision_indicator, range(*rows), schedule)
    inv, _ = se._run_outer(objs, inv_square, range(*rows), schedule)
    return {"rows": list(rows), "schedule": schedule, "count": cnt, "pairs": pairs, "inv_sum": inv}


def configs(ref):
    gen, se, lc = ref.generators, ref.spi_engine, ref.lattice_counter
    out = {}
    t0 = time.time()

    # config 1: N=4096 integer points, exact-coincidence all-pairs
    cloud = gen.normal_cloud(4096, 8.0, 64, 0)
    chain, ext = gen.random_chain(4096, 0)
    out["cfg1"] = {"cloud": {"args": [4096, 8.0, 64, 0], "sha256": digest(cloud),
                             "oracle_collisions": lc.oracle_collisions(cloud),
                             "oracle_contacts": lc.oracle_contacts(cloud)},
                   "chain": {"args": [4096, 0], "sha256": digest(chain), "extent": ext,
                             "oracle_collisions": lc.oracle_collisions(chain),
                             "oracle_contacts": lc.oracle_contacts(chain)}}
    print("cfg1", out["cfg1"], time.time() - t0, flush=True)

    # config 3 / 4: row samples (full runs take 12 h / 218 h on one core)
    def edge(n):
        return (4.0 * np.pi * n / 3.0) ** (1.0 / 3.0)

    n3 = 2**20
    s3 = (gen.random_spheres(n3, edge(n3), 1)).astype(np.float32)
    out["cfg3"] = {"args": [n3, edge(n3), 1], "sha256": digest(s3), "samples": []}
    for rows, sched in (((0, 32), "balanced"), ((524272, 524304), "balanced"), ((524272, 524304), "standard"),
                        ((0, 32), "standard"), ((1048560, 1048576), "balanced"), ((1048000, 1048576), "standard"),
                        ((300001, 300013), "balanced")):
        out["cfg3"]["samples"].append(run_outer_sample(ref, s3, rows, sched))
        print("cfg3", out["cfg3"]["samples"][-1], time.time() - t0, flush=True)

    n4 = 2**22
    s4 = gen.random_spheres(n4, edge(n4), 2).astype(np.float32)
    out["cfg4u"] = {"args": [n4, edge(n4), 2], "sha256": digest(s4), "samples": []}
    for rows, sched in (((0, 32), "balanced"), ((2097136, 2097168), "balanced"), ((0, 16), "standard")):
        out["cfg4u"]["samples"].append(run_outer_sample(ref, s4, rows, sched))
        print("cfg4u", out["cfg4u"]["samples"][-1], time.time() - t0, flush=True)
    rng = gen._rng(2, 6)
    centres = rng.random((1024, 3)) * edge(n4)
    assign = rng.integers(0, 1024, n4)
    off = gen._box_muller(rng, 3 * n4).reshape(n4, 3) * 2.0
    c4 = (centres[assign] + off).astype(np.float32)
    out["cfg4c"] = {"recipe": "SURVEY.md 8(d) row 4", "sha256": digest(c4), "samples": []}
    for rows, sched in (((0, 32), "balanced"), ((4194000, 4194304), "balanced"), ((77, 93), "standard")):
        out["cfg4c"]["samples"].append(run_outer_sample(ref, c4, rows, sched))
        print("cfg4c", out["cfg4c"]["samples"][-1], time.time() - t0, flush=True)
    del s4, c4

    # config 5: counting array on 2^26 points in [-512,512)^3
    p5 = gen._rng(0, 5).integers(-512, 512, size=(2**26, 3), dtype=np.int64)
    sp = lc.new_space(512)
    rep = lc.count_collisions(p5, sp)
    flat = sp._flatten(p5)
    occ = sp.cells.reshape(-1)[flat]
    out["cfg5"] = {"args": [2**26, 512, 0, 5], "sha256": digest(p5), "count": rep.count,
                   "beads_processed": rep.beads_processed, "cells_touched": rep.cells_touched,
                   "max_occupancy": int(occ.max())}
    print("cfg5", out["cfg5"], time.time() - t0, flush=True)
    del sp, p5, flat, occ

    # config 2: N=65536 fp32 spheres, full totals under both schedules (~5 min)
    n2 = 65536
    s2 = gen.random_spheres(n2, edge(n2), 0).astype(np.float32)
    out["cfg2"] = {"args": [n2, edge(n2), 0], "sha256": digest(s2), "samples": []}
    for rows, sched in (((0, 64), "standard"), ((0, 64), "balanced"), ((32700, 32800), "balanced"),
                        ((65000, 65536), "standard")):
        out["cfg2"]["samples"].append(run_outer_sample(ref, s2, rows, sched))
    for name, fn in (("standard", se.spi_standard), ("balanced", se.spi_balanced)):
        r = fn(s2, se.collision_indicator)
        out["cfg2"][name] = {"total": r.total, "pairs": r.pairs_evaluated, "depth": r.depth_per_worker}
        print("cfg2", name, out["cfg2"][name], time.time() - t0, flush=True)
    return out


def main(argv):
    ref = load_reference()
    which = argv[1] if len(argv) > 1 else "small"
    if which == "small":
        data = small(ref)
        path = HERE / "golden_small.json"
    elif which == "configs":
        data = configs(ref)
        path = HERE / "golden_configs.json"
    else:
        raise SystemExit(f"unknown fixture set {which!r}")
    data["_generated_by"] = "tests/golden/make_golden.py " + which + " (reference pkg/src/paircount, numpy " + np.__version__ + ")"
    path.write_text(json.dumps(data, indent=1) + "\n")
    print("wrote", path)


if __name__ == "__main__":
    main(sys.argv)
