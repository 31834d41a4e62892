"""Full-size oracle totals for the headline configs -> tests/golden/golden_full.json.

TEST INFRASTRUCTURE (dev container only; the GPU box reads the committed JSON).

The reference's own whole-triangle result (``_run_outer`` over every row,
spi_engine.py:109-120, summed over the partition, 191-230) is out of the
reference's CPU reach at 2^20 / 2^22 points (12 h / 218 h on one core,
SURVEY.md §8(d)).  These totals come from the C oracle's ``orc_total_f64``
(oracle/oracle.c): the reference's float64 predicate and term per pair, over
the same pair set, compiled here with -O3 -march=native (AVX-512) into /tmp.

Trust chain, checked by this script before it computes anything:
  1. the inputs are produced by the UNMODIFIED reference generators (loaded
     read-only as ``paircount_ref``, as make_golden.py does) and must match
     the SHA-256 digests already pinned in golden_configs.json;
  2. the fast build must reproduce the reference's own standard-schedule row
     samples in golden_configs.json (count exact, sum within 1e-12);
  3. the fast build must agree with the pinned ``orc_rows_f64`` (portable
     liboracle.so, tests/test_oracle.py) on the first pinned row range.

    python -B tests/golden/make_full_totals.py [cfg3 cfg4u cfg4c]
"""

from __future__ import annotations

import ctypes
import json
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))

from make_golden import digest, load_reference  # noqa: E402
from oracle import c_oracle  # noqa: E402

OUT = HERE / "golden_full.json"
FAST = Path("/tmp/liboracle_fast.so")


def fast_lib():
    subprocess.run(["gcc", "-O3", "-march=native", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared",
                    "-fPIC", str(ROOT / "oracle" / "oracle.c"), "-o", str(FAST)], check=True)
    lib = ctypes.CDLL(str(FAST))
    lib.orc_total_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)]
    return lib


def inputs(ref, which):
    gen = ref.generators

    def edge(n):
        return (4.0 * np.pi * n / 3.0) ** (1.0 / 3.0)

    if which == "cfg3":
        return gen.random_spheres(2**20, edge(2**20), 1).astype(np.float32)
    if which == "cfg4u":
        return gen.random_spheres(2**22, edge(2**22), 2).astype(np.float32)
    n4 = 2**22  # SURVEY.md §8(d) row 4 (make_golden.configs)
    rng = gen._rng(2, 6)
    centres = rng.random((1024, 3)) * edge(n4)
    assign = rng.integers(0, 1024, n4)
    off = gen._box_muller(rng, 3 * n4).reshape(n4, 3) * 2.0
    return (centres[assign] + off).astype(np.float32)


def main(argv):
    which = argv[1:] or ["cfg3", "cfg4u", "cfg4c"]
    ref = load_reference()
    cfgs = json.loads((HERE / "golden_configs.json").read_text())
    lib = fast_lib()
    out = json.loads(OUT.read_text()) if OUT.exists() else {}
    out["_provenance"] = ("orc_total_f64 (oracle/oracle.c, -O3 -march=native) over every pair i<j of the reference "
                          "generators' inputs; pinned to the reference's standard-schedule row samples in "
                          "golden_configs.json and to orc_rows_f64; tests/golden/make_full_totals.py")
    for name in which:
        t0 = time.time()
        x = inputs(ref, name)
        assert digest(x) == cfgs[name]["sha256"], f"{name}: input digest differs from the pinned reference input"
        n = len(x)
        for smp in cfgs[name]["samples"]:
            if smp["schedule"] != "standard":
                continue
            c, s = c_oracle.total(x, *smp["rows"], lib=lib)
            assert c == smp["count"] and abs(s - smp["inv_sum"]) <= 1e-12 * smp["inv_sum"], (name, smp, c, s)
        lo, hi = cfgs[name]["samples"][0]["rows"]
        c_p, s_p, _ = c_oracle.rows(x, lo, hi, "standard")
        c_f, s_f = c_oracle.total(x, lo, hi, lib=lib)
        assert c_p == c_f and abs(s_p - s_f) <= 1e-12 * s_p, (name, c_p, c_f, s_p, s_f)
        print(f"{name}: n={n} pinned checks ok ({time.time() - t0:.1f} s); computing the full triangle", flush=True)
        t1 = time.time()
        count, inv_sum = c_oracle.total(x, 0, n, lib=lib)
        out[name] = {"n": n, "sha256": cfgs[name]["sha256"], "pairs": n * (n - 1) // 2, "count": count,
                     "inv_sum": inv_sum, "seconds": round(time.time() - t1, 1)}
        print(name, out[name], flush=True)
        OUT.write_text(json.dumps(out, indent=1) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv))
