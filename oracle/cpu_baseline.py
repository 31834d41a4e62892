"""Timed CPU reference for bench.py -- TEST/BASELINE INFRASTRUCTURE ONLY.

Times the reference's own per-row algorithm -- ``_run_outer`` with its batch
evaluation (spi_engine.py:84-120) -- on a bounded sample of outer rows of the
bench workload, over a fork process pool on every host core (the reference's
own thread pool is GIL-bound and slower than one core), and
extrapolates to pair-tests/s.  Balanced rows all own (n-1)/2 (+-1) pairs, so
sampled rows are representative.

Which implementation is timed:
  * ``"reference"`` -- the UNMODIFIED reference package installed in
    ``baseline/_ref`` (``pip install --target baseline/_ref``),
    imported as ``paircount`` from there; the interactions are its own
    ``collision_indicator`` and the reference tests' softened inverse square
    (test_spi_engine.py:108-111, a user-supplied f);
  * ``"port"`` -- ``numpy_port.run_rows``, the restatement, when
    ``baseline/_ref`` is absent.
"""

from __future__ import annotations

import importlib
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

from . import numpy_port as npo

REF_DIR = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
_OBJ = None
_KIND = "port"


def inv_dist(a, b):
    """The reference tests' float interaction (test_spi_engine.py:108-111)."""
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return 1.0 / (1.0 + ((a - b) ** 2).sum(axis=-1))


def load_reference():
    """The unmodified reference's spi_engine from baseline/_ref, or None."""
    if not (REF_DIR / "paircount" / "spi_engine.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    mod = importlib.import_module("paircount.spi_engine")
    if not str(Path(mod.__file__).resolve()).startswith(str(REF_DIR.resolve())):
        return None  # another `paircount` shadows it
    return mod


def kind() -> str:
    return "reference" if load_reference() is not None else "port"


def _task(args):
    lo, hi, schedule, fns = args
    ref = load_reference() if _KIND == "reference" else None
    t0 = time.perf_counter()
    pairs = 0
    for name in fns:
        if ref is not None:
            f = ref.collision_indicator if name == "collision" else inv_dist
            _, p = ref._run_outer(_OBJ, f, range(lo, hi), schedule)
        else:
            f = npo.collision_indicator if name == "collision" else npo.inverse_square
            _, p = npo.run_rows(_OBJ, f, lo, hi, schedule)
        pairs = p
    return pairs, time.perf_counter() - t0


def sample_rows(n: int, count: int, rows_each: int = 1, offset: int = 0) -> list[tuple[int, int]]:
    """`count` row blocks of `rows_each` rows spread evenly over [0, n)."""
    starts = np.linspace(0, n - rows_each, count).astype(np.int64)
    return [(int((s + offset) % max(1, n - rows_each)), int((s + offset) % max(1, n - rows_each)) + rows_each)
            for s in starts]


def time_sample(obj: np.ndarray, rows: list[tuple[int, int]], schedule: str = "balanced",
                fns=("collision", "inverse_square"), processes: int | None = None, impl: str | None = None):
    """Evaluate every f of `fns` on every row block; returns
    (pair-tests done, wall seconds, processes used, kind).  A pair-test is one
    pair evaluated for every f in `fns` (the reference needs one pass per f)."""
    global _OBJ, _KIND
    _OBJ = obj
    _KIND = impl or kind()
    procs = processes or os.cpu_count() or 1
    tasks = [(lo, hi, schedule, tuple(fns)) for lo, hi in rows]
    t0 = time.perf_counter()
    if procs == 1:
        out = [_task(t) for t in tasks]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            out = pool.map(_task, tasks, chunksize=1)
    wall = time.perf_counter() - t0
    return sum(p for p, _ in out), wall, procs, _KIND


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
