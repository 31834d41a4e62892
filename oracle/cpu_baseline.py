"""Timed CPU reference for bench.py -- TEST/BASELINE INFRASTRUCTURE ONLY.

Times ``numpy_port.run_rows`` -- the reference's own per-row numpy algorithm
(spi_engine.py:84-120) -- on a bounded sample of outer rows of the bench
workload, over a fork process pool (the reference's thread pool is GIL-bound
and slower than one core), and extrapolates to pair-tests/s.
Balanced rows all own (n-1)/2 (+-1) pairs, so sampled rows are representative.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import numpy_port as npo

_OBJ = None


def _task(args):
    lo, hi, schedule, fns = args
    t0 = time.perf_counter()
    pairs = 0
    for name in fns:
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
                fns=("collision", "inverse_square"), processes: int | None = None):
    """Evaluate every f of `fns` on every row block; returns
    (pair-tests done, wall seconds, processes used).  A pair-test is one pair
    evaluated for every f in `fns` (the reference needs one pass per f)."""
    global _OBJ
    _OBJ = obj
    procs = processes or os.cpu_count() or 1
    tasks = [(lo, hi, schedule, tuple(fns)) for lo, hi in rows]
    t0 = time.perf_counter()
    if procs == 1:
        out = [_task(t) for t in tasks]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            out = pool.map(_task, tasks, chunksize=1)
    wall = time.perf_counter() - t0
    return sum(p for p, _ in out), wall, procs


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
