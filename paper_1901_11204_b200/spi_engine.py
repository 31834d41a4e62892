"""Symmetric pairwise interaction (SPI) engines on the B200.

Drop-in for the reference module ``pkg/src/paircount/spi_engine.py``: same
names, arguments, result record and exceptions.  The O(N^2) accumulation runs
in libpaircount.so (``pc_pairs_host``); the Python here only validates,
converts the object array, maps the interaction function onto a kernel and
assembles the ``SpiResult``.

Supported interaction functions (the GPU has no way to run an arbitrary
Python callable, and there is no CPU fallback):
  * ``collision_indicator``  -- integer contact count, bit-exact (the fp32
    filter + exact float64 re-check of csrc/paircount.cu);
  * ``inverse_square``       -- softened inverse square 1/(1+|a-b|^2) summed
    in fp32 per chunk and float64 across chunks (float64/integer coordinates
    enter as hi+lo fp32 pairs so separations keep ~2u relative accuracy);
    agrees with the float64 reference within 1e-5 relative
    (tests/test_gpu_parity.py).
Any other callable raises ``TypeError`` -- after the same argument checks the
reference performs and after the n < 2 short-circuit, where the reference
never calls ``f`` either.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib
from .pair_schedule import row_pairs

SCHEDULES = ("standard", "balanced")


class InteractionDomainError(ValueError):
    """An interaction function was handed a non-finite object."""


class AccumulationError(ArithmeticError):
    """An interaction function produced a non-finite contribution."""


class SymmetryViolationError(ValueError):
    """An interaction function returned different values for (a,b) and (b,a)."""


@dataclass(frozen=True)
class Sphere:
    """A point sphere of diameter 1 (spi_engine.py:44-50)."""

    x: float
    y: float
    z: float


@dataclass(frozen=True)
class SpiResult:
    """Same fields as the reference record (spi_engine.py:53-59)."""

    total: float | int
    partials: tuple
    pairs_evaluated: int
    depth_per_worker: int
    worker_pairs: tuple


# ---------------------------------------------------------------------------
# interaction functions.  Called directly they evaluate one object against a
# batch with numpy (they are the user-facing predicate objects); passed to the
# engines they select a GPU kernel and are never called per pair.
# ---------------------------------------------------------------------------

def collision_indicator(a, b):
    """1 if two unit-diameter spheres' centres are strictly closer than 1
    (float64 arithmetic, spi_engine.py:62-73); batches broadcast."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if not np.isfinite(a).all() or not np.isfinite(b).all():
        raise InteractionDomainError("sphere coordinates must be finite")
    diff = a - b
    return (np.sum(diff * diff, axis=-1) < 1.0).astype(np.int64)


def inverse_square(a, b):
    """Softened inverse square 1/(1 + |a-b|^2) (the float SPI of
    test_spi_engine.py:108-111; BASELINE config 3)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    diff = a - b
    return 1.0 / (1.0 + np.sum(diff * diff, axis=-1))


def _interaction_code(f) -> int:
    if f is collision_indicator:
        return _lib.PC_COLLISION
    if f is inverse_square:
        return _lib.PC_COLLISION_INVSQ
    # the reference's own function object (or another drop-in's) is accepted by name
    name = getattr(f, "__name__", "")
    module = getattr(f, "__module__", "") or ""
    if name == "collision_indicator" and module.endswith("spi_engine"):
        return _lib.PC_COLLISION
    raise TypeError(
        f"interaction {f!r} cannot run on the GPU; supported: spi_engine.collision_indicator "
        "(contact count) and spi_engine.inverse_square (softened inverse-square sum)")


# ---------------------------------------------------------------------------
# object arrays
# ---------------------------------------------------------------------------

def as_object_array(objects) -> np.ndarray:
    """ndarray passes through; Sphere sequences become float64 (n, 3)
    (spi_engine.py:76-81)."""
    if isinstance(objects, np.ndarray):
        return objects
    if len(objects) > 0 and isinstance(objects[0], Sphere):
        return np.array([[o.x, o.y, o.z] for o in objects], dtype=np.float64)
    return np.asarray(objects)


def _device_coords(obj: np.ndarray) -> np.ndarray:
    """(n, 3) C-contiguous array in a dtype the kernels read.  Fewer than
    three coordinates are zero-padded (exact: adds 0^2 terms); float32,
    float64, int32 and int64 pass through, anything else is widened to
    float64 exactly as collision_indicator's np.asarray(.., float64) would."""
    if obj.ndim == 1:
        # the reference's batch call sums over the partner axis, its scalar
        # fallback then reduces a 0-d array over axis -1 (spi_engine.py:87-92)
        raise np.exceptions.AxisError(-1, 0)
    if obj.ndim != 2 or obj.shape[1] > 3:
        raise TypeError(f"objects must be points with at most 3 coordinates, got shape {obj.shape}")
    if obj.dtype not in _lib.DTYPE_CODES:
        obj = obj.astype(np.float64)
    if obj.shape[1] < 3:
        pad = np.zeros((obj.shape[0], 3), dtype=obj.dtype)
        pad[:, : obj.shape[1]] = obj
        obj = pad
    return np.ascontiguousarray(obj)


def _window_len(n: int, rows: np.ndarray, schedule: str) -> np.ndarray:
    """Partners each row owns (pair_schedule.py:49-59)."""
    if schedule == "standard":
        return n - 1 - rows
    if n % 2:
        return np.full(len(rows), (n - 1) // 2, dtype=np.int64)
    return np.where(rows < n // 2, n // 2, n // 2 - 1)


def _first_bad_pair(xyz: np.ndarray, schedule: str, ranges, nan_only: bool):
    """Error path only (no interaction is evaluated): the first (row, partner)
    in the reference's evaluation order -- ranges in order, rows in order,
    partners in window order (spi_engine.py:102-120) -- that involves a
    non-finite point (``nan_only=False``: collision_indicator raises for
    such a batch, spi_engine.py:70-71) or whose softened inverse-square term
    is NaN (``nan_only=True``: a NaN coordinate, or the same infinity on the
    same axis of both points; 1/(1+inf) = 0 is finite, spi_engine.py:93-95).
    Returns (range index, i, j) or None."""
    n = len(xyz)
    finite = np.isfinite(xyz)
    bad = np.nonzero(~finite.all(axis=1))[0]
    if len(bad) == 0:
        return None
    nanrow = np.isnan(xyz).any(axis=1)
    bxyz = xyz[bad]
    for k, (lo, hi) in enumerate(ranges):
        for r0 in range(lo, hi, 4096):
            rows = np.arange(r0, min(hi, r0 + 4096), dtype=np.int64)
            wl = _window_len(n, rows, schedule)
            best = np.full(len(rows), np.iinfo(np.int64).max, dtype=np.int64)
            # a row whose own point is NaN (or any non-finite, for the count) fails at its first partner
            own_bad = nanrow[rows] if nan_only else ~finite[rows].all(axis=1)
            best[own_bad & (wl >= 1)] = 1
            for b0 in range(0, len(bad), 256):
                bs = bad[b0:b0 + 256]
                off = bs[None, :] - rows[:, None]
                if schedule == "balanced":
                    off %= n
                owned = (off >= 1) & (off <= wl[:, None])
                if nan_only:
                    pts = xyz[rows]
                    same_inf = (np.isinf(pts)[:, None, :] & (pts[:, None, :] == bxyz[None, b0:b0 + 256, :])).any(-1)
                    owned &= nanrow[bs][None, :] | same_inf
                best = np.minimum(best, np.where(owned, off, np.iinfo(np.int64).max).min(axis=1))
            hit = np.nonzero(best < np.iinfo(np.int64).max)[0]
            if len(hit):
                i = int(rows[hit[0]])
                j = i + int(best[hit[0]])
                return k, i, (j % n if schedule == "balanced" else j)
    return None


def _prepare(obj: np.ndarray, f, ranges: list[tuple[int, int]], schedule: str):
    """(interaction code, device-ready coordinates).  Non-finite coordinates
    are found by the device (prep statistics), not by a host scan: see
    _resolve_domain for how they map onto the reference's errors."""
    del ranges, schedule
    return _interaction_code(f), _device_coords(obj)


def _resolve_domain(xyz: np.ndarray, code: int, schedule: str, ranges, results, rerun):
    """Reference semantics for a call whose device result flags PC_ERR_DOMAIN.

    * collision_indicator: InteractionDomainError if some owned pair of the
      ranges touches a non-finite point (the reference's batch check,
      spi_engine.py:70-71); otherwise those points are in no evaluated pair
      and the call is rerun with them zeroed.
    * inverse_square: the device evaluated every term in float64 (isolated
      infinities give 0, as in the reference); a NaN sum means a NaN term, and
      the reference raises AccumulationError naming the first such pair
      (spi_engine.py:93-95)."""
    if not any(r.error == _lib.PC_ERR_DOMAIN for r in results):
        return results
    if code == _lib.PC_COLLISION_INVSQ:
        hit = _first_bad_pair(xyz, schedule, ranges, nan_only=True)
        if hit is None:
            raise AccumulationError("non-finite contribution (pair not located)")
        raise AccumulationError(f"non-finite contribution for pair ({hit[1]}, {hit[2]})")
    if xyz.dtype.kind != "f" or _first_bad_pair(xyz, schedule, ranges, nan_only=False) is not None:
        raise InteractionDomainError("sphere coordinates must be finite")
    clean = xyz.copy()
    clean[~np.isfinite(clean).all(axis=1)] = 0
    return rerun(clean)


def _partial_of(r, code: int, n: int, lo: int, hi: int, schedule: str):
    """Typed partial of one kernel result record (int count or float sum)."""
    if r.error == _lib.PC_ERR_DOMAIN:
        raise InteractionDomainError("sphere coordinates must be finite")
    pairs = row_pairs(n, lo, hi, schedule)
    if int(r.pairs) != pairs:
        raise RuntimeError(f"kernel pair count {r.pairs} != closed form {pairs}")
    partial = float(r.sum) if code == _lib.PC_COLLISION_INVSQ else int(r.count)
    return (partial if pairs else 0), pairs


def _run_ranges(obj: np.ndarray, f, ranges: list[tuple[int, int]], schedule: str):
    """(partial, pairs) per row range -- the GPU counterpart of calling
    _run_outer once per range (spi_engine.py:109-120)."""
    n = len(obj)
    if n < 2:
        return [(0, 0) for _ in ranges]
    code, xyz = _prepare(obj, f, ranges, schedule)
    bounds = [ranges[0][0]] + [hi for _, hi in ranges]
    sched = _lib.SCHEDULE_CODES[schedule]

    def run(x):
        return _lib.pairs_host(x, code, sched, bounds)

    results = _resolve_domain(xyz, code, schedule, ranges, run(xyz), run)
    return [_partial_of(r, code, n, lo, hi, schedule) for (lo, hi), r in zip(ranges, results)]


def _audit_symmetry(obj: np.ndarray, f, rng_seed: int = 0, samples: int = 16) -> None:
    """Debug probe f(a,b) == f(b,a) on sampled pairs (spi_engine.py:123-136)."""
    n = len(obj)
    if n < 2:
        return
    rng = np.random.Generator(np.random.PCG64(rng_seed))
    for _ in range(samples):
        i, j = rng.integers(0, n, size=2)
        if i == j:
            continue
        ab, ba = f(obj[i], obj[j]), f(obj[j], obj[i])
        if not np.all(np.asarray(ab) == np.asarray(ba)):
            raise SymmetryViolationError(
                f"f({i},{j})={ab} but f({j},{i})={ba}: interaction must be symmetric")


def _depth(n: int, schedule: str) -> int:
    """Depth metric (spi_engine.py:139-144): n-1 standard, n//2 balanced."""
    if n <= 1:
        return 0
    return n - 1 if schedule == "standard" else n // 2


def _partition(n: int, workers: int) -> list[range]:
    """Contiguous near-equal outer blocks (spi_engine.py:179-188)."""
    base, extra = divmod(n, workers)
    blocks, start = [], 0
    for w in range(workers):
        size = base + (1 if w < extra else 0)
        blocks.append(range(start, start + size))
        start += size
    return blocks


def _sequential(objects, f, audit_symmetry: bool, schedule: str) -> SpiResult:
    obj = as_object_array(objects)
    if audit_symmetry:
        _audit_symmetry(obj, f)
    n = len(obj)
    ((total, pairs),) = _run_ranges(obj, f, [(0, n)], schedule)
    return SpiResult(total=total, partials=(total,), pairs_evaluated=pairs,
                     depth_per_worker=_depth(n, schedule), worker_pairs=(pairs,))


def spi_standard(objects, f: Callable, audit_symmetry: bool = False) -> SpiResult:
    """Triangular schedule: row i with every j > i (Alg. 3; spi_engine.py:147-160)."""
    return _sequential(objects, f, audit_symmetry, "standard")


def spi_balanced(objects, f: Callable, audit_symmetry: bool = False) -> SpiResult:
    """Balanced circular schedule (Alg. 4; spi_engine.py:163-176)."""
    return _sequential(objects, f, audit_symmetry, "balanced")


def spi_parallel(objects, f: Callable, workers: int, schedule: str = "balanced",
                 audit_symmetry: bool = False) -> SpiResult:
    """Per-worker partials over contiguous outer blocks, summed in ascending
    worker order (spi_engine.py:191-230).  All blocks go to the GPU in one
    call; each block's partial is exactly the reference worker's."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if schedule not in SCHEDULES:
        raise ValueError(f"schedule must be one of {SCHEDULES}, got {schedule!r}")
    obj = as_object_array(objects)
    if audit_symmetry:
        _audit_symmetry(obj, f)
    n = len(obj)
    blocks = [(b.start, b.stop) for b in _partition(n, workers)]
    results = _run_ranges(obj, f, blocks, schedule)
    partials = tuple(p for p, _ in results)
    worker_pairs = tuple(c for _, c in results)
    total = partials[0] if partials else 0
    for p in partials[1:]:
        total = total + p
    return SpiResult(total=total, partials=partials, pairs_evaluated=sum(worker_pairs),
                     depth_per_worker=_depth(n, schedule), worker_pairs=worker_pairs)


def spi_rows(objects, f: Callable, rows: range | tuple, schedule: str = "balanced"):
    """(partial, pairs) owned by outer rows [lo, hi) -- the reference's
    ``_run_outer(obj, f, range(lo, hi), schedule)`` (spi_engine.py:109-120)."""
    if schedule not in SCHEDULES:
        raise ValueError(f"schedule must be one of {SCHEDULES}, got {schedule!r}")
    lo, hi = (rows.start, rows.stop) if isinstance(rows, range) else rows
    obj = as_object_array(objects)
    if not 0 <= lo <= hi <= len(obj):
        raise ValueError(f"row range [{lo}, {hi}) outside [0, {len(obj)}]")
    ((partial, pairs),) = _run_ranges(obj, f, [(lo, hi)], schedule)
    return partial, pairs


def spi_totals_batch(objects_list, f: Callable) -> list:
    """``[spi_balanced(obj, f).total for obj in objects_list]`` in one GPU launch
    (``pc_pairs_batch``: one CTA per object array, the pairs evaluated in
    float64 with the reference's own arithmetic, so counts are exact and sums
    are float64).  Meant for many small problems (the paper's 100-1000
    vectors per execution); arrays of more than 4096 objects fall back to
    ``spi_balanced``.  Same argument checks and errors as ``spi_balanced``."""
    arrays = [as_object_array(o) for o in objects_list]
    code = _interaction_code(f) if any(len(a) >= 2 for a in arrays) else None
    out = [None] * len(arrays)
    batch = []
    for idx, obj in enumerate(arrays):
        if len(obj) < 2:
            out[idx] = 0
            continue
        xyz = _device_coords(obj)
        if xyz.dtype.kind == "f" and not np.isfinite(xyz).all():
            out[idx] = spi_balanced(obj, f).total  # raises the reference's error for this array
            continue
        batch.append((idx, xyz.astype(np.float64) if xyz.dtype != np.float64 else xyz))
    if batch:
        results = _lib.pairs_batch([np.ascontiguousarray(x) for _, x in batch], code)
        for (idx, xyz), r in zip(batch, results):
            if r.error == _lib.PC_ERR_ARG:  # too many objects for one CTA: the full path
                out[idx] = spi_balanced(arrays[idx], f).total
            elif r.error:
                raise InteractionDomainError("sphere coordinates must be finite")
            else:
                out[idx] = float(r.sum) if code == _lib.PC_COLLISION_INVSQ else int(r.count)
    return out
