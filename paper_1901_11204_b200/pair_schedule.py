"""Balanced circular pair schedule (Alg. 4) -- host-side closed forms.

Same API as the reference module (``pkg/src/paircount/pair_schedule.py``).
These functions DEFINE the row ownership the GPU kernels implement in
closed form (``steps_for_dev`` and the ownership test in
``csrc/paircount.cu``); they are index arithmetic, not the counting hot path.
``pairs_array`` materialises O(n^2) indices and, as in the reference, exists
for tests and small n only.

Row i evaluates partner (i + s) mod n for s = 1 .. steps_for(n, i):
(n-1)/2 steps for odd n; for even n, n/2 steps for i < n/2 and n/2 - 1 for
the rest (the even-N rule).
"""

from __future__ import annotations

from typing import Iterator

import numpy as np


def _require_n(n: int) -> None:
    if n < 1:
        raise ValueError(f"need at least one index, got n={n}")


def _require_index(n: int, i: int) -> None:
    if i < 0 or i >= n:
        raise IndexError(f"index {i} out of range for n={n}")


def _require_step(s: int) -> None:
    if s < 1:
        raise ValueError(f"steps start at 1, got s={s}")


def reach(n: int, i: int, s: int) -> int:
    """Partner that i evaluates at step s: (i + s) mod n (pair_schedule.py:31-37)."""
    _require_n(n)
    _require_index(n, i)
    _require_step(s)
    return (i + s) % n


def reached(n: int, i: int, s: int) -> int:
    """Index that evaluates i at step s: (i - s) mod n (pair_schedule.py:40-46)."""
    _require_n(n)
    _require_index(n, i)
    _require_step(s)
    return (i - s) % n


def steps_for(n: int, i: int) -> int:
    """Inner steps of outer index i (pair_schedule.py:49-59)."""
    _require_n(n)
    _require_index(n, i)
    half = n // 2
    if n % 2:
        return half
    return half if i < half else half - 1


def step_counts(n: int) -> np.ndarray:
    """steps_for over all indices, int64 (pair_schedule.py:62-69)."""
    _require_n(n)
    half = n // 2
    if n % 2:
        return np.full(n, half, dtype=np.int64)
    counts = np.full(n, half - 1, dtype=np.int64)
    counts[:half] = half
    return counts


def total_pairs(n: int) -> int:
    return n * (n - 1) // 2


def pairs(n: int) -> Iterator[tuple[int, int]]:
    """Oriented pairs (i, (i+s) mod n) in schedule order (pair_schedule.py:76-85)."""
    _require_n(n)
    for i in range(n):
        for s in range(1, steps_for(n, i) + 1):
            yield i, (i + s) % n


def _rows_block(lo: int, hi: int, steps: int, n: int) -> np.ndarray:
    """(count*steps, 2) int32 oriented pairs for rows [lo, hi), `steps` each."""
    rows = np.arange(lo, hi, dtype=np.int32)
    cols = rows[:, None] + np.arange(1, steps + 1, dtype=np.int32)[None, :]
    cols -= n * (cols >= n)
    out = np.empty((2, (hi - lo) * steps), dtype=np.int32)
    out[0] = np.repeat(rows, steps)
    out[1] = cols.reshape(-1)
    return out


def pairs_array(n: int) -> np.ndarray:
    """All oriented pairs as an (n(n-1)/2, 2) int32 array in schedule order,
    each column contiguous (pair_schedule.py:101-114)."""
    _require_n(n)
    if n < 2:
        return np.empty((0, 2), dtype=np.int32)
    half = n // 2
    if n % 2:
        return _rows_block(0, n, half, n).T
    both = np.concatenate([_rows_block(0, half, half, n), _rows_block(half, n, half - 1, n)], axis=1)
    return both.T


def first_violation_step(n: int) -> int:
    """(n+1)/2: first step at which the odd-n ring would repeat a pair
    (pair_schedule.py:117-123; Eq. (3))."""
    if n < 3 or n % 2 == 0:
        raise ValueError(f"defined for odd n >= 3, got n={n}")
    return (n + 1) // 2


# --- row ownership helpers used by the engine and the distributed slabs ----

def row_pairs(n: int, lo: int, hi: int, schedule: str) -> int:
    """Pairs owned by outer rows [lo, hi) under `schedule` (closed form)."""
    if hi <= lo:
        return 0
    if schedule == "standard":
        return ((n - 1 - lo) + (n - 1 - (hi - 1))) * (hi - lo) // 2
    half = n // 2
    if n % 2:
        return (hi - lo) * half
    first = max(0, min(hi, half) - lo)
    return first * half + (hi - lo - first) * (half - 1)
