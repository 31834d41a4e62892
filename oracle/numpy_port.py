"""numpy restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Each function restates one reference function (``/root/reference/pkg/src/
paircount``; file:line in its docstring) with the same numpy arithmetic, so
results are bit-identical for integer outputs and ulp-identical for the
float64 per-row sums.  Pinned against the reference's outputs in
``tests/golden/golden_small.json`` / ``golden_configs.json``.
"""

from __future__ import annotations

import numpy as np

STANDARD, BALANCED = "standard", "balanced"


# ---------------------------------------------------------------- schedule --

def steps_for(n: int, i: int) -> int:
    """Inner steps of outer index i (pair_schedule.py:49-59)."""
    if n % 2:
        return (n - 1) // 2
    return n // 2 if i < n // 2 else n // 2 - 1


def depth(n: int, schedule: str) -> int:
    """Depth metric (spi_engine.py:139-144)."""
    if n <= 1:
        return 0
    return n - 1 if schedule == STANDARD else n // 2


def partners(n: int, i: int, schedule: str) -> np.ndarray:
    """Partner indices of row i (spi_engine.py:102-106)."""
    if schedule == STANDARD:
        return np.arange(i + 1, n, dtype=np.int64)
    return (i + np.arange(1, steps_for(n, i) + 1, dtype=np.int64)) % n


def row_pairs(n: int, lo: int, hi: int, schedule: str) -> int:
    """Pairs owned by rows [lo, hi): closed form of the reference's pair count
    (spi_engine.py:113-120)."""
    if hi <= lo:
        return 0
    if schedule == STANDARD:
        return sum(n - 1 - i for i in (lo, hi - 1)) * (hi - lo) // 2
    if n % 2:
        return (hi - lo) * ((n - 1) // 2)
    h = n // 2
    first = max(0, min(hi, h) - lo)
    return first * h + (hi - lo - first) * (h - 1)


def partition(n: int, workers: int) -> list[tuple[int, int]]:
    """Contiguous near-equal outer blocks (spi_engine.py:179-188)."""
    base, extra = divmod(n, workers)
    out, start = [], 0
    for w in range(workers):
        size = base + (w < extra)
        out.append((start, start + size))
        start += size
    return out


# ----------------------------------------------------------- interactions --

def collision_indicator(a, b):
    """1 iff float64 ((a-b)**2).sum(-1) < 1.0 (spi_engine.py:62-73)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d2 = ((a - b) ** 2).sum(axis=-1)
    return (d2 < 1.0).astype(np.int64)


def inverse_square(a, b):
    """Softened inverse square 1/(1+|a-b|^2) (test_spi_engine.py:108-111)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return 1.0 / (1.0 + ((a - b) ** 2).sum(axis=-1))


def run_rows(obj: np.ndarray, f, lo: int, hi: int, schedule: str):
    """Partial over outer rows [lo, hi) (spi_engine.py:109-120 with the
    batch evaluation of spi_engine.py:84-99): per row a numpy sum of f over
    its partner batch, accumulated as a Python int/float in row order."""
    n = len(obj)
    partial, pairs = 0, 0
    for i in range(lo, hi):
        js = partners(n, i, schedule)
        if len(js) == 0:
            continue
        vals = np.asarray(f(obj[i], obj[js]))
        s = vals.sum()
        partial = partial + (int(s) if np.issubdtype(vals.dtype, np.integer) else float(s))
        pairs += len(js)
    return partial, pairs


def spi_partials(obj: np.ndarray, f, workers: int, schedule: str):
    """Per-worker partials in ascending worker order (spi_engine.py:191-230)."""
    results = [run_rows(obj, f, lo, hi, schedule) for lo, hi in partition(len(obj), workers)]
    partials = tuple(p for p, _ in results)
    total = partials[0] if partials else 0
    for p in partials[1:]:
        total = total + p
    return total, partials, tuple(c for _, c in results)


# ----------------------------------------------------------------- lattice --

def _small_ints(beads) -> np.ndarray:
    """int32 downcast when |c| < 2^30 (lattice_counter.py:220-224)."""
    arr = np.asarray(beads, dtype=np.int64).reshape(-1, 3)
    if len(arr) and np.abs(arr).max() < 2**30:
        arr = arr.astype(np.int32)
    return arr


def oracle_collisions(beads) -> int:
    """Full N x N coincidence matrix, (sum - n) // 2 (lattice_counter.py:227-241)."""
    arr = _small_ints(beads)
    n = len(arr)
    if n < 2:
        return 0
    same = np.ones((n, n), dtype=bool)
    for k in range(3):
        same &= arr[:, k][:, None] == arr[:, k][None, :]
    return (int(same.sum()) - n) // 2


def oracle_contacts(beads) -> int:
    """Pairs at Manhattan distance exactly 1 (lattice_counter.py:244-255)."""
    arr = _small_ints(beads)
    n = len(arr)
    if n < 2:
        return 0
    man = np.zeros((n, n), dtype=arr.dtype)
    for k in range(3):
        man += np.abs(arr[:, k][:, None] - arr[:, k][None, :])
    return int((man == 1).sum()) // 2


def count_collisions(beads, half_extent: int):
    """Alg. 1 counting array (lattice_counter.py:125-156), evaluated through
    the per-cell occupancy: count = sum_beads (occ - 1) // 2, cells_touched =
    number of distinct occupied cells.  Returns (count, n, cells_touched)."""
    arr = np.asarray(beads, dtype=np.int64).reshape(-1, 3)
    if len(arr) == 0:
        return 0, 0, 0
    bad = np.abs(arr) > half_extent
    if bad.any():
        raise ValueError(f"bead {int(np.nonzero(bad.any(axis=1))[0][0])} out of range")
    side = 2 * half_extent + 3
    shifted = arr + (half_extent + 1)
    flat = (shifted[:, 0] * side + shifted[:, 1]) * side + shifted[:, 2]
    _, counts = np.unique(flat, return_counts=True)
    counts = counts.astype(np.int64)
    return int((counts * (counts - 1) // 2).sum()), len(arr), len(counts)


def new_dense_space(half_extent: int) -> np.ndarray:
    """Dense uint32 grid of side 2a+3 (LatticeSpace.__init__, lattice_counter.py:70-88)."""
    side = 2 * half_extent + 3
    return np.zeros((side, side, side), dtype=np.uint32)


def count_collisions_dense(beads, cells: np.ndarray, half_extent: int):
    """Alg. 1 exactly as the reference runs it on its dense numpy grid:
    validate, flatten, np.unique, np.add.at, overflow check, occ gather,
    sum(occ-1)//2, then reset_sparse through the unique cells
    (lattice_counter.py:98-156, 198-210).  Used as the timed CPU baseline of
    the counting-array rows.  Returns (count, n, cells_touched)."""
    arr = np.asarray(beads, dtype=np.int64).reshape(-1, 3)
    if len(arr) == 0:
        return 0, 0, 0
    if (np.abs(arr) > half_extent).any():
        raise ValueError("bead out of range")
    shifted = arr + (half_extent + 1)
    flat = np.ravel_multi_index((shifted[:, 0], shifted[:, 1], shifted[:, 2]), cells.shape)
    occupied = np.unique(flat)
    flat_cells = cells.reshape(-1)
    np.add.at(flat_cells, flat, 1)
    if flat_cells[occupied].max(initial=0) >= np.iinfo(np.uint32).max:
        raise OverflowError("cell occupancy overflow")
    occ = flat_cells[flat].astype(np.int64)
    count = int((occ - 1).sum()) // 2
    flat_cells[occupied] = 0
    return count, len(arr), len(occupied)


def count_contacts(beads, half_extent: int):
    """Alg. 2 (lattice_counter.py:159-195): doubled neighbour-occupancy sum
    over the six axial offsets, halved; cells_touched counts the distinct
    cells among each bead and its six neighbours."""
    arr = np.asarray(beads, dtype=np.int64).reshape(-1, 3)
    if len(arr) == 0:
        return 0, 0, 0
    side = 2 * half_extent + 3

    def flat(a):
        s = a + (half_extent + 1)
        return (s[:, 0] * side + s[:, 1]) * side + s[:, 2]

    keys, counts = np.unique(flat(arr), return_counts=True)
    offsets = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], dtype=np.int64)
    doubled = 0
    reads = [flat(arr)]
    for off in offsets:
        nk = flat(arr + off)
        reads.append(nk)
        pos = np.searchsorted(keys, nk)
        pos = np.minimum(pos, len(keys) - 1)
        hit = keys[pos] == nk
        doubled += int(counts[pos][hit].sum())
    return doubled // 2, len(arr), len(np.unique(np.concatenate(reads)))
