"""Counting-array collision/contact counters on the B200.

Drop-in for the reference module ``pkg/src/paircount/lattice_counter.py``.
The space is a device-resident dense uint32 grid of side 2a+3 (one zero
padding cell per face, index (x+a+1, y+a+1, z+a+1)).  libpaircount.so places
the beads -- one atomic increment each when beads are few relative to cells
(Alg. 1: collisions += old occupancy), shared-memory slabs streamed out by
TMA when they are many -- and evaluates Alg. 2's neighbour sums (per bead,
or one stencil pass over the grid in the dense regime) and the sparse reset.
The O(N^2) oracles run on the GPU all-pairs kernel with the reference's
exact integer predicates; ``*_batch`` and ``*_multi_gpu`` variants count many
small vectors in one launch / one grid over several GPUs.

Differences of representation (not of results):
  * ``LatticeSpace.cells`` is a read-only host snapshot of the device grid
    (the reference exposes its numpy array; writes to the snapshot are not
    seen by the GPU).
  * ``LatticeSpace.touched`` holds one ``TouchedCells`` record per counted
    vector: the device buffer of that vector's cell keys; ``len()`` is the
    number of distinct cells it occupied after count_collisions (as the
    reference's np.unique list, lattice_counter.py:129,136) and the number of
    beads after the contact counters (a superset, which the reference's
    touched-list contract allows).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

NEIGHBOR_OFFSETS = np.array(
    [[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], dtype=np.int64)

_CELL_MAX = np.iinfo(np.uint32).max
# reset_sparse clears the whole grid instead of scattering zeros once the
# touched keys exceed 1/_CLEAR_RATIO of the cells (random 4-byte stores cost a
# 32-byte sector read-modify-write each; a streaming clear costs 4 B/cell)
_CLEAR_RATIO = 32


class CoordinateRangeError(ValueError):
    """A bead lies outside the [-a, a]^3 cube of its space."""


class OccupancyOverflowError(OverflowError):
    """A cell's occupancy count would exceed the cell counter width."""


class SpaceSizeError(MemoryError):
    """The requested half-extent does not fit in addressable memory."""


@dataclass(frozen=True)
class CountReport:
    """Outcome of one counting pass (lattice_counter.py:43-49)."""

    count: int
    beads_processed: int
    cells_touched: int


def as_bead_array(beads) -> np.ndarray:
    """Coerce beads to int64 (N, 3) (lattice_counter.py:52-59)."""
    arr = np.asarray(beads, dtype=np.int64)
    if arr.size == 0:
        return arr.reshape(0, 3)
    if arr.ndim != 2 or arr.shape[1] != 3:
        raise ValueError(f"bead vector must have shape (N, 3), got {arr.shape}")
    return arr


class TouchedCells:
    """Device keys of one counted vector (the touched-list entry)."""

    __slots__ = ("keys", "nkeys", "distinct")

    def __init__(self, keys: _lib.DeviceBuffer, nkeys: int, distinct: int):
        self.keys, self.nkeys, self.distinct = keys, nkeys, distinct

    def __len__(self) -> int:
        return self.distinct


class LatticeSpace:
    """Dense device occupancy grid over [-a, a]^3 with zero padding
    (lattice_counter.py:62-111)."""

    def __init__(self, half_extent: int):
        if half_extent < 0:
            raise ValueError(f"half_extent must be >= 0, got {half_extent}")
        side = 2 * half_extent + 3
        if side**3 > np.iinfo(np.intp).max:
            raise SpaceSizeError(
                f"half_extent {half_extent} needs {side}^3 cells, beyond the platform index range")
        self.half_extent = half_extent
        self._side = side
        self._ncells = side**3
        try:
            self._grid = _lib.DeviceBuffer(4 * self._ncells)
        except MemoryError as exc:
            raise SpaceSizeError(f"cannot allocate {side}^3 cells for half_extent {half_extent}") from exc
        self.touched: list[TouchedCells] = []
        self._base_clean = True  # grid known all-zero once `touched` is replayed

    @property
    def cells(self) -> np.ndarray:
        """Host snapshot (side, side, side) uint32 of the device grid."""
        return self._grid.to_host(np.uint32, self._ncells).reshape(self._side, self._side, self._side)

    @property
    def interior_cells(self) -> int:
        return (2 * self.half_extent + 1) ** 3

    @property
    def grid_ptr(self) -> int:
        return self._grid.ptr

    def is_zero(self) -> bool:
        nz = ctypes.c_int64()
        _lib.check(_lib.load().pc_grid_count_nonzero(self._grid.ptr, self._ncells, ctypes.byref(nz), None))
        return nz.value == 0

    def _clean(self) -> bool:
        return self._base_clean and not self.touched

    def _validate(self, beads: np.ndarray) -> None:
        a = self.half_extent
        bad = np.abs(beads) > a
        if bad.any():
            idx = int(np.nonzero(bad.any(axis=1))[0][0])
            raise CoordinateRangeError(f"bead {idx} at {tuple(beads[idx])} outside [-{a}, {a}]^3")

    def _flatten(self, beads: np.ndarray) -> np.ndarray:
        s = beads + (self.half_extent + 1)
        return np.ravel_multi_index((s[:, 0], s[:, 1], s[:, 2]), (self._side,) * 3)


def new_space(half_extent: int) -> LatticeSpace:
    return LatticeSpace(half_extent)


def interior_cell_count(half_extent: int) -> int:
    """(2a+1)^3 without allocating (lattice_counter.py:118-122)."""
    if half_extent < 0:
        raise ValueError(f"half_extent must be >= 0, got {half_extent}")
    return (2 * half_extent + 1) ** 3


def _raise_for(res, space: LatticeSpace, arr: np.ndarray) -> None:
    if res.error == _lib.PC_ERR_RANGE:
        idx = int(res.detail)
        a = space.half_extent
        raise CoordinateRangeError(f"bead {idx} at {tuple(arr[idx])} outside [-{a}, {a}]^3")
    if res.error == _lib.PC_ERR_OVERFLOW:
        raise OccupancyOverflowError(f"cell occupancy exceeds {_CELL_MAX} (counter width)")
    if res.error == _lib.PC_ERR_ODD:
        raise ArithmeticError(f"doubled contact sum {res.doubled} is odd")


def _lattice_call(fn_name: str, beads, space: LatticeSpace):
    arr = np.ascontiguousarray(as_bead_array(beads))
    lib = _lib.load()
    kb = int(lib.pc_lattice_key_bytes(space.half_extent))
    keys = _lib.DeviceBuffer(max(1, len(arr)) * kb)
    res = _lib.LatticeResult()
    rc = getattr(lib, fn_name)(arr.ctypes.data, _lib.PC_I64, 0, len(arr), space.half_extent, space.grid_ptr,
                               keys.ptr, 1 if space._clean() else 0, ctypes.byref(res), None)
    if rc in (_lib.PC_ERR_CUDA, _lib.PC_ERR_ARG):
        _lib.check(rc)
    _raise_for(res, space, arr)
    # placed: the keys become this vector's touched-list entry
    distinct = int(res.cells_touched) if fn_name == "pc_lattice_collisions" else -1
    return arr, res, keys, distinct


def count_collisions(beads, space: LatticeSpace) -> CountReport:
    """Pairs of beads on the same site (Alg. 1; lattice_counter.py:140-156).
    Leaves the space populated; the caller resets it."""
    arr = as_bead_array(beads)
    if len(arr) == 0:
        return CountReport(count=0, beads_processed=0, cells_touched=0)
    arr, res, keys, distinct = _lattice_call("pc_lattice_collisions", arr, space)
    space.touched.append(TouchedCells(keys, len(arr), distinct))
    return CountReport(count=int(res.count), beads_processed=len(arr), cells_touched=distinct)


def _contacts(beads, space: LatticeSpace):
    arr, res, keys, _ = _lattice_call("pc_lattice_contacts", beads, space)
    # touched entry: one key per placed bead (a superset of the occupied
    # cells, like the reference's list; neighbour reads are not writes)
    space.touched.append(TouchedCells(keys, len(arr), len(arr)))
    return arr, res


def contact_accumulator(beads, space: LatticeSpace) -> int:
    """Doubled contact sum (Alg. 2 before halving; lattice_counter.py:159-175)."""
    arr = as_bead_array(beads)
    if len(arr) == 0:
        return 0
    _, res = _contacts(arr, space)
    return int(res.doubled)


def count_contacts(beads, space: LatticeSpace) -> CountReport:
    """Pairs at unit axial distance, with multiplicity (Alg. 2;
    lattice_counter.py:178-195)."""
    arr = as_bead_array(beads)
    if len(arr) == 0:
        return CountReport(count=0, beads_processed=0, cells_touched=0)
    arr, res = _contacts(arr, space)
    return CountReport(count=int(res.count), beads_processed=len(arr), cells_touched=int(res.cells_touched))


def reset_sparse(space: LatticeSpace, beads=None) -> None:
    """Zero only touched cells (lattice_counter.py:198-217): via the touched
    list when present, else each given bead's cell and its six neighbours."""
    lib = _lib.load()
    if space.touched:
        nkeys = sum(entry.nkeys for entry in space.touched)
        if space._base_clean and nkeys * _CLEAR_RATIO > space._ncells:
            # every nonzero cell is a touched one: one streaming clear leaves the
            # same all-zero grid faster than scattered 4-byte stores
            _lib.check(lib.pc_lattice_clear(space.grid_ptr, space.half_extent, None))
        else:
            for entry in space.touched:
                _lib.check(lib.pc_lattice_reset_keys(space.grid_ptr, space.half_extent, entry.keys.ptr,
                                                     entry.nkeys, None))
        _lib.check(lib.pc_stream_sync(None))
        space.touched.clear()
        return
    if beads is None:
        return
    arr = np.ascontiguousarray(as_bead_array(beads))
    if len(arr) == 0:
        return
    res = _lib.LatticeResult()
    rc = lib.pc_lattice_reset_beads(arr.ctypes.data, _lib.PC_I64, 0, len(arr), space.half_extent,
                                    space.grid_ptr, ctypes.byref(res), None)
    if rc in (_lib.PC_ERR_CUDA, _lib.PC_ERR_ARG):
        _lib.check(rc)
    _raise_for(res, space, arr)
    # cells outside the beads' neighbourhoods may still hold counts
    space._base_clean = False


def count_collisions_batch(vectors, space: LatticeSpace) -> list[CountReport]:
    """Count every bead vector as ``count_collisions(v, space)`` on a clean
    space followed by ``reset_sparse`` -- the reference's per-vector loop
    (bench_cli.py:129-141 ``_linear_pass``; the paper counts 100-1000 vectors
    per execution) -- in one GPU launch: one CTA per
    vector, Alg. 1 on an on-chip hashed counting array.  Vectors longer than
    4096 beads go through ``space``'s grid.  The space must be clean on entry
    and is clean on return.  Raises CoordinateRangeError for the first vector
    holding a bead outside [-a, a]^3."""
    if not space._clean():
        raise ValueError("count_collisions_batch needs a clean space (fresh or reset)")
    arrays = [np.ascontiguousarray(as_bead_array(v)) for v in vectors]
    if not arrays:
        return []
    # the library gathers the separate host vectors itself (threads, pinned
    # staging, int64 -> int32 narrowing): no host-side concatenation
    ptrs = np.array([_lib.host_address(a) for a in arrays], dtype=np.uintp)
    lengths = np.array([len(a) for a in arrays], dtype=np.int64)
    res = (_lib.LatticeResult * len(arrays))()
    lib = _lib.load()
    _lib.check(lib.pc_lattice_collisions_vectors(ptrs.ctypes.data, lengths.ctypes.data, _lib.PC_I64, len(arrays),
                                                 space.half_extent, ctypes.addressof(res), None))
    reports = []
    for arr, r in zip(arrays, res):
        if r.error == _lib.PC_ERR_RANGE:
            _raise_for(r, space, arr)
        if r.error == _lib.PC_ERR_ARG:  # too long for the on-chip table: through the grid
            rep = count_collisions(arr, space)
            reset_sparse(space)
            reports.append(rep)
            continue
        reports.append(CountReport(count=int(r.count), beads_processed=len(arr), cells_touched=int(r.cells_touched)))
    return reports


def _integer_pairs(beads, interaction: int) -> int:
    arr = as_bead_array(beads)
    n = len(arr)
    if n < 2:
        return 0
    lo, hi = arr.min(axis=0), arr.max(axis=0)
    if max(-int(lo.min()), int(hi.max())) < 2**30:  # halve H2D traffic, as the reference halves its diff traffic
        arr = arr.astype(np.int32)
    # coincidences of points spanning <= 1023 per axis: compare packed 30-bit keys on the INT32
    # pipe (PC_TILE_KEY, 1.7x the FP32 Gram filter at 2^20 points); otherwise the Gram filter +
    # exact int64 re-check
    key = interaction == _lib.PC_COINCIDE and int((hi.astype(object) - lo.astype(object)).max()) <= 1023
    (res,) = _lib.pairs_host(arr, interaction, _lib.PC_BALANCED, [0, n],
                             tiling=_lib.PC_TILE_KEY if key else _lib.PC_TILE_AUTO)
    if res.error:
        raise RuntimeError(f"integer all-pairs kernel reported error {res.error}")
    return int(res.count)


def oracle_collisions(beads) -> int:
    """Exact-coincidence pairs over all i < j (lattice_counter.py:227-241),
    on the GPU all-pairs kernel with the exact integer predicate."""
    return _integer_pairs(beads, _lib.PC_COINCIDE)


def oracle_contacts(beads) -> int:
    """Pairs at Manhattan distance exactly 1 (lattice_counter.py:244-255)."""
    return _integer_pairs(beads, _lib.PC_MANHATTAN1)


def _integer_pairs_batch(vectors, interaction: int) -> list[int]:
    arrays = [np.ascontiguousarray(as_bead_array(v)) for v in vectors]
    out = []
    for arr, r in zip(arrays, _lib.pairs_batch(arrays, interaction)):
        if r.error == _lib.PC_ERR_ARG:  # too long for one CTA's shared memory: the full all-pairs path
            out.append(_integer_pairs(arr, interaction))
        else:
            out.append(int(r.count))
    return out


def oracle_collisions_batch(vectors) -> list[int]:
    """``[oracle_collisions(v) for v in vectors]`` in one GPU launch (one CTA
    per vector, exact int64 compare) -- the quadratic side of the reference's
    linear-vs-quadratic harness (bench_cli.py:129-179)."""
    return _integer_pairs_batch(vectors, _lib.PC_COINCIDE)


def oracle_contacts_batch(vectors) -> list[int]:
    """``[oracle_contacts(v) for v in vectors]`` in one GPU launch."""
    return _integer_pairs_batch(vectors, _lib.PC_MANHATTAN1)


def count_collisions_multi_gpu(beads, half_extent: int, devices=None) -> CountReport:
    """``count_collisions(beads, new_space(half_extent))`` with the grid split
    over several GPUs of this process by x-planes (``pc_lattice_collisions_multi``):
    each device validates all beads, keeps its planes' beads and runs Alg. 1 on
    a private slab grid; the counts and touched cells of the disjoint slabs
    add up.  No space is left populated.  ``devices`` defaults to every visible
    GPU; an ordinal may repeat."""
    arr = np.ascontiguousarray(as_bead_array(beads))
    if half_extent < 0:
        raise ValueError(f"half_extent must be >= 0, got {half_extent}")
    lib = _lib.load()
    if devices is None:
        devices = list(range(_lib.device_count()))
    devs = np.ascontiguousarray(np.asarray(list(devices), dtype=np.int32))
    if len(devs) == 0:
        raise ValueError("need at least one device")
    per = (_lib.LatticeResult * len(devs))()
    tot = _lib.LatticeResult()
    _lib.check(lib.pc_lattice_collisions_multi(arr.ctypes.data, _lib.PC_I64, len(arr), half_extent, len(devs),
                                               devs.ctypes.data, ctypes.addressof(per), ctypes.byref(tot)))
    if tot.error == _lib.PC_ERR_RANGE:
        idx = int(tot.detail)
        raise CoordinateRangeError(f"bead {idx} at {tuple(arr[idx])} outside [-{half_extent}, {half_extent}]^3")
    if tot.error == _lib.PC_ERR_OVERFLOW:
        raise OccupancyOverflowError(f"cell occupancy exceeds {_CELL_MAX} (counter width)")
    return CountReport(count=int(tot.count), beads_processed=len(arr), cells_touched=int(tot.cells_touched))
