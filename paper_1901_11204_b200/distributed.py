"""Multi-GPU all-pairs: equal-work row splits + one NCCL int64 all-reduce.

One process per GPU (torchrun).  Two ways to split the pair triangle over the
ranks, both with no exchange but the final reduction:

* ``"slabs"`` -- rank r owns a contiguous slab of outer rows.  Under the
  balanced schedule every row owns (n-1)/2 (+-1) pairs, so the reference's own
  worker partition (``_partition``, spi_engine.py:179-188) is already an
  equal-work split and the per-rank partials equal
  ``spi_parallel(workers=world).partials``.  Under the standard schedule rows
  own n-1-i pairs and the cuts r_g = n - n*sqrt(1 - g/G) equalise the work.
* ``"tiles"`` -- the whole-range call's row tiles dealt round-robin in blocks
  of four (``pc_pairs_part_*``): rank r runs blocks r, r+G, r+2G, ...  For fp32
  spheres this is the path a single GPU takes (spatially sorted points,
  PC_TILE_SORTED: the inverse-square sum with tile-local Gram chunks, the
  contact count with box pruning) split G ways; on sorted points contiguous
  slabs are uneven (some regions of the sort order hold more near-field
  chunks than others) and interleaved tiles are not.  The parts add up to the
  whole-range result; they are not reference worker partials.

``"auto"`` takes tiles for fp32 inverse-square sums and contact counts under
the balanced schedule from 2^15 points (where one GPU would sort), slabs
otherwise.

The only exchange is the reduction: every rank writes (count, float64-sum
bits, flags, pairs) into its own four slots of a zeroed int64 vector of
length 4*world and one ``all_reduce(SUM)`` leaves every slot holding its owner's
exact value on every rank (x + 0 == x).  The float64 total is then summed in
ascending rank order -- deterministic, the same fold as the reference's
ascending-worker reduction (spi_engine.py:219-223).  The flags carry each
rank's partial type (the reference returns int 0 for an empty block even
for a float interaction) and whether the rank failed, so a domain error on
one rank raises on every rank instead of leaving the others in the
collective.
"""

from __future__ import annotations

import math
from typing import Callable

import numpy as np

from .pair_schedule import row_pairs

SPLITS = ("auto", "slabs", "tiles")
_FLOAT, _FAILED = 1, 2
SORTED_MIN_N = 1 << 15  # csrc/paircount.cu kSortedMinN: whole-range fp32 sums sort from here


def row_slabs(n: int, world: int, schedule: str = "balanced") -> list[tuple[int, int]]:
    """Contiguous outer-row slabs, one per rank, of (near-)equal work."""
    if world < 1:
        raise ValueError(f"world size must be >= 1, got {world}")
    if schedule == "balanced":
        base, extra = divmod(n, world)
        out, start = [], 0
        for r in range(world):
            size = base + (1 if r < extra else 0)
            out.append((start, start + size))
            start += size
        return out
    cuts = [0] + [min(n, int(round(n - n * math.sqrt(1.0 - g / world)))) for g in range(1, world)] + [n]
    for g in range(1, len(cuts)):
        cuts[g] = max(cuts[g], cuts[g - 1])
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def pack_partial(count: int, total: float, rank: int, world: int, is_float: bool = False,
                 failed: bool = False, pairs: int = 0) -> np.ndarray:
    slots = np.zeros(4 * world, dtype=np.int64)
    slots[4 * rank] = count
    slots[4 * rank + 1] = np.array([total], dtype=np.float64).view(np.int64)[0]
    slots[4 * rank + 2] = (_FLOAT if is_float else 0) | (_FAILED if failed else 0)
    slots[4 * rank + 3] = pairs
    return slots


def unpack_partials(slots: np.ndarray, world: int):
    """(counts, float64 sums, flags, pairs) per rank from the reduced slot vector."""
    slots = np.asarray(slots, dtype=np.int64).reshape(world, 4)
    return (slots[:, 0].tolist(), slots[:, 1].copy().view(np.float64).tolist(), slots[:, 2].tolist(),
            slots[:, 3].tolist())


def allreduce_partials(count: int, total: float, group=None, device=None, is_float: bool = False,
                       failed: bool = False, pairs: int = 0):
    """The one collective: int64 all-reduce of the packed slot vector."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = torch.from_numpy(pack_partial(count, total, rank, world, is_float, failed, pairs))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return unpack_partials(t.cpu().numpy(), world)


def choose_split(obj: np.ndarray, f, schedule: str, split: str = "auto") -> str:
    """"tiles" or "slabs" for this problem (see the module docstring)."""
    from . import _lib, spi_engine

    if split not in SPLITS:
        raise ValueError(f"split must be one of {SPLITS}, got {split!r}")
    if split != "auto":
        return split
    try:
        code = spi_engine._interaction_code(f)
    except TypeError:
        return "slabs"  # the engines raise the reference's TypeError on their own
    dt = getattr(obj, "dtype", None)
    sortable = dt == np.float32 or (dt == np.float64 and code == _lib.PC_COLLISION)  # the sorted kernels' inputs
    return ("tiles" if code in (_lib.PC_COLLISION, _lib.PC_COLLISION_INVSQ) and schedule == "balanced"
            and len(obj) >= SORTED_MIN_N and sortable and obj.ndim == 2 and obj.shape[1] == 3 else "slabs")


def rank_partial(obj: np.ndarray, f, schedule: str, rank: int, world: int, split: str):
    """(partial, pairs) of this rank's share of the triangle, on the calling
    thread's current CUDA device."""
    from . import _lib, spi_engine

    n = len(obj)
    if split == "slabs":
        lo, hi = row_slabs(n, world, schedule)[rank]
        return spi_engine.spi_rows(obj, f, (lo, hi), schedule)
    if n < 2:
        return 0, 0
    code, xyz = spi_engine._prepare(obj, f, [(0, n)], schedule)
    sortable = xyz.dtype == np.float32 or (xyz.dtype == np.float64 and code == _lib.PC_COLLISION)
    tiling = _lib.PC_TILE_SORTED if (code in (_lib.PC_COLLISION, _lib.PC_COLLISION_INVSQ) and sortable
                                     and schedule == "balanced" and n >= SORTED_MIN_N) else _lib.PC_TILE_AUTO
    sched = _lib.SCHEDULE_CODES[schedule]

    def run(x):
        return [_lib.pairs_part_host(x, code, sched, 0, n, rank, world, tiling)]

    (r,) = spi_engine._resolve_domain(xyz, code, schedule, [(0, n)], run(xyz), run)
    pairs = int(r.pairs)
    partial = float(r.sum) if code == _lib.PC_COLLISION_INVSQ else int(r.count)
    return (partial if pairs else 0), pairs


def spi_distributed(objects, f, schedule: str = "balanced", group=None,
                    compute: Callable | None = None, device=None, split: str = "auto"):
    """Total of f over all pairs, the triangle split over the process group.

    ``compute(obj, f, lo, hi, schedule) -> count_or_sum`` evaluates one
    contiguous slab (``split="slabs"`` only); it defaults to the GPU kernels,
    which run on the calling thread's current CUDA device -- one process per
    GPU sets it (``torch.cuda.set_device(local_rank)`` or ``PAIRCOUNT_DEVICE``).
    Returns (total, per-rank partials, per-rank pair counts)."""
    import torch.distributed as dist

    from . import spi_engine

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obj = spi_engine.as_object_array(objects)
    n = len(obj)
    if compute is not None:
        split = "slabs"
    split = choose_split(obj, f, schedule, split)
    err, part, pairs = None, 0, 0
    try:
        if compute is not None:
            lo, hi = row_slabs(n, world, schedule)[rank]
            part, pairs = compute(obj, f, lo, hi, schedule), row_pairs(n, lo, hi, schedule)
        else:
            part, pairs = rank_partial(obj, f, schedule, rank, world, split)
    except Exception as exc:  # noqa: BLE001 -- re-raised after the collective, on every rank
        err = exc
    is_float = isinstance(part, float)
    counts, sums, flags, pairs_per_rank = allreduce_partials(
        0 if is_float else int(part), float(part) if is_float else 0.0, group, device, is_float=is_float,
        failed=err is not None, pairs=int(pairs))
    if err is not None:
        raise err
    failed = [r for r, fl in enumerate(flags) if fl & _FAILED]
    if failed:
        raise RuntimeError(f"spi_distributed: rank(s) {failed} failed; see their error")
    partials = tuple(s if fl & _FLOAT else c for c, s, fl in zip(counts, sums, flags))
    total = partials[0]
    for p in partials[1:]:
        total = total + p
    return total, partials, tuple(pairs_per_rank)


def spi_multi_gpu(objects, f, schedule: str = "balanced", devices=None):
    """Total of f over all pairs with the rows split over several GPUs of ONE
    process (``pc_pairs_multi``: a host thread per device, partials combined
    in ascending device order).  ``devices`` defaults to every visible GPU;
    an ordinal may repeat.  Returns (total, per-device partials, per-device
    pair counts), like ``spi_distributed``."""
    from . import _lib, spi_engine

    if schedule not in spi_engine.SCHEDULES:
        raise ValueError(f"schedule must be one of {spi_engine.SCHEDULES}, got {schedule!r}")
    obj = spi_engine.as_object_array(objects)
    n = len(obj)
    if devices is None:
        devices = list(range(_lib.device_count()))
    devices = [int(d) for d in devices]
    if not devices:
        raise ValueError("need at least one device")
    slabs = row_slabs(n, len(devices), schedule)
    pairs = tuple(row_pairs(n, a, b, schedule) for a, b in slabs)
    if n < 2:
        return 0, tuple(0 for _ in devices), pairs
    code, xyz = spi_engine._prepare(obj, f, slabs, schedule)
    bounds = [slabs[0][0]] + [b for _, b in slabs]
    sched = _lib.SCHEDULE_CODES[schedule]

    def run(x):
        return _lib.pairs_multi(x, code, sched, devices, bounds)[0]

    per = spi_engine._resolve_domain(xyz, code, schedule, slabs, run(xyz), run)
    partials = tuple(spi_engine._partial_of(r, code, n, a, b, schedule)[0] for (a, b), r in zip(slabs, per))
    total = partials[0]
    for p in partials[1:]:
        total = total + p
    return total, partials, pairs
