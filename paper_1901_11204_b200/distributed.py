"""Multi-GPU all-pairs: equal-work row slabs + one NCCL int64 all-reduce.

One process per GPU (torchrun).  Rank r owns a contiguous slab of outer
rows; under the balanced schedule every row owns (n-1)/2 (+-1) pairs, so the
reference's own worker partition (``_partition``, spi_engine.py:179-188) is
already an equal-work split and the per-rank partials equal
``spi_parallel(workers=world).partials``.  Under the standard schedule rows
own n-1-i pairs and the cuts r_g = n - n*sqrt(1 - g/G) equalise the work.

The only exchange is the reduction of the partials: every rank writes its
(count, float64-sum bits) into its own two slots of a zeroed int64 vector of
length 2*world and one ``all_reduce(SUM)`` leaves every slot holding its
owner's exact value on every rank (x + 0 == x), so the float64 total is then
summed in ascending rank order -- deterministic and identical to the
reference's ascending-worker reduction (spi_engine.py:219-223).
"""

from __future__ import annotations

import math
from typing import Callable

import numpy as np

from .pair_schedule import row_pairs


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


def pack_partial(count: int, total: float, rank: int, world: int) -> np.ndarray:
    slots = np.zeros(2 * world, dtype=np.int64)
    slots[2 * rank] = count
    slots[2 * rank + 1] = np.array([total], dtype=np.float64).view(np.int64)[0]
    return slots


def unpack_partials(slots: np.ndarray, world: int):
    """(counts, float64 sums) per rank from the reduced slot vector."""
    slots = np.asarray(slots, dtype=np.int64).reshape(world, 2)
    return slots[:, 0].tolist(), slots[:, 1].copy().view(np.float64).tolist()


def allreduce_partials(count: int, total: float, group=None, device=None):
    """The one collective: int64 all-reduce of the packed slot vector."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = torch.from_numpy(pack_partial(count, total, rank, world))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return unpack_partials(t.cpu().numpy(), world)


def spi_distributed(objects, f, schedule: str = "balanced", group=None,
                    compute: Callable | None = None, device=None):
    """Total of f over all pairs, rows sharded over the process group.

    ``compute(obj, f, lo, hi, schedule) -> (count_or_sum)`` evaluates one
    slab; it defaults to the GPU kernels (``spi_engine.spi_rows``), which run
    on the calling thread's current CUDA device -- one process per GPU sets it
    (``torch.cuda.set_device(local_rank)`` or ``PAIRCOUNT_DEVICE``).  Returns
    (total, per-rank partials, per-rank pair counts)."""
    import torch.distributed as dist

    from . import spi_engine

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obj = spi_engine.as_object_array(objects)
    n = len(obj)
    lo, hi = row_slabs(n, world, schedule)[rank]
    if compute is None:
        part, _ = spi_engine.spi_rows(obj, f, (lo, hi), schedule)
    else:
        part = compute(obj, f, lo, hi, schedule)
    is_float = isinstance(part, float)
    counts, sums = allreduce_partials(0 if is_float else int(part), float(part) if is_float else 0.0,
                                      group, device)
    partials = tuple(sums) if is_float else tuple(counts)
    total = partials[0]
    for p in partials[1:]:
        total = total + p
    pairs = tuple(row_pairs(n, a, b, schedule) for a, b in row_slabs(n, world, schedule))
    return total, partials, pairs


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
        devices = list(range(int(_lib.load().pc_device_count())))
    devices = [int(d) for d in devices]
    if not devices:
        raise ValueError("need at least one device")
    slabs = row_slabs(n, len(devices), schedule)
    pairs = tuple(row_pairs(n, a, b, schedule) for a, b in slabs)
    if n < 2:
        return 0, tuple(0 for _ in devices), pairs
    code, xyz = spi_engine._prepare(obj, f, slabs, schedule)
    bounds = [slabs[0][0]] + [b for _, b in slabs]
    per, _ = _lib.pairs_multi(xyz, code, _lib.SCHEDULE_CODES[schedule], devices, bounds)
    partials = tuple(spi_engine._partial_of(r, code, n, a, b, schedule)[0] for (a, b), r in zip(slabs, per))
    total = partials[0]
    for p in partials[1:]:
        total = total + p
    return total, partials, pairs
