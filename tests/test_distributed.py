"""N>1 host path on CPU: world_size-2 gloo process group, slab split and the
single int64 all-reduce of partials.  The per-slab compute is injected (the
pinned C oracle), so this runs without a GPU; the GPU path differs only in
the compute callback."""

from __future__ import annotations

import functools
import operator
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_11204_b200 import distributed as D
from paper_1901_11204_b200.pair_schedule import row_pairs


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_compute(obj, f, lo, hi, schedule):
    from oracle import c_oracle

    c, s, _ = c_oracle.rows(obj, lo, hi, schedule)
    return c if f == "count" else s


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1901_11204_b200 import generators as gen

        objs = gen.random_spheres(3001, 14.0, 7).astype(np.float32)
        out = {}
        for sched in ("balanced", "standard"):
            out[sched] = (D.spi_distributed(objs, "count", sched, compute=_oracle_compute),
                          D.spi_distributed(objs, "sum", sched, compute=_oracle_compute))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_single_process():
    from oracle import c_oracle
    from paper_1901_11204_b200 import generators as gen

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    objs = gen.random_spheres(3001, 14.0, 7).astype(np.float32)
    n = len(objs)
    for sched in ("balanced", "standard"):
        want_c, want_s, _ = c_oracle.rows(objs, 0, n, sched)
        for rank in range(world):
            (tc, pc_, pairs), (ts, ps_, _) = results[rank][sched]
            assert tc == want_c
            assert ts == pytest.approx(want_s, rel=1e-12)
            assert sum(pairs) == n * (n - 1) // 2
            # every rank sees every partial, bit-identical
            assert (pc_, ps_) == (results[0][sched][0][1], results[0][sched][1][1])


def test_slabs_cover_and_balance():
    for n in (1, 2, 7, 1000, 2**20):
        for world in (1, 2, 4, 8):
            for sched in ("balanced", "standard"):
                slabs = D.row_slabs(n, world, sched)
                assert slabs[0][0] == 0 and slabs[-1][1] == n
                assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))
                if n >= 1000:
                    work = [row_pairs(n, a, b, sched) for a, b in slabs]
                    assert max(work) <= 1.01 * min(work) + n


def test_pack_roundtrip():
    s = D.pack_partial(12345, 0.1 + 0.2, 1, 3, is_float=True, pairs=77)
    counts, sums, flags, pairs = D.unpack_partials(s, 3)
    assert counts == [0, 12345, 0] and sums[1] == 0.1 + 0.2 and sums[0] == 0.0
    assert flags == [0, 1, 0] and pairs == [0, 77, 0]


def _ref_compute(obj, f, lo, hi, schedule):
    """The reference's _run_outer typing (spi_engine.py:109-120): an empty block is int 0."""
    from oracle import c_oracle

    if lo == hi:
        return 0
    c, s, _ = c_oracle.rows(obj, lo, hi, schedule)
    return c if f == "count" else s


def _empty_rank_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        objs = np.array([[0.0, 0.0, 0.0], [0.5, 0.0, 0.0]], dtype=np.float64)
        q.put((rank, D.spi_distributed(objs, "sum", "balanced", compute=_ref_compute)))
    finally:
        dist.destroy_process_group()


def test_empty_rank_float_sum_same_on_every_rank():
    """world 3, n = 2: one rank owns no rows and returns int 0 (as the
    reference's empty worker does); every rank still returns the float total
    (the partial type now travels with the partial)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_empty_rank_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = 1.0 / (1.0 + 0.25)
    for rank in range(world):
        total, partials, pairs = results[rank]
        assert total == want and isinstance(total, float)
        assert sum(pairs) == 1
        assert 0 in partials and any(isinstance(p, float) for p in partials)


def _gpu_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1901_11204_b200 import generators as gen
        from paper_1901_11204_b200 import spi_engine as se

        objs = gen.random_spheres(50_001, 30.0, 3).astype(np.float32)
        out = {}
        for sched in ("balanced", "standard"):
            out[sched] = (D.spi_distributed(objs, se.collision_indicator, sched, split="slabs"),
                          D.spi_distributed(objs, se.inverse_square, sched),
                          D.spi_distributed(objs, se.collision_indicator, sched))  # auto: tiles when balanced
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_real_kernels_gloo():
    """The N>1 path with the real kernels: 2 processes (gloo) share cuda:0, each
    runs its row slab; the partials meet in the one all-reduce.  (Kernels of
    different ranks never wait on each other, so sharing a GPU is safe.)"""
    from oracle import c_oracle
    from paper_1901_11204_b200 import generators as gen

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    objs = gen.random_spheres(50_001, 30.0, 3).astype(np.float32)
    for sched in ("balanced", "standard"):
        want_c, want_s, _ = c_oracle.rows(objs, 0, len(objs), sched)
        (tc, parts, pairs), (ts, _, _), (ta, aparts, apairs) = results[0][sched]
        assert tc == want_c and ts == pytest.approx(want_s, rel=1e-5) and ta == want_c
        assert sum(apairs) == len(objs) * (len(objs) - 1) // 2
        for (lo, hi), part in zip(D.row_slabs(len(objs), world, sched), parts):
            assert part == c_oracle.rows(objs, lo, hi, sched)[0]  # slabs: the reference workers' partials
        assert results[1][sched][0] == results[0][sched][0] and results[1][sched][2] == results[0][sched][2]


@pytest.mark.gpu
def test_single_process_multi_gpu_entry():
    """pc_pairs_multi (SURVEY.md §8(b) pc_multi_pairs): slabs on a device list,
    partials combined host-side in device order.  The box has one GPU, so the
    list repeats ordinal 0 -- the slabs are independent, nothing waits."""
    from oracle import c_oracle
    from paper_1901_11204_b200 import _lib
    from paper_1901_11204_b200 import generators as gen
    from paper_1901_11204_b200 import spi_engine as se

    objs = gen.random_spheres(30_001, 24.0, 8).astype(np.float32)
    n = len(objs)
    for sched in ("balanced", "standard"):
        want_c, want_s, _ = c_oracle.rows(objs, 0, n, sched)
        for devs in ([0], [0, 0], [0, 0, 0, 0]):
            tc, parts, pairs = D.spi_multi_gpu(objs, se.collision_indicator, sched, devs)
            assert tc == want_c and sum(pairs) == n * (n - 1) // 2
            for (lo, hi), part in zip(D.row_slabs(n, len(devs), sched), parts):
                assert part == c_oracle.rows(objs, lo, hi, sched)[0]
            ts, sparts, _ = D.spi_multi_gpu(objs, se.inverse_square, sched, devs)
            assert ts == pytest.approx(want_s, rel=1e-5)
            assert ts == functools.reduce(operator.add, sparts)  # left fold, as spi_engine.py:221-223
        if sched == "balanced":  # equal slabs == the reference's worker partition
            assert parts == se.spi_parallel(objs, se.collision_indicator, 4, "balanced").partials
    with pytest.raises(ValueError):
        _lib.pairs_multi(objs, _lib.PC_COLLISION, _lib.PC_BALANCED, [0, 99], [0, 5, n])
