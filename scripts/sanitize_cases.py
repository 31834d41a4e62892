"""Memory-safety cases: every path with asynchronous on-chip hand-offs, once.

compute-sanitizer is closed on this GPU pool ("runs under it have left GPUs
needing a reset"; profiles/r2_sanitizer.md), so the evidence is built from:
  * the bounds-checked build (``python -m paper_1901_11204_b200.build
    --checked``: PC_CHECK traps on every computed global index / claim slot);
  * poisoned scratch (PAIRCOUNT_POISON=<byte> fills the library's scratch
    before each call): results must not depend on the poison byte;
  * canaries after caller-owned device buffers (workspace, grid, keys): bytes
    past the end must be untouched;
  * every result checked against the C oracle.
``scripts/run_sanitize.sh`` runs this file three times (poison 0x00, 0xA5,
0xFF) under the checked build and diffs the JSON digests.

    PAIRCOUNT_LIB=build/checked/libpaircount.so PAIRCOUNT_POISON=0xA5 python scripts/sanitize_cases.py

Cases (sizes the checked build finishes in seconds):
  * sorted sum (Morton sort, TMA bulk staging on mbarriers, tile-local Gram)
  * FFMA2 Gram count, FLAT (claims) and PER_ROW_TILE (naive), standard schedule
  * tensor-core count (tcgen05 alloc / MMA / commit / TMEM drain, candidate queues)
  * compensated float64 sum and the integer predicates
  * counting array, dense regime (key partition + shared-memory slabs + TMA
    bulk stores) and sparse regime, Alg. 2, reset
  * the batch entry points (counting array and all-pairs)
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1901_11204_b200 as pc  # noqa: E402
from oracle import c_oracle  # noqa: E402
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402


def spheres(n, seed, f32=True):
    x = gen.random_spheres(n, gen.contact_box_edge(n), seed)
    return x.astype(np.float32) if f32 else x


DIGEST = {}


def check_pairs(tag, x, interaction, sched, tiling, lo=0, hi=None):
    hi = len(x) if hi is None else hi
    (r,) = _lib.pairs_host(x, interaction, _lib.SCHEDULE_CODES[sched], [lo, hi], tiling=tiling)
    c, s, p = c_oracle.rows(x, lo, hi, sched)
    assert r.error == 0 and r.count == c and r.pairs == p, (tag, r.count, c, r.pairs, p)
    if interaction == _lib.PC_COLLISION_INVSQ:
        assert abs(r.sum - s) <= 1e-6 * s, (tag, r.sum, s)
    DIGEST[tag] = [int(r.count), float(r.sum).hex(), int(r.exact_checks)]
    print(f"ok {tag}: count {r.count}", flush=True)


def canary_cases():
    """Caller-owned device buffers with 1 MiB canaries behind them: the device-pointer
    entries (pc_pairs_async / pc_pairs_part_async / pc_lattice_collisions) must write
    nothing past the sizes they ask for."""
    import ctypes

    import torch

    canary = 1 << 20
    pat = 0x5A

    def guarded(nbytes):
        buf = torch.full((nbytes + canary,), pat, dtype=torch.uint8, device="cuda")
        return buf

    def intact(buf, nbytes, what):
        tail = buf[nbytes:]
        assert bool((tail == pat).all()), f"{what}: {int((tail != pat).sum())} canary bytes overwritten"

    st = torch.cuda.current_stream()
    for n, inter, tiling in ((40001, _lib.PC_COLLISION_INVSQ, _lib.PC_TILE_AUTO),
                             (40001, _lib.PC_COLLISION, _lib.PC_TILE_FLAT),
                             (40000, _lib.PC_COLLISION, _lib.PC_TILE_TC),
                             (9000, _lib.PC_COLLISION_INVSQ, _lib.PC_TILE_PER_ROW_TILE)):
        x = spheres(n, 21)
        d = torch.from_numpy(x).cuda()
        wsb = _lib.workspace_bytes(n)
        ws = guarded(wsb)
        res = guarded(40)
        _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, inter, _lib.PC_BALANCED, np.array([0, n]), ws.data_ptr(),
                         wsb, res.data_ptr(), st.cuda_stream, tiling)
        torch.cuda.synchronize()
        intact(ws, wsb, f"workspace n={n} tiling={tiling}")
        intact(res, 40, "result record")
        for k in range(3):
            _lib.pairs_part_async(d.data_ptr(), _lib.PC_F32, n, inter, _lib.PC_BALANCED, 0, n, k, 3, ws.data_ptr(),
                                  wsb, res.data_ptr(), st.cuda_stream,
                                  tiling if tiling != _lib.PC_TILE_TC else _lib.PC_TILE_FLAT)
        torch.cuda.synchronize()
        intact(ws, wsb, f"workspace parts n={n}")
    lib = _lib.load()
    for a, nb in ((64, 2**21), (40, 3000)):  # dense (slab) and sparse regimes
        beads = gen._rng(31, 5).integers(-a, a + 1, size=(nb, 3), dtype=np.int64).astype(np.int32)
        db = torch.from_numpy(beads).cuda()
        cells = int(lib.pc_lattice_grid_cells(a))
        grid = guarded(cells * 4)
        grid[: cells * 4].zero_()
        keys = guarded(nb * 4)
        r = _lib.LatticeResult()
        _lib.check(lib.pc_lattice_collisions(db.data_ptr(), _lib.PC_I32, 1, nb, a, grid.data_ptr(), keys.data_ptr(), 1,
                                             ctypes.byref(r), ctypes.c_void_p(st.cuda_stream)))
        torch.cuda.synchronize()
        intact(grid, cells * 4, f"grid a={a}")
        intact(keys, nb * 4, f"keys a={a}")
        _, counts = np.unique(beads, axis=0, return_counts=True)
        assert int(r.count) == int((counts * (counts - 1) // 2).sum()) and int(r.cells_touched) == len(counts)
        DIGEST[f"canary lattice a={a}"] = [int(r.count), int(r.cells_touched)]
    print("ok canaries: workspace, result, grid and keys tails untouched", flush=True)


def main():
    t0 = time.time()
    x40 = spheres(40001, 3)
    check_pairs("sorted sum n=40001", x40, _lib.PC_COLLISION_INVSQ, "balanced", _lib.PC_TILE_AUTO)
    # PC_TILE_SORTED ranges index the sorted order: three slabs add up to the whole range
    slabs = [_lib.pairs_host(x40, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, b, tiling=_lib.PC_TILE_SORTED)[0]
             for b in ([0, 9000], [9000, 27000], [27000, 40001])]
    c, s, p = c_oracle.rows(x40, 0, 40001, "balanced")
    assert sum(r.count for r in slabs) == c and sum(r.pairs for r in slabs) == p
    assert abs(sum(r.sum for r in slabs) - s) <= 1e-6 * s
    DIGEST["sorted slabs n=40001"] = [[int(r.count), float(r.sum).hex()] for r in slabs]
    print("ok sorted slabs n=40001", flush=True)
    check_pairs("direct sum FLAT n=40001", x40, _lib.PC_COLLISION_INVSQ, "balanced", _lib.PC_TILE_FLAT)
    check_pairs("gram count FLAT n=40001", x40, _lib.PC_COLLISION, "balanced", _lib.PC_TILE_FLAT)
    x20 = spheres(20001, 4)
    check_pairs("gram count naive n=20001", x20, _lib.PC_COLLISION, "standard", _lib.PC_TILE_PER_ROW_TILE)
    check_pairs("direct sum naive n=20001", x20, _lib.PC_COLLISION_INVSQ, "standard", _lib.PC_TILE_PER_ROW_TILE)
    for n in (4097, 40000):
        check_pairs(f"tensor-core count n={n}", spheres(n, 5), _lib.PC_COLLISION, "balanced", _lib.PC_TILE_TC)
    check_pairs("tensor-core count rows n=40000", spheres(40000, 5), _lib.PC_COLLISION, "balanced",
                _lib.PC_TILE_TC, 1000, 21003)
    x64 = spheres(5000, 6, f32=False) + 1e4
    check_pairs("compensated f64 sum n=5000", x64, _lib.PC_COLLISION_INVSQ, "balanced", _lib.PC_TILE_AUTO)
    beads, ext = gen.random_chain(20000, 7)
    col, con = c_oracle.int_pairs(beads)
    assert pc.oracle_collisions(beads) == col and pc.oracle_contacts(beads) == con
    print(f"ok integer predicates n=20000: {col} / {con}", flush=True)

    # counting array: dense regime (2^21 beads on a = 64: 131^3 = 2.25M cells) and sparse
    a = 64
    dense = gen._rng(9, 5).integers(-a, a + 1, size=(2**21, 3), dtype=np.int64)
    space = pc.new_space(a)
    got = pc.count_collisions(dense, space)
    pc.reset_sparse(space)
    assert space.is_zero()
    got_c = pc.count_contacts(dense, space)
    pc.reset_sparse(space)
    assert space.is_zero()
    _, counts = np.unique(dense, axis=0, return_counts=True)
    want_col = int((counts * (counts - 1) // 2).sum())
    assert got.count == want_col and got.cells_touched == len(counts), (got, want_col, len(counts))
    print(f"ok counting array dense 2^21 beads a=64: {got.count} collisions, {got.cells_touched} cells; "
          f"contacts {got_c.count}", flush=True)
    sp2 = pc.new_space(ext)
    assert pc.count_collisions(beads, sp2).count == col
    pc.reset_sparse(sp2)
    assert sp2.is_zero()
    print("ok counting array sparse", flush=True)

    # batch entry points
    chains = [gen.random_chain(700 + 13 * v, 100 + v)[0] for v in range(64)]
    e = max(int(np.abs(c).max()) for c in chains)
    spb = pc.new_space(e)
    rb = pc.count_collisions_batch(chains, spb)
    ob = pc.oracle_collisions_batch(chains)
    cb = pc.oracle_contacts_batch(chains)
    for c, r, o, k in zip(chains, rb, ob, cb):
        w = c_oracle.int_pairs(c)
        assert r.count == w[0] and o == w[0] and k == w[1]
    objs = [spheres(300 + 7 * v, 200 + v) for v in range(32)]
    tb = pc.spi_totals_batch(objs, pc.collision_indicator)
    for o, t in zip(objs, tb):
        assert t == c_oracle.rows(o, 0, len(o), "balanced")[0]
    print(f"ok batch entry points ({time.time() - t0:.1f} s)", flush=True)
    DIGEST["batch"] = [[int(r.count) for r in rb], ob, cb, tb]
    DIGEST["lattice dense"] = [int(got.count), int(got.cells_touched), int(got_c.count)]
    canary_cases()
    import json

    print("SANITIZE CASES PASSED")
    print("DIGEST " + json.dumps(DIGEST, sort_keys=True))


if __name__ == "__main__":
    main()
