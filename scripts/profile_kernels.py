"""Run each hot kernel a few times on its benchmark size, for ncu captures.

    python scripts/profile_kernels.py [direct|sorted|gram|tc|tc4|gram_std|cfg2|cfg4|lattice|all] [--reps R]

Prints one timing line per case (CUDA events around the main kernel via
pc_kernel_timing); the numbers under ncu are not bench values.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402


def pairs_case(name, n, interaction, schedule, tiling, reps, seed=1, obj=None):
    if obj is None:
        obj = gen.random_spheres(n, gen.contact_box_edge(n), seed).astype(np.float32)
    d = torch.from_numpy(obj).cuda()
    ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    res = torch.zeros(8, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    b = np.array([0, n])
    _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, interaction, schedule, b, ws.data_ptr(), ws.numel(),
                     res.data_ptr(), s.cuda_stream, tiling)
    torch.cuda.synchronize()
    _lib.kernel_timing(True)
    for _ in range(reps):
        _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, interaction, schedule, b, ws.data_ptr(), ws.numel(),
                         res.data_ptr(), s.cuda_stream, tiling)
    ms, cnt = _lib.kernel_timing_read()
    _lib.kernel_timing(False)
    torch.cuda.synchronize()
    pairs = n * (n - 1) // 2
    r = res.cpu().numpy()
    print(json.dumps({"case": name, "n": n, "kernel_ms": ms / cnt, "Gpair_per_s": pairs / (ms / cnt * 1e-3) / 1e9,
                      "count": int(r[0]), "checks": int(r[3])}), flush=True)


def lattice_case(reps):
    lib = _lib.load()
    n5, a5 = 2**26, 512
    pts = gen.grid_points(n5, a5).astype(np.int32)
    d5 = torch.from_numpy(pts).cuda()
    grid = torch.zeros(int(lib.pc_lattice_grid_cells(a5)), dtype=torch.int32, device="cuda")
    keys = torch.empty(n5, dtype=torch.int32, device="cuda")
    r = _lib.LatticeResult()
    s = torch.cuda.current_stream()
    for step in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(lib.pc_lattice_collisions(d5.data_ptr(), _lib.PC_I32, 1, n5, a5, grid.data_ptr(), keys.data_ptr(),
                                             1, ctypes.byref(r), ctypes.c_void_p(s.cuda_stream)))
        _lib.check(lib.pc_lattice_clear(grid.data_ptr(), a5, ctypes.c_void_p(s.cuda_stream)))
        torch.cuda.synchronize()
        if step:
            print(json.dumps({"case": "lattice", "wall_ms": (time.perf_counter() - t0) * 1e3, "count": int(r.count),
                              "cells_touched": int(r.cells_touched)}), flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("what", nargs="?", default="all")
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    _lib.load()
    w = a.what
    if w in ("direct", "all"):
        pairs_case("direct_flat_2^20", 2**20, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, _lib.PC_TILE_FLAT, a.reps)
    if w in ("sorted", "all"):  # the headline's path: Morton-sorted points, tile-local Gram chunks
        pairs_case("direct_sorted_2^20", 2**20, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, _lib.PC_TILE_SORTED, a.reps)
    if w in ("gram", "all"):
        pairs_case("gram_flat_2^20", 2**20, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_FLAT, a.reps)
    if w in ("tc", "all"):
        pairs_case("tc_2^20", 2**20, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_TC, a.reps)
        pairs_case("tc_65536", 65536, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_TC, a.reps, seed=0)
    if w == "tc_small":
        for n in (4096, 8192, 16384, 32768):
            pairs_case(f"tc_{n}", n, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_TC, a.reps, seed=0)
            pairs_case(f"gram_flat_{n}", n, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_FLAT, a.reps, seed=0)
    if w in ("tc4", "all"):
        pairs_case("tc_clustered_2^22", 2**22, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_TC, a.reps,
                   obj=gen.clustered_spheres(2**22).astype(np.float32))
    if w == "tc4u":  # uniform 2^22 (config 4u) on both count kernels
        obj = gen.random_spheres(2**22, 259.9657721761944, 2).astype(np.float32)
        pairs_case("tc_uniform_2^22", 2**22, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_TC, a.reps, obj=obj)
        pairs_case("gram_flat_uniform_2^22", 2**22, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_FLAT, a.reps,
                   obj=obj)
    if w in ("gram_std", "all"):
        pairs_case("gram_naive_2^20", 2**20, _lib.PC_COLLISION, _lib.PC_STANDARD, _lib.PC_TILE_PER_ROW_TILE, a.reps)
    if w in ("cfg2", "all"):
        pairs_case("gram_flat_65536", 65536, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_FLAT, a.reps, seed=0)
    if w in ("cfg4", "all"):
        pairs_case("gram_flat_clustered_2^22", 2**22, _lib.PC_COLLISION, _lib.PC_BALANCED, _lib.PC_TILE_FLAT, a.reps,
                   obj=gen.clustered_spheres(2**22).astype(np.float32))
    if w in ("lattice", "all"):
        lattice_case(a.reps)
    if w in ("micro", "all"):
        for kind in (0, 1):
            rate, secs = _lib.microbench(kind)
            print(json.dumps({"case": f"microbench{kind}", "per_s": rate, "s": secs}), flush=True)


if __name__ == "__main__":
    main()
