#!/usr/bin/env python
"""Benchmark of the B200 all-pairs hot path (BASELINE.json metric: G pair-tests/s
at N=2^20, 1/2/4/8 B200, vs the CPU reference).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (config 3): N = 2^20 uniform fp32 unit-diameter
spheres (generators.random_spheres(2^20, (4*pi*N/3)^(1/3), 1)), one step =
one pass over all C(N,2) pairs computing the exact contact count and the
softened inverse-square sum (Morton sort + the sorted kernel, as spi_balanced
runs it).  With N>1 ranks, rank r runs row tiles r, r+N, ... of the sorted
order and the partials meet in one NCCL int64 all-reduce (strong scaling:
total work fixed).  Every run also reports north_star's scaling config
(2^22 clustered spheres, count + sum) under the same split
(``cfg4_clustered_n2^22``).

Rank 0 prints ONE JSON line.  `value` is device-resident throughput (inputs
already in HBM; CUDA events on the launching stream; max over ranks); `e2e`
is the same metric through the public API -- spi_balanced (N=1) or
distributed.spi_distributed (N>1) on a pageable numpy array, host copies in
the timed region; `roofline.frac` is the executed FMA-pipe work (path counters
x per-loop SASS cost) against the measured FFMA peak.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_POINTS = 2**20
FLOPS_PER_PAIR = 12  # reference formula: 3 sub, 3 mul, 2 add (d^2), compare, 1 add + 1 div (1/(1+d^2)), 1 accumulate
THROTTLE_BAD = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-secondary", action="store_true", help="skip the config-2/5 side measurements")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="gloo only to exercise the N>1 path with several ranks on one GPU (timings meaningless)")
    p.add_argument("--shared-gpu", action="store_true", help="all ranks use cuda:0 (with --dist-backend gloo)")
    p.add_argument("--cpu-rows-per-core", type=int, default=160)
    p.add_argument("--ref-rows-per-core", type=int, default=32, help="reference arm: rows per core per step")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_input():
    from paper_1901_11204_b200 import generators as gen

    return gen.random_spheres(N_POINTS, gen.contact_box_edge(N_POINTS), 1).astype(np.float32)


# ---------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi sampled every 200 ms while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        loaded = [r for r in rows if r[0] > 0.5 * r[1]] or rows
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for _, _, parts in loaded:
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median([r[0] for r in loaded])), "sm_max_mhz": max(r[1] for r in loaded),
                "samples": len(loaded), "reasons": sorted(reasons)}


# ------------------------------------------------------------ reference --
def run_reference(args):
    """The reference's own CPU implementation on this box's host cores: the
    unmodified package from baseline/_ref (``_run_outer`` per sampled row,
    fork pool over every core), or the oracle port when it is not installed."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import cpu_baseline as cb

    obj = workload_input()
    n = len(obj)
    cores = os.cpu_count() or 1
    per_step = cores * max(1, args.ref_rows_per_core)
    times, pairs, kind = [], [], cb.kind()
    for step in range(args.warmup + args.steps):
        rows = cb.sample_rows(n, per_step, 1, offset=step * 7919)
        p, wall, used, kind = cb.time_sample(obj, rows, "balanced", processes=cores)
        if step >= args.warmup:
            times.append(wall)
            pairs.append(p)
    rate = sum(pairs) / sum(times) / 1e9
    impl = ("unmodified reference paircount (baseline/_ref) _run_outer" if kind == "reference"
            else "oracle numpy port of the reference's _run_outer")
    line = {
        "impl": "reference", "metric": "G pair-tests/s at N=2^20 (contact count + inverse-square sum)",
        "value": rate, "unit": "Gpair/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg3: 2^20 uniform spheres, balanced schedule, {impl} per sampled row",
                   "n_points": n, "sample": f"{per_step} balanced rows per step x 2 interaction passes"},
        "cpu_baseline": {"value": rate, "unit": "Gpair/s", "cores": cores, "kind": kind,
                         "sample": f"{per_step} rows/step of {n} ({sum(pairs)} pair-tests timed)",
                         "cpu": cb.cpu_model(), "numpy": np.__version__},
        "e2e": {"value": rate, "unit": "Gpair/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- helpers --
def l2_flush(buf):
    buf.zero_()


def cpu_baseline_leg(obj, rows_per_core):
    from oracle import cpu_baseline as cb

    cores = os.cpu_count() or 1
    rows = cb.sample_rows(len(obj), cores * rows_per_core, 1)
    pairs, wall, used, kind = cb.time_sample(obj, rows, "balanced", processes=cores)
    who = ("the unmodified reference (baseline/_ref) _run_outer" if kind == "reference"
           else "the oracle port of the reference's _run_outer")
    return {"value": pairs / wall / 1e9, "unit": "Gpair/s", "cores": used, "kind": kind,
            "sample": f"{len(rows)} balanced rows of N=2^20 ({who}: collision_indicator + inverse-square "
                      f"passes, fork pool over all cores), {pairs} pair-tests in {wall:.1f} s",
            "cpu": cb.cpu_model(), "numpy": np.__version__}


def sass_model():
    """Per-pair FMA-pipe cycles of each inner loop, from the shipped kernels' SASS
    (scripts/sass_model.py; tests/test_sass_model.py keeps it in sync)."""
    f = ROOT / "profiles" / "sass_model.json"
    return json.loads(f.read_text())["kernels"] if f.exists() else {}


EDGE_FMA_CYCLES = 8.0  # masked scalar loop: 3 FADD + 3 FFMA + FADD + mask arithmetic per pair (not pinned)


def executed_roofline(prof, kern_s, clock_mhz, sms, kernel="sorted_sum"):
    """FMA-pipe busy fraction predicted from what the kernel executed (path
    counters x per-pair SASS cost) over the kernel's own duration."""
    m = sass_model().get(kernel, {})
    cyc = {"gram": m.get("gram", {}).get("fma_cycles_per_pair"),
           "near": m.get("near", {}).get("fma_cycles_per_pair"),
           "far": m.get("direct", {}).get("fma_cycles_per_pair"),
           "main": m.get("direct", {}).get("fma_cycles_per_pair")}
    if any(v is None for v in cyc.values()) or not prof.pairs_per_chunk:
        return None
    ppc = prof.pairs_per_chunk
    lane_cycles = ppc * (prof.chunks_gram * cyc["gram"] + prof.chunks_near * cyc["near"] +
                         prof.chunks_far * cyc["far"] + prof.chunks_main * cyc["main"] +
                         prof.chunks_edge * EDGE_FMA_CYCLES)
    # (the slow path's rescans -- rows_rescanned x W columns -- are < 0.1 % of the pairs and left out)
    smsp_cycles = lane_cycles / 32.0
    avail = kern_s * clock_mhz * 1e6 * sms * 4
    chunks = prof.chunks_gram + prof.chunks_near + prof.chunks_far + prof.chunks_main + prof.chunks_edge
    # a packed FFMA2/FADD2/FMUL2 is 2 lane-ops in 2 pipe cycles, a scalar FMA-pipe op 1 in 1: per lane,
    # pipe cycles per pair = FMA-pipe lane-ops per pair
    return {"frac": smsp_cycles / avail, "fma_lane_ops_per_pair": lane_cycles / max(1, prof.pairs),
            "fma_cycles_per_pair_by_loop": cyc, "clock_mhz": clock_mhz,
            "path_mix": {"gram": prof.chunks_gram / chunks, "near": prof.chunks_near / chunks,
                         "far_direct": prof.chunks_far / chunks, "main_direct": prof.chunks_main / chunks,
                         "edge": prof.chunks_edge / chunks},
            "chunks": chunks, "pairs_per_chunk": ppc, "rows_rescanned": prof.rows_rescanned,
            "exact_checks": prof.exact_checks, "claims": prof.claims}


def clock_ghz():
    return 1.965  # clocks.max.sm; the bench line's `clocks` records what the run saw


def secondary(torch, lib, stream):
    """Config 2 (naive vs balanced at N=65,536) and config 5 (counting array)."""
    import ctypes

    from paper_1901_11204_b200 import _lib
    from paper_1901_11204_b200 import generators as gen

    out = {}
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    # ---- config 1: N=4,096 integer points, exact-coincidence count (the reference's naive oracle)
    from oracle import numpy_port as npo1
    from paper_1901_11204_b200 import lattice_counter as lc1

    cloud = gen.normal_cloud(4096, 8.0, 64, 0)
    for _ in range(20):
        got1 = lc1.oracle_collisions(cloud)
    t0 = time.perf_counter()
    for _ in range(200):
        got1 = lc1.oracle_collisions(cloud)
    api_us = (time.perf_counter() - t0) / 200 * 1e6
    t0 = time.perf_counter()
    want1 = npo1.oracle_collisions(cloud)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    out["cfg1_integer_coincidence_n4096"] = {
        "count": got1, "expected": 356, "api_us_per_call": api_us,
        "api_path": "oracle_collisions(int64 host points): H2D, prep, all-pairs kernel with the exact int64 predicate, D2H",
        "cpu_oracle_ms": cpu_ms, "cpu": "numpy port of the reference's N x N coincidence matrix (1 core)",
        "matches_cpu": got1 == want1}

    # ---- integer all-pairs predicates at scale (oracle_collisions / oracle_contacts, lattice_counter.py:
    # 227-255) on 2^20 integer points: a normal cloud (std 64, so coordinates span < 1024 per axis)
    ni = 2**20
    cloud_i = gen.normal_cloud(ni, 64.0, 512, 3)
    di = torch.from_numpy(cloud_i.astype(np.int32)).cuda()
    wsi = torch.empty(_lib.workspace_bytes(ni), dtype=torch.uint8, device="cuda")
    resi = torch.zeros(8, dtype=torch.int64, device="cuda")
    pairs_i = ni * (ni - 1) // 2

    def int_leg(inter, tiling, reps=3):
        for _ in range(2):
            _lib.pairs_async(di.data_ptr(), _lib.PC_I32, ni, inter, _lib.PC_BALANCED, np.array([0, ni]),
                             wsi.data_ptr(), wsi.numel(), resi.data_ptr(), stream.cuda_stream, tiling)
        torch.cuda.synchronize()
        _lib.kernel_timing(True)
        for _ in range(reps):
            _lib.pairs_async(di.data_ptr(), _lib.PC_I32, ni, inter, _lib.PC_BALANCED, np.array([0, ni]),
                             wsi.data_ptr(), wsi.numel(), resi.data_ptr(), stream.cuda_stream, tiling)
        ms, cnt = _lib.kernel_timing_read()
        _lib.kernel_timing(False)
        torch.cuda.synchronize()
        ms /= cnt
        return {"kernel_ms": ms, "Tpair_per_s": pairs_i / (ms * 1e-3) / 1e12, "count": int(resi[0].item()),
                "exact_checks": int(resi[3].item())}

    _, occ = np.unique(cloud_i, axis=0, return_counts=True)
    want_col = int((occ * (occ - 1) // 2).sum())
    col = {"int32_key": int_leg(_lib.PC_COINCIDE, _lib.PC_TILE_KEY),
           "fp32_gram_filter": int_leg(_lib.PC_COINCIDE, _lib.PC_TILE_FLAT),
           "tensor_core_filter": int_leg(_lib.PC_COINCIDE, _lib.PC_TILE_TC)}
    con = {"fp32_gram_filter": int_leg(_lib.PC_MANHATTAN1, _lib.PC_TILE_FLAT),
           "tensor_core_filter": int_leg(_lib.PC_MANHATTAN1, _lib.PC_TILE_TC)}
    alu_ceiling = sms * 64 * clock_ghz() * 1e9 / 1.0  # one ISETP.EQ.OR per pair on the 64-lane/clk/SM INT pipe
    out["integer_predicates_n2^20"] = {
        "input": "normal_cloud(2^20, std 64, half-extent 512, seed 3) as int32",
        "oracle_collisions": col, "oracle_contacts": con, "coincidences_np_unique": want_col,
        "counts_exact": all(v["count"] == want_col for v in col.values()),
        "chosen": {"oracle_collisions": "int32_key when the bounding box spans <= 1023 per axis "
                                        "(lattice_counter._integer_pairs), else the Gram filter",
                   "oracle_contacts": "tensor-core filter (PC_TILE_AUTO) / FP32 Gram filter"},
        "int32_key_frac_of_int_pipe": col["int32_key"]["Tpair_per_s"] * 1e12 / alu_ceiling,
        "int_pipe_ceiling_basis": "1 ISETP.EQ.OR per pair (SASS of pairs_key_kernel's loop: 48 ISETP.EQ.OR + 8 LDG "
                                  "per 48 pairs) at 64 lanes/clk/SM x 148 SMs x the sampled SM clock"}
    del di, wsi

    # ---- float64 input (the reference generators' own dtype): the sum on the input order
    # (compensated hi + lo) vs on Morton-sorted points (what spi_balanced takes from 2^15 points)
    x64 = gen.random_spheres(2**20, gen.contact_box_edge(2**20), 1)
    d64 = torch.from_numpy(x64).cuda()
    ws64 = torch.empty(_lib.workspace_bytes(2**20), dtype=torch.uint8, device="cuda")
    res = torch.zeros(8, dtype=torch.int64, device="cuda")
    f64leg = {}
    for label, tiling in (("input_order_compensated", _lib.PC_TILE_FLAT), ("sorted_compensated", _lib.PC_TILE_AUTO)):
        _lib.pairs_async(d64.data_ptr(), _lib.PC_F64, 2**20, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED,
                         np.array([0, 2**20]), ws64.data_ptr(), ws64.numel(), res.data_ptr(), stream.cuda_stream, tiling)
        _lib.kernel_timing(True)
        for _ in range(2):
            _lib.pairs_async(d64.data_ptr(), _lib.PC_F64, 2**20, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED,
                             np.array([0, 2**20]), ws64.data_ptr(), ws64.numel(), res.data_ptr(), stream.cuda_stream,
                             tiling)
        (fm64, fc64), (tm64, tc64) = _lib.kernel_timing_read_split()
        _lib.kernel_timing(False)
        torch.cuda.synchronize()
        ms_call = (fm64 + tm64) / 2  # all-pairs kernels per call (the sorted call adds the tensor-core one)
        f64leg[label] = {"kernel_ms": ms_call, "ffma_kernel_ms": fm64 / 2, "tensor_core_kernel_ms": tm64 / 2,
                         "count": int(res[0].item()),
                         "Gpair_per_s": (2**20) * (2**20 - 1) / 2 / (ms_call * 1e-3) / 1e9}
    out["float64_points_sum_n2^20"] = f64leg
    del d64, ws64

    # ---- config 2
    n2 = 65536
    obj2 = gen.random_spheres(n2, gen.contact_box_edge(n2), 0).astype(np.float32)
    d2 = torch.from_numpy(obj2).cuda()
    ws = torch.empty(_lib.workspace_bytes(n2), dtype=torch.uint8, device="cuda")
    res = torch.zeros(8, dtype=torch.int64, device="cuda")
    pairs2 = n2 * (n2 - 1) // 2
    rows = {}
    for label, sched, tiling in (("naive_standard_per_row_tile", _lib.PC_STANDARD, _lib.PC_TILE_PER_ROW_TILE),
                                 ("balanced_per_row_tile", _lib.PC_BALANCED, _lib.PC_TILE_PER_ROW_TILE),
                                 ("balanced_uniform_tiles", _lib.PC_BALANCED, _lib.PC_TILE_FLAT),
                                 ("balanced_uniform_tiles_tensor_cores", _lib.PC_BALANCED, _lib.PC_TILE_TC)):
        for _ in range(3):
            _lib.pairs_async(d2.data_ptr(), _lib.PC_F32, n2, _lib.PC_COLLISION, sched, np.array([0, n2]),
                             ws.data_ptr(), ws.numel(), res.data_ptr(), stream.cuda_stream, tiling)
        _lib.kernel_timing(True)
        reps = 20
        for _ in range(reps):
            _lib.pairs_async(d2.data_ptr(), _lib.PC_F32, n2, _lib.PC_COLLISION, sched, np.array([0, n2]),
                             ws.data_ptr(), ws.numel(), res.data_ptr(), stream.cuda_stream, tiling)
        ms, cnt = _lib.kernel_timing_read()
        _lib.kernel_timing(False)
        torch.cuda.synchronize()
        count = int(res[0].item())
        rows[label] = {"kernel_ms": ms / cnt, "Gpair_per_s": pairs2 / (ms / cnt * 1e-3) / 1e9, "count": count}
    rows["naive_over_balanced_time"] = rows["naive_standard_per_row_tile"]["kernel_ms"] / \
        rows["balanced_uniform_tiles"]["kernel_ms"]
    rows["paper_reference_ratio"] = "1.12x on P100 for N > 525,000 (PAPER.md:419)"
    rows["tensor_cores_over_ffma_speedup"] = rows["balanced_uniform_tiles"]["kernel_ms"] / \
        rows["balanced_uniform_tiles_tensor_cores"]["kernel_ms"]
    out["cfg2_naive_vs_balanced_n65536"] = rows
    del d2, ws

    # ---- config 3, count only: the metric's "collision-count wall time at N=2^20"
    from paper_1901_11204_b200 import spi_engine as se

    n3 = 2**20
    obj3 = workload_input()
    d3 = torch.from_numpy(obj3).cuda()
    ws3 = torch.empty(_lib.workspace_bytes(n3), dtype=torch.uint8, device="cuda")
    pairs3 = n3 * (n3 - 1) // 2

    def count_leg(tiling, reps=5):
        for _ in range(2):
            _lib.pairs_async(d3.data_ptr(), _lib.PC_F32, n3, _lib.PC_COLLISION, _lib.PC_BALANCED, np.array([0, n3]),
                             ws3.data_ptr(), ws3.numel(), res.data_ptr(), stream.cuda_stream, tiling)
        torch.cuda.synchronize()
        _lib.kernel_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            _lib.pairs_async(d3.data_ptr(), _lib.PC_F32, n3, _lib.PC_COLLISION, _lib.PC_BALANCED, np.array([0, n3]),
                             ws3.data_ptr(), ws3.numel(), res.data_ptr(), stream.cuda_stream, tiling)
        e1.record(stream)
        torch.cuda.synchronize()
        ms, cnt = _lib.kernel_timing_read()
        _lib.kernel_timing(False)
        return ms / cnt, e0.elapsed_time(e1) / reps, int(res[0].item()), int(res[3].item())

    k_ffma, dev_ffma, count_ffma, checks_ffma = count_leg(_lib.PC_TILE_FLAT)
    k_tc, dev_tc, count_tc, checks_tc = count_leg(_lib.PC_TILE_TC)
    k_pr, dev_pr, count_pr, checks_pr = count_leg(_lib.PC_TILE_AUTO)  # whole range fp32: pruned sorted count
    prof_pr = _lib.profile_read(ws3.data_ptr(), n3, stream.cuda_stream)
    chunks_pr = (prof_pr.chunks_gram + prof_pr.chunks_main + prof_pr.chunks_near + prof_pr.chunks_far +
                 prof_pr.chunks_edge)
    evaluated_cells = (chunks_pr - prof_pr.chunks_far) * prof_pr.pairs_per_chunk
    t0 = time.perf_counter()
    r3 = se.spi_balanced(obj3, se.collision_indicator)
    api_ms = (time.perf_counter() - t0) * 1e3
    out["cfg3_collision_count_n2^20"] = {
        "count": count_tc, "api_count": int(r3.total), "ffma_count": count_ffma, "pruned_count": count_pr,
        "kernel_ms": k_tc, "device_ms_per_call": dev_tc, "exact_checks": checks_tc,
        "Gpair_per_s_kernel": pairs3 / (k_tc * 1e-3) / 1e9,
        "kernel": "pairs_tc_kernel (tcgen05.mma kind::tf32, 3xTF32 Gram filter, TMEM drained by 8 warps) + "
                  "tc_exact_kernel: every pair evaluated",
        "ffma_kernel": "pairs_kernel<128,12,192,GRAM,FLAT>", "ffma_kernel_ms": k_ffma,
        "ffma_device_ms_per_call": dev_ffma, "ffma_exact_checks": checks_ffma,
        "ffma_Gpair_per_s_kernel": pairs3 / (k_ffma * 1e-3) / 1e9,
        "pruned_sorted": {
            "kernel": "pairs_kernel<128,12,192,GRAM,FLAT,SORTED>: Morton-sorted points, claims and chunks whose "
                      "bounding boxes are beyond contact distance of the tile decided without evaluation "
                      "(PAPER.md:443: the all-pairs count composed with pruning); PC_TILE_AUTO for whole-range "
                      "fp32 counts from 2^15 points",
            "kernel_ms": k_pr, "device_ms_per_call": dev_pr, "count": count_pr, "exact_checks": checks_pr,
            "pairs_decided_by_boxes_not_evaluated": int(pairs3 - min(pairs3, evaluated_cells)),
            "pair_cells_evaluated": int(evaluated_cells),
            "evaluated_Gpair_per_s": evaluated_cells / (k_pr * 1e-3) / 1e9,
            "note": "not a pair-test rate: most pairs are decided by their boxes, reported apart"},
        "api_wall_ms": api_ms,
        "api_path": "spi_balanced(points, collision_indicator): numpy (n,3) f32 -> ctypes pc_pairs_host "
                    "(H2D, bbox, Morton sort, pruned Gram count, exact re-checks, finalize, D2H) -> SpiResult",
    }
    ms_k, cnt_k = k_ffma, 1  # the naive comparison below is against the same FFMA inner code
    # the paper's comparison in its large-N regime (N > 525,000): the straightforward
    # scheme (standard schedule, one warp per row tile) on the same inner code
    _lib.kernel_timing(True)
    _lib.pairs_async(d3.data_ptr(), _lib.PC_F32, n3, _lib.PC_COLLISION, _lib.PC_STANDARD, np.array([0, n3]),
                     ws3.data_ptr(), ws3.numel(), res.data_ptr(), stream.cuda_stream, _lib.PC_TILE_PER_ROW_TILE)
    ms_n, cnt_n = _lib.kernel_timing_read()
    _lib.kernel_timing(False)
    torch.cuda.synchronize()
    out["cfg3_collision_count_n2^20"].update({
        "naive_standard_per_row_tile_ms": ms_n / cnt_n, "naive_count": int(res[0].item()),
        "naive_over_balanced_time": (ms_n / cnt_n) / (ms_k / cnt_k)})
    # the paper's own experiment (>12 % at N > 525,000 on a P100): thread-per-row
    # kernels in 1024-row blocks, the straightforward (standard) vs the balanced schedule, same code
    paper = {}
    for sched_name, sched in (("straightforward_standard", _lib.PC_STANDARD), ("balanced", _lib.PC_BALANCED)):
        _lib.pairs_async(d3.data_ptr(), _lib.PC_F32, n3, _lib.PC_COLLISION, sched, np.array([0, n3]),
                         ws3.data_ptr(), ws3.numel(), res.data_ptr(), stream.cuda_stream, _lib.PC_TILE_THREAD_ROW)
        _lib.kernel_timing(True)
        for _ in range(2):
            _lib.pairs_async(d3.data_ptr(), _lib.PC_F32, n3, _lib.PC_COLLISION, sched, np.array([0, n3]),
                             ws3.data_ptr(), ws3.numel(), res.data_ptr(), stream.cuda_stream, _lib.PC_TILE_THREAD_ROW)
        ms_p, cnt_p = _lib.kernel_timing_read()
        _lib.kernel_timing(False)
        torch.cuda.synchronize()
        paper[sched_name] = {"kernel_ms": ms_p / cnt_p, "count": int(res[0].item()),
                             "Gpair_per_s": pairs3 / (ms_p / cnt_p * 1e-3) / 1e9}
    paper["straightforward_over_balanced_time"] = (paper["straightforward_standard"]["kernel_ms"] /
                                                   paper["balanced"]["kernel_ms"])
    paper["paper"] = "1.12x on a P100 for N > 525,000 (PAPER.md:416)"
    paper["kernel"] = "pairs_row_kernel (PC_TILE_THREAD_ROW): one thread per row, 1024-row blocks, shared-memory tiles"
    out["cfg3_collision_count_n2^20"]["paper_thread_per_row"] = paper
    del d3, ws3

    # ---- config 5: counting array, device-resident int32 coordinates
    n5, a5 = 2**26, 512
    pts = gen.grid_points(n5, a5)
    d5 = torch.from_numpy(pts.astype(np.int32)).cuda()
    ncell = int(lib.pc_lattice_grid_cells(a5))
    grid = torch.zeros(ncell, dtype=torch.int32, device="cuda")
    keys = torch.empty(n5, dtype=torch.int32, device="cuda")
    r = _lib.LatticeResult()
    times = []
    for step in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rc = lib.pc_lattice_collisions(d5.data_ptr(), _lib.PC_I32, 1, n5, a5, grid.data_ptr(), keys.data_ptr(), 1,
                                       ctypes.byref(r), ctypes.c_void_p(stream.cuda_stream))
        _lib.check(rc)
        # reset_sparse's policy (lattice_counter.py): 2^26 keys > cells/32 on a clean grid -> streaming clear
        if n5 * 32 > ncell:
            _lib.check(lib.pc_lattice_clear(grid.data_ptr(), a5, ctypes.c_void_p(stream.cuda_stream)))
        else:
            _lib.check(lib.pc_lattice_reset_keys(grid.data_ptr(), a5, keys.data_ptr(), n5,
                                                 ctypes.c_void_p(stream.cuda_stream)))
        e1.record(stream)
        torch.cuda.synchronize()
        if step >= 3:
            times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    # SURVEY.md §8(d) B_alg: 12 B coords + 8 B counter RMW per bead, 8 B per cell (write + clear)
    b_alg = 20 * n5 + 8 * ncell
    peaks = ROOT / "MEASURED_PEAKS.json"
    hbm = json.loads(peaks.read_text()).get("hbm_gbs", 6532.5) if peaks.exists() else 6532.5
    out["cfg5_counting_array_n2^26"] = {
        "wall_ms_per_step": ms, "count": int(r.count), "cells_touched": int(r.cells_touched),
        "expected_count": 2101067, "grid_cells": ncell,
        "step": "count_collisions (dense regime: validate+keys, bucket partition, Alg. 1 on shared-memory "
                "slabs, TMA bulk slab stores) + reset_sparse (streaming clear)",
        "alg_bytes_survey": b_alg, "achieved_GBps": b_alg / (ms * 1e-3) / 1e9,
        "hbm_frac_of_measured": b_alg / (ms * 1e-3) / 1e9 / hbm,
        "note": "scattered global atomics would cap this at ~21 G beads/s (scripts/microbench_l2atomic.cu)"}
    del d5, grid, keys
    # the same step through the drop-in API from host int64 beads (the reference's own input)
    from paper_1901_11204_b200 import lattice_counter as lc

    pts64 = np.ascontiguousarray(pts.astype(np.int64))
    sp5 = lc.new_space(a5)
    api_times = []
    for rep in range(3):
        t0 = time.perf_counter()
        rep5 = lc.count_collisions(pts64, sp5)
        lc.reset_sparse(sp5)
        api_times.append((time.perf_counter() - t0) * 1e3)
    api_ms = min(api_times[1:])  # first call pays the host pages' first touch
    out["cfg5_counting_array_n2^26"].update({
        "api_wall_ms": api_ms, "api_count": rep5.count,
        "api_path": "count_collisions(int64 host beads, space) + reset_sparse: host threads narrow the 1.61 GB "
                    "of int64 beads to int32 in pinned chunks streamed to the device (0.8 GB H2D) + the device step"})
    del sp5, pts64

    # ---- the headline workload split 2/4/8 ways the way the multi-GPU step splits it: row tiles of
    # the sorted order dealt round-robin (pc_pairs_part_async; what bench N>1 and spi_distributed run),
    # beside contiguous slabs of the sorted order (round 1's split).  Each share timed alone on this
    # GPU: the balance of the split and a projected per-GPU step (the exchange is one all-reduce).
    from paper_1901_11204_b200.distributed import row_slabs

    def split_legs(d, n_, ws_, res_, interaction, tiling, worlds=(2, 4, 8)):
        def timed(fn):
            _lib.kernel_timing(True)
            fn()
            ms_k, _ = _lib.kernel_timing_read()
            _lib.kernel_timing(False)
            torch.cuda.synchronize()
            return ms_k, int(res_[0].item()), int(res_[2].item())

        def whole():
            _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n_, interaction, _lib.PC_BALANCED, np.array([0, n_]),
                             ws_.data_ptr(), ws_.numel(), res_.data_ptr(), stream.cuda_stream, tiling)

        timed(whole)
        full_ms, full_count, _ = timed(whole)
        out_ = {"kernel_ms_1gpu": full_ms, "count": full_count}
        for g in worlds:
            parts = [timed(lambda k=k: _lib.pairs_part_async(
                d.data_ptr(), _lib.PC_F32, n_, interaction, _lib.PC_BALANCED, 0, n_, k, g, ws_.data_ptr(),
                ws_.numel(), res_.data_ptr(), stream.cuda_stream, tiling)) for k in range(g)]
            slabs = [timed(lambda lo=lo, hi=hi: _lib.pairs_async(
                d.data_ptr(), _lib.PC_F32, n_, interaction, _lib.PC_BALANCED, np.array([lo, hi]), ws_.data_ptr(),
                ws_.numel(), res_.data_ptr(), stream.cuda_stream, tiling)) for lo, hi in row_slabs(n_, g, "balanced")]
            out_[f"split{g}"] = {
                "tile_parts": {"ms_max": max(t for t, _, _ in parts), "ms_min": min(t for t, _, _ in parts),
                               "projected_speedup": full_ms / max(t for t, _, _ in parts),
                               "counts_add_up": sum(c for _, c, _ in parts) == full_count},
                "contiguous_slabs": {"ms_max": max(t for t, _, _ in slabs), "ms_min": min(t for t, _, _ in slabs),
                                     "projected_speedup": full_ms / max(t for t, _, _ in slabs),
                                     "counts_add_up": sum(c for _, c, _ in slabs) == full_count}}
        return out_

    d3s = torch.from_numpy(workload_input()).cuda()
    ws3s = torch.empty(_lib.workspace_bytes(n3), dtype=torch.uint8, device="cuda")
    res3s = torch.zeros(8, dtype=torch.int64, device="cuda")
    out["cfg3_headline_split"] = split_legs(d3s, n3, ws3s, res3s, _lib.PC_COLLISION_INVSQ, _lib.PC_TILE_SORTED)
    del d3s, ws3s

    # ---- config 4: 2^22 clustered points; the count (FFMA2 Gram filter) and the count + sum (sorted
    # pass) on one GPU and split 2/4/8 ways, each share timed alone (ranks never wait on each other)
    n4 = 2**22
    obj4 = gen.clustered_spheres(n4).astype(np.float32)
    d4 = torch.from_numpy(obj4).cuda()
    ws4 = torch.empty(_lib.workspace_bytes(n4), dtype=torch.uint8, device="cuda")
    res4 = torch.zeros(8, dtype=torch.int64, device="cuda")
    pairs4 = n4 * (n4 - 1) // 2
    c4 = split_legs(d4, n4, ws4, res4, _lib.PC_COLLISION, _lib.PC_TILE_FLAT)
    c4["Gpair_per_s_1gpu"] = pairs4 / (c4["kernel_ms_1gpu"] * 1e-3) / 1e9
    s4 = split_legs(d4, n4, ws4, res4, _lib.PC_COLLISION_INVSQ, _lib.PC_TILE_SORTED)
    s4["Gpair_per_s_1gpu"] = pairs4 / (s4["kernel_ms_1gpu"] * 1e-3) / 1e9
    _lib.kernel_timing(True)
    for _ in range(2):
        _lib.pairs_async(d4.data_ptr(), _lib.PC_F32, n4, _lib.PC_COLLISION, _lib.PC_BALANCED, np.array([0, n4]),
                         ws4.data_ptr(), ws4.numel(), res4.data_ptr(), stream.cuda_stream, _lib.PC_TILE_AUTO)
    ms_p4, cnt_p4 = _lib.kernel_timing_read()
    _lib.kernel_timing(False)
    torch.cuda.synchronize()
    prof4 = _lib.profile_read(ws4.data_ptr(), n4, stream.cuda_stream)
    tot4 = prof4.chunks_gram + prof4.chunks_main + prof4.chunks_near + prof4.chunks_far + prof4.chunks_edge
    p4 = {"kernel_ms": ms_p4 / cnt_p4, "count": int(res4[0].item()), "exact_checks": int(res4[3].item()),
          "chunks_decided_by_boxes": prof4.chunks_far, "chunks_total": tot4,
          "note": "pruned sorted count (PC_TILE_AUTO): pairs decided by their boxes are not evaluated"}
    out["cfg4_clustered_n2^22"] = {"count_ffma_gram": c4, "count_plus_sum_sorted": s4, "count_pruned_sorted": p4}
    del d4, ws4

    # ---- many small vectors: the paper's setting (1000 chain vectors per execution)
    from oracle import numpy_port as npo
    from paper_1901_11204_b200 import lattice_counter as lc

    chains = [gen.random_chain(1024, 7000 + v)[0] for v in range(1000)]
    ext = max(int(np.abs(c).max()) for c in chains)
    sp = lc.new_space(ext)
    for _ in range(2):
        lc.count_collisions_batch(chains, sp)
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        got = lc.count_collisions_batch(chains, sp)
    gpu_ms = (time.perf_counter() - t0) / reps * 1e3
    lc.oracle_collisions_batch(chains)  # warm-up: grows the pinned staging and the device arena
    t0 = time.perf_counter()
    for _ in range(reps):
        quad = lc.oracle_collisions_batch(chains)
    quad_ms = (time.perf_counter() - t0) / reps * 1e3
    assert quad == [r.count for r in got]
    cells_np = npo.new_dense_space(ext)
    t0 = time.perf_counter()
    cpu = [npo.count_collisions_dense(c, cells_np, ext)[0] for c in chains[:100]]  # reference _linear_pass step
    cpu_ms = (time.perf_counter() - t0) * 10 * 1e3
    assert [r.count for r in got[:100]] == cpu
    out["many_vectors_1000x1024_chains"] = {
        "gpu_ms_per_execution": gpu_ms, "path": "count_collisions_batch from host arrays (H2D + 1 launch + D2H)",
        "gpu_quadratic_ms_per_execution": quad_ms,
        "quadratic_path": "oracle_collisions_batch: all 1000 x C(1024,2) pairs, one launch (the linear-vs-quadratic "
                          "harness's other side; counts equal)",
        "cpu_baseline_ms_per_execution": cpu_ms, "cpu_baseline": "oracle numpy port of the reference's dense-grid "
        "count_collisions + reset_sparse, 100 of the 1000 vectors timed on 1 core, x10",
        "collisions_total": int(sum(r.count for r in got))}
    return out


# ------------------------------------------------------------------ ours --
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1901_11204_b200 import _lib
    from paper_1901_11204_b200 import distributed as D
    from paper_1901_11204_b200 import spi_engine as se
    from paper_1901_11204_b200.pair_schedule import row_pairs

    rank, world, local = dist_env()
    if args.shared_gpu:
        local = 0
    torch.cuda.set_device(local)
    os.environ["PAIRCOUNT_DEVICE"] = str(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    sms = torch.cuda.get_device_properties(local).multi_processor_count

    obj = workload_input()
    n = len(obj)
    total_pairs = n * (n - 1) // 2
    d_obj = torch.from_numpy(obj).cuda()
    ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    res = torch.zeros(8, dtype=torch.int64, device="cuda")  # pc_pairs_result (40 B)
    slots = torch.zeros(4 * world, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        # the whole-range sum on Morton-sorted points (what spi_balanced runs); with N ranks rank r
        # runs row tiles r, r+N, ... of the same sorted order (pc_pairs_part_async, D.choose_split)
        _lib.pairs_part_async(d_obj.data_ptr(), _lib.PC_F32, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, 0, n,
                              rank, world, ws.data_ptr(), ws.numel(), res.data_ptr(), stream.cuda_stream,
                              _lib.PC_TILE_SORTED)
        launches = _lib.launches()
        if world > 1:
            slots.zero_()
            slots[4 * rank: 4 * rank + 2].copy_(res[0:2])  # count, float64 sum bits
            slots[4 * rank + 3].copy_(res[2])                # pairs
            dist.all_reduce(slots)  # the one NCCL int64 all-reduce of the partials
        return launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    launches = 0
    elapsed = 0.0
    _lib.kernel_timing(True)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launches += step()
            e1.record(stream)
            e1.synchronize()
            elapsed += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    (ffma_ms, ffma_launches), (tc_ms, tc_launches) = _lib.kernel_timing_read_split()
    kern_ms, kern_launches = ffma_ms + tc_ms, ffma_launches + tc_launches
    _lib.kernel_timing(False)
    prof = _lib.profile_read(ws.data_ptr(), n, stream.cuda_stream)  # the last step's path counters
    if world > 1:
        dist.barrier()
        t = torch.tensor([elapsed, kern_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, kern_ms_max = float(t[0].item()), float(t[1].item())
        v = slots.view(world, 4)
        counts = int(v[:, 0].sum().item())
        psum = float(np.array(v[:, 1].cpu().numpy()).view(np.float64).sum())
        assert int(v[:, 3].sum().item()) == total_pairs
    else:
        counts = int(res[0].item())
        psum = float(np.array([res[1].item()], dtype=np.int64).view(np.float64)[0])
        kern_ms_max = kern_ms
    ms_per_step = elapsed / args.steps
    value = total_pairs / (ms_per_step * 1e-3) / 1e9

    # ---- end to end through the public API: a pageable numpy array in, the Python result out
    for _ in range(2):
        api_total = (se.spi_balanced(obj, se.inverse_square).total if world == 1 else
                     D.spi_distributed(obj, se.inverse_square, device="cuda")[0])
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_launches = 0
    for _ in range(args.steps):
        if world == 1:
            api_total = se.spi_balanced(obj, se.inverse_square).total
        else:
            api_total = D.spi_distributed(obj, se.inverse_square, device="cuda")[0]
        e2e_launches += _lib.launches()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    api_path = ("spi_engine.spi_balanced(points, inverse_square) on a pageable numpy (2^20, 3) float32 array: "
                "ctypes pc_pairs_host = H2D + bbox + Morton sort + kernel + float64 kernel (idle) + finalize + D2H"
                if world == 1 else
                "distributed.spi_distributed(points, inverse_square, device='cuda'): pc_pairs_part_host per rank "
                "(H2D + sort + this rank's row tiles + D2H) + one NCCL int64 all-reduce of the partials")
    e2e = {"value": total_pairs / e2e_s / 1e9, "unit": "Gpair/s", "h2d_bytes_per_step": int(obj.nbytes),
           "d2h_bytes_per_step": 40 + ctypes_sizeof_profile(), "ms_per_step": e2e_s * 1e3, "path": api_path,
           "api_total": api_total, "device_launches_per_step": e2e_launches / max(1, args.steps)}

    # ---- the north_star scaling config: 2^22 clustered spheres, count + sum (one pass per step)
    cfg4 = scaling_leg(torch, dist, _lib, rank, world, stream, min(args.steps, 3))

    if rank != 0:
        dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel: pairs_tcs_kernel (the tensor-core Gram chunks, ~93 % of the
    # pairs at 2^20), with the sorted FFMA kernel (the remaining near / far-direct / edge chunks) beside it
    steps_timed = max(1, args.steps)
    rank_pairs = int(prof.pairs)
    clocks = clk.summary()
    clock_mhz = clocks.get("sm_mhz") or 1965.0
    ffma_rate, _ = _lib.microbench(0)  # lane-FFMA/s over all SMs, measured live
    peak_tflops = 2.0 * ffma_rate / 1e12
    tinfo = {}
    tfile = ROOT / "profiles" / "kernel_traffic.json"
    if tfile.exists():
        try:
            tinfo = json.loads(tfile.read_text())
        except (ValueError, OSError):
            tinfo = {}
    peaks = {}
    pfile = ROOT / "MEASURED_PEAKS.json"
    if pfile.exists():
        try:
            peaks = json.loads(pfile.read_text())
        except (ValueError, OSError):
            peaks = {}
    ffma_ms_avg = ffma_ms / max(1, ffma_launches)
    tc_ms_avg = tc_ms / max(1, tc_launches)
    ppc = int(prof.pairs_per_chunk) or 65536
    pairs_tc = int(prof.chunks_tc) * ppc
    pairs_ffma = rank_pairs - pairs_tc
    exe = executed_roofline(prof, ffma_ms_avg * 1e-3, clock_mhz, sms)  # the FFMA kernel over its own chunks
    ffma_part = {
        "kernel": "pairs_kernel<4,8,256,DIRECT,FLAT,SORTED> (near, far-direct and edge chunks; skips the "
                  "tensor-core chunks)",
        "kernel_ms": ffma_ms_avg, "launches_per_step": ffma_launches / steps_timed, "pairs": pairs_ffma,
        "pairs_per_s": pairs_ffma / (ffma_ms_avg * 1e-3) if ffma_ms_avg else None,
        "executed": exe,
        "frac_fma_pipe": (exe["frac"] if exe else None),
        "frac_basis": "executed FMA-pipe work (its path counters x per-pair SASS cost of each inner loop, "
                      "profiles/sass_model.json) / the kernel's time x FMA-pipe capacity",
    }
    if tc_launches:
        mma_flops_per_pair = 64  # tcgen05.mma kind::f16, K = 32 bf16 products per pair, 2 flop each
        tc_s = tc_ms_avg * 1e-3
        pairs_tc_s = pairs_tc / tc_s
        bf16_peak = peaks.get("bf16_tflops") or 2250.0
        achieved = mma_flops_per_pair * pairs_tc_s / 1e12
        clk_hz = clock_mhz * 1e6
        per_clk_sm = pairs_tc_s / (sms * clk_hz)
        roofline = {
            "bound": "tensor", "unit": "TFLOP/s",
            "achieved": achieved, "peak": bf16_peak, "frac": achieved / bf16_peak,
            "frac_basis": "executed tcgen05.mma flops (64 per pair: K = 32 bf16 products) of the timed step / "
                          "pairs_tcs_kernel's CUDA-event time, against the measured dense bf16 peak "
                          "(MEASURED_PEAKS.json bf16_tflops, burst)",
            "traffic": tinfo.get("pairs_tcs_kernel_n2^20"),
            "traffic_basis": "dram read+write bytes per launch from the committed ncu --set full capture "
                             "(profiles/kernel_traffic.json), not measured in this run",
            "kernel": "pairs_tcs_kernel (tcgen05.mma kind::f16 M=128 N=256 K=32, TMEM drained by 8 warps)",
            "kernel_ms": tc_ms_avg, "pairs": pairs_tc, "pairs_per_s_kernel": pairs_tc_s,
            "pairs_per_clk_per_sm": per_clk_sm,
            "binding_resource": {
                "what": "the epilogue: each pair's accumulator word read from TMEM (4 B) and folded into the sum "
                        "with 2 FMA-pipe lane-ops + 1/4 MUFU.RCP (eight terms per two reciprocals)",
                "fma_mufu_ceiling_pairs_per_clk_sm": 64.0,
                "frac_of_fma_mufu_ceiling": per_clk_sm / 64.0,
                "tmem_drain_ceiling_pairs_per_clk_sm": 78.7,
                "frac_of_tmem_drain_ceiling": per_clk_sm / 78.7,
                "pipelined_proto_pairs_per_clk_sm": 35.7,
                "frac_of_pipelined_proto": per_clk_sm / 35.7,
                "basis": "FMA 128 lane-ops/clk/SM / 2 per pair; MUFU 16/clk/SM / 0.25 per pair; TMEM loads alone "
                         "78.7 pairs/clk/SM and the same epilogue on a static operand 35.7 "
                         "(scripts/tc_sum_proto.cu, B200); ncu of this kernel: FMA pipe 62 %, XU 62 %, "
                         "tensor 30 %, issue 50 % (profiles/r2_ncu_tcs_kernel.txt)",
            },
            "ffma_kernel": ffma_part,
            "step_kernels_ms": {"pairs_tcs_kernel": tc_ms_avg, "pairs_kernel_sorted": ffma_ms_avg},
            "normalised": {"flops_per_pair": FLOPS_PER_PAIR,
                           "tflops": FLOPS_PER_PAIR * rank_pairs / ((tc_ms_avg + ffma_ms_avg) * 1e-3) / 1e12,
                           "frac": FLOPS_PER_PAIR * rank_pairs / ((tc_ms_avg + ffma_ms_avg) * 1e-3) / 1e12 /
                           peak_tflops,
                           "basis": "12 reference-formula flops per pair over both kernels' time, against the "
                                    "measured FP32 FFMA peak (a normalisation: the tensor cores do the product)"},
        }
    else:  # PAIRCOUNT_TCSUM=0: the FFMA sorted kernel alone
        norm_tflops = FLOPS_PER_PAIR * rank_pairs / (ffma_ms_avg * 1e-3) / 1e12
        pairs_s = rank_pairs / (ffma_ms_avg * 1e-3)
        exec_lane_ops_s = (exe["fma_lane_ops_per_pair"] * pairs_s) if exe else None
        roofline = {
            "bound": "fp32 FMA pipe", "unit": "TFLOP/s",
            "achieved": (exec_lane_ops_s * 2.0 / 1e12) if exe else norm_tflops,
            "peak": peak_tflops,
            "frac": (exec_lane_ops_s / ffma_rate) if exe else norm_tflops / peak_tflops,
            "frac_basis": ffma_part["frac_basis"] + " (measured FFMA peak, pc_microbench)",
            "traffic": tinfo.get("pairs_kernel_direct_flat_n2^20"),
            "kernel": "pairs_kernel<4,8,256,DIRECT,FLAT,SORTED>", "kernel_ms": ffma_ms_avg,
            "pairs_per_s_kernel": pairs_s, "executed": exe,
        }
    kern_ms_avg = kern_ms / steps_timed

    line = {
        "metric": "G pair-tests/s at N=2^20 (contact count + inverse-square sum)",
        "value": value, "unit": "Gpair/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": "cfg3: N=2^20 uniform fp32 unit spheres, exact contact count + softened "
                               "inverse-square sum, balanced schedule on uniform tiles",
                   "n_points": n, "pairs_per_step": total_pairs, "schedule": "balanced",
                   "tiling": "flat, on Morton-sorted points (sort inside the step)",
                   "parallelism": (f"row tiles dealt round-robin over {world} ranks, one NCCL int64 all-reduce"
                                   if world > 1 else "1 GPU"),
                   "l2": "flushed between timed steps (256 MiB memset)", "contacts": counts, "inv_sum": psum},
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "cfg4_clustered_n2^22": cfg4,
    }
    if world > 1:
        line["kernel_ms_per_step_max_over_ranks"] = kern_ms_max / max(1, args.steps)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(obj, args.cpu_rows_per_core)
    if world == 1 and not args.no_secondary:
        line["secondary"] = secondary(torch, lib, stream)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def ctypes_sizeof_profile() -> int:
    import ctypes

    from paper_1901_11204_b200 import _lib

    return ctypes.sizeof(_lib.PairsProfile)


def scaling_leg(torch, dist, _lib, rank, world, stream, steps):
    """north_star's scaling config (BASELINE config 4): N = 2^22 clustered fp32
    spheres, one pass per step computing the exact contact count and the
    inverse-square sum (PC_TILE_SORTED), rank r on row tiles r, r+N, ...; the
    device time is the max over ranks.  Checked against golden_full.json."""
    from paper_1901_11204_b200 import generators as gen

    n4 = 2**22
    obj4 = gen.clustered_spheres(n4).astype(np.float32)
    d4 = torch.from_numpy(obj4).cuda()
    ws4 = torch.empty(_lib.workspace_bytes(n4), dtype=torch.uint8, device="cuda")
    res4 = torch.zeros(8, dtype=torch.int64, device="cuda")
    slots4 = torch.zeros(4 * world, dtype=torch.int64, device="cuda")

    def one():
        _lib.pairs_part_async(d4.data_ptr(), _lib.PC_F32, n4, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, 0, n4,
                              rank, world, ws4.data_ptr(), ws4.numel(), res4.data_ptr(), stream.cuda_stream,
                              _lib.PC_TILE_SORTED)
        slots4.zero_()
        slots4[4 * rank: 4 * rank + 2].copy_(res4[0:2])
        slots4[4 * rank + 3].copy_(res4[2])
        if world > 1:
            dist.all_reduce(slots4)

    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    v = slots4.view(world, 4).cpu().numpy()
    count = int(v[:, 0].sum())
    inv_sum = float(v[:, 1].copy().view(np.float64).sum())
    pairs = n4 * (n4 - 1) // 2
    gold = {}
    gfile = ROOT / "tests" / "golden" / "golden_full.json"
    if gfile.exists():
        gold = json.loads(gfile.read_text()).get("cfg4c", {})
    prof = _lib.profile_read(ws4.data_ptr(), n4, stream.cuda_stream)
    del d4, ws4
    return {"workload": "cfg4 clustered: 2^22 fp32 spheres (1024 Gaussian clusters), exact contact count + "
                        "inverse-square sum in one sorted pass", "n_gpus": world, "ms_per_step": ms,
            "Gpair_per_s": pairs / (ms * 1e-3) / 1e9, "steps": steps, "count": count, "inv_sum": inv_sum,
            "count_matches_oracle": count == gold.get("count"),
            "sum_rel_err_vs_oracle": (abs(inv_sum - gold["inv_sum"]) / gold["inv_sum"]) if gold else None,
            "split": f"row tiles round-robin over {world} rank(s)",
            "rank0_path_mix": {"gram": prof.chunks_gram, "near": prof.chunks_near, "far": prof.chunks_far,
                               "edge": prof.chunks_edge, "rows_rescanned": prof.rows_rescanned,
                               "exact_checks": prof.exact_checks}}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
