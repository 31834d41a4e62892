"""The GPU harness keeps the reference CLI's contract (test_bench_cli.py of the
reference: CSV schema, append safety, exit codes, verify determinism)."""

from __future__ import annotations

import csv

import pytest

from paper_1901_11204_b200 import bench_cli
from paper_1901_11204_b200.bench_cli import CSV_COLUMNS, BenchConfig, main


def _read(path):
    with open(path, newline="") as fh:
        return list(csv.DictReader(fh))


def test_config_error_exit_code(tmp_path):
    assert main(["bench", "linear-vs-quadratic", "--sizes", "", "--out", str(tmp_path / "r.csv")]) == bench_cli.EXIT_CONFIG
    with pytest.raises(ValueError):
        BenchConfig(sizes=[8], reps=0)


def test_csv_schema_matches_reference():
    assert CSV_COLUMNS == ["experiment", "algorithm", "n", "rep", "wall_ns", "result", "cells_touched", "space_cells"]
    assert (bench_cli.EXIT_OK, bench_cli.EXIT_MISMATCH, bench_cli.EXIT_CONFIG, bench_cli.EXIT_RESOURCE) == (0, 1, 2, 3)


@pytest.mark.gpu
def test_linear_vs_quadratic_rows_and_append(tmp_path):
    out = tmp_path / "raw.csv"
    cfg = BenchConfig(sizes=[16, 32], vectors=3, reps=2, seed=1, out=out)
    rows = bench_cli.run_linear_vs_quadratic(cfg)
    assert len(rows) == 8
    disk = _read(out)
    assert list(disk[0].keys()) == CSV_COLUMNS
    for lin, quad in zip(disk[::2], disk[1::2]):
        assert lin["algorithm"] == "linear" and quad["algorithm"] == "quadratic"
        assert lin["result"] == quad["result"]
    bench_cli.run_linear_vs_quadratic(cfg)
    with open(out) as fh:
        assert sum(line.startswith("experiment,") for line in fh) == 1


@pytest.mark.gpu
def test_realloc_locality_spi(tmp_path):
    out = tmp_path / "raw.csv"
    rows = bench_cli.run_realloc_sweep(BenchConfig(sizes=[32], vectors=10, reps=2, seed=3,
                                                   realloc_every=[1, 4, 0], out=out))
    by_k = {}
    for r in rows:
        by_k.setdefault(r["algorithm"], []).append(r["result"])
    assert len(by_k) == 3 and len({tuple(v) for v in by_k.values()}) == 1
    rows = bench_cli.run_locality_sweep(BenchConfig(sizes=[100], vectors=2, reps=1, seed=5, std_devs=[1.0, 10.0],
                                                    out=out))
    assert {r["algorithm"] for r in rows} == {"linear-std1", "linear-std10"}
    rows = bench_cli.run_spi_compare(BenchConfig(sizes=[60, 61], vectors=1, reps=2, workers=3, out=out))
    for n in (60, 61):
        assert len({r["result"] for r in rows if r["n"] == n}) == 1


@pytest.mark.gpu
def test_verify_quick_passes_and_is_deterministic(tmp_path, capsys):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert bench_cli.verify("quick", seed=7, out=a)
    assert "pass schedule-completeness" in capsys.readouterr().out
    assert bench_cli.verify("quick", seed=7, out=b)
    assert a.read_bytes() == b.read_bytes()
    assert main(["verify", "quick", "--out", str(tmp_path / "v.csv")]) == 0


@pytest.mark.gpu
def test_mismatch_exit_code(tmp_path, monkeypatch):
    monkeypatch.setattr(bench_cli, "oracle_collisions_batch", lambda vectors: [-1 for _ in vectors])
    rc = main(["bench", "linear-vs-quadratic", "--sizes", "8", "--vectors", "1", "--reps", "1",
               "--out", str(tmp_path / "raw.csv")])
    assert rc == bench_cli.EXIT_MISMATCH
