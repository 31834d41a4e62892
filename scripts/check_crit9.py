import sys, tempfile
sys.path.insert(0, '.')
import numpy as np
from pathlib import Path
from paper_1901_11204_b200.bench_cli import BenchConfig, run_linear_vs_quadratic
for trial in range(3):
    cfg = BenchConfig(sizes=[64,128,256,512,1024], vectors=10, reps=3, seed=0, out=Path(tempfile.mkdtemp())/"l.csv")
    rows = run_linear_vs_quadratic(cfg)
    means = {}
    for r in rows: means.setdefault((r["algorithm"], r["n"]), []).append(r["wall_ns"])
    print({n: round(np.mean(means[("quadratic", n)]) / np.mean(means[("linear", n)]),2) for n in cfg.sizes})
