"""Design estimate (CPU, numpy): the share of the sorted sum's chunks tcs_takes() accepts when the
tile centre o is replaced by the centre of a group of G consecutive tiles (the column operand of a
chunk could then serve the G items (t + k, c - k) along its diagonal).

    python scripts/sim_tcs_groups.py [cfg3|cfg4u|cfg4c] [G ...]
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from tests.helpers import config_input  # noqa: E402


def spread10(v):
    v = v.astype(np.uint32)
    v = (v | (v << 16)) & 0x030000FF
    v = (v | (v << 8)) & 0x0300F00F
    v = (v | (v << 4)) & 0x030C30C3
    v = (v | (v << 2)) & 0x09249249
    return v


def morton_sorted(x):
    mn, mx = x.min(0).astype(np.float64), x.max(0).astype(np.float64)
    sc = np.where(mx > mn, 1023.0 / (mx - mn), 0.0).astype(np.float32)
    c = np.clip(((x - mn.astype(np.float32)) * sc), 0, 1023).astype(np.uint32)
    key = spread10(c[:, 0]) | (spread10(c[:, 1]) << 1) | (spread10(c[:, 2]) << 2)
    return x[np.argsort(key, kind="stable")]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    gs = [int(g) for g in sys.argv[2:]] or [1, 2, 4, 8]
    cfgs = json.loads((ROOT / "tests" / "golden" / "golden_configs.json").read_text())
    x = morton_sorted(config_input(cfgs, name))
    n = len(x)
    T = W = 256
    blk = x[: n // 32 * 32].reshape(-1, 32, 3)
    bmin, bmax = blk.min(1), blk.max(1)
    nt = n // T
    tmin, tmax = bmin.reshape(nt, 8, 3).min(1), bmax.reshape(nt, 8, 3).max(1)
    L = T - 1 + n // 2
    steps_min = (n - 1) // 2 if n & 1 else n // 2 - 1
    cpw = (L + W - 1) // W
    offs = np.arange(cpw) * W
    dense = (offs + W <= L) & (offs + 1 >= T) & (offs + W <= steps_min)
    nblk = len(bmin)
    # chunk boxes: chunk starting at column 256 m + 1 covers blocks 8m .. 8m + 8
    idx = (8 * np.arange(n // W)[:, None] + np.arange(9)[None, :]) % nblk
    cmin, cmax = bmin[idx].min(1), bmax[idx].max(1)
    f = np.float32
    for G in gs:
        ng = nt // G
        gmin = tmin[: ng * G].reshape(ng, G, 3).min(1)
        gmax = tmax[: ng * G].reshape(ng, G, 3).max(1)
        taken = 0
        total = 0
        for t in range(ng * G):
            o = f(0.5) * (gmin[t // G] + gmax[t // G])
            rt = np.maximum(np.abs(tmin[t] - o), np.abs(tmax[t] - o))
            rt2 = f((rt * rt).sum())
            m = (t * T // W + np.arange(cpw)) % (n // W)  # chunk c starts at 256 (t + c) + 1
            cl, ch = cmin[m], cmax[m]
            d = np.maximum(0, np.maximum(cl - tmax[t], tmin[t] - ch))
            gap2 = (d * d).sum(1, dtype=f)
            bb = np.maximum(np.abs(cl - o), np.abs(ch - o))
            ab = np.sqrt(rt2) + np.sqrt((bb * bb).sum(1, dtype=f))
            ok = dense & (gap2 > 4.5) & (ab <= 3e4) & (f(2.98023223876953125e-07) * ab * ab <= f(3.125e-6) * (1 + gap2))
            taken += int(ok.sum())
            total += int(dense.sum())
        print(json.dumps({"workload": name, "G": G, "dense_chunks": total, "taken": taken, "frac": round(taken / total, 4)}),
              flush=True)


if __name__ == "__main__":
    main()
