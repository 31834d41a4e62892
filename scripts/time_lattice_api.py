"""Wall time of count_collisions + reset_sparse from host int64 beads (config 5:
2^26 beads, a = 512), next to a plain pageable H2D copy of the same array."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_1901_11204_b200 import generators as gen
from paper_1901_11204_b200 import lattice_counter as lc

n, a = 2**26, 512
pts = np.ascontiguousarray(gen.grid_points(n, a).astype(np.int64))
sp = lc.new_space(a)
for label, fn in (
    ("count_collisions + reset_sparse", lambda: (lc.count_collisions(pts, sp), lc.reset_sparse(sp))),
    ("count_contacts + reset_sparse", lambda: (lc.count_contacts(pts, sp), lc.reset_sparse(sp))),
    ("pageable torch H2D of the int64 array", lambda: torch.from_numpy(pts).cuda()),
):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{label}: min {min(ts[1:]):.1f} ms (all {[round(t, 1) for t in ts]})")
