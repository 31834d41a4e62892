"""spi_balanced(points, inverse_square) end to end at 2^20 from a pageable numpy array."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import generators as gen  # noqa: E402
from paper_1901_11204_b200 import spi_engine as se  # noqa: E402

n = 2**20
x = gen.random_spheres(n, gen.contact_box_edge(n), 1).astype(np.float32)
for _ in range(2):
    se.spi_balanced(x, se.inverse_square)
ts = []
for _ in range(8):
    t0 = time.perf_counter()
    r = se.spi_balanced(x, se.inverse_square)
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"e2e spi_balanced inverse_square: median {np.median(ts):.2f} ms min {min(ts):.2f} ms total {r.total!r}")
