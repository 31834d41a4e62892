"""Per-call latency of the drop-in API at small N (launch-bound regime)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402
from paper_1901_11204_b200 import spi_engine as se  # noqa: E402

for n in (64, 1024, 4096):
    pts = gen.random_spheres(n, 10.0, 1).astype(np.float32)
    for _ in range(20):
        se.spi_balanced(pts, se.collision_indicator)
    t0 = time.perf_counter()
    for _ in range(200):
        se.spi_balanced(pts, se.collision_indicator)
    api = (time.perf_counter() - t0) / 200 * 1e6
    t0 = time.perf_counter()
    for _ in range(200):
        _lib.pairs_host(pts, _lib.PC_COLLISION, _lib.PC_BALANCED, [0, n])
    abi = (time.perf_counter() - t0) / 200 * 1e6
    print(f"n={n}: spi_balanced {api:.1f} us/call, pc_pairs_host via ctypes {abi:.1f} us/call, launches {_lib.launches()}")
