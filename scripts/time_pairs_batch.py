"""Time oracle_collisions_batch (1000 chains x 1024 beads): end to end and the kernel under ncu."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1901_11204_b200 import generators as gen  # noqa: E402
from paper_1901_11204_b200 import lattice_counter as lc  # noqa: E402

chains = [gen.random_chain(1024, 7000 + v)[0] for v in range(1000)]
lc.oracle_collisions_batch(chains[:8])
for _ in range(3):
    t0 = time.perf_counter()
    got = lc.oracle_collisions_batch(chains)
    print(f"e2e {1e3 * (time.perf_counter() - t0):.2f} ms, total {sum(got)}", flush=True)
