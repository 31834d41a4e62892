"""One headline-size call per kernel (for ncu): sorted sum, then the FFMA2 Gram count.

    PAIRCOUNT_LIB=... python scripts/one_call.py [n]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2**20
x = gen.random_spheres(n, gen.contact_box_edge(n), 1).astype(np.float32)
(r1,) = _lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n], tiling=_lib.PC_TILE_SORTED)
(r2,) = _lib.pairs_host(x, _lib.PC_COLLISION, _lib.PC_BALANCED, [0, n], tiling=_lib.PC_TILE_FLAT)
print(r1.count, r1.sum, r2.count)
