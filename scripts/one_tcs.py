"""One headline sum call through PC_TILE_AUTO (sorted FFMA kernel + tensor-core Gram chunks): ncu target."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

n = 2**20
x = gen.random_spheres(n, gen.contact_box_edge(n), 1).astype(np.float32)
(r,) = _lib.pairs_host(x, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
print(r.count, r.sum, _lib.last_profile().kernel)
