import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1901_11204_b200 import _lib, generators as gen, spi_engine as se
objs = gen.random_spheres(2**20, 163.7681743084811, 1).astype(np.float32)
n=len(objs)
b = se.spi_balanced(objs, se.collision_indicator).total
sums=set(); counts=set()
for k in range(12):
    (r,) = _lib.pairs_host(objs, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n])
    sums.add(r.sum); counts.add(r.count)
print("count ref", b, "counts", counts, "distinct sums", len(sums), sorted(sums)[:3])
(rf,) = _lib.pairs_host(objs, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, n], tiling=_lib.PC_TILE_FLAT)
print("flat", rf.count, rf.sum)
