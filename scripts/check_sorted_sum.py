import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1901_11204_b200 import _lib, generators as gen
from oracle import c_oracle
rng = np.random.default_rng(3)
cases = []
n = 65536
cases.append(("uniform cfg2", gen.random_spheres(n, gen.contact_box_edge(n), 0).astype(np.float32)))
cases.append(("uniform big box", (rng.random((n, 3)) * 500).astype(np.float32)))
k = 64
cent = rng.random((k, 3)) * 300
cases.append(("clustered", (cent[rng.integers(0, k, n)] + rng.normal(size=(n, 3)) * 2.0).astype(np.float32)))
p = rng.random((n, 3)) * 20; p[n // 2:] += 1e4
cases.append(("two far clusters", p.astype(np.float32)))
cases.append(("offset 1e4", (rng.random((n, 3)) * 60 + 1e4).astype(np.float32)))
cases.append(("thin slab", (rng.random((n, 3)) * np.array([400, 400, 1.0])).astype(np.float32)))
for name, pts in cases:
    t = time.time()
    wc, ws, _ = c_oracle.rows(pts, 0, len(pts), "balanced")
    (r,) = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, len(pts)])
    (rf,) = _lib.pairs_host(pts, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, [0, len(pts)], tiling=_lib.PC_TILE_FLAT)
    print(f"{name:18s} count {r.count} want {wc} {'OK' if r.count == wc else 'BAD'}  sum rel err {abs(r.sum - ws) / ws:.2e} "
          f"(unsorted path? {abs(rf.sum - ws) / ws:.2e})  oracle {time.time() - t:.1f}s", flush=True)
