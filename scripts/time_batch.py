import time, numpy as np, sys
sys.path.insert(0, '.')
from paper_1901_11204_b200 import generators as gen, lattice_counter as lc
chains=[gen.random_chain(1024, 7000+v)[0] for v in range(1000)]
ext=max(int(np.abs(c).max()) for c in chains); sp=lc.new_space(ext)
for _ in range(3): lc.count_collisions_batch(chains, sp)
t=time.perf_counter()
for _ in range(10): r=lc.count_collisions_batch(chains, sp)
print("vectors path ms/exec", (time.perf_counter()-t)/10*1e3, sum(x.count for x in r))
