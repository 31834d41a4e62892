"""count_contacts (Alg. 2) at config-5 size: device time of the lattice call + reset."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

lib = _lib.load()
for n, a in ((2**26, 512), (2**22, 512), (2**20, 64)):
    pts = torch.from_numpy(gen.grid_points(n, a).astype(np.int32)).cuda() if a == 512 else \
        torch.from_numpy(np.random.default_rng(0).integers(-a, a + 1, size=(n, 3)).astype(np.int32)).cuda()
    grid = torch.zeros(int(lib.pc_lattice_grid_cells(a)), dtype=torch.int32, device="cuda")
    keys = torch.empty(n, dtype=torch.int32, device="cuda")
    r = _lib.LatticeResult()
    s = torch.cuda.current_stream()
    for fn in ("pc_lattice_collisions", "pc_lattice_contacts"):
        times = []
        for rep in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _lib.check(getattr(lib, fn)(pts.data_ptr(), _lib.PC_I32, 1, n, a, grid.data_ptr(), keys.data_ptr(), 1,
                                        ctypes.byref(r), ctypes.c_void_p(s.cuda_stream)))
            _lib.check(lib.pc_lattice_clear(grid.data_ptr(), a, ctypes.c_void_p(s.cuda_stream)))
            e1.record(s)
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1))
        print(f"{fn} n={n} a={a}: {np.median(times):.3f} ms (count {r.count}, cells {r.cells_touched})", flush=True)
