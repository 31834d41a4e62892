"""Device-pointer pc_lattice_collisions, dense regime, caller-owned keys (debug)."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

lib = _lib.load()
for a, nb, pad in ((64, 2**21, 0), (64, 2**21, 1 << 20), (40, 3000, 0)):
    beads = gen._rng(31, 5).integers(-a, a + 1, size=(nb, 3), dtype=np.int64).astype(np.int32)
    db = torch.from_numpy(beads).cuda()
    cells = int(lib.pc_lattice_grid_cells(a))
    grid = torch.zeros(cells + pad, dtype=torch.int32, device="cuda")
    keys = torch.zeros(nb + pad, dtype=torch.int32, device="cuda")
    r = _lib.LatticeResult()
    rc = lib.pc_lattice_collisions(db.data_ptr(), _lib.PC_I32, 1, nb, a, grid.data_ptr(), keys.data_ptr(), 1,
                                   ctypes.byref(r), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    print(a, nb, pad, rc, _lib.last_error() if rc else "", r.count, r.cells_touched, flush=True)
    if rc:
        break
