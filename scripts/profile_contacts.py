import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_1901_11204_b200 import _lib, generators as gen
lib = _lib.load()
n, a = 2**26, 512
pts = torch.from_numpy(gen.grid_points(n, a).astype(np.int32)).cuda()
grid = torch.zeros(int(lib.pc_lattice_grid_cells(a)), dtype=torch.int32, device="cuda")
keys = torch.empty(n, dtype=torch.int32, device="cuda")
r = _lib.LatticeResult()
s = torch.cuda.current_stream()
for _ in range(2):
    _lib.check(lib.pc_lattice_contacts(pts.data_ptr(), _lib.PC_I32, 1, n, a, grid.data_ptr(), keys.data_ptr(), 1, ctypes.byref(r), ctypes.c_void_p(s.cuda_stream)))
    _lib.check(lib.pc_lattice_clear(grid.data_ptr(), a, ctypes.c_void_p(s.cuda_stream)))
torch.cuda.synchronize()
print(r.count, r.cells_touched)
