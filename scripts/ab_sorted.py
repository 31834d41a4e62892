"""A/B timing of library builds on the headline workload (one process per build).

    PAIRCOUNT_LIB=path python scripts/ab_sorted.py [reps]
Prints the sorted-sum kernel time (CUDA events on the launching stream) and the
count kernels at N = 2^20."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = 2**20
x = gen.random_spheres(n, gen.contact_box_edge(n), 1).astype(np.float32)
d = torch.from_numpy(x).cuda()
ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
res = torch.zeros(8, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
out = {}
for label, inter, tiling in (("sorted_sum", _lib.PC_COLLISION_INVSQ, _lib.PC_TILE_SORTED),
                             ("flat_sum", _lib.PC_COLLISION_INVSQ, _lib.PC_TILE_FLAT),
                             ("gram_count", _lib.PC_COLLISION, _lib.PC_TILE_FLAT)):
    for _ in range(2):
        _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, inter, _lib.PC_BALANCED, np.array([0, n]), ws.data_ptr(),
                         ws.numel(), res.data_ptr(), st.cuda_stream, tiling)
    torch.cuda.synchronize()
    _lib.kernel_timing(True)
    for _ in range(reps):
        _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, inter, _lib.PC_BALANCED, np.array([0, n]), ws.data_ptr(),
                         ws.numel(), res.data_ptr(), st.cuda_stream, tiling)
    ms, cnt = _lib.kernel_timing_read()
    _lib.kernel_timing(False)
    torch.cuda.synchronize()
    out[label] = round(ms / cnt, 3)
    out[label + "_count"] = int(res[0].item())
print(os.environ.get("PAIRCOUNT_LIB", "default"), out, flush=True)
