"""Per-launch overhead of the FLAT kernels: one whole-range call vs the same
work as G tile parts (pc_pairs_part_async), kernel time summed over the parts."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2**20
x = gen.random_spheres(n, gen.contact_box_edge(n), 1).astype(np.float32)
d = torch.from_numpy(x).cuda()
ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
res = torch.zeros(8, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
for label, inter, tiling in (("sorted_sum", _lib.PC_COLLISION_INVSQ, _lib.PC_TILE_SORTED),
                             ("flat_sum", _lib.PC_COLLISION_INVSQ, _lib.PC_TILE_FLAT),
                             ("gram_count", _lib.PC_COLLISION, _lib.PC_TILE_FLAT)):
    row = {}
    for g in (1, 2, 8):
        for rep in range(2):
            _lib.kernel_timing(True)
            for k in range(g):
                _lib.pairs_part_async(d.data_ptr(), _lib.PC_F32, n, inter, _lib.PC_BALANCED, 0, n, k, g, ws.data_ptr(),
                                      ws.numel(), res.data_ptr(), st.cuda_stream, tiling)
            ms, cnt = _lib.kernel_timing_read()
            _lib.kernel_timing(False)
            torch.cuda.synchronize()
        prof = _lib.profile_read(ws.data_ptr(), n, st.cuda_stream)
        row[g] = round(ms, 3)
        row[f"claims{g}"] = prof.claims
    print(label, row, flush=True)
