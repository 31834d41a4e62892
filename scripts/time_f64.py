"""Float64 inputs at 2^20: the compensated sum (input order) vs the sorted compensated sum,
and the f32 sorted sum for reference."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

n = 2**20
x64 = gen.random_spheres(n, gen.contact_box_edge(n), 1)
st = torch.cuda.current_stream()
for label, x, code, tiling in (("f64 flat (compensated)", x64, _lib.PC_F64, _lib.PC_TILE_FLAT),
                               ("f64 sorted (compensated)", x64, _lib.PC_F64, _lib.PC_TILE_SORTED),
                               ("f32 sorted", x64.astype(np.float32), _lib.PC_F32, _lib.PC_TILE_SORTED)):
    d = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    res = torch.zeros(8, dtype=torch.int64, device="cuda")
    _lib.pairs_async(d.data_ptr(), code, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, np.array([0, n]),
                     ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, tiling)
    torch.cuda.synchronize()
    _lib.kernel_timing(True)
    for _ in range(3):
        _lib.pairs_async(d.data_ptr(), code, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, np.array([0, n]),
                         ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, tiling)
    ms, cnt = _lib.kernel_timing_read()
    _lib.kernel_timing(False)
    prof = _lib.profile_read(ws.data_ptr(), n, st.cuda_stream)
    s = float(np.array([res[1].item()], dtype=np.int64).view(np.float64)[0])
    tot = max(1, prof.chunks_gram + prof.chunks_main + prof.chunks_near + prof.chunks_far + prof.chunks_edge)
    print(f"{label:26s} {ms / cnt:8.2f} ms  {n * (n - 1) / 2 / (ms / cnt * 1e-3) / 1e12:5.2f} Tpair/s  count "
          f"{int(res[0].item())}  sum {s!r}  gram {prof.chunks_gram / tot:.3f}", flush=True)
