"""Per-warp start/end of the FLAT sum kernels (debug build -DPC_TIMELINE): where a
launch's time goes besides the work -- ramp-up and tail."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

n = 2**20
x = gen.random_spheres(n, gen.contact_box_edge(n), 1).astype(np.float32)
d = torch.from_numpy(x).cuda()
wsb = _lib.workspace_bytes(n)
ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
res = torch.zeros(8, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
# claim area offset: read it from a profile-free route -- the layout places it after the slots
import ctypes  # noqa: E402
for tiling, label in ((_lib.PC_TILE_SORTED, "sorted"), (_lib.PC_TILE_FLAT, "flat")):
    for g in (1, 8):
        for k in range(min(g, 2)):
            ws.zero_()
            _lib.pairs_part_async(d.data_ptr(), _lib.PC_F32, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, 0, n, k, g,
                                  ws.data_ptr(), wsb, res.data_ptr(), st.cuda_stream, tiling)
            torch.cuda.synchronize()
            def al(v, a):
                return (v + a - 1) // a * a
            pair_bytes = al((n // 2 + 1) * 3 * 16, 256)
            slots = 2 * pair_bytes + 512
            max_slots = 148 * 64 + n // (32 * 2 * 4) + 64
            claims = al(slots + max_slots * 64, 256)
            off = claims + ((1 << 20) - 2 * 8192) * 8
            buf = ws[off: off + 2 * 2368 * 8].cpu().numpy().view(np.uint64)
            tl = buf.reshape(-1, 2).astype(np.float64)
            tl = tl[tl[:, 0] > 0]
            t0 = tl[:, 0].min()
            s, e = (tl[:, 0] - t0) / 1e6, (tl[:, 1] - t0) / 1e6
            print(f"{label} part {k}/{g}: warps {len(tl)}  start spread {s.max():.3f} ms  end min {e.min():.3f} "
                  f"p10 {np.percentile(e, 10):.3f} p50 {np.median(e):.3f} p90 {np.percentile(e, 90):.3f} max {e.max():.3f} ms",
                  flush=True)
