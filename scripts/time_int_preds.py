"""Integer all-pairs predicates at scale: oracle_collisions /
oracle_contacts at N = 2^20 integer points, per tiling, kernel time + counts."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

n = 2**20
st = torch.cuda.current_stream()
for std in (64.0, 16.0):
    pts = gen.normal_cloud(n, std, 512, 3)
    d = torch.from_numpy(pts.astype(np.int32)).cuda()
    ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    res = torch.zeros(8, dtype=torch.int64, device="cuda")
    _, counts = np.unique(pts, axis=0, return_counts=True)
    want = int((counts * (counts - 1) // 2).sum())
    for inter, name in ((_lib.PC_COINCIDE, "coincide"), (_lib.PC_MANHATTAN1, "manhattan1")):
        for tiling, tname in ((_lib.PC_TILE_FLAT, "ffma_gram"), (_lib.PC_TILE_TC, "tensor_cores"),
                              (getattr(_lib, "PC_TILE_KEY", None), "int32_key")):
            if tiling is None or (tname == "int32_key" and inter != _lib.PC_COINCIDE):
                continue
            try:
                for _ in range(2):
                    _lib.pairs_async(d.data_ptr(), _lib.PC_I32, n, inter, _lib.PC_BALANCED, np.array([0, n]),
                                     ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, tiling)
                torch.cuda.synchronize()
                _lib.kernel_timing(True)
                for _ in range(3):
                    _lib.pairs_async(d.data_ptr(), _lib.PC_I32, n, inter, _lib.PC_BALANCED, np.array([0, n]),
                                     ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, tiling)
                ms, cnt = _lib.kernel_timing_read()
                _lib.kernel_timing(False)
                torch.cuda.synchronize()
                c = int(res[0].item())
                print(f"std={std} {name:10s} {tname:12s} {ms / cnt:8.3f} ms  {n * (n - 1) / 2 / (ms / cnt * 1e-3) / 1e12:6.3f} Tpair/s"
                      f"  count {c}  checks {int(res[3].item())}" + (f"  unique-oracle {want}" if name == "coincide" else ""),
                      flush=True)
            except Exception as e:  # noqa: BLE001
                print(std, name, tname, "ERROR", e, flush=True)
