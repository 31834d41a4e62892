"""Sorted sum at 2^20: kernel time, path mix and accuracy vs the full-size oracle total."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402

gold = json.loads((Path(__file__).resolve().parent.parent / "tests/golden/golden_full.json").read_text())
for name, n, mk in (("cfg3", 2**20, lambda: gen.random_spheres(2**20, gen.contact_box_edge(2**20), 1)),
                    ("cfg4c", 2**22, lambda: gen.clustered_spheres(2**22))):
    x = mk().astype(np.float32)
    d = torch.from_numpy(x).cuda()
    ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    res = torch.zeros(8, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    reps = 5 if n == 2**20 else 2
    for _ in range(2):
        _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, np.array([0, n]),
                         ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, _lib.PC_TILE_SORTED)
    torch.cuda.synchronize()
    _lib.kernel_timing(True)
    for _ in range(reps):
        _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, np.array([0, n]),
                         ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, _lib.PC_TILE_SORTED)
    ms, cnt = _lib.kernel_timing_read()
    _lib.kernel_timing(False)
    prof = _lib.profile_read(ws.data_ptr(), n, st.cuda_stream)
    s = float(np.array([res[1].item()], dtype=np.int64).view(np.float64)[0])
    tot = prof.chunks_gram + prof.chunks_near + prof.chunks_far + prof.chunks_main + prof.chunks_edge
    print(os.environ.get("PAIRCOUNT_LIB", "default"), name, f"{ms / cnt:.3f} ms", f"gram {prof.chunks_gram / tot:.4f}",
          f"far {prof.chunks_far / tot:.4f}", f"near {prof.chunks_near / tot:.4f}",
          f"count_ok {int(res[0].item()) == gold[name]['count']}",
          f"rel_err {abs(s - gold[name]['inv_sum']) / gold[name]['inv_sum']:.3e}", flush=True)
    del d, ws
