"""Tile parts of the 2^20 headline sum, each part timed alone (CUDA events): max / min ms per part count.

    [PAIRCOUNT_LIB=...] python scripts/part_split_timing2.py
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1901_11204_b200 import _lib  # noqa: E402
from tests.helpers import config_input  # noqa: E402

cfgs = json.loads((ROOT / "tests" / "golden" / "golden_configs.json").read_text())
x = config_input(cfgs, "cfg3")
n = len(x)
d = torch.from_numpy(x).cuda()
ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
res = torch.zeros(6, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
for g in (1, 2, 4, 8):
    ts = [timed(lambda k=k: _lib.pairs_part_async(d.data_ptr(), _lib.PC_F32, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED,
                                                  0, n, k, g, ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream,
                                                  _lib.PC_TILE_SORTED)) for k in range(g)]
    out[g] = (round(max(ts), 3), round(min(ts), 3))
print(json.dumps(out))
