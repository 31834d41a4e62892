"""Tensor-core count kernel timing at 2^20 (PC_TILE_TC, balanced, whole range): device time per call
(CUDA events around the call) and the count.   PAIRCOUNT_LIB=... python scripts/time_tc_count.py"""
import json, os, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1901_11204_b200 import _lib  # noqa: E402
from tests.helpers import config_input  # noqa: E402
cfgs = json.loads((ROOT / "tests" / "golden" / "golden_configs.json").read_text())
x = config_input(cfgs, "cfg3"); n = len(x)
d = torch.from_numpy(x).cuda()
ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
res = torch.zeros(6, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
def call():
    _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, _lib.PC_COLLISION, _lib.PC_BALANCED, np.array([0, n]),
                     ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, _lib.PC_TILE_TC)
for _ in range(2): call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): call()
e1.record(); torch.cuda.synchronize()
print(os.environ.get("PAIRCOUNT_LIB", "default"), "tc count 2^20 ms/call", round(e0.elapsed_time(e1) / 5, 3), "count", int(res[0].item()))
