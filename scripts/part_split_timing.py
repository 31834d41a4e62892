import sys, json
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1901_11204_b200 import _lib
from tests.helpers import config_input
cfgs = json.load(open("tests/golden/golden_configs.json"))
x = config_input(cfgs, "cfg3"); n = len(x)
d = torch.from_numpy(x).cuda()
ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
res = torch.zeros(8, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
for g in (1, 8):
    for rep in range(2):
        _lib.kernel_timing(True)
        for k in range(g):
            _lib.pairs_part_async(d.data_ptr(), _lib.PC_F32, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, 0, n, k, g,
                                  ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, _lib.PC_TILE_SORTED)
        (fm, fc), (tm, tc) = _lib.kernel_timing_read_split()
        _lib.kernel_timing(False)
    print(g, "ffma per part", round(fm / g, 3), "tc per part", round(tm / g, 3))
