"""Sorted fp32 sum with / without the tensor-core Gram chunks (PAIRCOUNT_TCSUM=0 turns them off).

    [PAIRCOUNT_TCSUM=0] python scripts/ab_tcsum.py [reps]
Per workload: the step time (CUDA events around the whole call on the launching stream),
the summed time of the timed kernels, the path profile, and the result against the
full-size float64 oracle totals (tests/golden/golden_full.json)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1901_11204_b200 import _lib  # noqa: E402
from tests.helpers import config_input  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
gold = json.loads((ROOT / "tests" / "golden" / "golden_full.json").read_text())
cfgs = json.loads((ROOT / "tests" / "golden" / "golden_configs.json").read_text())
work = ["cfg3"] + (["cfg4u", "cfg4c"] if os.environ.get("AB_CFG4") else [])
st = torch.cuda.current_stream()
for name in work:
    x = config_input(cfgs, name)
    if os.environ.get("AB_F64"):  # the float64 points the reference's generators return
        x = x.astype(np.float64)
    n = len(x)
    d = torch.from_numpy(x).cuda()
    ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    res = torch.zeros(6, dtype=torch.int64, device="cuda")

    def call():
        _lib.pairs_async(d.data_ptr(), _lib.PC_F64 if x.dtype == np.float64 else _lib.PC_F32, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, np.array([0, n]),
                         ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, _lib.PC_TILE_AUTO)

    for _ in range(2):
        call()
    torch.cuda.synchronize()
    _lib.kernel_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    (fms, fcnt), (tms, tcnt) = _lib.kernel_timing_read_split()
    kms, cnt = fms + tms, fcnt + tcnt
    _lib.kernel_timing(False)
    step = e0.elapsed_time(e1) / reps
    r = _lib.PairsResult.from_buffer_copy(res.cpu().numpy().tobytes())
    prof = _lib.profile_read(ws.data_ptr(), n, st.cuda_stream).as_dict()
    g = gold[name]
    rel = abs(r.sum - g["inv_sum"]) / g["inv_sum"]
    print(json.dumps({"workload": name + (" f64" if x.dtype == np.float64 else ""), "tcsum": os.environ.get("PAIRCOUNT_TCSUM", "1"), "step_ms": round(step, 3),
                      "timed_kernels_ms": round(kms / reps, 3), "ffma_ms": round(fms / reps, 3), "tc_ms": round(tms / reps, 3), "launches_per_step": cnt / reps,
                      "count": r.count, "count_ok": r.count == g["count"], "sum": r.sum, "sum_rel_err": rel,
                      "pairs": r.pairs, "error": r.error, "profile": prof}), flush=True)
