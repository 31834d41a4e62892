"""Whole-range contact counts at 2^20 (cfg3) and 2^22 clustered (cfg4c): the AUTO path
(pruned sorted count), the tensor cores and the FFMA2 Gram filter; kernel and call time."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_11204_b200 import _lib  # noqa: E402
from paper_1901_11204_b200 import generators as gen  # noqa: E402
from paper_1901_11204_b200 import spi_engine as se  # noqa: E402

st = torch.cuda.current_stream()
for name, n, mk in (("cfg3", 2**20, lambda: gen.random_spheres(2**20, gen.contact_box_edge(2**20), 1)),
                    ("cfg4c", 2**22, lambda: gen.clustered_spheres(2**22))):
    x = mk().astype(np.float32)
    d = torch.from_numpy(x).cuda()
    ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    res = torch.zeros(8, dtype=torch.int64, device="cuda")
    for tname, tiling in (("auto(pruned)", _lib.PC_TILE_AUTO), ("tensor_cores", _lib.PC_TILE_TC),
                          ("ffma_gram", _lib.PC_TILE_FLAT)):
        if name == "cfg4c" and tiling == _lib.PC_TILE_TC:
            continue
        for _ in range(2):
            _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, _lib.PC_COLLISION, _lib.PC_BALANCED, np.array([0, n]),
                             ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, tiling)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _lib.kernel_timing(True)
        e0.record(st)
        reps = 3
        for _ in range(reps):
            _lib.pairs_async(d.data_ptr(), _lib.PC_F32, n, _lib.PC_COLLISION, _lib.PC_BALANCED, np.array([0, n]),
                             ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, tiling)
        e1.record(st)
        torch.cuda.synchronize()
        ms, cnt = _lib.kernel_timing_read()
        _lib.kernel_timing(False)
        prof = _lib.profile_read(ws.data_ptr(), n, st.cuda_stream)
        tot = max(1, prof.chunks_gram + prof.chunks_main + prof.chunks_near + prof.chunks_far + prof.chunks_edge)
        print(f"{name} {tname:13s} kernel {ms / cnt:9.3f} ms  call {e0.elapsed_time(e1) / reps:9.3f} ms  "
              f"count {int(res[0].item())}  pruned {prof.chunks_far / tot:.4f} of {tot} chunks  "
              f"checks {prof.exact_checks}", flush=True)
    t0 = time.perf_counter()
    r = se.spi_balanced(x, se.collision_indicator)
    print(f"{name} spi_balanced(collision_indicator) {1e3 * (time.perf_counter() - t0):.1f} ms total {r.total}",
          flush=True)
    del d, ws
