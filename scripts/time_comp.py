"""Kernel time of the sum path for f32 (plain direct) vs f64 (compensated) input, N=2^20."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_1901_11204_b200 import _lib, generators as gen

n = 2**20
base = gen.random_spheres(n, gen.contact_box_edge(n), 1)
for dt, code in ((np.float32, _lib.PC_F32), (np.float64, _lib.PC_F64)):
    obj = torch.from_numpy(base.astype(dt)).cuda()
    ws = torch.empty(_lib.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    res = torch.zeros(8, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(2):
        _lib.pairs_async(obj.data_ptr(), code, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, np.array([0, n]),
                         ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, _lib.PC_TILE_FLAT)
    torch.cuda.synchronize()
    _lib.kernel_timing(True)
    for _ in range(3):
        _lib.pairs_async(obj.data_ptr(), code, n, _lib.PC_COLLISION_INVSQ, _lib.PC_BALANCED, np.array([0, n]),
                         ws.data_ptr(), ws.numel(), res.data_ptr(), st.cuda_stream, _lib.PC_TILE_FLAT)
    ms, cnt = _lib.kernel_timing_read()
    _lib.kernel_timing(False)
    torch.cuda.synchronize()
    r = res.cpu().numpy()
    pairs = n * (n - 1) // 2
    print(f"{np.dtype(dt).name}: kernel {ms / cnt:.2f} ms  {pairs / (ms / cnt * 1e-3) / 1e12:.3f} Tpair/s  "
          f"count {int(r[0])} sum {r[1:2].view(np.float64)[0]:.10f}")
