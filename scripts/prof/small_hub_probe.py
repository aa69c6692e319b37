"""Small R-MAT SpMV: hub table on/off and staging modes (where does the hub
table start to pay?).  python scripts/prof/small_hub_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_07391_b200 as mb  # noqa: E402

ctx = mb.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
for scale, trans in [(19, False), (20, False), (21, False), (21, True), (22, False)]:
    A = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=trans, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(A, c)
    x = torch.rand(A.n_cols, device="cuda")
    y = torch.empty(A.n_rows, device="cuda")
    out = []
    for hubs, pf in [(-1, 0), (0, 0), (0, 2), (0, 1)]:
        ctx.set_tuning(32, 1, hubs, smem_per_sm=-1, prefetch=pf)
        A.build_xcache(hubs)
        for _ in range(3):
            mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(100):
            mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        e1.record(s)
        torch.cuda.synchronize()
        out.append(f"hubs {hubs:>2} pf {pf}: {e0.elapsed_time(e1) / 100 * 1e3:7.1f} us")
    print(f"s{scale} {'trans' if trans else 'U01'} nnz {A.nnz}: " + " | ".join(out), flush=True)
    ctx.set_tuning(32, 1, -1, smem_per_sm=-1, prefetch=-1)
