"""SpMV time with and without the x hub table: python scripts/prof/hub_gain.py
(C1: R-MAT s20 fp32 U[0,1); s22/s24 natural transition fp32)."""
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
for name, scale, trans in [("c1_s20", 20, False), ("s22", 22, True), ("s24", 24, True)]:
    A = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=trans, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(A, c)
    x = torch.rand(A.n_cols, device="cuda")
    y = torch.empty(A.n_rows, device="cuda")
    res = []
    for hubs in (-1, 0):
        A.build_xcache(hubs)
        for _ in range(3):
            mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(50):
            mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        e1.record(s)
        torch.cuda.synchronize()
        res.append((A.xcache_info()[0], e0.elapsed_time(e1) / 50 * 1e3))
    print(name, "hubs", res[0][0], f"{res[0][1]:.1f} us", "| no hubs", f"{res[1][1]:.1f} us", flush=True)
