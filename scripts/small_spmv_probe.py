"""Small-matrix SpMV probe (BASELINE C1 scale and below): K2+K3 time with the
default launch vs the next-tile L2 prefetch and without the hub table."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402
from bench import time_device  # noqa: E402

st = torch.cuda.Stream()
torch.cuda.set_stream(st)
for scale in (18, 20, 22):
    for name, kw in (("default", {}), ("prefetch", {"prefetch": 1}), ("no_hubs", {"max_hubs": 0})):
        ctx = mb.Context(0)
        ctx.set_stream(st.cuda_stream)
        ctx.set_tuning(**kw)
        A = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, dtype=np.float32)
        c = mb.SimtConfig.make(32, 14, 128)
        t = mb.generate_tile_for(A, c)
        A.build_xcache(0 if kw.get("max_hubs") == 0 else -1)
        x = torch.rand(A.n_cols, device="cuda")
        y = torch.empty(A.n_rows, device="cuda")
        for _ in range(3):
            mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        ts = time_device(st, lambda: mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr()), 100)
        print(scale, name, round(ts * 1e6, 1), "us", flush=True)
        del A, t, ctx
