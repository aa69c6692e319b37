"""ncu target: BASELINE C1 (R-MAT s20 fp32) -- TILE generation, hub table,
slot copy and a few SpMVs, so the per-kernel split of a small SpMV shows."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

ctx = mb.Context(0)
A = mb.DeviceMatrix.rmat(ctx, 20, 16, seed=1, dtype=np.float32)
c = mb.SimtConfig.make(32, 14, 128)
t = mb.generate_tile_for(A, c)
A.build_xcache()
x = torch.rand(A.n_cols, device="cuda")
y = torch.empty(A.n_rows, device="cuda")
for _ in range(4):
    mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
print("done")
