"""ncu target: SpMV (K2+K3) on the BASELINE C5 27-point stencil (400^3) and the
C3 power-law matrix, a few launches each."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c5"
dt = np.float64 if (len(sys.argv) < 3 or sys.argv[2] == "f64") else np.float32
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
A = (mb.DeviceMatrix.stencil27(ctx, 400, dt) if which == "c5"
     else mb.DeviceMatrix.powerlaw(ctx, 22, seed=3, dtype=dt))
c = mb.SimtConfig.make(32, 7 if dt == np.float64 else 14, 128)
t = mb.generate_tile_for(A, c)
A.build_xcache()
tdt = torch.float64 if dt == np.float64 else torch.float32
x = torch.rand(A.n_cols, device="cuda", dtype=tdt)
y = torch.empty(A.n_rows, device="cuda", dtype=tdt)
for _ in range(4):
    mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
print("done")
