"""K2 launch shape x staging mode sweep of the plain SpMV on a bench matrix:
  python scripts/prof/spmv_shape.py c5|c3|s24 f32|f64"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_07391_b200 as mb  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c5"
dt = np.float64 if (len(sys.argv) < 3 or sys.argv[2] == "f64") else np.float32
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
A = (mb.DeviceMatrix.stencil27(ctx, 400, dt) if which == "c5"
     else mb.DeviceMatrix.powerlaw(ctx, 22, seed=3, dtype=dt) if which == "c3"
     else mb.DeviceMatrix.rmat(ctx, 24, 16, seed=1, transition=True, dtype=dt))
c = mb.SimtConfig.make(32, 7 if dt == np.float64 else 14, 128)
t = mb.generate_tile_for(A, c)
tdt = torch.float64 if dt == np.float64 else torch.float32
x = torch.rand(A.n_cols, device="cuda", dtype=tdt)
y = torch.empty(A.n_rows, device="cuda", dtype=tdt)
reps = 20
for rep in range(2):
    for (w, cps, mode) in [(0, 0, -1), (32, 1, 0), (32, 1, 1), (32, 1, 2), (16, 2, 0),
                           (16, 2, 1), (16, 2, 2), (24, 1, 1)]:
        ctx.set_tuning(w, cps, -1, prefetch=mode)
        A.build_xcache()
        for _ in range(2):
            mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        e1.record(s)
        torch.cuda.synchronize()
        print(f"{which} {sys.argv[2] if len(sys.argv) > 2 else 'f64'} {w}x{cps} mode {mode} "
              f"hubs {A.xcache_info()[0]}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us", flush=True)
