"""C1 (R-MAT s20 fp32 SpMV, no hub table) across K2 launch shapes:
  python scripts/prof/c1_shape.py"""
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
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dt = np.float64 if os.environ.get("F64") else np.float32
A = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, dtype=dt)
tdt = torch.float64 if dt == np.float64 else torch.float32
x = torch.rand(A.n_cols, device="cuda", dtype=tdt)
y = torch.empty(A.n_rows, device="cuda", dtype=tdt)
c = mb.SimtConfig.make(32, 14 if dt == np.float32 else 7, 128)
t = mb.generate_tile_for(A, c)
for rep in range(2):
    for (w, cps) in [tuple(int(v) for v in s.split("x")) for s in os.environ.get("SHAPES", "0x0,32x1,16x2,8x4").split(",")]:
        ctx.set_tuning(w, cps, -1, prefetch=int(os.environ.get("MODE", -1)))
        A.build_xcache()
        for _ in range(3):
            mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(200):
            mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
        e1.record(s)
        torch.cuda.synchronize()
        print(f"s{scale} mode {os.environ.get('MODE', '-')} {w}x{cps} hubs {A.xcache_info()[0]}: "
              f"{e0.elapsed_time(e1) / 200 * 1e3:.1f} us", flush=True)
