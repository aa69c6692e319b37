"""BiCGSTAB (the paper's second workload) on the device: the C5-style
27-point stencil (diagonally dominant, fp64) at a given grid, b = A * x_true,
reporting passes, device seconds per pass and the SpMV share (3 per pass)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402
from paper_2605_07391_b200 import _lib  # noqa: E402
import ctypes as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=200)
ap.add_argument("--dtype", default="f64")
ap.add_argument("--tol", type=float, default=1e-10)
ap.add_argument("--max-iters", type=int, default=200)
args = ap.parse_args()
dt = np.float64 if args.dtype == "f64" else np.float32
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = mb.Context(0)
ctx.set_stream(stream.cuda_stream)  # events below time the library's own stream
A = mb.DeviceMatrix.stencil27(ctx, args.grid, dt)
c = mb.SimtConfig.make(32, 7 if dt == np.float64 else 14, 128)
t = mb.generate_tile_for(A, c)
n = A.n_rows
rng = np.random.default_rng(1)
x_true = rng.uniform(-1, 1, n).astype(dt)
tdt = torch.float64 if dt == np.float64 else torch.float32
xd = torch.from_numpy(x_true).cuda()
yd = torch.empty(n, dtype=tdt, device="cuda")
mb.spmv_device(A, t, c, xd.data_ptr(), yd.data_ptr())
torch.cuda.synchronize()
b = yd.cpu().numpy()
# SpMV time for the share
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    mb.spmv_device(A, t, c, xd.data_ptr(), yd.data_ptr())
e1.record()
torch.cuda.synchronize()
spmv_s = e0.elapsed_time(e1) * 1e-3 / 10
be = type("B", (), {})()
be.matrix, be.tile_, be.c = A, t, c
r = mb.bicgstab(None, b, mb.BicgstabConfig(tol=args.tol, max_iters=args.max_iters), backend=be)
err = float(np.abs(r.x.astype(np.float64) - x_true).max())
print(json.dumps({"grid": args.grid, "n": n, "nnz": A.nnz, "dtype": args.dtype,
                  "status": r.status, "passes": r.iterations, "final_residual": r.final_residual,
                  "iterate_s": r.iterate_seconds,
                  "ms_per_pass": 1e3 * r.iterate_seconds / max(r.iterations, 1),
                  "spmv_ms": spmv_s * 1e3,
                  "spmv_share": 3 * spmv_s * r.iterations / max(r.iterate_seconds, 1e-30),
                  "max_abs_err_vs_x_true": err}))
