"""A-B driver for one SpMV (K2 + K3) on R-MAT: python scripts/prof/spmv_iter.py
[scale] [f32|f64] [reps] [transition 0|1] [relabel 0|1].  Env SMEM / MODE set
the K2 shared-memory budget and staging mode (0 LDG, 1 L2 prefetch, 2 TMA)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_07391_b200 as mb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dt = np.float64 if (len(sys.argv) > 2 and sys.argv[2] == "f64") else np.float32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 100
trans = int(sys.argv[4]) if len(sys.argv) > 4 else 0
relabel = int(sys.argv[5]) if len(sys.argv) > 5 else 0
ctx = mb.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
if os.environ.get("SMEM") or os.environ.get("MODE"):
    ctx.set_tuning(32, 1, -1, smem_per_sm=int(os.environ.get("SMEM", -1)),
                   prefetch=int(os.environ.get("MODE", -1)))
A = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=bool(trans), dtype=dt)
if relabel:
    A, _ = A.relabel_by_degree(want_rank=False)
c = mb.SimtConfig.make(32, 14 if dt == np.float32 else 7, 128)
t = mb.generate_tile_for(A, c)
A.build_xcache()
tdt = torch.float32 if dt == np.float32 else torch.float64
x = torch.rand(A.n_cols, device="cuda", dtype=tdt)
y = torch.empty(A.n_rows, device="cuda", dtype=tdt)
for _ in range(5):
    mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(reps):
    mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
e1.record(s)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
m, n = A.nnz, A.n_rows
vs = 4 if dt == np.float32 else 8
b = m * (vs + 4) + 2 * n * vs + 4 * (n + 1)
print(f"spmv s{scale} {'f32' if vs == 4 else 'f64'} trans {trans} relabel {relabel} smem "
      f"{os.environ.get('SMEM', '-')} mode {os.environ.get('MODE', '-')} hubs {A.xcache_info()[0]}: "
      f"{us:.1f} us, {b / us / 1e3:.0f} GB/s, ysum {float(y.double().sum()):.6e}", flush=True)
