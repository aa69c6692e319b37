import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2605_07391_b200 as mb
ctx = mb.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
A = mb.DeviceMatrix.rmat(ctx, 20, 16, seed=1, dtype=np.float32)
x = torch.rand(A.n_cols, device="cuda"); y = torch.empty(A.n_rows, device="cuda")
for b in (128, 256, 512, 1024):
  c = mb.SimtConfig.make(32, 14, b)
  t = mb.generate_tile_for(A, c)
  for (w, cps) in [(32, 1), (16, 2), (8, 4)]:
    ctx.set_tuning(w, cps, -1)
    A.build_xcache()
    for _ in range(3): mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(200): mb.spmv_device(A, t, c, x.data_ptr(), y.data_ptr())
    e1.record(s); torch.cuda.synchronize()
    print(b, w, cps, A.xcache_info()[0], f"{e0.elapsed_time(e1)/200*1e3:.1f} us", flush=True)
