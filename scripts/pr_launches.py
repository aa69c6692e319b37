"""Target for an ncu launch list of the fused PageRank loop (s24, 5 iterations)
and of the plain SpMV, so per-kernel shares can be read off."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
if os.environ.get("MBX_VERTEX_ORDER", "degree") == "degree":  # as bench.py
    P, _ = P.relabel_by_degree()
c = mb.SimtConfig.make(32, 14, 128)
t = mb.generate_tile_for(P, c)
P.build_xcache()
plan = mb.PageRankPlan(P, t, c, mb.PageRankConfig(0.85, 1e-30, 5, 0))
plan.run()
x = torch.rand(P.n_rows, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    mb.spmv_device(P, t, c, x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
print("done")
