"""Probe: does spreading x's 128-byte lines over the L2 slices help the
gather-bound SpMV?  Re-labels columns by a line-level bijection
(c -> perm[c >> 5] * 32 + (c & 31)), which keeps the 32 columns of a line
together but scatters R-MAT's hot (low-popcount) lines, then times K2+K3 on
the original and the relabeled matrix (y is bitwise the same up to the
permutation of x)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
P = mb.DeviceMatrix.rmat(ctx, 24, 16, seed=1, transition=True, dtype=np.float32)
ro, cols, vals = P.download()
n = P.n_cols
lines = (n + 31) // 32
rng = np.random.default_rng(7)
perm = rng.permutation(lines).astype(np.int64)
c2 = (perm[cols.astype(np.int64) >> 5] * 32 + (cols & 31)).astype(np.int32)
Q = mb.DeviceMatrix.upload(ctx, P.n_rows, lines * 32, ro, c2, vals)
c = mb.SimtConfig.make(32, 14, 128)
x = torch.rand(n, device="cuda")
x2 = torch.zeros(lines * 32, device="cuda")
idx = torch.from_numpy(perm).cuda()
x2.view(lines, 32)[idx] = torch.nn.functional.pad(x, (0, lines * 32 - n)).view(lines, 32)
out = {}
for name, M, xx in (("natural", P, x), ("line_permuted", Q, x2)):
    t = mb.generate_tile_for(M, c)
    M.build_xcache()
    y = torch.empty(M.n_rows, device="cuda")
    for _ in range(3):
        mb.spmv_device(M, t, c, xx.data_ptr(), y.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        mb.spmv_device(M, t, c, xx.data_ptr(), y.data_ptr())
    e1.record(s)
    torch.cuda.synchronize()
    out[name] = {"ms": e0.elapsed_time(e1) / 20, "hubs": M.xcache_info()[0],
                 "y_sum": float(y.double().sum())}
print(json.dumps(out))
