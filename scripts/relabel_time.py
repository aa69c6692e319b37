"""Wall time of mbx_matrix_relabel_by_degree at R-MAT s24: first call vs
repeat (pool growth, module loading) -- preprocessing cost in bench.py."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
mode = sys.argv[2] if len(sys.argv) > 2 else "plain"
if mode in ("torch", "stream"):
    torch.cuda.init()
if mode == "stream":
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
ctx = mb.Context(0)
if mode == "stream":
    ctx.set_stream(st.cuda_stream)
t = time.perf_counter()
P = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
ctx.synchronize()
print("generate", time.perf_counter() - t)
for k in range(3):
    t = time.perf_counter()
    Q, _ = P.relabel_by_degree(want_rank=False)
    ctx.synchronize()
    print("relabel", k, time.perf_counter() - t)
    del Q
