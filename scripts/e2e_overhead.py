"""Where the end-to-end mbx_pagerank call (host pi0 in, pi out, original
vertex order) spends time beyond the device loop, R-MAT s24 relabelled:
plan creation, H2D + D2H of pi (pinned), vertex-map permutations."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402
from paper_2605_07391_b200 import _lib  # noqa: E402

st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = mb.Context(0)
ctx.set_stream(st.cuda_stream)
P0 = mb.DeviceMatrix.rmat(ctx, 24, 16, seed=1, transition=True, dtype=np.float32)
P, _ = P0.relabel_by_degree()
del P0
n = P.n_rows
cfg = mb.SimtConfig.make(32, 14, 128)
tile = mb.generate_tile_for(P, cfg)
P.build_xcache()
L = _lib.lib()
pi0 = torch.full((n,), 1.0 / n, dtype=torch.float32).pin_memory()
pi_out = torch.empty(n, dtype=torch.float32).pin_memory()
dev = torch.empty(n, dtype=torch.float32, device="cuda")


def wall(fn, k=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e3


for iters in (1, 100):
    prc = mb.PageRankConfig(0.85, 1e-30, iters, 0)
    cc, pc = cfg._c(), prc._c()
    rr = _lib.mbx_pagerank_result()

    def e2e():
        assert L.mbx_pagerank(ctx.h, P.h, tile.h, C.byref(cc), C.byref(pc), pi0.data_ptr(),
                              pi_out.data_ptr(), None, None, C.byref(rr)) == 0
    plan = mb.PageRankPlan(P, tile, cfg, prc)
    print(iters, "e2e_ms", round(wall(e2e), 3), "plan_run_ms", round(wall(plan.run), 3))
    plan.close()
print("h2d_ms", round(wall(lambda: dev.copy_(pi0, non_blocking=True)), 3),
      "d2h_ms", round(wall(lambda: pi_out.copy_(dev, non_blocking=True)), 3))
t = time.perf_counter()
for _ in range(5):
    plan = mb.PageRankPlan(P, tile, cfg, mb.PageRankConfig(0.85, 1e-30, 100, 0))
    plan.close()
torch.cuda.synchronize()
print("plan_create_destroy_ms", round((time.perf_counter() - t) / 5 * 1e3, 3))
