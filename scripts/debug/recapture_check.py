"""Repeats test_plan_recaptures_after_matrix_buffers_change's sequence and
reports which comparison differs (debugging an intermittent failure)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O  # noqa: E402
import paper_2605_07391_b200 as mb  # noqa: E402

ctx = mb.Context(0)
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    c = mb.SimtConfig.make(32, 14, 128)
    c2 = mb.SimtConfig.make(32, 14, 64)
    P = mb.DeviceMatrix.rmat(ctx, 13, 16, seed=5, transition=True, dtype=np.float32)
    n = P.n_rows
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, mb.generate_tile_for(P, c), c
    t2 = mb.generate_tile_for(P, c2)
    cfg = mb.PageRankConfig(0.85, 1e-30, 20, 0)
    a = mb.pagerank(None, cfg, backend=be)
    x = O.hash_uniform(3, n, 0.0, 1.0, np.float32)
    y2 = mb.spmv_merbit(P, t2, c2, x, mb.DualBuffer(n, np.float32))
    b = mb.pagerank(None, cfg, backend=be)
    ab = np.array_equal(a.pi.view(np.uint32), b.pi.view(np.uint32))
    plan = mb.PageRankPlan(P, be.tile_, c, cfg)
    xd = torch.empty(n, dtype=torch.float32, device="cuda")
    yd = torch.empty(n, dtype=torch.float32, device="cuda")
    plan.run()
    r1, h1 = plan.result(want_history=True)
    P.build_xcache()
    torch.cuda.synchronize()
    mb.spmv_device(P, t2, c2, xd.data_ptr(), yd.data_ptr())
    ctx.synchronize()
    plan.run()
    r2, h2 = plan.result(want_history=True)
    hh = np.array_equal(h1, h2) and r1.l1_residual == r2.l1_residual
    y2b = mb.spmv_merbit(P, t2, c2, x, mb.DualBuffer(n, np.float32))
    yy = np.array_equal(y2.view(np.uint32), y2b.view(np.uint32))
    d = np.nonzero(y2 != y2b)[0]
    print(f"trial {trial}: a==b {ab} hist {hh} y2==y2b {yy} hubs {P.xcache_info()[0]} "
          f"ndiff {d.size} rows {d[:6]} y2 {y2[d[:3]]} y2b {y2b[d[:3]]}", flush=True)
    plan.close()
