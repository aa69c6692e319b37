"""PageRank fp32 iteration time vs R-MAT scale (s20 .. s27) on one B200,
degree-relabelled (bench.py's configuration) and natural order: shows where
pi leaves L2 (s24: 64 MB fits the 126 MB L2; s25+: it does not) and how the
scattered-gather bound moves.  One JSON line per (scale, order)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

scales = [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "20,21,22,23,24,25,26,27").split(",")]
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = mb.Context(0)
ctx.set_stream(st.cuda_stream)
c = mb.SimtConfig.make(32, 14, 128)
iters = 20
for s in scales:
    P0 = mb.DeviceMatrix.rmat(ctx, s, 16, seed=1, transition=True, dtype=np.float32)
    for order in ("degree", "natural"):
        P = P0.relabel_by_degree()[0] if order == "degree" else P0
        t = mb.generate_tile_for(P, c)
        P.build_xcache()
        hubs, cov = P.xcache_info()
        plan = mb.PageRankPlan(P, t, c, mb.PageRankConfig(0.85, 1e-30, iters, 0))
        plan.run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            plan.run()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / (3 * iters)
        n, m = P.n_rows, P.nnz
        print(json.dumps({"scale": s, "order": order, "n": n, "nnz": m, "ms_per_iteration": ms,
                          "iters_per_s": 1e3 / ms, "hbm_gbs": (8 * m + 16 * n + 4) / ms / 1e6,
                          "hub_coverage": cov, "non_hub_gathers_per_s": m * (1 - cov) / ms * 1e3}),
              flush=True)
        plan.close()
        del plan, t
        if order == "degree":
            del P
    del P0
    torch.cuda.synchronize()
