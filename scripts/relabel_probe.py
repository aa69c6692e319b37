"""Degree relabelling probe: PageRank fp32 on R-MAT at a scale, natural vertex
order vs the device-side symmetric relabel P' = Q P Q^T (vertices by
descending column count).  Prints ms/iteration for both and the L1 distance
of the two answers (pi'[rank] vs pi)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
P = mb.DeviceMatrix.rmat(ctx, args.scale, 16, seed=1, transition=True, dtype=np.float32)
c = mb.SimtConfig.make(32, 14, 128)
cfg = mb.PageRankConfig(0.85, 1e-30, args.iters, 0)
out = {"scale": args.scale, "n": P.n_rows, "nnz": P.nnz}
pis = {}
for name in ("natural", "relabel"):
    t0 = time.perf_counter()
    if name == "relabel":
        M, rank = P.relabel_by_degree()
        torch.cuda.synchronize()
        out["relabel_s"] = time.perf_counter() - t0
    else:
        M, rank = P, None
    t = mb.generate_tile_for(M, c)
    M.build_xcache()
    plan = mb.PageRankPlan(M, t, c, cfg)
    plan.run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    plan.run()
    e1.record(s)
    torch.cuda.synchronize()
    plan.close()
    out[name + "_ms_per_iter"] = e0.elapsed_time(e1) / args.iters
    out[name + "_hubs"], out[name + "_hub_cov"] = M.xcache_info()
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = M, t, c
    pis[name] = (mb.pagerank(None, cfg, backend=be).pi, rank)
nat = pis["natural"][0].astype(np.float64)
rel, rank = pis["relabel"]  # mbx_pagerank returns pi in the original vertex order
out["l1_natural_vs_relabel"] = float(np.abs(nat - rel.astype(np.float64)).sum())
print(json.dumps(out))
