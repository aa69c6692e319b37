"""(Historical: needs the mbx_context_set_l2_hot knob, measured and reverted.)
L2 hot-head probe: PageRank fp32 on the degree-relabelled R-MAT at a scale
with the x gathers of the first H columns marked L2 evict_last (the rest
evict_first), for several H (0 = plain gathers, -1 = auto)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--hot", default="0,-1,8000000,24000000")
args = ap.parse_args()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
P0 = mb.DeviceMatrix.rmat(ctx, args.scale, 16, seed=1, transition=True, dtype=np.float32)
P, _ = P0.relabel_by_degree()
del P0
c = mb.SimtConfig.make(32, 14, 128)
t = mb.generate_tile_for(P, c)
P.build_xcache()
cfg = mb.PageRankConfig(0.85, 1e-30, args.iters, 0)
out = {"scale": args.scale}
for h in [int(v) for v in args.hot.split(",")]:
    ctx.set_l2_hot(h)
    plan = mb.PageRankPlan(P, t, c, cfg)
    plan.run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    plan.run()
    e1.record(s)
    torch.cuda.synchronize()
    res, hist = plan.result(want_history=True)
    out[str(h)] = {"ms_per_iter": e0.elapsed_time(e1) / args.iters, "resid_last": float(hist[-1])}
    plan.close()
print(json.dumps(out))
