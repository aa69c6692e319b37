"""A/B timing of the two K2 data layouts (slot copy vs staged CSR order) on
R-MAT: plain SpMV (K2+K3) and fused PageRank iterations, plus shared-memory
budgets.  Prints one JSON line per variant."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--variants", default="1:131072:32,0:131072:32",
                help="layout:smem_per_sm:warps[:prefetch],...")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()

s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
dt = np.float32 if args.dtype == "f32" else np.float64
tdt = torch.float32 if dt == np.float32 else torch.float64
P = mb.DeviceMatrix.rmat(ctx, args.scale, 16, seed=1, transition=True, dtype=dt)
c = mb.SimtConfig.make(32, 14 if dt == np.float32 else 7, 128)
t = mb.generate_tile_for(P, c)
x = torch.rand(P.n_rows, device="cuda", dtype=tdt)
yref = None


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for v in args.variants.split(","):
    fs = [int(f) for f in v.split(":")] + [0]
    layout, smem, warps, pf = fs[:4]
    ctx.set_layout(layout)
    ctx.set_tuning(warps, 1, -1, smem, pf)
    xs = P.build_xcache()
    y = torch.empty_like(x)
    ms = timed(lambda: mb.spmv_device(P, t, c, x.data_ptr(), y.data_ptr()), args.reps)
    if yref is None:
        yref = y.clone()
    rel = float(((y.double() - yref.double()).abs().max() / yref.double().abs().max()).item())
    plan = mb.PageRankPlan(P, t, c, mb.PageRankConfig(0.85, 1e-30, args.iters, 0))
    plan.run()
    pr_ms = timed(plan.run, 3) / args.iters
    res, _ = plan.result(want_history=True)
    m, n = P.nnz, P.n_rows
    vs = 4 if dt == np.float32 else 8
    b = m * (vs + 4) + 2 * n * vs + 4 * (n + 1)
    print(json.dumps({"layout": layout, "smem_per_sm": smem, "warps": warps, "prefetch": pf,
                      "hubs": P.xcache_info()[0], "coverage": P.xcache_info()[1],
                      "slot_build_s": P.slot_info()[1], "spmv_ms": ms, "spmv_gbs": b / ms / 1e6,
                      "pr_ms_per_iter": pr_ms, "pr_it_s": 1e3 / pr_ms,
                      "rel_vs_first": rel, "pr_mass": res.mass}), flush=True)
    del plan
