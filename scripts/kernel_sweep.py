"""Time the SpMV (K2+K3) and one fused PageRank iteration on R-MAT inputs over
kernel launch shapes (warps/CTA : CTAs/SM : hub cap) and block sizes
(chunks per warp range = block_size / 32).  Checks that every variant gives
the bitwise-identical y.  Also the target for ncu captures (--reps small)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_07391_b200 as mb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--blocks", default="128")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--transition", type=int, default=1)
ap.add_argument("--pr-iters", type=int, default=20)
ap.add_argument("--tunings", default="16:2:-1", help="warps:ctas_per_sm:max_hubs,...")
args = ap.parse_args()

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = mb.Context(0)
ctx.set_stream(stream.cuda_stream)
dt = np.float32 if args.dtype == "f32" else np.float64
tdt = torch.float32 if dt == np.float32 else torch.float64
sigma = 14 if dt == np.float32 else 7
P = mb.DeviceMatrix.rmat(ctx, args.scale, 16, seed=1, transition=bool(args.transition), dtype=dt)
n, m = P.n_rows, P.nnz
vs = 4 if dt == np.float32 else 8
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
x = torch.rand(n, device="cuda", dtype=tdt)
y = torch.empty_like(x)
yref = None
tiles = {}
combos = []
for tu in args.tunings.split(","):
    f = [int(v) for v in tu.split(":")] + [144, 1]
    for b in [int(v) for v in args.blocks.split(",")]:
        combos.append((f[0], f[1], f[2], f[3], f[4], b))
for (wpc, cps, hubs, smem_kb, pf, b) in combos:
    ctx.set_tuning(wpc, cps, hubs, smem_kb * 1024, pf)
    xc_s = P.build_xcache(hubs)
    nh, cov = P.xcache_info()
    c = mb.SimtConfig.make(32, sigma, b)
    if b not in tiles:
        tiles[b] = mb.generate_tile_for(P, c)
    t = tiles[b]
    for _ in range(3):
        mb.spmv_device(P, t, c, x.data_ptr(), y.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.reps):
        mb.spmv_device(P, t, c, x.data_ptr(), y.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    ts = e0.elapsed_time(e1) / args.reps * 1e-3
    bs = m * (vs + 4) + 2 * n * vs + 4 * (n + 1)
    same = None
    if b == 128:
        if yref is None:
            yref = y.clone()
        else:
            same = bool(torch.equal(y.view(torch.int32 if vs == 4 else torch.int64),
                                    yref.view(torch.int32 if vs == 4 else torch.int64)))
    row = {"warps": wpc, "ctas_per_sm": cps, "smem_kb": smem_kb, "pf": pf, "hubs": nh, "hub_cov": round(cov, 3),
           "xcache_ms": round(xc_s * 1e3, 3), "block": b, "spmv_us": round(ts * 1e6, 1),
           "spmv_gbs": round(bs / ts / 1e9, 1), "spmv_frac": round(bs / ts / 1e9 / peak, 4),
           "gflops": round(2 * m / ts / 1e9, 1), "tile_ms": round(t.preprocess_seconds * 1e3, 3),
           "bitwise_same_as_first": same}
    if args.transition and args.pr_iters:
        plan = mb.PageRankPlan(P, t, c, mb.PageRankConfig(0.85, 1e-30, args.pr_iters, 0))
        plan.run()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            plan.run()
        e1.record(stream)
        torch.cuda.synchronize()
        ti = e0.elapsed_time(e1) * 1e-3 / (3 * args.pr_iters)
        bi = m * (vs + 4) + 3 * n * vs + 4 * (n + 1)
        res, hist = plan.result(want_history=True)
        row.update({"pr_iter_us": round(ti * 1e6, 1), "pr_gbs": round(bi / ti / 1e9, 1),
                    "pr_frac": round(bi / ti / 1e9 / peak, 4),
                    "resid_last": float(hist[args.pr_iters - 1]), "mass": res.mass})
        plan.close()
    print(json.dumps(row), flush=True)
print(json.dumps({"n": n, "nnz": m, "scale": args.scale, "dtype": args.dtype}))
