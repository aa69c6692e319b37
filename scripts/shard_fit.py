"""Row-shard balance study (one GPU, virtual shard group): per-shard K2+K3
times of the degree-relabelled R-MAT PageRank for a cut, then re-cuts that
spread each shard's MEASURED time over its rows in proportion to the
nnz + w*rows cost and cut the resulting time curve evenly (a few rounds).
Prints one JSON line per round with the bounds, shard times and per-shard
degree-bucket features (rows and nonzeros per bucket) for fitting a cost
model.  python scripts/shard_fit.py --scale 27 --parts 8 --rounds 3"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402
from paper_2605_07391_b200.merbit import ShardGroup, row_slice  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from shard_projection_lib import shard_kernel_ms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--parts", type=int, default=8)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--row-weight", type=float, default=1.5)
ap.add_argument("--proxy", action="store_true",
                help="re-cut from each shard's plain SpMV time (+ its rows' K3 stream) "
                     "instead of the measured PageRank shard times")
args = ap.parse_args()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
P0 = mb.DeviceMatrix.rmat(ctx, args.scale, 16, seed=1, transition=True, dtype=np.float32)
P, _ = P0.relabel_by_degree()
del P0
n, m = P.n_rows, P.nnz
c = mb.SimtConfig.make(32, 14, 128)
cfg = mb.PageRankConfig(0.85, 1e-30, args.iters, 0)
ro = P.row_offsets().astype(np.int64)
deg = np.diff(ro)
EDGES = [0, 1, 2, 4, 8, 16, 32, 128, 1 << 40]
# column buckets (relabelled: small ids = most referenced): per row, how many
# of its nonzeros fall in each prefix band of x
CEDGES = np.array([0, 1 << 15, 1 << 18, 1 << 21, 1 << 23, 1 << 25, 1 << 40])
_, cols, _ = P.download(want_values=False)
cb = np.searchsorted(CEDGES, cols, side="right").astype(np.int8) - 1
del cols
# per-row counts would be n x 6; keep prefix sums over nonzeros per bucket
cpre = np.zeros((len(CEDGES) - 1, m + 1), np.int64)
for k in range(len(CEDGES) - 1):
    np.cumsum(cb == k, out=cpre[k, 1:])
del cb


def features(r0, r1):
    d = deg[r0:r1]
    b = np.searchsorted(EDGES, d, side="right") - 1
    return {"rows": int(r1 - r0), "nnz": int(ro[r1] - ro[r0]),
            "rows_b": np.bincount(b, minlength=len(EDGES) - 1).tolist(),
            "nnz_b": np.bincount(b, weights=d, minlength=len(EDGES) - 1).astype(np.int64).tolist(),
            "cols_b": [int(cpre[k, ro[r1]] - cpre[k, ro[r0]]) for k in range(cpre.shape[0])]}


def measure(bounds):
    g = len(bounds) - 1
    shards = []
    for r in range(g):
        L = row_slice(P, int(bounds[r]), int(bounds[r + 1]))
        shards.append((L, mb.generate_tile_for(L, c)))
    prox = [mb.merbit.shard_cost_probe(L, t, c) * 1e3 for L, t in shards]
    grp = ShardGroup(ctx, n, g, bounds, 0, shards, c, cfg, None)
    grp.run()
    t = shard_kernel_ms(grp.run, g)
    grp.close()
    del grp, shards
    torch.cuda.synchronize()
    return t, prox


w = args.row_weight
bounds = mb.plan_row_shards(ro, n, m, args.parts, w)
cost = ro.astype(np.float64) + w * np.arange(n + 1)  # cumulative nnz + w*rows
for rnd in range(args.rounds + 1):
    t, prox = measure(bounds)
    print(json.dumps({"scale": args.scale, "round": rnd, "w": w, "bounds": bounds.tolist(),
                      "shard_ms": [round(v, 4) for v in t], "max_ms": max(t),
                      "proxy_ms": [round(v, 4) for v in prox],
                      "mean_ms": float(np.mean(t)),
                      "features": [features(int(bounds[i]), int(bounds[i + 1]))
                                   for i in range(len(t))]}), flush=True)
    if rnd == args.rounds:
        break
    bounds = mb.recut_row_shards(ro, bounds, prox if args.proxy else t, w)
