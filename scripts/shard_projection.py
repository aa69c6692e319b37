"""Measured ingredients of the multi-GPU projection (only one GPU is available
in this run): PageRank fp32 on R-MAT at a scale (degree-relabelled, as
bench.py), (1) the single-GPU plan, (2) the same graph as G row shards run
back to back on this one GPU by the virtual shard group (the sharded kernels,
remap and combine, no exchange).  Per-GPU compute at G GPUs ~ (2) / G; the
exchange per iteration is the compacted chunk bytes each GPU receives,
(G-1)/G * total, over NVLink at the measured 770 GB/s peer bandwidth
(B200_PROFILING).  Prints the measured times and the projection."""
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
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--parts", default="2,4,8")
ap.add_argument("--row-weight", type=float, default=0.0, help="0: pagerank_row_weight(n)")
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


def timed(fn):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.iters


t = mb.generate_tile_for(P, c)
P.build_xcache()
plan = mb.PageRankPlan(P, t, c, cfg)
single = timed(plan.run)
plan.close()
del t
ro, cols, _ = P.download(want_values=False)
nondangling = int(np.count_nonzero(np.bincount(cols, minlength=n)))
del cols
out = {"scale": args.scale, "n": n, "nnz": m, "single_gpu_ms_per_iter": single,
       "nondangling_vertices": nondangling}
for g in [int(x) for x in args.parts.split(",")]:
    w = args.row_weight or mb.merbit.pagerank_row_weight(n)
    bounds = mb.plan_row_shards(ro, n, m, g, w)
    shards = []
    for r in range(g):
        L = row_slice(P, int(bounds[r]), int(bounds[r + 1]))
        shards.append((L, mb.generate_tile_for(L, c)))
    grp = ShardGroup(ctx, n, g, bounds, 0, shards, c, cfg, None)
    virt = timed(grp.run)
    per_shard = shard_kernel_ms(grp.run, g)
    grp.close()
    del grp, shards
    torch.cuda.synchronize()
    xbytes = nondangling * 4 * (g - 1) / g  # received per GPU per iteration
    exch = xbytes / 770e9 * 1e3
    slowest = max(per_shard)
    proj = slowest + exch + 0.02  # + NCCL/launch latency allowance
    out[f"G{g}"] = {"virtual_all_shards_ms_per_iter": virt, "mean_gpu_compute_ms": virt / g,
                    "shard_kernel_ms": [round(v, 4) for v in per_shard],
                    "per_gpu_compute_ms": slowest,
                    "exchange_ms_at_770GBps": exch, "projected_ms_per_iter": proj,
                    "projected_speedup": single / proj}
print(json.dumps(out))
