"""ncu target: the virtual shard group (G row shards of the relabelled R-MAT on
one GPU), a few PageRank iterations -- per-kernel shares of a sharded
iteration (K2 and K3 per shard, the combine kernel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_07391_b200 as mb  # noqa: E402
from paper_2605_07391_b200.merbit import ShardGroup, row_slice  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = int(sys.argv[2]) if len(sys.argv) > 2 else 8
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = mb.Context(0)
ctx.set_stream(s.cuda_stream)
P0 = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
P, _ = P0.relabel_by_degree()
del P0
c = mb.SimtConfig.make(32, 14, 128)
ro, _, _ = P.download(want_values=False)
w = float(os.environ.get("MBX_ROW_WEIGHT", "3.4"))  # 1.0 = merge-path cut
bounds = mb.plan_row_shards(ro, P.n_rows, P.nnz, g, w)
for r in range(g):
    print("shard", r, int(bounds[r + 1] - bounds[r]), int(ro[bounds[r + 1]] - ro[bounds[r]]), file=sys.stderr)
shards = []
for r in range(g):
    L = row_slice(P, int(bounds[r]), int(bounds[r + 1]))
    shards.append((L, mb.generate_tile_for(L, c)))
grp = ShardGroup(ctx, P.n_rows, g, bounds, 0, shards, c, mb.PageRankConfig(0.85, 1e-30, 3, 0))
grp.run()
torch.cuda.synchronize()
print("done")
