"""Debug: peer shard groups with several ranks in one process (own contexts
of device 0).  argv: scale world iters relabel(0/1) weighted(0/1)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2605_07391_b200 as mb  # noqa: E402
from paper_2605_07391_b200.merbit import PeerShardGroup, prepare_rank_shard, row_slice  # noqa: E402

scale, world, iters, relabel, weighted = map(int, sys.argv[1:6])
c = mb.SimtConfig.make(32, 14, 128)
cfg = mb.PageRankConfig(0.85, 1e-30, iters, 0)
groups, keep = [], []
for r in range(world):
    cx = mb.Context(0)
    P = mb.DeviceMatrix.rmat(cx, scale, 16, seed=1, transition=True, dtype=np.float32)
    Q = P.relabel_by_degree(want_rank=False)[0] if relabel else P
    if weighted:
        b, L, t, w = prepare_rank_shard(Q, world, r, c)
    else:
        ro, _, _ = Q.download(want_values=False)
        b = mb.plan_row_shards(ro, Q.n_rows, Q.nnz, world, 1.0)
        L = row_slice(Q, int(b[r]), int(b[r + 1]))
        t = mb.generate_tile_for(L, c)
    print("rank", r, "bounds", list(b), flush=True)
    groups.append(PeerShardGroup(cx, Q.n_rows, world, b, r, L, t, c, cfg))
    keep.append((cx, P, Q, L, t))
blobs = [g.export() for g in groups]
for g in groups:
    g.connect(blobs)
t0 = time.time()
for g in groups:
    g.run()
print("enqueued", time.time() - t0, flush=True)
for g in groups:
    try:
        res, _ = g.result()
        print("ok", res.iterations, res.mass, time.time() - t0, flush=True)
    except Exception as e:
        print("ERR", e, time.time() - t0, flush=True)
for g in groups:
    g.quiesce()
for g in groups:
    g.close()
print("closed", flush=True)
