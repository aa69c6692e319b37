"""One rank of tests/test_gpu_shards_peer.py::test_peer_groups_across_two_processes:
builds its row shard, publishes its IPC blob over a gloo bootstrap, connects
to the other rank's buffers and runs the fused-exchange PageRank twice."""
import os
import sys

import numpy as np
import torch.distributed as dist

import paper_2605_07391_b200 as mb
from paper_2605_07391_b200.merbit import PeerShardGroup, row_slice


def main():
    out, iters = sys.argv[1], int(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = np.load(os.path.join(out, "bounds.npy"))
    ctx = mb.Context(0)
    P = mb.DeviceMatrix.rmat(ctx, 11, 16, seed=5, transition=True, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    L = row_slice(P, int(b[rank]), int(b[rank + 1]))
    t = mb.generate_tile_for(L, c)
    g = PeerShardGroup(ctx, P.n_rows, world, b, rank, L, t, c,
                       mb.PageRankConfig(0.85, 1e-30, iters, 0))
    blobs = [None] * world
    dist.all_gather_object(blobs, g.export())
    g.connect(blobs)
    for _ in range(2):
        g.run()
        res, _ = g.result()
        assert res.iterations == iters
        pi = g.gather_pi()  # the next run's entry barrier protects these reads
    np.save(os.path.join(out, f"pi{rank}.npy"), pi)
    np.save(os.path.join(out, f"resid{rank}.npy"), np.float64(res.l1_residual))
    g.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
