"""GPU: bench.py's N > 1 path, exactly as the bench runs it -- R-MAT
transition matrix -> degree relabelling on the device -> prepare_rank_shard
(cost-weighted cut with pagerank_row_weight, row slice, TILE) -> the FUSED
exchange (PeerShardGroup: commit stores into every peer's buffer + device
barrier) -- with 2 / 3 ranks on their own contexts of the one GPU, checked
against the fp64 oracle (north-star gate L1 <= 1e-6, 100 iterations) in the
original vertex order.

And BASELINE C4's own matrix (R-MAT scale 27, 2.1 G nonzeros): the one-GPU
PageRank vs the same matrix cut into 8 shards by the bench's weighted cut
(virtual shard group, every shard on this GPU, re-cut from the shards'
measured cost as the bench does): L1 <= 1e-6.  No CPU oracle
finishes 100 iterations over 2.1 G nonzeros in a test's time; the one-GPU
path is itself gated against the fp64 oracle at scale 24
(test_gpu_scale.py) and against the compiled reference at scale 20
(test_gpu_scale_ref.py).

References: the loop being sharded is pagerank<T> (solvers.hpp:154-218);
the cut restates merge_search's diagonal split (merge_path.cpp:8-36) with a
row weight."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb
from paper_2605_07391_b200.merbit import (PeerShardGroup, ShardGroup, pagerank_row_weight,
                                          prepare_rank_shard, recut_rank_shard,
                                          shard_cost_probe)

pytestmark = pytest.mark.gpu
NT = os.cpu_count() or 1


@pytest.mark.parametrize("scale,world,recut", [(16, 2, False), (18, 3, True), (20, 2, True)])
def test_bench_sharded_path_vs_fp64_oracle(scale, world, recut):
    iters = 100
    c = mb.SimtConfig.make(32, 14, 128)
    cfg = mb.PageRankConfig(0.85, 1e-30, iters, 0)
    groups, keep, ranks = [], [], []
    bounds0 = None
    for r in range(world):
        cx = mb.Context(0)  # own stream per rank: the ranks' loops overlap
        P = mb.DeviceMatrix.rmat(cx, scale, 16, seed=1, transition=True, dtype=np.float32)
        Q, rank_of = P.relabel_by_degree(want_rank=True)
        bounds, L, t, w = prepare_rank_shard(Q, world, r, c)
        assert w == pagerank_row_weight(Q.n_rows, 4)
        if bounds0 is None:
            bounds0, rank0_of, P0 = bounds, rank_of, P
        assert np.array_equal(bounds, bounds0)  # every rank cuts the same way
        ranks.append([cx, Q, bounds, L, t, w])
    if recut:
        # bench.py's measured re-cut: probe every first-cut shard, share the
        # times, re-cut identically on every rank
        times = [shard_cost_probe(L, t, c) for _, _, _, L, t, _ in ranks]
        for r, rk in enumerate(ranks):
            rk[2], rk[3], rk[4] = recut_rank_shard(rk[1], rk[2], times, r, c, rk[5])
        assert all(np.array_equal(rk[2], ranks[0][2]) for rk in ranks)
        assert ranks[0][2][0] == 0 and ranks[0][2][-1] == ranks[0][1].n_rows
    for r, (cx, Q, bounds, L, t, _) in enumerate(ranks):
        groups.append(PeerShardGroup(cx, Q.n_rows, world, bounds, r, L, t, c, cfg))
        keep.append((cx, Q, L, t))
    blobs = [g.export() for g in groups]
    for g in groups:
        g.connect(blobs)
    for g in groups:
        g.run()
    for g in groups:
        res, hist = g.result(want_history=True)
        assert res.iterations == iters and abs(res.mass - 1.0) <= 1e-5
    pi_rel = groups[0].gather_pi()
    for g in groups[1:]:
        assert np.array_equal(g.gather_pi().view(np.uint32), pi_rel.view(np.uint32))
    pi = pi_rel[rank0_of]  # original vertex order
    ro, cols, _ = P0.download(want_values=False)
    n = P0.n_rows
    p64 = O.Csr(n, n, ro, cols, O.transition_values(n, cols, np.float64))
    want = O.pagerank(p64, 0.85, 1e-300, iters, 0, nthreads=NT)
    l1 = float(np.abs(pi.astype(np.float64) - want["pi"]).sum())
    assert l1 <= 1e-6, l1
    for g in groups:
        g.quiesce()
    for g in groups:
        g.close()


@pytest.mark.slow
def test_c4_s27_one_gpu_vs_8_weighted_shards():
    cx = mb.Context(0)
    c = mb.SimtConfig.make(32, 14, 128)
    iters = 100
    cfg = mb.PageRankConfig(0.85, 1e-30, iters, 0)
    P = mb.DeviceMatrix.rmat(cx, 27, 16, seed=1, transition=True, dtype=np.float32)
    n = P.n_rows
    Q, rank_of = P.relabel_by_degree(want_rank=True)
    del P
    # one GPU, the bench's configuration (pi in the original order)
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = Q, mb.generate_tile_for(Q, c), c
    Q.build_xcache()
    one = mb.pagerank(None, cfg, backend=be)
    assert one.iterations == iters and abs(one.mass - 1.0) <= 1e-5
    del be
    cx.release_cache()
    Q.release_caches()
    # eight shards cut exactly as bench.py --gpus 8 cuts them: the weighted
    # cut, every shard probed, the measured re-cut
    shards, bounds = [], None
    for r in range(8):
        b, L, t, w = prepare_rank_shard(Q, 8, r, c)
        assert bounds is None or np.array_equal(b, bounds)
        bounds = b
        shards.append((L, t))
    times = [shard_cost_probe(L, t, c) for L, t in shards]
    del shards
    shards = []
    for r in range(8):
        b, L, t = recut_rank_shard(Q, bounds, times, r, c, w)
        shards.append((L, t))
    bounds = b
    g = ShardGroup(cx, n, 8, bounds, 0, shards, c, cfg)
    g.run()
    res, _ = g.result()
    assert res.iterations == iters and abs(res.mass - 1.0) <= 1e-5
    pi = g.gather_pi()[rank_of]
    g.close()
    l1 = float(np.abs(pi.astype(np.float64) - one.pi.astype(np.float64)).sum())
    assert l1 <= 1e-6, l1
