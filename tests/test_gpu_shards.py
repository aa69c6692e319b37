"""GPU: the row-sharded multi-GPU PageRank path (shard.cu) checked on one
GPU: G shards in one process share the padded exchange buffer, so the remap,
per-shard TILEs, fused commit, chunk-tail scalars and rank-order combine run
exactly as on G GPUs (only the ncclAllGather is absent).  Gate: L1 <= 1e-6
against the fp64 oracle, same as the single-GPU path."""
import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb
from helpers import FORCE_HUBS
from paper_2605_07391_b200.merbit import ShardGroup, row_slice

pytestmark = pytest.mark.gpu


def sharded_pagerank(ctx, P, parts, iters, c, row_weight=1.0):
    ro, _, _ = P.download(want_values=False)
    b = mb.plan_row_shards(ro, P.n_rows, P.nnz, parts, row_weight)
    shards = []
    for g in range(parts):
        m = row_slice(P, int(b[g]), int(b[g + 1]))
        shards.append((m, mb.generate_tile_for(m, c)))
    grp = ShardGroup(ctx, P.n_rows, parts, b, 0, shards, c,
                     mb.PageRankConfig(0.85, 1e-30, iters, 0))
    grp.run()
    res, hist = grp.result(want_history=True)
    return grp.gather_pi(), res, hist, b


@pytest.mark.parametrize("hubs", [False, True])
@pytest.mark.parametrize("row_weight", [1.0, mb.merbit.PAGERANK_ROW_WEIGHT])
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_sharded_matches_fp64_oracle_and_single_gpu(ctx, parts, row_weight, hubs):
    """hubs: every shard view builds a (forced) x hub table over its remapped
    columns, as the large shards of the bench do automatically."""
    if hubs:
        ctx.set_tuning(32, 1, FORCE_HUBS)
    try:
        _sharded_vs_oracle(ctx, parts, row_weight, hubs)
    finally:
        ctx.set_tuning()


def _sharded_vs_oracle(ctx, parts, row_weight, hubs):
    P = mb.DeviceMatrix.rmat(ctx, 14, 16, seed=7, transition=True, dtype=np.float32)
    ro, cols, _ = P.download(want_values=False)
    c = mb.SimtConfig.make(32, 14, 128)
    pi, res, hist, b = sharded_pagerank(ctx, P, parts, 60, c, row_weight)
    assert res.iterations == 60
    p64 = O.Csr(P.n_rows, P.n_cols, ro, cols, O.transition_values(P.n_rows, cols, np.float64))
    want = O.pagerank(p64, 0.85, 1e-300, 60, 0, nthreads=8)
    l1 = np.abs(pi.astype(np.float64) - want["pi"]).sum()
    assert l1 <= 1e-6, l1
    assert abs(res.mass - 1.0) <= 1e-5
    # same answer as the single-GPU fused loop, to fp32 rounding
    t = mb.generate_tile_for(P, c)
    if hubs:
        P.build_xcache(FORCE_HUBS)
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, t, c
    single = mb.pagerank(None, mb.PageRankConfig(0.85, 1e-30, 60, 0), backend=be)
    assert np.abs(pi.astype(np.float64) - single.pi).sum() <= 1e-6
    if parts == 1:
        # one shard is the single-GPU computation: bitwise identical
        assert np.array_equal(pi.view(np.uint32), single.pi.view(np.uint32))
    # deterministic run to run
    pi2, _, _, _ = sharded_pagerank(ctx, P, parts, 60, c, row_weight)
    assert np.array_equal(pi.view(np.uint32), pi2.view(np.uint32))


def test_sharded_convergence_exit(ctx):
    """2-cycle split over 2 shards: pi = [0.5, 0.5] equals the zero-iteration
    yardstick, so the combined ERR is 0 and the loop stops at iteration 1
    (test_solvers.cpp:61-73) -- the stop decision is made after the exchange."""
    two = O.Csr(2, 2, np.array([0, 1, 2]), np.array([1, 0], np.int32), np.ones(2))
    p = O.build_transition(two)
    P = mb.DeviceMatrix.from_csr(ctx, p)
    c = mb.SimtConfig.make(4, 4, 4)
    shards = []
    for g in range(2):
        m = row_slice(P, g, g + 1)
        shards.append((m, mb.generate_tile_for(m, c)))
    grp = ShardGroup(ctx, 2, 2, [0, 1, 2], 0, shards, c, mb.PageRankConfig(0.85, 1e-10, 210, 0))
    grp.run()
    res, _ = grp.result()
    assert res.status == 0 and res.iterations == 1 and res.final_err == 0.0
    assert grp.gather_pi().tolist() == [0.5, 0.5]


@pytest.mark.parametrize("parts", [1, 3])
def test_shards_with_yardstick_run(ctx, parts):
    """reference_iters > 0 (the reference's default config runs a 210-step
    CSR yardstick, solvers.hpp:178-191): the shard group runs it through the
    same exchange and stops on ERR against it like the single-GPU loop."""
    P = mb.DeviceMatrix.rmat(ctx, 12, 16, seed=5, transition=True, dtype=np.float64)
    c = mb.SimtConfig.make(32, 7, 128)
    cfg = mb.PageRankConfig(0.85, 1e-6, 210, 40)
    t = mb.generate_tile_for(P, c)
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, t, c
    single = mb.pagerank(None, cfg, backend=be)
    assert single.status == "converged" and 1 < single.iterations < 210
    ro, _, _ = P.download(want_values=False)
    b = mb.plan_row_shards(ro, P.n_rows, P.nnz, parts)
    shards = [(m, mb.generate_tile_for(m, c)) for m in
              (row_slice(P, int(b[g]), int(b[g + 1])) for g in range(parts))]
    grp = ShardGroup(ctx, P.n_rows, parts, b, 0, shards, c, cfg)
    grp.run()
    res, _ = grp.result()
    pi = grp.gather_pi()
    assert res.status == 0 and abs(res.iterations - single.iterations) <= 1
    if parts == 1:  # the same yardstick and TILE: bitwise
        assert res.iterations == single.iterations and res.final_err == single.final_err
        assert np.array_equal(pi, single.pi)
    else:
        assert np.abs(pi - single.pi).sum() <= 1e-6

def test_start_vector_path_is_bitwise_equal(ctx):
    import torch
    P = mb.DeviceMatrix.rmat(ctx, 12, 16, seed=2, transition=True, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    ro, _, _ = P.download(want_values=False)
    b = mb.plan_row_shards(ro, P.n_rows, P.nnz, 3)
    shards = [(m, mb.generate_tile_for(m, c)) for m in
              (row_slice(P, int(b[g]), int(b[g + 1])) for g in range(3))]
    grp = ShardGroup(ctx, P.n_rows, 3, b, 0, shards, c, mb.PageRankConfig(0.85, 1e-30, 20, 0))
    grp.run()
    a = grp.gather_pi()
    pi0 = torch.full((P.n_rows,), 1.0 / P.n_rows, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    grp.run(pi0.data_ptr())
    assert np.array_equal(a.view(np.uint32), grp.gather_pi().view(np.uint32))
    out = np.zeros(P.n_rows, np.float32)
    grp.download_local(out.ctypes.data)
    assert np.array_equal(out, a)


def test_single_rank_nccl_group(ctx):
    """The NCCL path (comm init, all-reduce of column flags, all-gather inside
    the captured graph) with a world of one rank."""
    from paper_2605_07391_b200.merbit import nccl_unique_id
    P = mb.DeviceMatrix.rmat(ctx, 12, 16, seed=2, transition=True, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(P, c)
    grp = ShardGroup(ctx, P.n_rows, 1, [0, P.n_rows], 0, [(P, t)], c,
                     mb.PageRankConfig(0.85, 1e-30, 20, 0), nccl_unique_id())
    grp.run()
    res, _ = grp.result()
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, t, c
    single = mb.pagerank(None, mb.PageRankConfig(0.85, 1e-30, 20, 0), backend=be)
    assert res.iterations == 20
    assert np.array_equal(grp.gather_pi().view(np.uint32), single.pi.view(np.uint32))


def test_single_rank_nccl_group_with_yardstick(ctx):
    """The NCCL exchange carries the yardstick phase too (1-rank world)."""
    from paper_2605_07391_b200.merbit import nccl_unique_id
    P = mb.DeviceMatrix.rmat(ctx, 11, 16, seed=2, transition=True, dtype=np.float64)
    c = mb.SimtConfig.make(32, 7, 128)
    t = mb.generate_tile_for(P, c)
    cfg = mb.PageRankConfig(0.85, 1e-6, 210, 30)
    grp = ShardGroup(ctx, P.n_rows, 1, [0, P.n_rows], 0, [(P, t)], c, cfg, nccl_unique_id())
    grp.run()
    res, _ = grp.result()
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, t, c
    single = mb.pagerank(None, cfg, backend=be)
    assert res.iterations == single.iterations and res.final_err == single.final_err
    assert np.array_equal(grp.gather_pi(), single.pi)


@pytest.mark.parametrize("parts", [1, 2])
def test_shard_group_device_loop_long_run(ctx, parts):
    """The shard groups' WHILE-node loop: 5000 iterations (beyond any
    unrolled graph) equal the single-GPU loop (bitwise with one shard)."""
    P = mb.DeviceMatrix.rmat(ctx, 8, 16, seed=3, transition=True, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    cfg = mb.PageRankConfig(0.85, 1e-30, 5000, 0)
    pi, res, hist, _ = sharded_pagerank(ctx, P, parts, 5000, c)
    t = mb.generate_tile_for(P, c)
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, t, c
    single = mb.pagerank(None, cfg, backend=be)
    assert res.iterations == single.iterations == 5000
    if parts == 1:
        assert np.array_equal(pi.view(np.uint32), single.pi.view(np.uint32))
    else:
        assert np.abs(pi.astype(np.float64) - single.pi).sum() <= 1e-6
