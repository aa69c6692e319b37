"""GPU fused PageRank (solvers.hpp:154-218) against the reference's golden
results and the fp64 oracle (north-star gate: L1 <= 1e-6)."""
import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb
from helpers import FORCE_HUBS

pytestmark = pytest.mark.gpu


def backend(ctx, p, w=32, s=None, b=128):
    dt = p.values.dtype
    s = s or (14 if dt == np.float32 else 7)
    return mb.MerbitB200Backend(p, mb.SimtConfig.make(w, s, b), ctx)


def test_two_cycle_exact_fixed_point(ctx):
    # test_solvers.cpp:61-73
    two = O.Csr(2, 2, np.array([0, 1, 2]), np.array([1, 0], np.int32), np.ones(2))
    p = O.build_transition(two)
    r = mb.pagerank(p, mb.PageRankConfig(), backend(ctx, p))
    assert r.status == "converged" and r.iterations == 1
    assert r.pi.tolist() == [0.5, 0.5] and r.final_err == 0.0
    assert np.array_equal(r.reference_pi, r.pi)


def test_dangling_closed_form(ctx):
    # test_solvers.cpp:75-99
    dang = O.Csr(2, 2, np.array([0, 1, 1]), np.array([1], np.int32), np.ones(1))
    p = O.build_transition(dang)
    r = mb.pagerank(p, mb.PageRankConfig(), backend(ctx, p))
    c = 0.85
    assert r.status == "converged"
    assert abs(r.pi[0] - 1 / (2 + c)) <= 1e-10 and abs(r.pi[1] - (1 + c) / (2 + c)) <= 1e-10
    assert abs(r.mass - 1.0) <= 1e-13


def test_ring_matches_reference(ctx, golden):
    # test_solvers.cpp:101-124, acceptance c9: agreement <= 1e-12 relative
    g = golden["pagerank"]["ring_100_260_42"]
    p = O.build_transition(O.ring_with_chords(100, 260, 42))
    for (w, s, b) in [(32, 7, 128), (4, 4, 16)]:
        r = mb.pagerank(p, mb.PageRankConfig(), backend(ctx, p, w, s, b))
        assert r.status == "converged" and r.iterations <= 210 and r.final_err < 1e-10
        want = np.array(g["pi"])
        assert np.all(np.abs(r.pi - want) <= 1e-12 * np.abs(want))
        assert abs(r.mass - 1.0) <= 1e-12


def test_ring_fp32_fixed_iterations(ctx, golden):
    g = golden["pagerank"]["ring_f32_50it"]
    p = O.build_transition(O.ring_with_chords(100, 260, 42), np.float32)
    r = mb.pagerank(p, mb.PageRankConfig(0.85, 1e-30, 50, 0), backend(ctx, p))
    assert r.iterations == 50 and r.status == "max_iterations"
    assert np.abs(r.pi - np.array(g["pi"])).sum() <= 1e-6


def test_bad_configs(ctx):
    # test_solvers.cpp:126-139
    p = O.build_transition(O.ring_with_chords(8, 4, 3))
    be = backend(ctx, p)
    with pytest.raises(mb.ConfigError):
        mb.pagerank(p, mb.PageRankConfig(damping=1.5), be)
    with pytest.raises(mb.ConfigError):
        mb.pagerank(p, mb.PageRankConfig(err_tol=0.0), be)
    rect = O.single_dense_row(4, 1)
    with pytest.raises(mb.DimensionError):
        mb.pagerank(rect, mb.PageRankConfig(), backend(ctx, rect))


@pytest.mark.parametrize("scale", [14, 18])
def test_rmat_fp32_l1_vs_fp64_oracle(ctx, scale):
    """North-star gate on R-MAT: 100 fixed iterations (reference_iters=0),
    L1(pi_gpu_fp32, pi_fp64) <= 1e-6; residual history is monotone-ish and
    the device L1 residual matches the host recomputation."""
    m = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=True, dtype=np.float32)
    ro, cols, _ = m.download(want_values=False)
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(m, c)
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = m, t, c
    r = mb.pagerank(None, mb.PageRankConfig(0.85, 1e-30, 100, 0), backend=be)
    p64 = O.Csr(m.n_rows, m.n_cols, ro, cols, O.transition_values(m.n_rows, cols, np.float64))
    want = O.pagerank(p64, 0.85, 1e-300, 100, 0, nthreads=8)
    l1 = np.abs(r.pi.astype(np.float64) - want["pi"]).sum()
    assert r.iterations == 100 and l1 <= 1e-6, l1
    assert abs(r.mass - 1.0) <= 1e-5
    assert r.residual_history[-1] < r.residual_history[0]
    r2 = mb.pagerank(None, mb.PageRankConfig(0.85, 1e-30, 100, 0), backend=be)
    assert np.array_equal(r.pi.view(np.uint32), r2.pi.view(np.uint32))  # deterministic


def test_short_rows_transition_fp32(ctx):
    """Transition matrix of a sparse graph (0-3 out-edges, many dangling
    vertices): tiles close > 64 rows, so the slot kernel's lane-by-lane
    commit carries the fused update.  L1 vs the fp64 oracle <= 1e-6."""
    rng = np.random.default_rng(4)
    n = 50000
    lens = rng.integers(0, 4, n)
    ro = np.zeros(n + 1, np.int64)
    ro[1:] = np.cumsum(lens)
    cols = np.concatenate([np.sort(rng.choice(n, l, replace=False)) if l else
                           np.zeros(0, np.int64) for l in lens]).astype(np.int32)
    adj = O.Csr(n, n, ro, cols, np.ones(len(cols)))
    p32 = O.build_transition(adj, np.float32)
    p64 = O.build_transition(adj, np.float64)
    r = mb.pagerank(p32, mb.PageRankConfig(0.85, 1e-30, 60, 0), backend(ctx, p32))
    want = O.pagerank(p64, 0.85, 1e-300, 60, 0)
    l1 = np.abs(r.pi.astype(np.float64) - want["pi"]).sum()
    assert r.iterations == 60 and l1 <= 1e-6, l1


def test_degree_relabel_preprocessing(ctx):
    """mbx_matrix_relabel_by_degree: P' = Q P Q^T with vertices ranked by
    descending column count (numpy restatement below), TILE of P'
    byte-identical to the oracle's, and PageRank through the relabelled
    matrix returns pi in the ORIGINAL vertex order within 1e-6 L1 of the fp64
    oracle on P."""
    P = mb.DeviceMatrix.rmat(ctx, 18, 16, seed=6, transition=True, dtype=np.float32)
    ro, cols, vals = P.download()
    n = P.n_rows
    Q, rank = P.relabel_by_degree()
    cnt = np.bincount(cols, minlength=n)
    order = np.argsort(-cnt.astype(np.int64), kind="stable")
    want_rank = np.empty(n, np.int64)
    want_rank[order] = np.arange(n)
    assert np.array_equal(rank, want_rank)
    rows = np.repeat(np.arange(n), np.diff(ro))
    key = want_rank[rows] * n + want_rank[cols]
    o = np.argsort(key, kind="stable")
    qro, qcols, qvals = Q.download()
    assert np.array_equal(qcols, (key[o] % n).astype(np.int32))
    assert np.array_equal(qvals, vals[o])
    assert np.array_equal(qro, np.searchsorted(key[o] // n, np.arange(n + 1)))
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(Q, c)
    for got, want in zip(t.download(), O.generate_tile(qro, n, Q.nnz, 32, 14)):
        assert np.array_equal(got, want)
    # host-facing SpMV on the relabelled matrix: x and y in the original order
    x = O.hash_uniform(2, n, -1.0, 1.0, np.float32)
    y = mb.spmv_merbit(Q, t, c, x, mb.DualBuffer(n, np.float32))
    wy, mag = O.spmv_csr_f32_acc64(O.Csr(n, n, ro, cols, vals), x)
    assert (np.abs(y.astype(np.float64) - wy) / np.where(mag > 0, mag, 1)).max() <= 1e-5
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = Q, t, c
    r = mb.pagerank(None, mb.PageRankConfig(0.85, 1e-30, 50, 0), backend=be)
    p64 = O.Csr(n, n, ro, cols, O.transition_values(n, cols, np.float64))
    want = O.pagerank(p64, 0.85, 1e-300, 50, 0)
    assert np.abs(r.pi.astype(np.float64) - want["pi"]).sum() <= 1e-6


def test_pagerank_plan_cache(ctx):
    """mbx_pagerank keeps its plan between calls: repeated calls are bitwise
    equal, a changed config / tuning / matrix rebuilds it, and a destroyed
    matrix never leaves a stale plan behind."""
    def backend(P, c):
        be = type("B", (), {})()
        be.matrix, be.tile_, be.c = P, mb.generate_tile_for(P, c), c
        return be

    c = mb.SimtConfig.make(32, 14, 128)
    P = mb.DeviceMatrix.rmat(ctx, 12, 16, seed=3, transition=True, dtype=np.float32)
    be = backend(P, c)
    cfg = mb.PageRankConfig(0.85, 1e-30, 30, 0)
    a = mb.pagerank(None, cfg, backend=be)
    b = mb.pagerank(None, cfg, backend=be)  # cached plan
    assert np.array_equal(a.pi.view(np.uint32), b.pi.view(np.uint32))
    assert a.iterations == b.iterations == 30
    pi0 = np.random.default_rng(1).random(P.n_rows).astype(np.float32)
    pi0 /= pi0.sum()
    c0 = mb.pagerank(None, cfg, backend=be, pi0=pi0)  # same plan, other start
    ctx.release_cache()
    c1 = mb.pagerank(None, cfg, backend=be, pi0=pi0)  # fresh plan
    assert np.array_equal(c0.pi.view(np.uint32), c1.pi.view(np.uint32))
    d = mb.pagerank(None, mb.PageRankConfig(0.5, 1e-30, 7, 2), backend=be)  # new config
    ctx.release_cache()
    e = mb.pagerank(None, mb.PageRankConfig(0.5, 1e-30, 7, 2), backend=be)
    assert d.iterations == e.iterations and np.array_equal(d.pi, e.pi)
    ctx.set_tuning(32, 1, 0)  # no hub table: plan rebuilt, result unchanged
    f = mb.pagerank(None, cfg, backend=be)
    ctx.set_tuning()
    assert np.array_equal(a.pi.view(np.uint32), f.pi.view(np.uint32))
    # a new matrix (possibly at the freed address) gets its own plan
    del be, P
    Q = mb.DeviceMatrix.rmat(ctx, 11, 16, seed=4, transition=True, dtype=np.float32)
    beq = backend(Q, c)
    g = mb.pagerank(None, cfg, backend=beq)
    ctx.release_cache()
    h = mb.pagerank(None, cfg, backend=beq)
    assert g.pi.shape == (Q.n_rows,)
    assert np.array_equal(g.pi.view(np.uint32), h.pi.view(np.uint32))


@pytest.mark.parametrize("relabel", [False, True])
def test_pagerank_on_iteration_observes_every_iterate(ctx, relabel):
    """on_iteration (solvers.hpp:157-158, 209): called once per iteration
    with the iterate in the ORIGINAL vertex order and its ERR; the mass
    invariant holds for each; the observed run equals the fused one bitwise;
    an exception in the hook propagates."""
    c = mb.SimtConfig.make(32, 14, 128)
    P = mb.DeviceMatrix.rmat(ctx, 12, 16, seed=6, transition=True, dtype=np.float32)
    if relabel:
        P, _ = P.relabel_by_degree()
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, mb.generate_tile_for(P, c), c
    cfg = mb.PageRankConfig(0.85, 1e-30, 25, 0)
    seen = []

    def hook(r, pi, err):
        seen.append((r, pi, err))
    a = mb.pagerank(None, cfg, backend=be, on_iteration=hook)
    b = mb.pagerank(None, cfg, backend=be)
    assert [r for r, _, _ in seen] == list(range(1, 26))
    assert np.array_equal(a.pi.view(np.uint32), b.pi.view(np.uint32))
    assert np.array_equal(seen[-1][1].view(np.uint32), b.pi.view(np.uint32))
    for r, pi, err in seen:
        assert abs(pi.astype(np.float64).sum() - 1.0) <= 1e-5
        assert err >= 0.0
    assert np.array_equal(a.residual_history, b.residual_history)

    calls = []

    def boom(r, pi, err):
        calls.append(r)
        if r == 3:
            raise RuntimeError("stop here")
    with pytest.raises(RuntimeError, match="stop here"):
        mb.pagerank(None, cfg, backend=be, on_iteration=boom)
    assert calls == [1, 2, 3]  # the run stops at the raising iterate


@pytest.mark.parametrize("iters", [1, 2, 7, 5000])
def test_device_driven_loop_matches_host_unrolled(ctx, iters):
    """The CUDA-graph WHILE loop (iteration number, scalar slots and the
    stop / max_iters guards read on the device) equals the host-unrolled
    eager loop of the observed path bitwise -- odd and even counts, a single
    iteration, and a count far beyond what an unrolled graph would hold."""
    c = mb.SimtConfig.make(32, 14, 128)
    P = mb.DeviceMatrix.rmat(ctx, 9 if iters > 100 else 11, 16, seed=4, transition=True,
                             dtype=np.float32)
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, mb.generate_tile_for(P, c), c
    cfg = mb.PageRankConfig(0.85, 1e-30, iters, 0)
    a = mb.pagerank(None, cfg, backend=be)
    n_seen = []
    b = mb.pagerank(None, cfg, backend=be, on_iteration=lambda r, pi, e: n_seen.append(r))
    assert a.iterations == b.iterations == iters == len(n_seen)
    assert np.array_equal(a.pi.view(np.uint32), b.pi.view(np.uint32))
    assert np.array_equal(a.residual_history, b.residual_history)


def test_device_driven_loop_early_stop(ctx):
    """Converged at iteration 1 (a directed ring keeps pi uniform, ERR vs the
    uniform yardstick is 0): the WHILE loop ends there, pi and the result
    match the observed (eager) path."""
    n = 4096
    ring = O.Csr(n, n, np.arange(n + 1, dtype=np.int64),
                 np.array([(i - 1) % n for i in range(n)], np.int32), np.ones(n, np.float32))
    P = mb.DeviceMatrix.from_csr(ctx, ring)
    c = mb.SimtConfig.make(32, 14, 128)
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, mb.generate_tile_for(P, c), c
    cfg = mb.PageRankConfig(0.85, 1e-6, 210, 0)
    a = mb.pagerank(None, cfg, backend=be)
    b = mb.pagerank(None, cfg, backend=be, on_iteration=lambda r, pi, e: None)
    assert a.status == "converged" and a.iterations == 1 == b.iterations
    assert np.array_equal(a.pi, b.pi)



def test_plan_recaptures_after_matrix_buffers_change(ctx):
    """A captured PageRank plan holds raw pointers to the matrix's slot copy
    and x hub cache.  Rebuilding either -- an SpMV with another TILE rebuilds
    the slot copy; build_xcache frees and rebuilds the hub encoding -- bumps
    the matrix's buffer generation, and the plan (here the one mbx_pagerank
    keeps on the context, and a PageRankPlan) re-captures before its next
    replay: results stay bitwise equal to the first run."""
    import torch
    c = mb.SimtConfig.make(32, 14, 128)
    c2 = mb.SimtConfig.make(32, 14, 64)
    P = mb.DeviceMatrix.rmat(ctx, 13, 16, seed=5, transition=True, dtype=np.float32)
    n = P.n_rows
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = P, mb.generate_tile_for(P, c), c
    t2 = mb.generate_tile_for(P, c2)
    cfg = mb.PageRankConfig(0.85, 1e-30, 20, 0)
    a = mb.pagerank(None, cfg, backend=be)  # plan cached on the context
    x = O.hash_uniform(3, n, 0.0, 1.0, np.float32)
    y2 = mb.spmv_merbit(P, t2, c2, x, mb.DualBuffer(n, np.float32))  # slot copy for t2
    b = mb.pagerank(None, cfg, backend=be)  # cached plan, slot copy rebuilt for t1
    assert np.array_equal(a.pi.view(np.uint32), b.pi.view(np.uint32))
    # the plan object: run, rebuild the hub cache + slots, run again
    plan = mb.PageRankPlan(P, be.tile_, c, cfg)
    xd = torch.zeros(n, dtype=torch.float32, device="cuda")
    yd = torch.empty(n, dtype=torch.float32, device="cuda")
    ro0, cols0, vals0 = P.download()
    plan.run()
    r1, h1 = plan.result(want_history=True)
    P.build_xcache(FORCE_HUBS)
    assert P.xcache_info()[0] > 0
    torch.cuda.synchronize()
    mb.spmv_device(P, t2, c2, xd.data_ptr(), yd.data_ptr())
    ctx.synchronize()
    plan.run()
    r2, h2 = plan.result(want_history=True)
    assert np.array_equal(h1, h2) and r1.l1_residual == r2.l1_residual
    # the re-captured plan's workspace grew with the hub table (it used to
    # write the gathered hub values past its end, into whatever followed)
    ro1, cols1, vals1 = P.download()
    assert np.array_equal(cols0, cols1) and np.array_equal(vals0.view(np.uint32),
                                                           vals1.view(np.uint32))
    y2b = mb.spmv_merbit(P, t2, c2, x, mb.DualBuffer(n, np.float32))
    assert np.array_equal(y2.view(np.uint32), y2b.view(np.uint32))
    plan.close()


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_default_config_stop_iteration_matches_reference(ctx, dtype):
    """PageRankConfig() defaults (err_tol 1e-10, 210 yardstick iterations)
    against the compiled reference's pagerank<T> over its own MerbitBackend
    (the backend this library replaces): the same stop decision at the same
    iteration -- fp64 converges (17 / 34 iterations here), fp32 runs to
    max_iters in both, because MERBIT's summation order and the CSR
    yardstick's round differently, leaving ERR ~1e-7 -- and the final
    iterates agree.  The yardstick sums each row left to right in T like
    spmv_csr_reference (reference.hpp:28-37); its base term uses the fp64
    dangling mass where rank_update (solvers.hpp:104-109) sums in T."""
    for adj in (O.ring_with_chords(100, 260, 42), O.rmat(10, 16, 3)):
        p = O.build_transition(adj, dtype)
        r = mb.pagerank(p, mb.PageRankConfig(), backend(ctx, p))
        eng = O.RefEngine(p, 32, 14 if dtype == np.float32 else 7, 128, 4)
        want = eng.pagerank(0.85, 1e-10, 210, 210, want_pi=True)
        eng.close()
        assert r.iterations == want["iterations"]
        assert (r.status == "converged") == (want["iterations"] < 210)
        tol = 1e-12 if dtype == np.float64 else 1e-6
        assert np.abs(r.pi.astype(np.float64) - want["pi"].astype(np.float64)).sum() <= tol
