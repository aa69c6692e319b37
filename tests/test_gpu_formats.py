"""GPU side of the file formats: coo_to_csr<T> on the
device (mbx_matrix_from_coo) against the reference's own coo_to_csr, and MBTL
caches written from / loaded into device TILEs."""
import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb
from paper_2605_07391_b200 import formats as F

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built")


def _dup_heavy_coo(seed, n_rows=300, n_cols=200, n=6000):
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, n_rows, n)
    cols = rng.integers(0, n_cols, n)
    # force long duplicate runs with values of very different magnitude, so
    # a different summation order would change the low bits
    rows[:600] = 5
    cols[:600] = 7
    vals = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-8, 9, n)
    return F.CooTriples(n_rows, n_cols, rows, cols, vals)


@needs_ref
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_from_coo_matches_reference_coo_to_csr(ctx, dt):
    for seed in range(3):
        coo = _dup_heavy_coo(seed)
        m = F.matrix_from_coo(coo, dt, ctx)
        ro, cols, vals = m.download()
        want = O.ref().coo_to_csr(dict(n_rows=coo.n_rows, n_cols=coo.n_cols, rows=coo.rows,
                                       cols=coo.cols, vals=coo.vals))
        assert (m.n_rows, m.n_cols, m.nnz) == (want.n_rows, want.n_cols, want.nnz)
        assert np.array_equal(ro, want.row_offsets)
        assert np.array_equal(cols, want.col_indices)
        # coo_to_csr<T>: the fp64 duplicate sum, rounded to T once
        assert np.array_equal(vals, want.values.astype(dt))


def test_from_coo_edges_and_errors(ctx):
    empty = F.CooTriples(4, 3, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    m = F.matrix_from_coo(empty, np.float64, ctx)
    ro, cols, _ = m.download()
    assert m.nnz == 0 and ro.tolist() == [0, 0, 0, 0, 0]
    trailing = F.CooTriples(6, 6, np.array([0, 2]), np.array([1, 5]), np.array([1.0, 2.0]))
    ro, cols, vals = F.matrix_from_coo(trailing, np.float64, ctx).download()
    assert ro.tolist() == [0, 1, 1, 2, 2, 2, 2] and cols.tolist() == [1, 5]
    bad = F.CooTriples(2, 2, np.array([0, 3]), np.array([1, 1]), np.array([1.0, 1.0]))
    with pytest.raises(mb.DimensionError, match=r"coo entry \(3, 1\) outside 2x2"):
        F.matrix_from_coo(bad, np.float64, ctx)


def test_matrix_market_to_spmv(ctx, tmp_path):
    """Matrix Market file -> device CSR -> TILE -> SpMV within the reference's
    ToleranceBound of the CSR oracle."""
    lap = O.five_point_laplacian(20)
    rows = np.repeat(np.arange(lap.n_rows), np.diff(lap.row_offsets))
    coo = F.CooTriples(lap.n_rows, lap.n_cols, rows, lap.col_indices.astype(np.int64),
                       lap.values)
    path = str(tmp_path / "lap.mtx")
    F.write_matrix_market_file(path, coo)
    m = F.matrix_from_coo(F.load_matrix_any(path), np.float64, ctx)
    c = mb.SimtConfig.make(32, 7, 128)
    t = mb.generate_tile_for(m, c)
    x = O.seed_test_vector(m.n_cols, -1, 1, 3)
    y = mb.spmv_merbit(m, t, c, x, mb.DualBuffer(m.n_rows))
    assert np.allclose(y, O.spmv_csr_f64(lap, x), rtol=0, atol=1e-13)


@needs_ref
def test_tile_cache_device_round_trip(ctx, tmp_path):
    m = mb.DeviceMatrix.rmat(ctx, 14, 16, seed=2, dtype=np.float32)
    ro, _, _ = m.download(want_values=False)
    for (w, s) in ((32, 14), (32, 7), (4, 4)):
        c = mb.SimtConfig.make(w, s, 128 if w == 32 else 16)
        t = mb.generate_tile_for(m, c)
        path = str(tmp_path / f"t{w}_{s}.mbtl")
        F.write_tile_cache(path, t, "f32")
        # the reference's reader sees exactly its own generate_tile
        got = O.ref().tile_cache_read(path)
        want = O.generate_tile(ro, m.n_rows, m.nnz, w, s)
        for k, v in zip(("tile_x", "tile_y", "lane_desc"), want):
            assert np.array_equal(got[k], v)
        # and the reference's file loads back into an identical device TILE
        ref_path = str(tmp_path / f"r{w}_{s}.mbtl")
        O.ref().tile_cache_write(ref_path, ro, m.n_rows, m.nnz, w, s, False)
        t2, prec = F.load_tile_cache(ref_path, ctx)
        assert prec == "f32"
        for a, b in zip(t.download(), t2.download()):
            assert np.array_equal(a, b)
        x = O.hash_uniform(4, m.n_cols, -1, 1, np.float32)
        y1 = mb.spmv_merbit(m, t, c, x, mb.DualBuffer(m.n_rows, np.float32)).copy()
        y2 = mb.spmv_merbit(m, t2, c, x, mb.DualBuffer(m.n_rows, np.float32))
        assert np.array_equal(y1.view(np.uint32), y2.view(np.uint32))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_build_transition_is_the_reference(ctx, dt):
    """build_transition on the device == the oracle's restatement (pinned to
    the reference), bitwise: pattern, ascending sources, T(1)/T(outdeg)."""
    g = mb.DeviceMatrix.rmat(ctx, 12, 16, seed=5, dtype=np.float64)
    ro, cols, vals = g.download()
    rmat12 = O.Csr(g.n_rows, g.n_cols, ro, cols, vals)
    for adj in (O.ring_with_chords(100, 260, 42), rmat12, O.walkthrough()):
        a = adj.astype(dt)
        P = mb.DeviceMatrix.from_csr(ctx, a).build_transition()
        ro, cols, vals = P.download()
        want = O.build_transition(a, dt)
        assert np.array_equal(ro, want.row_offsets)
        assert np.array_equal(cols, want.col_indices)
        assert np.array_equal(vals, want.values)
    rect = O.single_dense_row(4, 1)
    with pytest.raises(mb.DimensionError):
        mb.DeviceMatrix.from_csr(ctx, rect).build_transition()


def test_degree_stats_reference_cases(ctx):
    """test_sparse_core.cpp:95-113: the walkthrough fixture (34 nonzeros over
    8 rows) and a 2-row matrix with 16 nonzeros; no rows -> dimension_error."""
    a = O.walkthrough()
    m = mb.DeviceMatrix.from_csr(ctx, a)
    single = m.degree_stats(14)
    assert abs(single.mean_degree - 4.25) <= 1e-12 and single.low_degree
    dbl = m.degree_stats(7)
    assert dbl.low_degree and dbl.max_degree == 7 and dbl.empty_rows == 1
    cols = np.array(list(range(0, 16, 2)) + list(range(1, 16, 2)), np.int32)
    wide = O.Csr(2, 16, np.array([0, 8, 16], np.int64), cols, np.ones(16))
    assert not mb.DeviceMatrix.from_csr(ctx, wide).degree_stats(7).low_degree
    empty = mb.DeviceMatrix.from_csr(ctx, O.Csr(0, 4, np.zeros(1, np.int64),
                                                np.zeros(0, np.int32), np.zeros(0)))
    with pytest.raises(mb.DimensionError):
        empty.degree_stats(7)


@pytest.mark.parametrize("case", ["rmat", "empty_rows", "one_dense_row", "long_row", "mid_rows",
                                  "single", "no_nnz"])
def test_relabel_by_degree_structure(ctx, case):
    """P' = Q P Q^T exactly: rank = vertices by descending column count (ties
    by id), row rank[r] of P' holds row r of P with columns renamed and sorted
    ascending, values carried along -- checked against numpy."""
    rng = np.random.default_rng(11)
    if case == "rmat":
        a = O.rmat(11, 8, 2, transposed=True)
        a = O.Csr(a.n_rows, a.n_cols, a.row_offsets, a.col_indices,
                  rng.random(a.col_indices.size))
    elif case == "empty_rows":
        n = 300
        lens = rng.integers(0, 6, n)
        lens[rng.random(n) < 0.4] = 0
        ro = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        cols = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]
                              ).astype(np.int32)
        a = O.Csr(n, n, ro, cols, rng.random(cols.size))
    elif case == "one_dense_row":
        n = 2000
        ro = np.zeros(n + 1, np.int64)
        ro[1:] = n  # row 0 holds every column, the rest are empty
        a = O.Csr(n, n, ro, np.arange(n, dtype=np.int32), rng.random(n))
    elif case == "long_row":
        # a row beyond the segmented sort's long-row cut (65536): sorted on its own
        n = 70000
        lens = np.zeros(n, np.int64)
        lens[0] = n
        lens[1:200] = rng.integers(1, 40, 199)
        ro = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        cols = np.concatenate([np.arange(n)] + [np.sort(rng.choice(n, l, replace=False))
                                                for l in lens[1:200]]).astype(np.int32)
        a = O.Csr(n, n, ro, cols, rng.random(cols.size))
    elif case == "mid_rows":
        # every sort route: CUB small (<= 128), shared-memory bitonic (129..1024
        # and 1025..8192), CUB large (8193..65535)
        n = 30000
        lens = rng.integers(0, 20, n)
        for i, l in enumerate([128, 129, 257, 1000, 1024, 1025, 3000, 8192, 8193, 16385, 20000]):
            lens[5 + 37 * i] = l
        ro = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        cols = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]
                              ).astype(np.int32)
        a = O.Csr(n, n, ro, cols, rng.random(cols.size))
    elif case == "single":
        a = O.Csr(1, 1, np.array([0, 1], np.int64), np.array([0], np.int32), np.array([2.5]))
    else:
        a = O.Csr(5, 5, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0))
    m = mb.DeviceMatrix.from_csr(ctx, a)
    q, rank = m.relabel_by_degree()
    n = a.n_rows
    cnt = np.bincount(a.col_indices, minlength=n)
    want_rank = np.empty(n, np.int64)
    want_rank[np.lexsort((np.arange(n), -cnt))] = np.arange(n)
    assert np.array_equal(rank, want_rank)
    ro2, c2, v2 = q.download()
    lens = np.diff(a.row_offsets)
    assert np.array_equal(np.diff(ro2)[want_rank], lens)
    for r in np.nonzero(lens)[0]:
        seg = slice(a.row_offsets[r], a.row_offsets[r + 1])
        newc = want_rank[a.col_indices[seg]]
        order = np.argsort(newc, kind="stable")
        s2 = slice(ro2[want_rank[r]], ro2[want_rank[r] + 1])
        assert np.array_equal(c2[s2], newc[order])
        assert np.array_equal(v2[s2], a.values[seg][order])
