"""GPU K2+K3 SpMV parity (merbit_spmv.hpp:136-352) against the oracle, with the
reference's own test cases (test_kernel.cpp) and BASELINE-size R-MAT inputs.
Tolerances: ToleranceBound 4 eps len max|A| max|x| on the fuzz corpus
(checks.hpp:20-42); north-star 1e-5 (fp32) / 1e-12 (fp64) relative to the
row-sum magnitude sum|a||x| at scale."""
import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb
from helpers import CONFIGS, FORCE_HUBS, first_violation, h, tolerance_bound

pytestmark = pytest.mark.gpu


def run(ctx, a, c, x, trace=None):
    m = mb.DeviceMatrix.from_csr(ctx, a)
    t = mb.generate_tile_for(m, c)
    buf = mb.DualBuffer(a.n_rows, a.values.dtype)
    return mb.spmv_merbit(m, t, c, x, buf, trace).copy()


def test_walkthrough_exact(ctx):
    # test_kernel.cpp:30-46
    a = O.walkthrough()
    for (w, s, b) in [(4, 4, 4), (4, 4, 8), (32, 7, 64), (32, 14, 128)]:
        for dt in (np.float64, np.float32):
            y = run(ctx, a.astype(dt), mb.SimtConfig.make(w, s, b), np.ones(8, dt))
            assert y.tolist() == [15, 0, 40, 36, 119, 141, 177, 67]


def test_fuzz_corpus_within_bound(ctx, golden):
    """test_kernel.cpp:48-77 / acceptance c1 over the whole 504-matrix corpus."""
    for e in golden["fuzz_corpus"]:
        m64 = O.random_matrix(e["shape"], e["seed"])
        x64 = O.seed_test_vector(m64.n_cols, -1.0, 1.0, e["seed"])
        for dt in (np.float64, np.float32):
            a = m64.astype(dt)
            x = x64.astype(dt)
            want = O.spmv_csr_f64(a.astype(np.float64), x.astype(np.float64))
            bound = tolerance_bound(a, x, dt)
            for (w, s, b) in CONFIGS:
                got = run(ctx, a, mb.SimtConfig.make(w, s, b), x)
                assert first_violation(bound, want, got) == -1, (e["shape"], e["seed"], w, s, dt)


def test_block_sizes_bound_and_bitwise_repeat(ctx):
    # test_kernel.cpp:79-99
    for shape in O.SHAPES:
        a = O.random_matrix(shape, 202)
        x = O.seed_test_vector(a.n_cols, -1, 1, 17)
        want = O.spmv_csr_f64(a, x)
        bound = tolerance_bound(a, x, np.float64)
        for block in (32, 128, 256, 992):
            c = mb.SimtConfig.make(32, 7, block)
            got = run(ctx, a, c, x)
            assert first_violation(bound, want, got) == -1
            assert np.array_equal(got.view(np.uint64), run(ctx, a, c, x).view(np.uint64))


def test_dual_buffer_alternating_matches_fresh(ctx):
    # test_kernel.cpp:116-134
    a = O.random_matrix("uniform", 404)
    c = mb.SimtConfig.make(32, 7, 128)
    m = mb.DeviceMatrix.from_csr(ctx, a)
    t = mb.generate_tile_for(m, c)
    alt = mb.DualBuffer(a.n_rows)
    for it in range(10):
        x = O.seed_test_vector(a.n_cols, -1, 1, 1000 + it)
        mb.spmv_merbit(m, t, c, x, alt)
        fresh = mb.DualBuffer(a.n_rows)
        mb.spmv_merbit(m, t, c, x, fresh)
        assert np.array_equal(alt.last_output(), fresh.last_output())
        assert not alt.active().any()


def test_long_row_fast_path(ctx):
    # test_kernel.cpp:160-176 / acceptance c6
    for s in (7, 14):
        c = mb.SimtConfig.make(32, s, 128)
        width = 10 * c.steps_per_tile()
        a = O.single_dense_row(width, 11)
        x = O.seed_test_vector(width, 0.25, 1.75, 13)
        tr = mb.SpmvTrace()
        y = run(ctx, a, c, x, tr)
        assert tr.fast_tiles == 10
        want = O.spmv_csr_f64(a, x)
        assert abs(y[0] - want[0]) / abs(want[0]) <= 1e-12


def test_trace_counts_match_reference(ctx, golden):
    for e in golden["fuzz_corpus"][:120]:
        m = O.random_matrix(e["shape"], e["seed"])
        c = mb.SimtConfig.make(32, 14, 128)
        t = mb.generate_tile_for(mb.DeviceMatrix.from_csr(ctx, m), c)
        tr = mb.trace_counts(t)
        assert [tr.fast_tiles, tr.normal_tiles, tr.skipped_tiles] == e["tiles"]["32,14"]["trace"]


def test_edge_shapes(ctx):
    # test_kernel.cpp:220-239
    c = mb.SimtConfig.make(4, 4, 8)
    empty = O.Csr(37, 5, np.zeros(38, np.int64), np.zeros(0, np.int32), np.zeros(0))
    y = run(ctx, empty, c, np.full(5, 3.0))
    assert y.shape == (37,) and not y.any()
    none = O.Csr(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    assert run(ctx, none, c, np.zeros(0)).size == 0


def test_error_paths(ctx):
    # test_kernel.cpp:241-267
    a = O.walkthrough()
    c = mb.SimtConfig.make(4, 4, 4)
    m = mb.DeviceMatrix.from_csr(ctx, a)
    t = mb.generate_tile_for(m, c)
    x = np.ones(8)
    with pytest.raises(mb.ConfigError):
        mb.spmv_merbit(m, t, mb.SimtConfig.make(32, 7, 64), x, mb.DualBuffer(8))
    stale = mb.generate_tile_for(mb.DeviceMatrix.from_csr(ctx, O.single_dense_row(16, 3)), c)
    with pytest.raises(mb.ConfigError):
        mb.spmv_merbit(m, stale, c, x, mb.DualBuffer(8))
    with pytest.raises(mb.DimensionError):
        mb.spmv_merbit(m, t, c, np.ones(7), mb.DualBuffer(8))
    with pytest.raises(mb.DimensionError):
        mb.spmv_merbit(m, t, c, x, mb.DualBuffer(7))
    with pytest.raises(mb.ConfigError):
        mb.SimtConfig.make(32, 20, 32)
    bad = O.Csr(2, 2, np.array([0, 1, 2]), np.array([0, 5], np.int32), np.ones(2))
    with pytest.raises(mb.DimensionError):
        mb.DeviceMatrix.upload(ctx, 2, 2, bad.row_offsets, bad.col_indices.astype(np.int64),
                               bad.values)


def _rel_err(y, want, mag):
    return np.abs(np.asarray(y, np.float64) - want) / np.where(mag > 0, mag, 1.0)


@pytest.mark.parametrize("scale", [16, 20])
def test_rmat_fp32_within_1e5(ctx, scale):
    """C1 (scale 20): y within 1e-5 of the fp64-accumulated oracle relative to
    sum|a||x| per row; also reports the reference fp32 sequential distance."""
    m = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, dtype=np.float32)
    ro, cols, vals = m.download()
    a = O.Csr(m.n_rows, m.n_cols, ro, cols, vals)
    x = O.hash_uniform(1, m.n_cols, -1.0, 1.0, np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(m, c)
    buf = mb.DualBuffer(m.n_rows, np.float32)
    y = mb.spmv_merbit(m, t, c, x, buf).copy()
    want, mag = O.spmv_csr_f32_acc64(a, x, nthreads=8)
    assert _rel_err(y, want, mag).max() <= 1e-5
    empty = np.diff(ro) == 0
    assert not y[empty].any()
    y2 = mb.spmv_merbit(m, t, c, x, buf)
    assert np.array_equal(y.view(np.uint32), y2.view(np.uint32))  # deterministic


@pytest.mark.parametrize("scale", [16, 20])
def test_rmat_fp64_within_1e12(ctx, scale):
    m = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, dtype=np.float64, lo=-1.0, hi=1.0)
    ro, cols, vals = m.download()
    a = O.Csr(m.n_rows, m.n_cols, ro, cols, vals)
    x = O.hash_uniform(1, m.n_cols, -1.0, 1.0, np.float64)
    c = mb.SimtConfig.make(32, 7, 128)
    t = mb.generate_tile_for(m, c)
    y = mb.spmv_merbit(m, t, c, x, mb.DualBuffer(m.n_rows, np.float64))
    want, mag = O.spmv_csr_f64(a, x, nthreads=8, want_abs=True)
    assert _rel_err(y, want, mag).max() <= 1e-12


def test_power_law_long_and_empty_rows_fp64(ctx):
    """C3-style: Zipf row lengths with rows of >= 100*omega*sigma nonzeros and
    exactly 10% empty rows (small analogue of BASELINE config 3)."""
    rng = np.random.default_rng(5)
    n = 1 << 14
    lens = np.minimum((40000 / (np.arange(n) + 1) ** 0.9).astype(np.int64) + 1, n)
    lens[rng.permutation(n)[: n // 10]] = 0
    ro = np.zeros(n + 1, np.int64)
    ro[1:] = np.cumsum(lens)
    cols = np.concatenate([np.sort(rng.choice(n, l, replace=False)) if l else
                           np.zeros(0, np.int64) for l in lens]).astype(np.int32)
    vals = rng.uniform(-1, 1, ro[-1])
    a = O.Csr(n, n, ro, cols, vals)
    x = rng.uniform(-1, 1, n)
    c = mb.SimtConfig.make(32, 7, 128)
    tr = mb.SpmvTrace()
    y = run(ctx, a, c, x, tr)
    want, mag = O.spmv_csr_f64(a, x, want_abs=True)
    assert _rel_err(y, want, mag).max() <= 1e-12
    assert tr.fast_tiles >= 100 and tr.skipped_tiles >= 0
    assert not y[lens == 0].any()


def _short_rows(n, seed, dt):
    """Rows of 0-3 nonzeros (30 % forced empty): ~180 rows per 32x14 tile,
    more than the slot kernel's 64-row commit buffer."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 4, n)
    lens[rng.random(n) < 0.3] = 0
    ro = np.zeros(n + 1, np.int64)
    ro[1:] = np.cumsum(lens)
    cols = rng.integers(0, n, int(ro[-1])).astype(np.int32)
    for r in range(0, n):  # CSR order: ascending columns within a row
        a0, a1 = ro[r], ro[r + 1]
        if a1 - a0 > 1:
            cols[a0:a1] = np.sort(cols[a0:a1])
    vals = rng.uniform(-1, 1, int(ro[-1])).astype(dt)
    return O.Csr(n, n, ro, cols, vals)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_many_rows_per_tile(ctx, dt):
    """Tiles closing more rows than the 64-row commit buffer commit lane by
    lane (slot layout) -- same bound, zero on every empty row."""
    a = _short_rows(30000, 21, dt)
    x = O.seed_test_vector(a.n_cols, -1, 1, 5).astype(dt)
    want = O.spmv_csr_f64(a.astype(np.float64), x.astype(np.float64))
    bound = tolerance_bound(a, x, dt)
    for (w, s, b) in [(32, 14 if dt == np.float32 else 7, 128), (32, 7, 32)]:
        got = run(ctx, a, mb.SimtConfig.make(w, s, b), x)
        assert first_violation(bound, want, got) == -1
        assert not got[np.diff(a.row_offsets) == 0].any()


def test_slot_and_staged_layouts_agree(ctx):
    """Both K2 layouts on one R-MAT matrix: within 1e-5 of each other relative
    to sum|a||x| (they differ only in the fast-tile summation order), and the
    slot copy is cached on the matrix after the first SpMV."""
    m = mb.DeviceMatrix.rmat(ctx, 16, 16, seed=8, dtype=np.float32)
    ro, cols, vals = m.download()
    a = O.Csr(m.n_rows, m.n_cols, ro, cols, vals)
    x = O.hash_uniform(3, m.n_cols, -1.0, 1.0, np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(m, c)
    ys = []
    for layout in (1, 0):
        ctx.set_layout(layout)
        ys.append(mb.spmv_merbit(m, t, c, x, mb.DualBuffer(m.n_rows, np.float32)).copy())
        if layout == 1:
            assert m.slot_info()[0] >= m.nnz
    ctx.set_layout(1)
    _, mag = O.spmv_csr_f32_acc64(a, x)
    assert _rel_err(ys[0], ys[1].astype(np.float64), mag).max() <= 1e-5


@pytest.mark.parametrize("tuning", [(32, 1, 0, 147456, 1), (16, 2, 0, 147456, 0),
                                    (8, 4, 0, 147456, 1), (32, 1, FORCE_HUBS, 131072, 1),
                                    (16, 2, FORCE_HUBS, 147456, 0)])
@pytest.mark.parametrize("layout", [1, 0])
def test_launch_shapes_and_hub_cache_are_bitwise_invariant(tuning, layout):
    """Every K2 launch shape, the L2 prefetch and the shared-memory x hub cache
    change only speed: y is bitwise identical to the default launch."""
    ctx = mb.Context(0)
    ctx.set_layout(layout)
    m = mb.DeviceMatrix.rmat(ctx, 16, 16, seed=4, dtype=np.float32)
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(m, c)
    x = O.hash_uniform(9, m.n_cols, -1.0, 1.0, np.float32)
    y0 = mb.spmv_merbit(m, t, c, x, mb.DualBuffer(m.n_rows, np.float32)).copy()
    w, cps, hubs, smem, pf = tuning
    ctx.set_tuning(w, cps, hubs, smem, pf)
    m.build_xcache(hubs)
    if hubs != 0:
        assert m.xcache_info()[0] > 0
    y1 = mb.spmv_merbit(m, t, c, x, mb.DualBuffer(m.n_rows, np.float32))
    assert np.array_equal(y0.view(np.uint32), y1.view(np.uint32))


@pytest.mark.parametrize("dtype,relabel", [(np.float32, False), (np.float32, True),
                                           (np.float64, False)])
def test_compact_matrix_round_trip(ctx, dtype, relabel):
    """mbx_matrix_compact: the CSR values and columns are freed once the slot
    copy exists (resident bytes drop to about the slot copy), SpMVs keep
    running bitwise-equal from the slots, and any CSR reader (download here,
    then a row slice and a relabelling) gets the CSR rebuilt bit-for-bit from
    the slot copy -- hub-encoded columns decoded, both hub encodings."""
    from paper_2605_07391_b200.merbit import row_slice
    A = mb.DeviceMatrix.rmat(ctx, 13, 16, seed=8, dtype=dtype, lo=-1.0, hi=1.0)
    if relabel:
        A, _ = A.relabel_by_degree(want_rank=False)
    ro, cols, vals = A.download()
    c = mb.SimtConfig.make(32, 14 if dtype == np.float32 else 7, 128)
    t = mb.generate_tile_for(A, c)
    A.build_xcache(FORCE_HUBS)
    x = O.hash_uniform(9, A.n_cols, -1.0, 1.0, dtype)
    y1 = mb.spmv_merbit(A, t, c, x, mb.DualBuffer(A.n_rows, dtype)).copy()
    if A.slot_info()[0] == 0:  # staged K2 layout: no slot copy to compact onto
        with pytest.raises(mb.ConfigError):
            A.compact(t)
        return
    full = A.resident_bytes()
    A.compact(t)
    csr_bytes = A.nnz * (np.dtype(dtype).itemsize + 4)
    tile_copy = 4 * (2 * (t.tile_num + 1) + t.lane_num)  # the compact form's TILE
    assert A.resident_bytes() == full - csr_bytes + tile_copy
    y2 = mb.spmv_merbit(A, t, c, x, mb.DualBuffer(A.n_rows, dtype))
    assert np.array_equal(y1.view(np.uint8), y2.view(np.uint8))
    ro2, cols2, vals2 = A.download()  # rebuilt from the slot copy
    assert np.array_equal(ro2, ro) and np.array_equal(cols2, cols)
    assert np.array_equal(vals2.view(np.uint8), vals.view(np.uint8))
    # compact again, then CSR readers of other kinds
    A.compact(t)
    half = A.n_rows // 2
    S = row_slice(A, 0, half)
    rs, cs, vs_ = S.download()
    assert np.array_equal(cs, cols[:ro[half]]) and np.array_equal(vs_, vals[:ro[half]])


@pytest.mark.parametrize("cfg", [(4, 4, 16), (32, 7, 64), (32, 14, 128)])
def test_trace_deposits_conserve_every_product(ctx, cfg):
    """tests/test_kernel.cpp:136-158 on the device: with collect_deposits the
    trace holds every (row, partial) contribution the decomposition forms;
    per-row totals reproduce y within the reference's ToleranceBound, rows in
    [0, n_rows] (the terminal row may appear), every shape of the corpus --
    and the same for a degree-relabelled matrix (rows in the original
    vertex order)."""
    w, s, b = cfg
    for shape in O.SHAPES:
        a = O.random_matrix(shape, 505)
        x = O.seed_test_vector(a.n_cols, -1, 1, 31)
        m = mb.DeviceMatrix.from_csr(ctx, a)
        c = mb.SimtConfig.make(w, s, b)
        t = mb.generate_tile(a.row_offsets, a.n_rows, a.nnz, c, ctx)
        tr = mb.SpmvTrace(collect_deposits=True)
        mb.spmv_merbit(m, t, c, x, mb.DualBuffer(a.n_rows, np.float64), tr)
        totals = np.zeros(a.n_rows)
        for row, amount in tr.deposits:
            assert 0 <= row <= a.n_rows
            if row < a.n_rows:
                totals[row] += amount
        want = O.spmv_csr_f64(a, x)
        assert first_violation(tolerance_bound(a, x, np.float64), want, totals) == -1, shape
        assert tr.normal_tiles + tr.fast_tiles + tr.skipped_tiles == t.tile_num
    P = mb.DeviceMatrix.rmat(ctx, 10, 16, seed=3, dtype=np.float64, lo=-1.0, hi=1.0)
    ro, cols, vals = P.download()
    Q, _ = P.relabel_by_degree(want_rank=False)
    c = mb.SimtConfig.make(32, 7, 128)
    tq = mb.generate_tile_for(Q, c)
    x = O.seed_test_vector(P.n_cols, -1, 1, 7)
    tr = mb.SpmvTrace(collect_deposits=True)
    y = mb.spmv_merbit(Q, tq, c, x, mb.DualBuffer(P.n_rows, np.float64), tr)
    totals = np.zeros(P.n_rows)
    for row, amount in tr.deposits:
        if row < P.n_rows:
            totals[row] += amount
    a = O.Csr(P.n_rows, P.n_cols, ro, cols, vals)
    want, mag = O.spmv_csr_f64(a, x, want_abs=True)
    assert (np.abs(totals - want) <= 1e-12 * np.where(mag > 0, mag, 1)).all()
    assert (np.abs(y - want) <= 1e-12 * np.where(mag > 0, mag, 1)).all()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_automatic_launch_shape(dtype):
    """set_tuning(0, 0): the automatic K2 launch shape (16 x 2 and no TMA
    staging for a small matrix without a hub table) -- bitwise the result of
    an explicit 32 x 1 launch; a half-automatic shape is a config error."""
    ctx = mb.Context(0)
    m = mb.DeviceMatrix.rmat(ctx, 15, 16, seed=6, dtype=dtype)
    c = mb.SimtConfig.make(32, 14 if dtype == np.float32 else 7, 128)
    t = mb.generate_tile_for(m, c)
    x = O.hash_uniform(3, m.n_cols, -1.0, 1.0, dtype)
    ys = []
    for shape in ((0, 0), (32, 1), (0, 0)):
        ctx.set_tuning(*shape, -1)
        m.build_xcache()
        assert m.xcache_info()[0] == 0  # small: no automatic hub table
        ys.append(mb.spmv_merbit(m, t, c, x, mb.DualBuffer(m.n_rows, dtype)).copy())
    u = np.uint32 if dtype == np.float32 else np.uint64
    assert np.array_equal(ys[0].view(u), ys[1].view(u))
    assert np.array_equal(ys[0].view(u), ys[2].view(u))
    with pytest.raises(mb.ConfigError):
        ctx.set_tuning(0, 1, -1)
