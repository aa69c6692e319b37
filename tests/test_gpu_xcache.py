"""The x hub cache's column selection (xcache.cu): the hub set is the top-h
columns by reference count, ties in ascending column order, stored in
ascending column order (a column's slot is its rank).  Below kSampleRuns
runs of 32 nonzeros the sample stride is 1, so the counts the device ranks
are the exact column counts and the set can be checked on the host."""
import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb
from helpers import FORCE_HUBS

pytestmark = pytest.mark.gpu


def top_by_count(cols, n, h):
    cnt = np.bincount(cols, minlength=n)
    order = np.lexsort((np.arange(n), -cnt))  # count desc, column asc
    return np.sort(order[:h]), cnt


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("scale", [14, 16])
def test_hub_set_is_top_h_by_count(ctx, dtype, scale):
    A = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=2, transition=True, dtype=dtype)
    A.build_xcache(FORCE_HUBS)
    hubs = A.hub_columns()
    h = hubs.size
    assert h > 0
    assert np.all(np.diff(hubs) > 0)  # ascending, unique
    _, cols, _ = A.download(want_values=False)
    want, cnt = top_by_count(cols, A.n_cols, h)
    assert np.array_equal(hubs, want)
    # and the SpMV through the table is bitwise the one without it
    c = mb.SimtConfig.make(32, 14 if dtype == np.float32 else 7, 128)
    t = mb.generate_tile_for(A, c)
    x = O.hash_uniform(5, A.n_cols, -1.0, 1.0, dtype)
    y1 = mb.spmv_merbit(A, t, c, x, mb.DualBuffer(A.n_rows, dtype)).copy()
    A.build_xcache(0)
    y0 = mb.spmv_merbit(A, t, c, x, mb.DualBuffer(A.n_rows, dtype))
    assert np.array_equal(y0.view(np.uint8), y1.view(np.uint8))


def test_capped_counts_rank_exactly(ctx):
    """Counts past the selection histogram's last bin (>= 8191): the device
    falls back to sorting them, still the exact top-h.  Column c is
    referenced 8200 + c times (c < 300); a 100-hub cap picks 200..299."""
    counts = 8200 + np.arange(300)
    n_rows = int(counts.max())
    rows = [np.nonzero(counts > r)[0].astype(np.int32) for r in range(n_rows)]
    ro = np.zeros(n_rows + 1, np.int64)
    ro[1:] = np.cumsum([len(r) for r in rows])
    cols = np.concatenate(rows)
    vals = np.ones(cols.size, np.float32)
    A = mb.DeviceMatrix.from_csr(ctx, O.Csr(n_rows, 300, ro, cols, vals))
    A.build_xcache(100)
    assert np.array_equal(A.hub_columns(), np.arange(200, 300))
    A.build_xcache(300)
    assert np.array_equal(A.hub_columns(), np.arange(300))


def test_automatic_mode_skips_small_matrices(ctx):
    """build_xcache() (automatic): no table below 4096 nonzeros per resident
    K2 warp (148 x 32 warps: ~19.4 M nonzeros), where K2 is latency-bound;
    a table above it."""
    A = mb.DeviceMatrix.rmat(ctx, 16, 16, seed=2, transition=True, dtype=np.float32)
    A.build_xcache()
    assert A.xcache_info()[0] == 0
    A.build_xcache(FORCE_HUBS)
    assert A.xcache_info()[0] > 0
    B = mb.DeviceMatrix.rmat(ctx, 21, 16, seed=2, transition=True, dtype=np.float32)
    B.build_xcache()
    assert B.xcache_info()[0] > 0


def test_gather_profile_picks_the_staging(ctx):
    """The hub sample also measures gather locality (distinct 32-byte x
    sectors per 32 consecutive nonzeros): a 27-point stencil ~11, R-MAT ~31.
    Below 16 the fp32 K2 prefetches each next tile into L2 -- results are
    bitwise those of the unprefetched kernel."""
    S = mb.DeviceMatrix.stencil27(ctx, 64, np.float32)
    S.build_xcache(FORCE_HUBS)
    assert S.xcache_info()[0] == 0  # no column can be a hub (27 references)
    assert 0.0 < S.gather_sectors() < 16.0
    R = mb.DeviceMatrix.rmat(ctx, 16, 16, seed=2, transition=True, dtype=np.float32)
    R.build_xcache(FORCE_HUBS)
    assert R.gather_sectors() > 24.0
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(S, c)
    x = O.hash_uniform(7, S.n_cols, -1.0, 1.0, np.float32)
    y_auto = mb.spmv_merbit(S, t, c, x, mb.DualBuffer(S.n_rows, np.float32)).copy()
    ctx.set_tuning(32, 1, -1, prefetch=0)
    try:
        y0 = mb.spmv_merbit(S, t, c, x, mb.DualBuffer(S.n_rows, np.float32))
    finally:
        ctx.set_tuning(prefetch=-1)
    assert np.array_equal(y0.view(np.uint32), y_auto.view(np.uint32))


def test_automatic_mode_skips_local_matrices(ctx):
    """build_xcache() (automatic) on a matrix big enough for a table: a
    device pilot of distinct x sectors per run finds the stencil's gathers
    local (< 16) and no column is counted -- no table, the locality kept for
    K2's staging; R-MAT (~31 sectors) goes on to the counted selection.
    SpMV results are bitwise those of a forced table."""
    S = mb.DeviceMatrix.stencil27(ctx, 100, np.float32)  # 27 M nonzeros
    S.build_xcache()
    assert S.xcache_info()[0] == 0
    assert 0.0 < S.gather_sectors() < 16.0
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(S, c)
    x = O.hash_uniform(5, S.n_cols, -1.0, 1.0, np.float32)
    y_auto = mb.spmv_merbit(S, t, c, x, mb.DualBuffer(S.n_rows, np.float32)).copy()
    S.build_xcache(FORCE_HUBS)
    y_forced = mb.spmv_merbit(S, t, c, x, mb.DualBuffer(S.n_rows, np.float32))
    assert np.array_equal(y_auto.view(np.uint32), y_forced.view(np.uint32))
    R = mb.DeviceMatrix.rmat(ctx, 21, 16, seed=2, transition=True, dtype=np.float32)
    R.build_xcache()
    assert R.xcache_info()[0] > 0 and R.gather_sectors() > 24.0


def test_hub_budget_shrinks_as_x_outgrows_l2():
    """K2's shared-memory budget per SM depends on x's size (160 KB up to
    192 MB of fp32 x, 128 KB to 384 MB, 96 KB beyond): the same 40,000
    columns referenced 1024 times each (a table needs > 4 x 148 references)
    fill 38,652 hub slots when x has 1 M entries, 30,460 at 64 M entries
    (256 MB) and 22,268 at 120 M (480 MB) -- with the default K2 layout (the
    slot copy; the staged layout's larger per-warp buffers leave fewer)."""
    ctx = mb.Context(0)
    hot, refs = 40000, 1024
    n_rows = hot * refs // 32
    # row r: hot columns (7919 r + 1249 i) mod 40000, i < 32 -- distinct in a
    # row, each column exactly `refs` times, and no aliasing with the
    # selection's every-S-th-run sample
    r = np.arange(n_rows, dtype=np.int64)[:, None]
    i = np.arange(32, dtype=np.int64)[None, :]
    cols = (((7919 * r + 1249 * i) % hot) * 25).astype(np.int32)
    cols.sort(axis=1)
    ro = np.arange(n_rows + 1, dtype=np.int64) * 32
    got = []
    for n_cols in (1 << 20, 64 << 20, 120 << 20):
        A = mb.DeviceMatrix.from_csr(ctx, O.Csr(n_rows, n_cols, ro, cols.reshape(-1),
                                                np.ones(cols.size, np.float32)))
        A.build_xcache(FORCE_HUBS)
        got.append(A.xcache_info()[0])
        del A
    assert got == [38652, 30460, 22268], got
