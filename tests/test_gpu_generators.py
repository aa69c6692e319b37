"""GPU: the device generators behind BASELINE configs C3 (power-law, long
and empty rows, fp64) and C5 (27-point stencil), and MERBIT parity on them."""
import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb
from helpers import FORCE_HUBS

pytestmark = pytest.mark.gpu


def stencil_reference(g):
    rows, cols, vals = [], [], []
    for i in range(g):
        for j in range(g):
            for k in range(g):
                r = (i * g + j) * g + k
                for di in (-1, 0, 1):
                    for dj in (-1, 0, 1):
                        for dk in (-1, 0, 1):
                            a, b, c = i + di, j + dj, k + dk
                            if 0 <= a < g and 0 <= b < g and 0 <= c < g:
                                cc = (a * g + b) * g + c
                                rows.append(r)
                                cols.append(cc)
                                vals.append(26.0 if cc == r else -1.0)
    n = g ** 3
    ro = np.zeros(n + 1, np.int64)
    np.add.at(ro, np.array(rows) + 1, 1)
    return np.cumsum(ro), np.array(cols, np.int32), np.array(vals)


@pytest.mark.parametrize("g", [1, 2, 5, 9])
def test_stencil27_structure_and_spmv(ctx, g):
    m = mb.DeviceMatrix.stencil27(ctx, g, np.float64)
    ro, cols, vals = m.download()
    wro, wcols, wvals = stencil_reference(g)
    assert np.array_equal(ro, wro) and np.array_equal(cols, wcols) and np.array_equal(vals, wvals)
    assert m.nnz == (3 * g - 2) ** 3 if g > 1 else m.nnz == 1
    c = mb.SimtConfig.make(32, 7, 128)
    t = mb.generate_tile_for(m, c)
    for a_, b_ in zip(t.download(), O.generate_tile(ro, m.n_rows, m.nnz, 32, 7)):
        assert np.array_equal(a_, b_)
    x = O.hash_uniform(3, m.n_cols, -1.0, 1.0)
    y = mb.spmv_merbit(m, t, c, x, mb.DualBuffer(m.n_rows, np.float64))
    want, mag = O.spmv_csr_f64(O.Csr(m.n_rows, m.n_cols, ro, cols, vals), x, want_abs=True)
    assert np.all(np.abs(y - want) <= 1e-12 * np.maximum(mag, 1e-300))


def test_stencil27_c5_nnz_formula():
    # BASELINE C5 at g = 400 has (3g-2)^3 = 1198^3 = 1,719,374,392 nonzeros
    assert (3 * 400 - 2) ** 3 == 1719374392


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_powerlaw_c3_structure_and_spmv(ctx, dtype):
    log2n = 15
    m = mb.DeviceMatrix.powerlaw(ctx, log2n, seed=3, dtype=dtype)
    ro, cols, vals = m.download()
    n = 1 << log2n
    lens = np.diff(ro)
    assert int((lens == 0).sum()) == n - (n - n // 10)  # exactly 10 % empty rows
    assert lens.max() == n  # hub rows saturate at n columns
    for r in np.nonzero(lens > 1)[0][:2000]:
        seg = cols[ro[r]:ro[r + 1]]
        assert np.all(np.diff(seg) > 0)  # strictly increasing, valid CSR
    assert np.all(vals >= -1.0) and np.all(vals < 1.0)
    sigma = 7 if dtype == np.float64 else 14
    c = mb.SimtConfig.make(32, sigma, 128)
    t = mb.generate_tile_for(m, c)
    m.build_xcache(FORCE_HUBS)
    tr = mb.trace_counts(t)
    assert tr.fast_tiles > 0 and tr.skipped_tiles >= 0
    x = O.hash_uniform(5, n, -1.0, 1.0, dtype)
    y = mb.spmv_merbit(m, t, c, x, mb.DualBuffer(n, dtype))
    a = O.Csr(n, n, ro, cols, vals)
    if dtype == np.float64:
        want, mag = O.spmv_csr_f64(a, x, want_abs=True)
        tol = 1e-12
    else:
        want, mag = O.spmv_csr_f32_acc64(a, x)
        tol = 1e-5
    assert np.all(np.abs(y.astype(np.float64) - want) <= tol * np.maximum(mag, 1e-300))
    assert not y[lens == 0].any()
