"""GPU parity at the benchmark's sizes pinned to the COMPILED reference
(oracle/_ref = the unmodified reference built from its sources), not only
to the C restatement:

* TILE at R-MAT scale 20 (C1) and 24 (C2): byte-identical to the
  reference's own generate_tile (src/tile.cpp:17-85);
* PageRank at scale 20: the device fp32 run (bench configuration: degree
  relabelled, hub table) within 1e-6 L1 of the reference's pagerank<double>
  (solvers.hpp:154-218) on the same transition matrix;
* C5 (27-point stencil, 64 M rows, fp32 and fp64) with a RANDOM x against
  the stencil's closed form accumulated in fp64 on the host (pinned to the
  CSR oracle on a small grid first), at the north-star tolerances 1e-5 /
  1e-12 relative to sum |a||x| per row.

Marked slow: the reference runs single-threaded (a few seconds per case)."""
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2605_07391_b200 as mb
from helpers import FORCE_HUBS

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
NT = os.cpu_count() or 1


@pytest.fixture(scope="module")
def cx():
    return mb.Context(0)  # default K2 layout (slot copy), the bench's


def need_ref():
    if O.ref() is None:
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    return O.ref()


@pytest.mark.parametrize("scale", [20, 24])
def test_rmat_tile_is_the_compiled_reference(cx, scale):
    ref = need_ref()
    P = mb.DeviceMatrix.rmat(cx, scale, 16, seed=1, transition=True, dtype=np.float32)
    ro = P.row_offsets()
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile_for(P, c)
    want = ref.generate_tile(ro, P.n_rows, P.nnz, 32, 14)
    for got, w in zip(t.download(), want):
        assert got.dtype == w.dtype and np.array_equal(got, w)


def test_s20_pagerank_vs_reference_pagerank_double(cx):
    """bench.py's configuration at scale 20 (device relabelling + hub table,
    100 fixed iterations, fp32) vs the reference's pagerank<double> over its
    csr backend with reference_iters = 0: L1 <= 1e-6 in the original
    vertex order."""
    ref = need_ref()
    P = mb.DeviceMatrix.rmat(cx, 20, 16, seed=1, transition=True, dtype=np.float32)
    ro, cols, _ = P.download(want_values=False)
    n = P.n_rows
    c = mb.SimtConfig.make(32, 14, 128)
    Q, _ = P.relabel_by_degree(want_rank=False)
    be = type("B", (), {})()
    be.matrix, be.tile_, be.c = Q, mb.generate_tile_for(Q, c), c
    Q.build_xcache(FORCE_HUBS)  # the bench's hub path (automatic mode skips s20)
    r = mb.pagerank(None, mb.PageRankConfig(0.85, 1e-30, 100, 0), backend=be)
    p64 = O.Csr(n, n, ro, cols, O.transition_values(n, cols, np.float64))
    want = ref.pagerank_csr(p64, 0.85, 1e-300, 100, 0)
    assert want["iterations"] == 100
    l1 = float(np.abs(r.pi.astype(np.float64) - want["pi"]).sum())
    assert r.iterations == 100 and l1 <= 1e-6, l1
    # and the restatement agrees with the reference itself here
    mine = O.pagerank(p64, 0.85, 1e-300, 100, 0, nthreads=NT)
    assert float(np.abs(mine["pi"] - want["pi"]).sum()) <= 1e-12


def stencil_closed_form(g, x):
    """y = A x for the 27-point stencil (diagonal 26, in-grid neighbours -1)
    in fp64, and sum |a||x| per row, from shifted copies of x."""
    x3 = x.astype(np.float64).reshape(g, g, g)
    pad = np.zeros((g + 2, g + 2, g + 2))
    pad[1:-1, 1:-1, 1:-1] = x3
    apad = np.abs(pad)
    nb = np.zeros((g, g, g))
    mag = np.zeros((g, g, g))
    for di in range(3):
        for dj in range(3):
            for dk in range(3):
                nb += pad[di:di + g, dj:dj + g, dk:dk + g]
                mag += apad[di:di + g, dj:dj + g, dk:dk + g]
    # nb and mag include the centre once
    y = 27.0 * x3 - nb
    mag = 25.0 * np.abs(x3) + mag
    return y.reshape(-1), mag.reshape(-1)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_stencil_closed_form_is_the_csr_oracle(cx, dtype):
    """Pins the closed form used below to the CSR oracle on a 24^3 grid."""
    g = 24
    A = mb.DeviceMatrix.stencil27(cx, g, dtype)
    ro, cols, vals = A.download()
    x = O.hash_uniform(11, A.n_cols, -1.0, 1.0, dtype)
    want, mag = O.spmv_csr_f64(O.Csr(A.n_rows, A.n_cols, ro, cols, vals.astype(np.float64)),
                               x.astype(np.float64), want_abs=True)
    y, m2 = stencil_closed_form(g, x)
    assert np.allclose(y, want, rtol=0, atol=1e-13) and np.allclose(m2, mag, rtol=1e-15)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_c5_full_size_random_x(cx, dtype):
    """BASELINE C5 at full size (400^3 = 64 M rows, 1.72e9 nonzeros) with a
    random x in [-1, 1): y within 1e-5 (fp32) / 1e-12 (fp64) of the fp64
    closed form relative to sum |a||x| per row."""
    g = 400
    A = mb.DeviceMatrix.stencil27(cx, g, dtype)
    c = mb.SimtConfig.make(32, 14 if dtype == np.float32 else 7, 128)
    t = mb.generate_tile_for(A, c)
    A.build_xcache()
    x = O.hash_uniform(13, A.n_cols, -1.0, 1.0, dtype)
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    xd = torch.from_numpy(x).to("cuda")
    yd = torch.empty(A.n_rows, dtype=tdt, device="cuda")
    torch.cuda.synchronize()  # x is on the device before the library's stream reads it
    mb.spmv_device(A, t, c, xd.data_ptr(), yd.data_ptr())
    cx.synchronize()  # and y is complete before torch's stream copies it out
    y = yd.cpu().numpy().astype(np.float64)
    del A, t, xd, yd
    torch.cuda.synchronize()
    want, mag = stencil_closed_form(g, x)
    tol = 1e-5 if dtype == np.float32 else 1e-12
    rel = np.abs(y - want) / np.where(mag > 0, mag, 1.0)
    assert rel.max() <= tol, rel.max()
