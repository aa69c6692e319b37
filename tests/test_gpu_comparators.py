"""GPU comparators: the paper's baselines on the same
device -- csr_vector, coo_atomic (CooReferenceBackend), merge_runtime (the
reference's spmv_merge_runtime, merge_spmv.hpp:21-82), merge_cub and the
paper's own baseline, cuSPARSE SpMV (COO / CSR, ALG1 / ALG2) -- each
within the reference's ToleranceBound; merge_runtime bitwise equal to the
reference's own implementation where no carry run exceeds one warp."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2605_07391_b200 as mb
from paper_2605_07391_b200.merbit import spmv_baseline_device
from helpers import first_violation, tolerance_bound

pytestmark = pytest.mark.gpu
KINDS = ["csr_vector", "coo_atomic", "merge_runtime", "merge_cub", "cusparse_coo_alg1",
         "cusparse_coo_alg2", "cusparse_csr_alg1", "cusparse_csr_alg2"]


def run(ctx, a, kind, x, sigma=0):
    m = mb.DeviceMatrix.from_csr(ctx, a)
    tdt = torch.float64 if a.values.dtype == np.float64 else torch.float32
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    yd = torch.full((max(a.n_rows, 1),), float("nan"), dtype=tdt, device="cuda")
    torch.cuda.synchronize()  # torch's stream is done with x and y
    spmv_baseline_device(m, kind, xd.data_ptr(), yd.data_ptr(), sigma)
    ctx.synchronize()  # the library's stream is done with y
    return yd.cpu().numpy()[:a.n_rows]


@pytest.mark.parametrize("kind", KINDS)
def test_corpus_within_bound(ctx, kind):
    for shape in O.SHAPES:
        for seed in (1, 2, 3):
            for dt in (np.float64, np.float32):
                a = O.random_matrix(shape, seed).astype(dt)
                x = O.seed_test_vector(a.n_cols, -1, 1, seed).astype(dt)
                want = O.spmv_csr_f64(a.astype(np.float64), x.astype(np.float64))
                got = run(ctx, a, kind, x)
                assert first_violation(tolerance_bound(a, x, dt), want, got) == -1, (shape, seed)


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built")
def test_merge_runtime_is_the_reference(ctx):
    for shape in O.SHAPES:
        for seed in (4, 5):
            a = O.random_matrix(shape, seed)
            if np.diff(a.row_offsets).max(initial=0) >= 32 * 7:
                continue  # carry runs longer than a warp fold in a different order
            x = O.seed_test_vector(a.n_cols, -1, 1, seed)
            for sigma in (7, 4):
                want = O.ref().spmv_merge_runtime(a, x, sigma)
                got = run(ctx, a, "merge_runtime", x, sigma)
                assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (shape, seed)


@pytest.mark.parametrize("kind", KINDS)
def test_rmat_and_long_rows(ctx, kind):
    m = mb.DeviceMatrix.rmat(ctx, 16, 16, seed=1, dtype=np.float32)
    ro, cols, vals = m.download()
    a = O.Csr(m.n_rows, m.n_cols, ro, cols, vals)
    x = O.hash_uniform(1, m.n_cols, -1.0, 1.0, np.float32)
    want, mag = O.spmv_csr_f32_acc64(a, x)
    got = run(ctx, a, kind, x)
    assert (np.abs(got.astype(np.float64) - want) / np.where(mag > 0, mag, 1)).max() <= 1e-5
    row = O.single_dense_row(20000, 3)
    xr = O.seed_test_vector(20000, -1, 1, 3)
    got = run(ctx, row, kind, xr)
    want = O.spmv_csr_f64(row, xr)
    assert abs(got[0] - want[0]) <= 1e-12 * np.abs(row.values * xr).sum()
