"""GPU BiCGSTAB (solvers.hpp:224-373) through K2/K3 and the
device dot/axpy kernels, checked with the reference's own test cases
(test_solvers.cpp:141-200, acceptance criterion 10) and against the oracle
restatement (pinned bitwise to the reference in test_oracle.py)."""
import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb

pytestmark = pytest.mark.gpu


def backend(ctx, a, w=32, s=None, b=128):
    s = s or (14 if a.values.dtype == np.float32 else 7)
    return mb.MerbitB200Backend(a, mb.SimtConfig.make(w, s, b), ctx)


def recomputed_residual(a, x, b):
    ax = O.spmv_csr_f64(a.astype(np.float64), np.asarray(x, np.float64))
    return float(np.sqrt(((ax - b) ** 2).sum() / (np.asarray(b, np.float64) ** 2).sum()))


@pytest.mark.parametrize("cfg", [(32, 7, 128), (4, 4, 16), (32, 7, 32)])
def test_five_point_laplacian(ctx, cfg):
    # test_solvers.cpp:141-166
    a = O.five_point_laplacian(8)
    b = O.seed_test_vector(a.n_rows, -1.0, 1.0, 97)
    r = mb.bicgstab(a, b, mb.BicgstabConfig(), backend(ctx, a, *cfg))
    assert r.status == "converged" and r.final_residual < 1e-10
    assert r.residual_history.size == r.iterations
    assert r.residual_history[-1] == r.final_residual
    assert abs(recomputed_residual(a, r.x, b) - r.final_residual) <= 1e-12
    want = O.bicgstab(a, b)
    assert abs(r.iterations - want["iterations"]) <= 1
    assert np.abs(r.x - want["x"]).max() <= 1e-9


def test_acceptance_criterion_10(ctx):
    # acceptance.cpp:401-443: 1024 x 1024 Laplacian, x_true known
    a = O.five_point_laplacian(32)
    x_true = O.seed_test_vector(a.n_rows, -1.0, 1.0, 77)
    b = O.spmv_csr_f64(a, x_true)
    r = mb.bicgstab(a, b, mb.BicgstabConfig(), backend(ctx, a))
    assert r.status == "converged" and r.iterations <= 20000 and r.final_residual < 1e-10
    assert abs(recomputed_residual(a, r.x, b) - r.final_residual) <= 1e-12
    # ||x - x_true|| is bounded by cond(A) (~400) times the 1e-10 residual
    assert np.abs(r.x - x_true).max() <= 1e-7
    want = O.bicgstab(a, b)
    assert abs(r.iterations - want["iterations"]) <= 2
    # deterministic: bitwise identical on a rerun
    r2 = mb.bicgstab(a, b, mb.BicgstabConfig(), backend(ctx, a))
    assert np.array_equal(r.x.view(np.uint64), r2.x.view(np.uint64))
    assert np.array_equal(r.residual_history, r2.residual_history)


def test_fp32_laplacian(ctx):
    a = O.five_point_laplacian(32, np.float32)
    x_true = O.seed_test_vector(a.n_rows, -1.0, 1.0, 77)
    b = O.spmv_csr_f64(a.astype(np.float64), x_true).astype(np.float32)
    r = mb.bicgstab(a, b, mb.BicgstabConfig(tol=1e-6), backend(ctx, a))
    want = O.bicgstab(a, b, 1e-6)
    assert r.status == want["status"] == "converged"
    assert r.final_residual < 1e-6
    assert abs(r.iterations - want["iterations"]) <= 3
    assert np.abs(r.x.astype(np.float64) - x_true).max() <= 1e-3  # cond(A) * 1e-6


def test_singular_breakdown(ctx):
    # test_solvers.cpp:168-179: <r_hat, v> vanishes at iteration 2
    a = O.singular_diagonal()
    r = mb.bicgstab(a, np.ones(2), mb.BicgstabConfig(), backend(ctx, a, 4, 4, 4))
    want = O.bicgstab(a, np.ones(2))
    assert r.status == "breakdown" and r.breakdown_reason == "rhat_dot_v"
    assert r.iterations == 2 == want["iterations"]
    assert np.array_equal(r.x, want["x"])
    assert np.array_equal(r.residual_history, want["residual_history"])


def test_trivial_and_dimension_checks(ctx):
    # test_solvers.cpp:181-200
    a = O.five_point_laplacian(3)
    be = backend(ctx, a)
    r = mb.bicgstab(a, np.zeros(a.n_rows), mb.BicgstabConfig(), be)
    assert r.status == "converged" and r.iterations == 0 and r.final_residual == 0.0
    assert not r.x.any()
    with pytest.raises(mb.DimensionError):
        mb.bicgstab(a, np.ones(3), mb.BicgstabConfig(), be)
    rect = O.single_dense_row(4, 1)
    with pytest.raises(mb.DimensionError):
        mb.bicgstab(rect, np.ones(3), mb.BicgstabConfig(), backend(ctx, rect))


def test_max_iterations_status(ctx):
    a = O.five_point_laplacian(32)
    b = O.seed_test_vector(a.n_rows, -1.0, 1.0, 5)
    r = mb.bicgstab(a, b, mb.BicgstabConfig(max_iters=5), backend(ctx, a))
    want = O.bicgstab(a, b, 1e-10, 5)
    assert r.status == want["status"] == "max_iterations" and r.iterations == 5
    assert np.allclose(r.residual_history, want["residual_history"], rtol=1e-9)
