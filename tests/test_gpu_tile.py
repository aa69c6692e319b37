"""GPU K1 (generate_tile on sm_100a) vs the oracle and the reference's golden
TILEs: byte-identical arrays (src/tile.cpp:17-85)."""
import numpy as np
import pytest

import oracle as O
import paper_2605_07391_b200 as mb
from helpers import CONFIGS, h

pytestmark = pytest.mark.gpu


def gpu_tile(ctx, a, w, s, b=None):
    c = mb.SimtConfig.make(w, s, b or w)
    return mb.generate_tile(a.row_offsets, a.n_rows, a.nnz, c, ctx)


def test_walkthrough_tile(ctx, golden):
    a = O.walkthrough()
    for key, t in golden["walkthrough"]["tiles"].items():
        w, s = map(int, key.split(","))
        tile = gpu_tile(ctx, a, w, s)
        assert (tile.tile_num, tile.lane_num) == ((42 + w * s - 1) // (w * s), (42 + s - 1) // s)
        assert [x.tolist() for x in tile.download()] == [t["tile_x"], t["tile_y"], t["lane_desc"]]
    tile = gpu_tile(ctx, a, 4, 4)
    tx, ty, ld = tile.download()
    assert tx.tolist() == [0, 13, 26, 34] and (ty & 0x7FFFFFFF).tolist() == [0, 3, 6, 8]
    assert tile.long_row_fraction() == 0.0
    steps = O.reconstruct_path(tx, ty, ld, 8, 34, 4, 4)
    assert np.array_equal(steps, O.sequential_path(a.row_offsets, 8, 34))


def test_fuzz_corpus_tiles_match_reference(ctx, golden):
    """acceptance.cpp c2/c4: all 504 corpus matrices x 3 configs."""
    for e in golden["fuzz_corpus"]:
        m = O.random_matrix(e["shape"], e["seed"])
        for (w, s, b) in CONFIGS:
            t = gpu_tile(ctx, m, w, s, b).download()
            assert h(*t) == e["tiles"][f"{w},{s}"]["tile"], (e["shape"], e["seed"], w, s)


@pytest.mark.parametrize("omega,sigma", [(1, 1), (1, 22), (2, 9), (3, 5), (8, 6), (16, 7),
                                         (32, 1), (32, 13), (64, 3), (128, 1)])
def test_odd_configs_match_oracle(ctx, omega, sigma):
    for shape in O.SHAPES:
        m = O.random_matrix(shape, 77)
        got = gpu_tile(ctx, m, omega, sigma).download()
        want = O.generate_tile(m.row_offsets, m.n_rows, m.nnz, omega, sigma)
        for g_, w_ in zip(got, want):
            assert np.array_equal(g_, w_), (shape, omega, sigma)


def test_single_dense_row_marks():
    # test_format.cpp:134-147
    ctx = mb.default_context()
    a = O.single_dense_row(64, 7)
    t = gpu_tile(ctx, a, 4, 4, 16)
    _, ty, _ = t.download()
    assert t.tile_num == 5
    assert all(ty[i] & 0x80000000 and (ty[i] & 0x7FFFFFFF) == 0 for i in range(4))
    assert not ty[4] & 0x80000000
    assert abs(t.long_row_fraction() - 0.8) < 1e-12


def test_capacity_errors_before_touching_data(ctx):
    # test_format.cpp:149-158
    c = mb.SimtConfig.make(4, 4, 4)
    with pytest.raises(mb.CapacityError):
        mb.generate_tile(None, 1 << 31, 0, c, ctx)
    with pytest.raises(mb.CapacityError):
        mb.generate_tile(None, 4, 1 << 32, c, ctx)


def test_empty_shapes(ctx):
    c = mb.SimtConfig.make(32, 14, 128)
    t = mb.generate_tile(np.zeros(1, np.int64), 0, 0, c, ctx)
    assert (t.tile_num, t.lane_num) == (0, 0)
    tx, ty, ld = t.download()
    assert tx.tolist() == [0] and ty.tolist() == [0] and ld.size == 0
    t = mb.generate_tile(np.zeros(38, np.int64), 37, 0, c, ctx)
    want = O.generate_tile(np.zeros(38, np.int64), 37, 0, 32, 14)
    assert all(np.array_equal(a, b) for a, b in zip(t.download(), want))


@pytest.mark.parametrize("scale,transposed", [(14, False), (16, True), (18, False)])
def test_rmat_tiles_byte_identical(ctx, scale, transposed):
    m = mb.DeviceMatrix.rmat(ctx, scale, 16, seed=1, transition=transposed)
    ro, cols, _ = m.download(want_values=False)
    cpu = O.rmat(scale, 16, 1, transposed=transposed)
    assert np.array_equal(ro, cpu.row_offsets) and np.array_equal(cols, cpu.col_indices)
    for (w, s) in [(32, 14), (32, 7)]:
        t = mb.generate_tile_for(m, mb.SimtConfig.make(w, s, 128))
        want = O.generate_tile(ro, m.n_rows, m.nnz, w, s)
        for g_, w_ in zip(t.download(), want):
            assert np.array_equal(g_, w_)


@pytest.mark.slow
def test_rmat_s20_tile_byte_identical(ctx):
    """C1 preprocessing at full size: R-MAT scale 20."""
    m = mb.DeviceMatrix.rmat(ctx, 20, 16, seed=1)
    ro, _, _ = m.download(want_values=False)
    for (w, s) in [(32, 14), (32, 7)]:
        t = mb.generate_tile_for(m, mb.SimtConfig.make(w, s, 128))
        want = O.generate_tile(ro, m.n_rows, m.nnz, w, s)
        for g_, w_ in zip(t.download(), want):
            assert np.array_equal(g_, w_)
