"""CPU: pin the oracle restatement (oracle/merbit_oracle.c) against the real
reference's outputs committed in tests/golden/ (written by make_golden.py from
oracle/_ref), and against the reference's own known-answer tests."""
import numpy as np
import pytest

import oracle as O
from helpers import CONFIGS, h


def test_walkthrough_known_answers(golden):
    g = golden["walkthrough"]
    a = O.walkthrough()
    assert a.row_offsets.tolist() == g["row_offsets"]
    # test_merge_path.cpp:142-150
    path = "".join("RD"[s] for s in O.sequential_path(a.row_offsets, 8, 34))
    assert path == g["path"] == ("RRRRR" "DD" "RRRRR" "D" "RRR" "D" "RRRRRRR" "D" "RRRRRR" "D"
                                 "RRRRRR" "D" "RR" "D")
    # test_merge_path.cpp:110-140
    starts = [list(O.merge_search(a.row_offsets, 8, 34, d)[:2]) for d in range(0, 42, 4)]
    assert starts == g["lane_starts_4_4"] == [[0, 0], [4, 0], [6, 2], [10, 2], [13, 3], [16, 4],
                                              [20, 4], [23, 5], [26, 6], [30, 6], [33, 7]]
    # test_format.cpp:59-110
    tx, ty, ld = O.generate_tile(a.row_offsets, 8, 34, 4, 4)
    assert tx.tolist() == [0, 13, 26, 34]
    assert (ty & 0x7FFFFFFF).tolist() == [0, 3, 6, 8]
    ob = O.config_make(4, 4, 4)
    assert [int(d) & 15 for d in ld[4:8]] == [0, 3, 7, 10]
    assert [(int(d) >> ob) & 15 for d in ld[4:8]] == [0, 1, 1, 2]
    assert int(ld[4]) >> (2 * ob) == 0b0001
    assert not np.any(ty[:-1] & 0x80000000)
    for key, t in g["tiles"].items():
        w, s = map(int, key.split(","))
        got = O.generate_tile(a.row_offsets, 8, 34, w, s)
        assert [x.tolist() for x in got] == [t["tile_x"], t["tile_y"], t["lane_desc"]]
    # test_kernel.cpp:30-46: bitwise for four configs
    assert g["y_unit"] == [15, 0, 40, 36, 119, 141, 177, 67]
    for (w, s, b) in [(4, 4, 4), (4, 4, 8), (32, 7, 64), (32, 14, 128)]:
        t = O.generate_tile(a.row_offsets, 8, 34, w, s)
        y, _ = O.spmv_merbit(a, np.ones(8), t, w, s, b)
        assert y.tolist() == g["y_unit"]


def test_descriptor_word_262659():
    # test_format.cpp:37-42: pack(3, 1, 0b1) at (32, 14) == 262659
    ob = O.config_make(32, 14, 32)
    assert (1 << (2 * ob)) | (1 << ob) | 3 == 262659


def test_fuzz_corpus_matches_reference_bitwise(golden):
    """504 matrices (acceptance.cpp:49-57) x 3 configs: CSR, x, TILE, CSR-y and
    MERBIT-y (f64) bit-identical to the compiled reference's."""
    for e in golden["fuzz_corpus"]:
        m = O.random_matrix(e["shape"], e["seed"])
        assert (m.n_rows, m.n_cols, m.nnz) == (e["n_rows"], e["n_cols"], e["nnz"])
        assert h(m.row_offsets, m.col_indices, m.values) == e["csr"], (e["shape"], e["seed"])
        x = O.seed_test_vector(m.n_cols, -1.0, 1.0, e["seed"])
        assert h(x) == e["x"]
        assert h(O.spmv_csr_f64(m, x)) == e["y_csr_f64"]
        for (w, s, b) in CONFIGS:
            t = O.generate_tile(m.row_offsets, m.n_rows, m.nnz, w, s)
            g = e["tiles"][f"{w},{s}"]
            assert h(*t) == g["tile"], (e["shape"], e["seed"], w, s)
            y, cnt = O.spmv_merbit(m, x, t, w, s, b)
            assert h(y) == g["y_merbit_f64"]
            assert cnt.tolist() == g["trace"]


def test_reconstruct_path_equals_walk():
    for shape in O.SHAPES:
        m = O.random_matrix(shape, 41)
        walked = O.sequential_path(m.row_offsets, m.n_rows, m.nnz)
        for (w, s, _) in CONFIGS:
            t = O.generate_tile(m.row_offsets, m.n_rows, m.nnz, w, s)
            assert np.array_equal(O.reconstruct_path(*t, m.n_rows, m.nnz, w, s), walked)


def test_merge_search_exhaustive_with_probe_budget():
    # test_merge_path.cpp:75-108
    for shape in O.SHAPES:
        used = 0
        for seed in range(31, 91):
            m = O.random_matrix(shape, seed)
            if m.nnz + m.n_rows > 2000:
                continue
            used += 1
            path = O.sequential_path(m.row_offsets, m.n_rows, m.nnz)
            budget = int(np.ceil(np.log2(m.n_rows + 1))) + 1
            x = y = 0
            for d in range(m.nnz + m.n_rows + 1):
                fx, fy, probes = O.merge_search(m.row_offsets, m.n_rows, m.nnz, d)
                assert (fx, fy) == (x, y) and probes <= budget
                if d < path.size:
                    x, y = (x + 1, y) if path[d] == 0 else (x, y + 1)
            if used == 3:
                break


def test_config_feasibility_formula():
    # acceptance.cpp:483-502
    for omega in (1, 2, 4, 8, 16, 32):
        for sigma in range(1, 41):
            ob = int(np.ceil(np.log2(omega * sigma))) if omega * sigma > 1 else 0
            infeasible = 2 * ob + sigma > 32
            try:
                O.config_make(omega, sigma, 4 * omega)
                threw = False
            except O.OracleError:
                threw = True
            assert threw == infeasible


def test_pagerank_ring_matches_reference(golden):
    g = golden["pagerank"]["ring_100_260_42"]
    p = O.build_transition(O.ring_with_chords(100, 260, 42))
    assert h(p.row_offsets, p.col_indices, p.values) == g["p_hash"]
    r = O.pagerank(p)
    assert r["iterations"] == g["iterations"] and r["status"] == "converged"
    assert np.array_equal(r["pi"], np.array(g["pi"]))
    g32 = golden["pagerank"]["ring_f32_50it"]
    r32 = O.pagerank(p.astype(np.float32), 0.85, 1e-30, 50, 0)
    assert np.array_equal(r32["pi"].astype(np.float64), np.array(g32["pi"]))


def test_pagerank_closed_forms():
    # test_solvers.cpp:61-99
    two = O.Csr(2, 2, np.array([0, 1, 2]), np.array([1, 0], np.int32), np.ones(2))
    r = O.pagerank(O.build_transition(two))
    assert r["iterations"] == 1 and r["pi"].tolist() == [0.5, 0.5]
    dang = O.Csr(2, 2, np.array([0, 1, 1]), np.array([1], np.int32), np.ones(1))
    r = O.pagerank(O.build_transition(dang))
    c = 0.85
    assert r["status"] == "converged"
    assert abs(r["pi"][0] - 1 / (2 + c)) < 1e-10 and abs(r["pi"][1] - (1 + c) / (2 + c)) < 1e-10


def test_rmat_generator_transposed_is_transition_pattern():
    a = O.rmat(12, 16, 5, transposed=False)
    p = O.rmat(12, 16, 5, transposed=True)
    q = O.build_transition(a, np.float32)
    assert np.array_equal(q.row_offsets, p.row_offsets)
    assert np.array_equal(q.col_indices, p.col_indices)
    assert np.array_equal(q.values, O.transition_values(p.n_rows, p.col_indices, np.float32))
    assert 0 < a.nnz <= 16 << 12


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref needs /root/reference to build")
def test_restatement_vs_live_reference_f32():
    R = O.ref()
    for seed in (3, 17):
        for shape in O.SHAPES:
            m = O.random_matrix(shape, seed).astype(np.float32)
            x = O.seed_test_vector(m.n_cols, -1, 1, seed).astype(np.float32)
            for (w, s, b) in CONFIGS:
                t = O.generate_tile(m.row_offsets, m.n_rows, m.nnz, w, s)
                y1, c1 = O.spmv_merbit(m, x, t, w, s, b)
                y2, c2 = R.spmv_merbit(m, x, w, s, b)
                assert np.array_equal(y1.view(np.uint32), y2.view(np.uint32))
                assert np.array_equal(c1, c2)


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref (the compiled reference) not built")
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_bicgstab_restatement_is_the_reference(dt):
    """mo_bicgstab (C restatement of solvers.hpp:268-373) == the reference's own
    bicgstab<T> over CsrReferenceBackend, bitwise: x, history, counts, reason."""
    cases = []
    a = O.five_point_laplacian(8, dt)
    cases.append((a, O.seed_test_vector(a.n_rows, -1, 1, 97).astype(dt), 1e-10))
    a = O.five_point_laplacian(32, dt)
    xt = O.seed_test_vector(a.n_rows, -1, 1, 77)
    cases.append((a, O.spmv_csr_f64(a.astype(np.float64), xt).astype(dt),
                  1e-10 if dt == np.float64 else 1e-6))
    cases.append((O.singular_diagonal(dt), np.ones(2, dt), 1e-10))
    cases.append((O.five_point_laplacian(3, dt), np.zeros(9, dt), 1e-10))
    for a, b, tol in cases:
        got = O.bicgstab(a, b, tol, 500)
        want = O.ref().bicgstab_csr(a, b, tol, 500)
        assert got["iterations"] == want["iterations"]
        assert got["status"] == want["status"]
        assert got["breakdown_reason"] == want["breakdown_reason"]
        assert np.array_equal(got["x"], want["x"])
        assert np.array_equal(got["residual_history"], want["residual_history"])
        assert got["final_residual"] == want["final_residual"] or (
            np.isinf(got["final_residual"]) and np.isinf(want["final_residual"]))
